"""NEXT f3: quality metrics (Table 1) -- the SPEC boundary examples,
invariants, and recovery on synthetic ground truth (oracle on CPU; the CUDA
path on GPU)."""
import numpy as np
import pytest

from inputs import synth
from paper_1610_04124_b200 import quality as Q
from tests import modelparams as mp

G, O, S_ = 0, 1, 2


def _col(H, obj_rows=(), ground_rows=()):
    """One reduced column of model-row labels: -2 sky by default."""
    lab = np.full(H, -2, np.int32)
    lab[list(ground_rows)] = -1
    for v in obj_rows:
        lab[v] = 0
    return lab[None, :]


def test_detection_boundary_strict():
    lab = _col(40, obj_rows=range(10, 20), ground_rows=range(0, 10))
    six = [(0, 9, G, 0.0), (10, 15, O, 5.0), (16, 39, S_, 0.0)]    # 6 of 10 rows covered
    five = [(0, 9, G, 0.0), (10, 14, O, 5.0), (15, 39, S_, 0.0)]   # exactly half
    assert Q.evaluate_frame([six], lab, 1)["detected"] == 1
    assert Q.evaluate_frame([five], lab, 1)["detected"] == 0


def test_empty_gt_rate_is_one():
    lab = _col(20, ground_rows=range(0, 8))
    r = Q.summarize([Q.evaluate_frame([[(0, 7, G, 0.0), (8, 19, S_, 0.0)]], lab, 1)])
    assert r["detection_rate"] == 1.0 and r["gt_stixels"] == 0


def test_false_positive_boundary():
    lab = _col(80, obj_rows=range(60, 70), ground_rows=range(0, 60))
    fp31 = [(0, 30, O, 3.0), (31, 79, G, 0.0)]        # 31 free-space pixels (s = 1)
    fp30 = [(0, 29, O, 3.0), (30, 79, G, 0.0)]        # 30: not a false positive
    assert Q.evaluate_frame([fp31], lab, 1)["false_positives"] == 1
    assert Q.evaluate_frame([fp30], lab, 1)["false_positives"] == 0
    assert Q.evaluate_frame([[(0, 79, G, 0.0)]], lab, 1)["false_positives"] == 0
    # width s multiplies the pixel count: 10 rows x s = 4 -> 40 > 30
    assert Q.evaluate_frame([[(0, 9, O, 3.0), (10, 79, G, 0.0)]], lab, 4)["false_positives"] == 1


def test_free_space_is_below_the_lowest_obstacle():
    lab = _col(50, obj_rows=range(20, 30), ground_rows=list(range(0, 20)) + list(range(30, 35)))
    fs = Q.free_space(lab)
    assert fs[0, :20].all() and not fs[0, 20:].any()


def test_detection_monotone_in_object_coverage():
    rng = np.random.default_rng(5)
    H = 60
    lab = np.full((1, H), -1, np.int32)
    lab[0, 10:25] = 0
    lab[0, 30:50] = 1
    base = [(0, 59, G, 0.0)]
    prev = Q.evaluate_frame([base], lab, 1)["detected"]
    cover = np.zeros(H, bool)
    for _ in range(20):
        a = int(rng.integers(0, H))
        b = int(rng.integers(a, H))
        cover[a:b + 1] = True
        lst, v = [], 0
        while v < H:                                   # re-tile: object runs where covered
            t = v
            while t + 1 < H and cover[t + 1] == cover[v]:
                t += 1
            lst.append((v, t, O if cover[v] else G, 0.0))
            v = t + 1
        cur = Q.evaluate_frame([lst], lab, 1)["detected"]
        assert cur >= prev
        prev = cur


def test_gt_labels_and_column_majority():
    sc = synth.c1_scene()
    lab = synth.gt_labels(sc)
    cl = Q.column_labels(lab, 5)
    st = Q.gt_stixels(cl)
    # box 0 spans image columns 10-24, rows 27-40 -> reduced columns 2-4, model rows 7-20
    assert (7, 20, 0) in st[2] and (7, 20, 0) in st[3]
    assert all(len(x) == 0 for x in st[:2])


def test_oracle_recovers_c1_scene_quality():
    """The oracle's segmentation of the noiseless C1 scene detects every GT
    stixel and has no false positive."""
    from tests.gpuharness import run_oracle
    sc = synth.c1_scene()
    img = synth.render(sc, 1, noise=False)
    p = mp.make(max_disparity=32, ground_slope=sc.alpha)
    lists, _ = run_oracle(p, img[None])
    cl = Q.column_labels(synth.gt_labels(sc), 5)
    r = Q.summarize([Q.evaluate_frame(lists[0], cl, 5)])
    assert r["detection_rate"] == 1.0 and r["total_false_positives"] == 0


@pytest.mark.gpu
def test_gpu_quality_on_noisy_c2_frames():
    """CUDA path on noisy C2-distribution frames: the metrics are those of the
    oracle's lists (exact parity) and the detection rate is high."""
    from tests.gpuharness import run_gpu, run_oracle
    frames, labs = [], []
    for i in range(3):
        sc = synth.random_scene(4000 + i, 1024, 440, 128)
        frames.append(synth.render(sc, 4000 + i))
        labs.append(Q.column_labels(synth.gt_labels(sc), 5))
    frames = np.stack(frames)
    p = mp.make()
    g, _, _, _ = run_gpu(p, frames)
    o, _ = run_oracle(p, frames)
    rg = Q.summarize([Q.evaluate_frame(g[b], labs[b], 5) for b in range(3)])
    ro = Q.summarize([Q.evaluate_frame(o[b], labs[b], 5) for b in range(3)])
    assert rg == ro
    assert rg["detection_rate"] >= 0.85
