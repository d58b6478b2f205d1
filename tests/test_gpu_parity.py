"""Parity of the CUDA path (through the C ABI) with the oracle, element by
element, on the same seeded inputs.  Exact mode (L#22): identical stixel lists
and identical column costs on EVERY column.  Continuous mode: BASELINE
north_star tolerance (column cost within 1e-4 relative; identical lists except
on columns whose GPU segmentation re-scores within 1e-4 of the oracle minimum).
"""
import numpy as np
import pytest

from inputs import synth
from tests import modelparams as mp
from tests.gpuharness import compare_exact, run_gpu, run_oracle

pytestmark = pytest.mark.gpu


def _frames_c2(n, seed0=2000, W=1024, H=440, D=128):
    return np.stack([synth.render(synth.random_scene(seed0 + i, W, H, D), seed0 + i)
                     for i in range(n)])


def _assert_exact(p, frames, **kw):
    """Both DP launch plans (4 and 8 warps per column) against the oracle."""
    o, oc = run_oracle(p, frames)
    for plan in (4, 8):
        g, gc, cnt, hd = run_gpu(p, frames, plan=plan, **kw)
        bad = compare_exact(g, gc, o, oc, p["cost_frac_bits"])
        assert not bad, f"plan {plan}: {len(bad)} mismatching columns, first: {bad[:2]}"
    return g, gc, cnt, hd


def test_single_frame_latency_plan_exact():
    """One 1024x440 frame (BASELINE configs[1]): the automatic plan gives each
    column 8 warps (at most 2 columns per SM) and is exact on every column."""
    frames = _frames_c2(1, seed0=2100)
    p = mp.make()
    g, gc, cnt, hd = run_gpu(p, frames)
    assert hd.last_launch_shape() == (8, 2)
    o, oc = run_oracle(p, frames)
    bad = compare_exact(g, gc, o, oc, p["cost_frac_bits"])
    assert not bad, f"{len(bad)} mismatching columns, first: {bad[:2]}"
    _, _, _, h4 = run_gpu(p, _frames_c2(4, seed0=2100))
    assert h4.last_launch_shape() == (4, 4)     # a batch filling the GPU keeps 4 x 4


def test_reduce_bit_exact():
    import torch
    from oracle import oracle as orc
    from paper_1610_04124_b200 import stixels as S
    frames = _frames_c2(3, W=1027)          # ragged tail: 1027 mod 5 = 2 dropped
    p = mp.make()
    B, H, W = frames.shape
    hd = S.Handle(S.params_from_dict(p, H), W, H, B)
    cols = torch.empty((B, hd.n_cols, H), dtype=torch.int16, device="cuda")   # u16 storage
    hd.reduce(torch.from_numpy(frames.view(np.int16)).cuda(), cols)
    hd.sync()
    got = cols.cpu().numpy().view(np.uint16).astype(np.int32)
    got[got == 0xFFFF] = -1
    for b in range(B):
        want = orc.reduce(frames[b], 5, 4, 0xFFFF, 128)
        assert (got[b] == want).all()


@pytest.mark.parametrize("s", [1, 2, 5, 8, 13])
def test_reduce_median_bit_exact(s):
    """Median reduction (NEXT f4): every reduced value equals the oracle's
    (sort-based) median, odd and even valid counts, invalid and >= D pixels."""
    import torch
    from oracle import oracle as orc
    from paper_1610_04124_b200 import stixels as S
    rng = np.random.default_rng(40 + s)
    H, W, D = 75, 13 * s + 3, 64
    f = rng.integers(0, (D + 3) * 16, size=(2, H, W)).astype(np.uint16)
    f[rng.random(f.shape) < 0.15] = 0xFFFF
    p = mp.make(max_disparity=D, stixel_width=s, reduce_mode=1)
    hd = S.Handle(S.params_from_dict(p, H), W, H, 2)
    cols = torch.empty((2, hd.n_cols, H), dtype=torch.int16, device="cuda")
    hd.reduce(torch.from_numpy(f.view(np.int16)).cuda(), cols)
    hd.sync()
    got = cols.cpu().numpy().view(np.uint16).astype(np.int32)
    got[got == 0xFFFF] = -1
    for b in range(2):
        assert (got[b] == orc.reduce(f[b], s, 4, 0xFFFF, D, mode=1)).all()


def test_median_mode_end_to_end_exact():
    """Whole path with the median reduction: identical lists and costs."""
    frames = _frames_c2(2, seed0=2500)
    p = mp.make(reduce_mode=1)
    _assert_exact(p, frames)


def _sigma_tables(seed, D, H):
    rng = np.random.default_rng(seed)
    f = np.arange(D)
    so = 0.7 + 1.4 / (1.0 + np.exp(-(f - D / 2) / (D / 10)))        # a sigmoid in f
    so = (so * rng.uniform(0.9, 1.1, D)).astype(np.float32)
    sg = rng.uniform(0.8, 3.0, H).astype(np.float32)
    return so, sg


def test_noise_model_tables_exact():
    """NEXT f2: sigma_O(f) (2-D pair table) and sigma_G(v) (per-row ground
    tables): identical lists and costs on C2 frames."""
    frames = _frames_c2(2, seed0=2700)
    so, sg = _sigma_tables(1, 128, 440)
    p = mp.make(sigma_object_f=so, sigma_ground_v=sg)
    _assert_exact(p, frames)


@pytest.mark.parametrize("H,W,D", [(33, 61, 128), (100, 70, 256), (65, 96, 200)])
def test_noise_model_tables_shapes_exact(H, W, D):
    so, sg = _sigma_tables(H + D, D, H)
    frames = np.stack([synth.uniform_random_image(55, W, H, D),
                       synth.render(synth.random_scene(56, W, H, D, alpha=0.9 * D / H), 56)])
    p = mp.make(max_disparity=D, ground_slope=0.9 * D / H, sigma_object_f=so, sigma_ground_v=sg)
    _assert_exact(p, frames)


def test_constant_noise_tables_equal_scalar_model():
    """Tables filled with the class constants give the scalar model's bytes."""
    frames = _frames_c2(1, seed0=2800)
    p0 = mp.make()
    p1 = mp.make(sigma_object_f=np.full(128, 1.0, np.float32),
                 sigma_ground_v=np.full(440, 2.0, np.float32))
    a = run_gpu(p0, frames)
    b = run_gpu(p1, frames)
    assert a[0] == b[0] and (a[1] == b[1]).all()


@pytest.mark.parametrize("W,s,fmt", [(1024, 3, "u16"), (1024, 7, "u16"), (1040, 5, "u8"),
                                      (512, 10, "u8"), (64, 64, "u16")])
def test_reduce_vector_path_bit_exact(W, s, fmt):
    """16-byte-load path of reduce_kernel (pitch and base 16-byte aligned): ragged
    tails (W mod s), tiles not aligned to 16 bytes, u8 and u16, mean and median."""
    import torch
    from oracle import oracle as orc
    from paper_1610_04124_b200 import stixels as S
    H, D = 70, 64
    rng = np.random.default_rng(W + s)
    if fmt == "u16":
        f = rng.integers(0, (D + 2) * 16, size=(2, H, W)).astype(np.uint16)
        f[rng.random(f.shape) < 0.1] = 0xFFFF
        kw = dict(invalid_value=0xFFFF, disp_frac_bits=4)
        dev = torch.from_numpy(f.view(np.int16)).cuda()
        dt = torch.int16
    else:
        f = rng.integers(0, 256, size=(2, H, W)).astype(np.uint8)
        kw = dict(invalid_value=255, disp_frac_bits=2, disp_format=S.U8)
        dev = torch.from_numpy(f).cuda()
        dt = torch.int16
    for mode in (0, 1):
        p = mp.make(max_disparity=D, stixel_width=s, reduce_mode=mode, **kw)
        hd = S.Handle(S.params_from_dict(p, H), W, H, 2)
        cols = torch.empty((2, hd.n_cols, H), dtype=dt, device="cuda")
        hd.reduce(dev, cols)
        hd.sync()
        got = cols.cpu().numpy().view(np.uint16).astype(np.int32)
        got[got == 0xFFFF] = -1
        for b in range(2):
            want = orc.reduce(f[b], s, kw["disp_frac_bits"], kw["invalid_value"], D, mode=mode)
            assert (got[b] == want).all(), (mode, b)
        hd.destroy()


@pytest.mark.parametrize("W,s", [(1024, 5), (1027, 3), (64, 64)])
def test_reduce_f32_bit_exact(W, s):
    """f32 input (L#28): NaN / inf / negative / >= D invalid, half-up conversion to
    1/256, mean and median; vector (W = 1024) and scalar (odd pitch) load paths."""
    import torch
    from oracle import oracle as orc
    from paper_1610_04124_b200 import stixels as S
    H, D = 50, 64
    rng = np.random.default_rng(W + s)
    f = rng.uniform(-2.0, D + 2.0, size=(2, H, W)).astype(np.float32)
    f[rng.random(f.shape) < 0.05] = np.nan
    f[rng.random(f.shape) < 0.02] = np.inf
    f[:, :, :7] = np.round(f[:, :, :7] * 256) / 256 + np.float32(1 / 512)   # exact half-way values
    for mode in (0, 1):
        p = mp.make(max_disparity=D, stixel_width=s, reduce_mode=mode, disp_format=S.F32)
        hd = S.Handle(S.params_from_dict(p, H), W, H, 2)
        cols = torch.empty((2, hd.n_cols, H), dtype=torch.int16, device="cuda")
        hd.reduce(torch.from_numpy(f).cuda(), cols)
        hd.sync()
        got = cols.cpu().numpy().view(np.uint16).astype(np.int32)
        got[got == 0xFFFF] = -1
        for b in range(2):
            assert (got[b] == orc.reduce(f[b], s, 0, 0, D, mode=mode)).all(), (mode, b)
        hd.destroy()


def test_f32_input_end_to_end_exact():
    frames = _frames_c2(1, seed0=2900)
    f = np.where(frames == 0xFFFF, np.nan, frames.astype(np.float64) / 16).astype(np.float32)
    from paper_1610_04124_b200 import stixels as S
    p = mp.make(disp_format=S.F32)
    _assert_exact(p, f)


def test_c1_scene_exact():
    sc = synth.c1_scene()
    frames = np.stack([synth.render(sc, 1, noise=False), synth.render(sc, 2)])
    p = mp.make(max_disparity=32, ground_slope=sc.alpha)
    _assert_exact(p, frames)


def test_c2_frames_exact():
    frames = _frames_c2(3)
    p = mp.make()
    g, gc, cnt, hd = _assert_exact(p, frames)
    assert hd.last_launch_count() == 2      # reduce_kernel + dp_kernel


def test_full_batch_path_exact_sampled():
    """The headline path at a batch large enough for the strip reduction (48 frames
    of 1024x440: 672 strips of 32 rows >= 4 per SM) and the int32 kernel with the
    chunk bound, through stixels_compute: every column of 6 sampled frames equals
    the oracle exactly."""
    frames = _frames_c2(48, seed0=3500)
    p = mp.make()
    g, gc, cnt, hd = run_gpu(p, frames)
    assert hd.skipped_cells() > 0
    pick = [0, 9, 17, 30, 41, 47]
    o, oc = run_oracle(p, frames[pick])
    bad = compare_exact([g[i] for i in pick], gc[pick], o, oc, p["cost_frac_bits"])
    assert not bad, f"{len(bad)} mismatching columns, first: {bad[:2]}"


def test_chunk_bound_skips_and_stays_exact():
    """The int32 kernel's exact chunk bound (columns of >= 320 rows): on C2 frames
    it skips a substantial share of the rectangle cells (stixels_skipped_cells) and
    the lists and costs stay identical to the oracle's under both launch plans; on
    two-valued striped columns (many equal-cost candidates in different chunks, so
    the nearest-first chunk order must still resolve ties to the lower bottom, L#17)
    and at h = 352 (a ragged last block) as well."""
    frames = _frames_c2(2, seed0=3300)
    p = mp.make()
    g, gc, cnt, hd = _assert_exact(p, frames)
    cells = hd.n_cols * 440 * 441 // 2 * frames.shape[0]
    # (the handle of the last plan, 8 warps per column, ran once on these frames)
    assert hd.skipped_cells() > 0.1 * cells
    rng = np.random.default_rng(3301)
    H, W = 352, 320
    stripes = np.where(rng.random((2, H, 1)) < 0.5, 10 * 16, 40 * 16).astype(np.uint16)
    fr = np.repeat(stripes, W, axis=2)
    fr[:, rng.random(H) < 0.05, :] = 0xFFFF              # a few invalid rows
    _assert_exact(mp.make(ground_slope=0.3), fr)


@pytest.mark.parametrize("H,W", [(440, 1024), (160, 400), (96, 300)])
def test_chunk_bound_on_off_identical(H, W):
    """stixels_set_chunk_bound: the int32 kernel with the chunk bound forced on and
    forced off gives byte-identical lists and costs, under both launch plans, and
    both equal the oracle's; the bound is forced on also below its automatic
    threshold (320 rows), where it is off by default, so short columns with few
    chunks exercise it as well."""
    frames = _frames_c2(2, seed0=3400 + H, W=W, H=H)
    p = mp.make()
    o, oc = run_oracle(p, frames)
    for plan in (4, 8):
        res = {}
        for bound in (1, 2):
            g, gc, cnt, hd = run_gpu(p, frames, plan=plan, bound=bound)
            bad = compare_exact(g, gc, o, oc, p["cost_frac_bits"])
            assert not bad, f"plan {plan} bound {bound}: {len(bad)} mismatching columns, first: {bad[:2]}"
            res[bound] = (g, gc.tobytes(), hd.skipped_cells())
        assert res[1][0] == res[2][0] and res[1][1] == res[2][1]
        assert res[1][2] == 0                            # off: nothing skipped


def test_chunk_bound_mode_errors():
    """stixels_set_chunk_bound rejects modes outside 0..2, and forcing it on for a
    model without the int32 kernel (continuous mode) is UNSUPPORTED."""
    from paper_1610_04124_b200 import stixels as S
    H, W = 440, 200
    hd = S.Handle(S.params_from_dict(mp.make(), H), W, H, 1)
    with pytest.raises(Exception):
        hd.set_chunk_bound(3)
    hd.set_chunk_bound(2)
    hd.set_chunk_bound(0)
    hd.destroy()
    hc = S.Handle(S.params_from_dict(mp.make(cost_frac_bits=0), H), W, H, 1)
    with pytest.raises(Exception):
        hc.set_chunk_bound(2)
    hc.set_chunk_bound(1)
    hc.destroy()


def test_dp_variants_exact():
    """Each DP kernel variant stixels_create picks is exact against
    the oracle: the int32 atomic-band path (band <= 3, the default model), the
    fp32 sparse band rounds (band 4..7) and the fp32 dense W-row ring (band > 7),
    chosen here through sigma_O; continuous mode never takes the int32 path."""
    from paper_1610_04124_b200 import stixels as S
    frames = _frames_c2(2, seed0=2600, W=320, H=200)
    seen = {}
    for sig_o in (1.0, 1.6, 2.2, 3.0, 4.5, 6.0):
        p = mp.make(sigma=(2.0, sig_o, 0.5))
        g, gc, cnt, hd = _assert_exact(p, frames)
        seen.setdefault(hd.dp_variant, sig_o)
    assert seen.get(S.DP_INT32) == 1.0
    assert {S.DP_INT32, S.DP_SPARSE, S.DP_DENSE} <= set(seen), seen
    _, _, _, hd = run_gpu(mp.make(cost_frac_bits=0), frames[:1])
    assert hd.dp_variant == S.DP_SPARSE


@pytest.mark.parametrize("H,W,D,s", [(1, 40, 16, 5), (31, 64, 16, 3), (32, 50, 64, 5),
                                     (33, 61, 128, 1), (65, 96, 200, 7), (100, 70, 256, 10)])
def test_shapes_and_disparity_ranges_exact(H, W, D, s):
    """Ragged column heights (1, 31, 32, 33, 65: partial 32-row blocks), D up to
    256 (the 256-slot kernel), s in {1,3,5,7,10}, ragged widths."""
    frames = np.stack([synth.uniform_random_image(77 + i, W, H, D) for i in range(2)] +
                      [synth.render(synth.random_scene(90, W, H, D, alpha=0.9 * D / max(H, 2)),
                                    90)])
    p = mp.make(max_disparity=D, stixel_width=s, ground_slope=0.9 * D / max(H, 2))
    _assert_exact(p, frames)


def test_max_height_c5_shape_exact():
    """Maximum column height h = 1024 with D = 256 (config C5's shape, q = 10 per
    L#22): 2 frames of 9 columns, every column exact."""
    H, W, D = 1024, 47, 256
    p = mp.make(max_disparity=D, ground_slope=0.35, cost_frac_bits=10)
    frames = np.stack([synth.render(synth.random_scene(700 + i, W, H, D, alpha=0.35), 700 + i)
                       for i in range(2)])
    _assert_exact(p, frames)


def test_degenerate_columns_exact():
    """All-invalid frame, all-zero frame, saturated (d = D - 1/16) frame."""
    H, W, D = 70, 40, 64
    f0 = np.full((H, W), 0xFFFF, np.uint16)
    f1 = np.zeros((H, W), np.uint16)
    f2 = np.full((H, W), D * 16 - 1, np.uint16)
    p = mp.make(max_disparity=D)
    _assert_exact(p, np.stack([f0, f1, f2]))


def test_u8_input_exact():
    H, W, D = 120, 100, 64
    rng = np.random.default_rng(8)
    sc = synth.random_scene(8, W, H, D, alpha=0.5, q_bits=2)
    f16 = synth.render(sc, 8)
    f8 = np.where(f16 == 0xFFFF, 255, np.minimum(f16, 254)).astype(np.uint8)
    p = mp.make(max_disparity=D, disp_frac_bits=2, invalid_value=255, ground_slope=0.5)
    _assert_exact(p, f8[None])


def test_random_priors_exact():
    """Random (structurally valid) prior weights, margins and sigmas."""
    rng = np.random.default_rng(12)
    H, W, D = 96, 80, 48
    for it in range(4):
        t = mp.default_trans()
        for a, b in [(0, 1), (0, 2), (1, 0), (1, 1), (1, 2)]:
            t[a][b] = float(rng.choice([1.0, 0.3, 0.05, 0.0]))
        p = mp.make(max_disparity=D, p_trans=t, p_ord=float(rng.uniform(0.01, 0.5)),
                    p_grav=float(rng.uniform(0, 0.4)), p_blg=float(rng.uniform(0, 0.4)),
                    p_exist=float(rng.choice([1.0, 0.1, 0.01])),
                    p_first=(1.0, float(rng.choice([1.0, 0.1, 0.0])), 0.0),
                    ord_margin=int(rng.integers(0, 4)), grav_margin=int(rng.integers(0, 4)),
                    sigma=tuple(float(x) for x in rng.choice([0.5, 1.0, 1.5, 3.0], 3)),
                    ground_slope=float(rng.uniform(0.2, 0.8)), cost_frac_bits=int(rng.integers(6, 12)))
        frames = np.stack([synth.render(synth.random_scene(300 + it, W, H, D, alpha=p["ground_slope"]),
                                        300 + it), synth.uniform_random_image(400 + it, W, H, D)])
        _assert_exact(p, frames)


def test_continuous_mode_tolerance():
    """cost_frac_bits = 0 (the paper-literal fp32 Eq. 4) vs double on
    3 C2 frames: column cost within 1e-4 relative; full stixel tuples (bounds,
    class, disparity) identical except where the GPU's segmentation is
    co-optimal (re-scored within 1e-4 of the oracle minimum), BASELINE
    north_star."""
    from oracle import oracle as orc
    frames = _frames_c2(3, seed0=2100)
    p = mp.make(cost_frac_bits=0)
    g, gc, cnt, hd = run_gpu(p, frames)
    o, oc = run_oracle(p, frames)
    m = mp.oracle_model(p, 440)
    ties = total = 0
    for b in range(3):
        cols = orc.reduce(frames[b], 5, 4, 0xFFFF, 128)
        for c in range(len(o[b])):
            total += 1
            assert abs(gc[b][c] - oc[b][c]) <= 1e-4 * abs(oc[b][c])
            og = [(a, z, k, float(np.float32(d))) for a, z, k, d in o[b][c]]
            if og != g[b][c]:
                ties += 1
                rs = orc.rescore(m, cols[c], g[b][c])
                assert abs(rs - oc[b][c]) <= 1e-4 * abs(oc[b][c]), (b, c)
    assert ties <= total // 10


def test_capacity_overflow_reported():
    from paper_1610_04124_b200 import stixels as S
    frames = _frames_c2(1)
    p = mp.make(max_stixels=3)
    with pytest.raises(S.StixelsError) as ei:
        run_gpu(p, frames)
    assert ei.value.status == S.ERR_CAPACITY


def test_host_path_matches_device_path():
    frames = _frames_c2(70, seed0=5000, W=200, H=150)   # several host-path stages
    p = mp.make(ground_slope=0.6)
    a, ac, an, _ = run_gpu(p, frames)
    b, bc, bn, _ = run_gpu(p, frames, host=True)
    assert a == b and (ac == bc).all() and (an == bn).all()


def test_host_path_pinned_overlapping_stages():
    """stixels_compute_host with PINNED buffers (asynchronous copies, so
    consecutive stages overlap on the GPU) at the GPU-filling C2 shape, 4 stages
    of 29 frames, right after a device-path call still queued on the handle's
    stream: byte-identical to the device path, sampled columns exact against
    the oracle (per-stage DP scratch, entry wait on the stream)."""
    import torch
    from oracle import oracle as orc
    from paper_1610_04124_b200 import stixels as S
    from tests.gpuharness import compare_exact
    n = 116
    pool = _frames_c2(8, seed0=5100)
    frames = pool[np.arange(n) % 8]
    p = mp.make()
    hd = S.Handle(S.params_from_dict(p, 440), 1024, 440, n)
    dev = torch.from_numpy(frames.view(np.int16)).cuda()
    o1, c1, k1 = hd.alloc_outputs(n)
    hin = torch.from_numpy(frames.view(np.int16)).pin_memory()
    hout = torch.zeros((n, hd.n_cols, hd.cap, 12), dtype=torch.uint8).pin_memory()
    hcnt = torch.zeros((n, hd.n_cols), dtype=torch.int32).pin_memory()
    hcost = torch.zeros((n, hd.n_cols), dtype=torch.float32).pin_memory()
    for rep in range(2):
        hd.compute(dev, o1, c1, k1)            # queued, not synchronised
        hd.compute_host_ptr(hin.data_ptr(), 1024 * 2, n, hout.data_ptr(), hcnt.data_ptr(),
                            hcost.data_ptr())
        hd.sync()
        cnt = c1.cpu()
        assert torch.equal(hcnt, cnt) and torch.equal(hcost, k1.cpu())
        for f in range(n):                     # entries past count are undefined
            for c in range(0, hd.n_cols, 7):
                m = int(cnt[f, c])
                assert torch.equal(hout[f, c, :m], o1[f, c, :m].cpu())
    got = S.decode(hout.numpy(), hcnt.numpy())
    m = mp.oracle_model(p, 440)
    rng = np.random.default_rng(3)
    for f in (0, 57, 115):
        ci = rng.choice(hd.n_cols, 10, replace=False)
        st, oc = orc.solve_frame(m, orc.reduce(frames[f], 5, 4, 0xFFFF, 128)[ci])
        assert not compare_exact([[got[f][c] for c in ci]], [hcost.numpy()[f][ci]], [st], [oc], 11)


def test_noise_model_wide_band_dense_exact():
    """NEXT f2 with a wide sigma_O(f) sigmoid (reaching ~5 px, pair-cost band
    > 7): the dense ring over the 2-D table runs and is exact; a
    per-row ground table alone with a wide scalar sigma_O also runs (formerly
    UNSUPPORTED)."""
    from paper_1610_04124_b200 import stixels as S
    frames = _frames_c2(2, seed0=2750, W=400, H=220)
    f = np.arange(128)
    so = (1.0 + 4.0 / (1.0 + np.exp(-(f - 64) / 12.0))).astype(np.float32)
    _, sg = _sigma_tables(7, 128, 220)
    p = mp.make(sigma_object_f=so, sigma_ground_v=sg)
    _, _, _, hd = _assert_exact(p, frames)
    assert hd.dp_variant == S.DP_PAIR2D_DENSE
    p = mp.make(sigma=(2.0, 4.0, 0.5), sigma_ground_v=sg)
    _, _, _, hd = _assert_exact(p, frames)
    assert hd.dp_variant == S.DP_PAIR2D_DENSE


def test_camera_derived_ground_slope_exact():
    """ground_slope <= 0: alpha = B cos(theta) / H_cam, theta = atan((c_y -
    v_hor) / f) (L#21), computed on both sides independently."""
    H, W, D = 440, 1024, 128
    p = mp.make(ground_slope=0.0, focal_px=1200.0, baseline_m=0.5, camera_height_m=1.5,
                principal_row=250.0)
    hz = p["horizon_frac"] * H
    th = np.arctan((p["principal_row"] - hz) / p["focal_px"])
    alpha = float(p["baseline_m"] * np.cos(th) / p["camera_height_m"])
    frames = np.stack([synth.render(synth.random_scene(2950 + i, W, H, D, alpha=alpha), 2950 + i)
                       for i in range(2)])
    _assert_exact(p, frames)


def test_deterministic_bytes():
    import torch
    from paper_1610_04124_b200 import stixels as S
    frames = _frames_c2(2)
    p = mp.make()
    params = S.params_from_dict(p, 440)
    hd = S.Handle(params, 1024, 440, 2)
    t = torch.from_numpy(frames.view(np.int16)).cuda()
    o1, c1, k1 = hd.alloc_outputs(2)
    o2, c2, k2 = hd.alloc_outputs(2)
    o1.zero_(); o2.zero_()
    hd.compute(t, o1, c1, k1)
    hd.compute(t, o2, c2, k2)
    hd.sync()
    assert torch.equal(o1, o2) and torch.equal(c1, c2) and torch.equal(k1, k2)


@pytest.mark.parametrize("fmt,mode,W,s", [("u16", 0, 1027, 5), ("u16", 1, 1024, 5), ("u8", 0, 1040, 3),
                                          ("f32", 0, 333, 7), ("u16", 1, 128, 13)])
def test_stage_calls_equal_compute(fmt, mode, W, s):
    """The stage entry points (stixels_reduce -> stixels_solve) give the same bytes
    as stixels_compute, and both equal the oracle (exact mode), per input format
    and reduction."""
    import torch
    from paper_1610_04124_b200 import stixels as S
    H, D = 120, 128
    rng = np.random.default_rng(77 + s)
    base = _frames_c2(2, seed0=2300, W=W, H=H)
    if fmt == "u8":
        f = (base >> 4).astype(np.uint8)
        f[base == 0xFFFF] = 255
        p = mp.make(stixel_width=s, reduce_mode=mode, disp_frac_bits=0, invalid_value=255)
    elif fmt == "f32":
        f = np.where(base == 0xFFFF, np.nan, base.astype(np.float32) / 16.0).astype(np.float32)
        f[rng.random(f.shape) < 0.01] = -1.0
        p = mp.make(stixel_width=s, reduce_mode=mode, disp_format=S.F32)
    else:
        f = base
        p = mp.make(stixel_width=s, reduce_mode=mode)
    g, gc, cnt, hd = run_gpu(p, f)
    assert hd.last_launch_count() == 2
    # the stage calls on the same handle
    B = f.shape[0]
    t = torch.from_numpy(f.view(np.int16) if f.dtype == np.uint16 else f).cuda()
    cols = torch.empty((B, hd.n_cols, H), dtype=torch.int16, device="cuda")
    out, cnt2, cost2 = hd.alloc_outputs(B)
    hd.reduce(t, cols)
    hd.solve(cols, out, cnt2, cost2)
    hd.sync()
    g2 = S.decode(out.cpu().numpy(), cnt2.cpu().numpy())
    assert g2 == g
    assert (cost2.cpu().numpy() == gc).all()
    o, oc = run_oracle(p, f)
    bad = compare_exact(g, gc, o, oc, p["cost_frac_bits"])
    assert not bad, f"{len(bad)} mismatching columns, first: {bad[:2]}"


@pytest.mark.parametrize("fmt", ["u16", "u8", "f32"])
@pytest.mark.parametrize("s", [3, 5, 7, 10])
@pytest.mark.parametrize("pad", [0, 48])
def test_reduce_rows_kernel_bit_exact(fmt, s, pad):
    """The row-wise register reduction (reduce_rows_kernel: s in {3, 5, 7, 10}, 16-byte
    aligned frames), bit-exact against the oracle for mean and median: widths whose
    last column group overruns a tight row (element loads), padded rows (pitch >
    W bpp), ragged tails, invalid / out-of-range / negative / NaN pixels."""
    import torch
    from oracle import oracle as orc
    from paper_1610_04124_b200 import stixels as S
    H, D = 70, 64
    bpp = {"u16": 2, "u8": 1, "f32": 4}[fmt]
    W = (16 * 37) // bpp + s - 1                     # a multiple of 16 bytes + a ragged tail
    W -= ((W * bpp) % 16) // bpp                     # tight rows: W bpp a multiple of 16
    rng = np.random.default_rng(100 * s + bpp + pad)
    Wp = W + pad // bpp                              # padded row (pitch)
    if fmt == "u16":
        full = rng.integers(0, (D + 2) * 16, size=(2, H, Wp)).astype(np.uint16)
        full[rng.random(full.shape) < 0.1] = 0xFFFF
        kw = dict(invalid_value=0xFFFF, disp_frac_bits=4)
        dev = torch.from_numpy(full.view(np.int16)).cuda()
    elif fmt == "u8":
        full = rng.integers(0, 256, size=(2, H, Wp)).astype(np.uint8)
        kw = dict(invalid_value=255, disp_frac_bits=2, disp_format=S.U8)
        dev = torch.from_numpy(full).cuda()
    else:
        full = (rng.random((2, H, Wp)) * (D + 2) - 1).astype(np.float32)
        full[rng.random(full.shape) < 0.05] = np.nan
        kw = dict(disp_format=S.F32)
        dev = torch.from_numpy(full).cuda()
    f = np.ascontiguousarray(full[:, :, :W])
    assert (Wp * bpp) % 16 == 0
    for mode in (0, 1):
        p = mp.make(max_disparity=D, stixel_width=s, reduce_mode=mode, **kw)
        hd = S.Handle(S.params_from_dict(p, H), W, H, 2)
        cols = torch.empty((2, hd.n_cols, H), dtype=torch.int16, device="cuda")
        hd.reduce(dev, cols, row_pitch_bytes=Wp * bpp)
        hd.sync()
        got = cols.cpu().numpy().view(np.uint16).astype(np.int32)
        got[got == 0xFFFF] = -1
        for b in range(2):
            if fmt == "f32":
                want = orc.reduce(f[b], s, 0, 0, D, mode=mode)
            else:
                want = orc.reduce(f[b], s, kw["disp_frac_bits"], kw["invalid_value"], D, mode=mode)
            assert (got[b] == want).all(), (mode, b, np.argwhere(got[b] != want)[:3])
        hd.destroy()


@pytest.mark.parametrize("fmt", ["u16", "u8", "f32"])
@pytest.mark.parametrize("s", [5, 7])
@pytest.mark.parametrize("pad", [0, 48])
def test_reduce_strip_kernel_bit_exact(fmt, s, pad):
    """The strip reduction (reduce_strip_kernel: whole rows streamed into shared
    memory by bulk copies, used when a batch has >= 4 strips of 32 rows per SM),
    bit-exact against the oracle for mean and median on 240 frames of 70 rows (a
    ragged 6-row last strip), tight and padded rows, invalid / out-of-range / NaN
    pixels, integer sentinels below and above the range limit."""
    import torch
    from oracle import oracle as orc
    from paper_1610_04124_b200 import stixels as S
    H, D, B = 70, 64, 240
    bpp = {"u16": 2, "u8": 1, "f32": 4}[fmt]
    W = (16 * 37) // bpp + s - 1
    W -= ((W * bpp) % 16) // bpp
    rng = np.random.default_rng(7 * s + bpp + pad)
    Wp = W + pad // bpp
    if fmt == "u16":
        full = rng.integers(0, (D + 2) * 16, size=(B, H, Wp)).astype(np.uint16)
        full[rng.random(full.shape) < 0.1] = 0xFFFF
        kws = [dict(invalid_value=0xFFFF, disp_frac_bits=4), dict(invalid_value=7, disp_frac_bits=4)]
        dev = torch.from_numpy(full.view(np.int16)).cuda()
    elif fmt == "u8":
        full = rng.integers(0, 256, size=(B, H, Wp)).astype(np.uint8)
        kws = [dict(invalid_value=255, disp_frac_bits=2, disp_format=S.U8),
               dict(invalid_value=3, disp_frac_bits=2, disp_format=S.U8)]
        dev = torch.from_numpy(full).cuda()
    else:
        full = (rng.random((B, H, Wp)) * (D + 2) - 1).astype(np.float32)
        full[rng.random(full.shape) < 0.05] = np.nan
        kws = [dict(disp_format=S.F32)]
        dev = torch.from_numpy(full).cuda()
    f = np.ascontiguousarray(full[:, :, :W])
    for kw in kws:
        for mode in (0, 1):
            p = mp.make(max_disparity=D, stixel_width=s, reduce_mode=mode, **kw)
            hd = S.Handle(S.params_from_dict(p, H), W, H, B)
            cols = torch.empty((B, hd.n_cols, H), dtype=torch.int16, device="cuda")
            hd.reduce(dev, cols, row_pitch_bytes=Wp * bpp)
            hd.sync()
            got = cols.cpu().numpy().view(np.uint16).astype(np.int32)
            got[got == 0xFFFF] = -1
            for b in range(0, B, 7):
                if fmt == "f32":
                    want = orc.reduce(f[b], s, 0, 0, D, mode=mode)
                else:
                    want = orc.reduce(f[b], s, kw["disp_frac_bits"], kw["invalid_value"], D, mode=mode)
                assert (got[b] == want).all(), (kw, mode, b, np.argwhere(got[b] != want)[:3])
            hd.destroy()


def test_reduce_strip_kernel_short_frames():
    """The strip reduction on frames shorter than one strip (20 rows: every strip
    is a ragged one) over 640 frames, u16 with an even number of 16-byte units per
    row (the shared-memory row stride then gets its 16-byte pad): bit-exact."""
    import torch
    from oracle import oracle as orc
    from paper_1610_04124_b200 import stixels as S
    H, D, B, s = 20, 64, 640, 5
    W = 160                                            # 320 bytes = 20 units of 16
    rng = np.random.default_rng(4242)
    full = rng.integers(0, (D + 2) * 16, size=(B, H, W)).astype(np.uint16)
    full[rng.random(full.shape) < 0.1] = 0xFFFF
    p = mp.make(max_disparity=D, stixel_width=s, invalid_value=0xFFFF, disp_frac_bits=4)
    hd = S.Handle(S.params_from_dict(p, H), W, H, B)
    cols = torch.empty((B, hd.n_cols, H), dtype=torch.int16, device="cuda")
    hd.reduce(torch.from_numpy(full.view(np.int16)).cuda(), cols, row_pitch_bytes=W * 2)
    hd.sync()
    got = cols.cpu().numpy().view(np.uint16).astype(np.int32)
    got[got == 0xFFFF] = -1
    for b in range(0, B, 37):
        want = orc.reduce(full[b], s, 4, 0xFFFF, D)
        assert (got[b] == want).all(), (b, np.argwhere(got[b] != want)[:3])
    hd.destroy()


@pytest.mark.parametrize("D,q", [(64, 4), (256, 8)])
def test_top_of_range_pixels_exact(D, q):
    """L#27: pixels in [D - 1/2, D) keep their value for the ground and sky terms
    and are clamped below D - 1/2 only by the object model (its LUT index and span
    mean); at D = 256 with 8 fractional bits the 16-bit top value is 0xFFFE.
    Exact against the oracle on frames whose objects sit at the top of the range."""
    H, W = 96, 160
    rng = np.random.default_rng(31 + D)
    top = (D << q) - 1
    f = rng.integers((D - 2) << q, top + 1, size=(2, H, W)).astype(np.uint16)   # in [D-2, D)
    f[:, : H // 3] = rng.integers(0, 4 << q, size=(2, H // 3, W))               # a low band
    f[rng.random(f.shape) < 0.05] = 0xFFFF if q < 8 else 0                       # invalid
    f[:, :, :20] = top                                                           # d' = D - 2^-q
    p = mp.make(max_disparity=D, disp_frac_bits=q, invalid_value=0xFFFF if q < 8 else 0,
                ground_slope=D / (2.0 * H), cost_frac_bits=10 if D > 128 else 11)
    _assert_exact(p, f)


def test_launch_plan_api():
    """stixels_set_launch_plan / stixels_query_launch: the shape is 0 before the
    first launch, a forced plan is reported back, other values are ARG errors."""
    from paper_1610_04124_b200 import stixels as S
    frames = _frames_c2(1, seed0=2200, W=320, H=120)
    p = mp.make()
    hd = S.Handle(S.params_from_dict(p, 120), 320, 120, 1)
    assert hd.last_launch_shape() == (0, 0)
    for bad in (1, 5, 16, -4):
        with pytest.raises(S.StixelsError):
            hd.set_launch_plan(bad)
    hd.destroy()
    for plan in (4, 8):
        _, _, _, h2 = run_gpu(p, frames, plan=plan)
        assert h2.last_launch_shape()[0] == plan
