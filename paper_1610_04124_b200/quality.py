"""Quality metrics of a stixel segmentation against ground truth (NEXT row f3,
SURVEY 8(f); Table 1 of the paper), computed on the host from the
library's output lists.  Host-side evaluation downstream of a7: no part of the
hot path runs here.

Definitions (readings L#25 in DESIGN.md):
- GT object stixels: per reduced column c (image columns [c s, c s + s)), each
  row takes the label of the majority of its s pixels (ties: the lower label
  id); maximal runs of rows with the same box id are the GT stixels.
- Detection rate: a GT stixel is detected iff the pixels it shares with the
  estimated OBJECT stixels of its column exceed 0.5 of its area (strict).
  Rate = detected / total (1.0 when there is no GT stixel).
- False positive: an estimated OBJECT stixel with more than 30 of its pixels
  (rows x s) inside the GT free space of its column -- the ground rows below
  the lowest GT obstacle (all ground rows if the column has none).
Rows are model rows (v = 0 at the bottom, image row = H - 1 - v).
"""
from __future__ import annotations

import numpy as np

OBJECT = 1


def column_labels(labels: np.ndarray, s: int) -> np.ndarray:
    """[H][W] label map -> [n_cols][H] per-reduced-column labels in model row
    order (majority over the s pixels; ties to the smaller label)."""
    H, W = labels.shape
    n = W // s
    out = np.empty((n, H), np.int32)
    for c in range(n):
        band = labels[:, c * s:(c + 1) * s]
        for r in range(H):
            vals, cnt = np.unique(band[r], return_counts=True)
            out[c, H - 1 - r] = vals[np.argmax(cnt)]        # unique() sorts: ties -> smaller
    return out


def gt_stixels(col_labels: np.ndarray):
    """Per column: list of (vb, vt, box_id) runs of object rows."""
    res = []
    for lab in col_labels:
        runs, v = [], 0
        H = len(lab)
        while v < H:
            if lab[v] >= 0:
                t = v
                while t + 1 < H and lab[t + 1] == lab[v]:
                    t += 1
                runs.append((v, t, int(lab[v])))
                v = t + 1
            else:
                v += 1
        res.append(runs)
    return res


def free_space(col_labels: np.ndarray) -> np.ndarray:
    """[n_cols][H] bool: GT ground rows below the lowest obstacle of the column."""
    n, H = col_labels.shape
    fs = np.zeros((n, H), bool)
    for c in range(n):
        obj = np.nonzero(col_labels[c] >= 0)[0]
        top = obj[0] if len(obj) else H
        fs[c, :top] = col_labels[c, :top] == -1
    return fs


def evaluate_frame(est, col_labels: np.ndarray, s: int) -> dict:
    """est: per column list of (vb, vt, cls, disparity) (stixels.decode).
    Returns counts for one frame."""
    gts = gt_stixels(col_labels)
    fs = free_space(col_labels)
    n_gt = det = fp = n_obj = 0
    for c, lst in enumerate(est):
        cover = np.zeros(col_labels.shape[1], bool)
        for (vb, vt, cls, _d) in lst:
            if cls == OBJECT:
                n_obj += 1
                cover[vb:vt + 1] = True
                if int(fs[c, vb:vt + 1].sum()) * s > 30:
                    fp += 1
        for (vb, vt, _k) in gts[c]:
            n_gt += 1
            if 2 * int(cover[vb:vt + 1].sum()) > (vt - vb + 1):     # ratio > 0.5, strict
                det += 1
    return {"n_gt": n_gt, "detected": det, "false_positives": fp, "n_est_objects": n_obj}


def summarize(per_frame: list) -> dict:
    """Table 1 quantities over frames."""
    n_gt = sum(f["n_gt"] for f in per_frame)
    det = sum(f["detected"] for f in per_frame)
    fp = sum(f["false_positives"] for f in per_frame)
    return {"frames": len(per_frame), "detection_rate": det / n_gt if n_gt else 1.0,
            "gt_stixels": n_gt, "detected": det, "total_false_positives": fp,
            "frames_with_fp": sum(1 for f in per_frame if f["false_positives"] > 0),
            "pct_frames_with_fp": 100.0 * sum(1 for f in per_frame if f["false_positives"] > 0)
            / max(1, len(per_frame))}
