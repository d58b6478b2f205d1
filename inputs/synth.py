"""Seeded synthetic disparity scenes -- the ONLY module shared by the oracle side
and the CUDA side (it generates inputs; it contains none of the method's
arithmetic: no reduction, no cost, no DP).

Scene recipe: a road scene as the paper's
workload ("images including cars, pedestrians, trees, and traffic
signals", P:255 SGM disparities): a ground plane whose disparity grows linearly
below the horizon row, fronto-parallel boxes standing on the ground (nearest
wins), sky (disparity 0, half of it invalid), Gaussian noise, uniform outliers
and randomly invalid pixels.  Disparities are stored as u16 fixed point with
`q_bits` fractional bits; invalid pixels hold `invalid`.

Everything is drawn from numpy's PCG64 seeded per (config, frame) so the same
bytes feed both the oracle and the GPU path.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

INVALID_U16 = 0xFFFF


@dataclass
class Box:
    x0: int          # first image column (inclusive)
    x1: int          # last image column (exclusive)
    base_row: int    # image row of the box's bottom edge (standing on the ground)
    height: int      # rows
    disp: float      # disparity (= ground disparity at base_row)


@dataclass
class Scene:
    W: int
    H: int
    D: int
    alpha: float
    horizon_row: float
    boxes: list = field(default_factory=list)
    noise_sigma: float = 0.5
    outlier_frac: float = 0.02
    invalid_frac: float = 0.05
    sky_invalid_frac: float = 0.5
    q_bits: int = 4


def ground_disparity_image_row(alpha: float, horizon_row: float, r: np.ndarray) -> np.ndarray:
    """Scene geometry: a flat road seen by a level camera has disparity
    alpha * (r - horizon_row) at image row r (0 = top), zero at and above the
    horizon."""
    return np.maximum(0.0, alpha * (r - horizon_row))


def random_scene(seed: int, W: int, H: int, D: int, alpha: float = 0.4,
                 horizon_frac: float = 0.3, n_boxes=(6, 20), min_w: int = 10,
                 max_w: int = 150, **kw) -> Scene:
    """Random ground-standing boxes: column span 10-150 px, height uniform in
    [10, base row] rows, base row uniform below the horizon."""
    rng = np.random.Generator(np.random.PCG64(seed))
    horizon_row = horizon_frac * H
    sc = Scene(W=W, H=H, D=D, alpha=alpha, horizon_row=horizon_row, **kw)
    nb = int(rng.integers(n_boxes[0], n_boxes[1] + 1))
    r_min = int(np.ceil(horizon_row)) + 2
    if r_min >= H:          # degenerate (tiny) frames: no room for boxes
        nb = 0
    for _ in range(nb):
        w = int(rng.integers(min(min_w, W), min(max_w, W) + 1))
        x0 = int(rng.integers(0, max(1, W - w + 1)))
        base = int(rng.integers(r_min, H))
        hgt = int(rng.integers(min(10, base), base + 1))
        disp = float(ground_disparity_image_row(alpha, horizon_row, np.array([base]))[0])
        sc.boxes.append(Box(x0, x0 + w, base, hgt, disp))
    return sc


def c1_scene() -> Scene:
    """C1: 64x48, D=32, flat ground + 2 box obstacles + sky (BASELINE configs[0])."""
    H, W, D = 48, 64, 32
    alpha = 0.6
    horizon_row = 0.3 * H
    sc = Scene(W=W, H=H, D=D, alpha=alpha, horizon_row=horizon_row)
    for (x0, x1, base, hgt) in ((10, 25, 40, 14), (40, 55, 30, 10)):
        disp = float(ground_disparity_image_row(alpha, horizon_row, np.array([base]))[0])
        sc.boxes.append(Box(x0, x1, base, hgt, disp))
    return sc


def clean_disparity(sc: Scene) -> np.ndarray:
    """Noise-free float disparity [H][W]; NaN marks sky."""
    r = np.arange(sc.H, dtype=np.float64)[:, None]
    d = np.broadcast_to(ground_disparity_image_row(sc.alpha, sc.horizon_row, r),
                        (sc.H, sc.W)).copy()
    d[np.arange(sc.H) <= sc.horizon_row, :] = np.nan        # sky above the horizon
    for b in sc.boxes:
        r0 = max(0, b.base_row - b.height + 1)
        blk = d[r0:b.base_row + 1, b.x0:b.x1]
        nearer = np.isnan(blk) | (blk <= b.disp)            # nearest wins
        blk[nearer] = b.disp
    return d


def gt_labels(sc: Scene) -> np.ndarray:
    """Ground-truth label map [H][W] of the scene (for the NEXT f3 quality
    metrics): -1 = ground, -2 = sky, k >= 0 = the box k visible at that pixel
    (the same nearest-wins painting as clean_disparity)."""
    r = np.arange(sc.H, dtype=np.float64)[:, None]
    d = np.broadcast_to(ground_disparity_image_row(sc.alpha, sc.horizon_row, r),
                        (sc.H, sc.W)).copy()
    sky = np.broadcast_to(np.arange(sc.H)[:, None] <= sc.horizon_row, (sc.H, sc.W))
    d[sky] = np.nan
    lab = np.where(sky, -2, -1).astype(np.int32)
    for k, b in enumerate(sc.boxes):
        r0 = max(0, b.base_row - b.height + 1)
        blk = d[r0:b.base_row + 1, b.x0:b.x1]
        nearer = np.isnan(blk) | (blk <= b.disp)
        blk[nearer] = b.disp
        lab[r0:b.base_row + 1, b.x0:b.x1][nearer] = k
    return lab


def render(sc: Scene, seed: int, noise: bool = True) -> np.ndarray:
    """u16 fixed-point disparity image [H][W] with `q_bits` fractional bits."""
    rng = np.random.Generator(np.random.PCG64(seed ^ 0x5EED))
    d = clean_disparity(sc)
    sky = np.isnan(d)
    d = np.where(sky, 0.0, d)
    invalid = np.zeros(d.shape, bool)
    if noise:
        d = d + rng.normal(0.0, sc.noise_sigma, d.shape)
        out_mask = rng.random(d.shape) < sc.outlier_frac
        d = np.where(out_mask, rng.uniform(0, sc.D, d.shape), d)
        invalid |= rng.random(d.shape) < sc.invalid_frac
        invalid |= sky & (rng.random(d.shape) < sc.sky_invalid_frac)
    Q = 1 << sc.q_bits
    u = np.clip(np.rint(d * Q), 0, sc.D * Q - 1).astype(np.uint16)
    u[invalid] = INVALID_U16
    return u


def uniform_random_image(seed: int, W: int, H: int, D: int, q_bits: int = 4,
                         invalid_frac: float = 0.05) -> np.ndarray:
    """Stress variant: uniform random disparities over [0, D) (widens the range of
    object means a column can produce)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    u = rng.integers(0, D << q_bits, size=(H, W)).astype(np.uint16)
    u[rng.random((H, W)) < invalid_frac] = INVALID_U16
    return u


def frame(cfg_id: int, index: int, W: int, H: int, D: int, alpha: float = 0.4,
          **kw) -> np.ndarray:
    """Frame `index` of config `cfg_id`: seed = 1000*cfg + frame."""
    seed = 1000 * cfg_id + index
    sc = random_scene(seed, W, H, D, alpha=alpha, **kw)
    return render(sc, seed)


def frames(cfg_id: int, n: int, W: int, H: int, D: int, alpha: float = 0.4, **kw) -> np.ndarray:
    return np.stack([frame(cfg_id, i, W, H, D, alpha, **kw) for i in range(n)])
