"""Seeded synthetic stereo MRFs for the BASELINE configurations.

The paper's Tsukuba pair is not available, so the benchmark and parity
workloads are seeded random-dot stereograms with a piecewise-constant planted
disparity (BASELINE.json configs):

* disparity: zeros, then 8 axis-aligned rectangles whose corners are uniform
  on the grid, each with a uniform integer disparity in [0, min(15, M-1)];
  later rectangles overwrite earlier ones;
* left image: uniform integers in [0, 255];
* right image: R(r, c) = L(r, c + d(r, c)) inside the frame, fresh noise
  outside it -- a restatement of the reference ``random_dot_pair``
  (``stereo.py:157-183``, checked bit-for-bit against it by the golden
  fixtures) -- plus Gaussian noise N(0, sigma^2), rounded and clipped;
* unaries: the reference stereo field (``stereo.py:82-99,120-125``) on
  right-image pixels, ``exp(-beta * min(|R(r,c) - L(r,c+x)|, T_u))`` with
  out-of-frame hypotheses at the full penalty; log unaries analytic.
  BASELINE uses beta = 0.1 untruncated, i.e. T_u = 255 (F7).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .model import GridMrf, sparse_from_dense, truncated_linear_potential

__all__ = [
    "rect_disparity",
    "random_dot_pair",
    "noisy_stereo_pair",
    "stereo_unary_field",
    "StereoConfig",
    "CONFIGS",
    "build_config_model",
    "quadratic_potential",
]


def rect_disparity(height: int, width: int, M: int, rng: np.random.Generator,
                   n_rects: int = 8, dmax: int = 15) -> np.ndarray:
    disp = np.zeros((height, width), dtype=np.int64)
    top = min(dmax, M - 1)
    for _ in range(n_rects):
        r0, r1 = np.sort(rng.integers(0, height + 1, size=2))
        c0, c1 = np.sort(rng.integers(0, width + 1, size=2))
        disp[r0:r1, c0:c1] = int(rng.integers(0, top + 1))
    return disp


def random_dot_pair(height: int, width: int, disparity, seed: int = 0, levels: int = 256):
    """(left, right) uint8 arrays; same RNG draws as the reference."""
    if not 2 <= levels <= 256:
        raise ValueError(f"levels must be in [2, 256], got {levels}")
    rng = np.random.default_rng(seed)
    step = 256 // levels
    left = (rng.integers(0, levels, size=(height, width)) * step).astype(np.uint8)
    d = np.broadcast_to(np.asarray(disparity, dtype=np.int64), (height, width))
    if d.min() < 0:
        raise ValueError("planted disparities must be nonnegative")
    src_col = np.arange(width)[None, :] + d
    right = (rng.integers(0, levels, size=(height, width)) * step).astype(np.uint8)
    ok = src_col < width
    rr, cc = np.nonzero(ok)
    right[rr, cc] = left[rr, src_col[rr, cc]]
    return left, right


def noisy_stereo_pair(height: int, width: int, M: int, sigma: float, seed: int):
    """Planted-disparity pair with Gaussian sensor noise on the right image."""
    disp = rect_disparity(height, width, M, np.random.default_rng(seed))
    left, right = random_dot_pair(height, width, disp, seed=seed + 1)
    if sigma > 0:
        noise = np.random.default_rng(seed + 2).normal(0.0, sigma, size=(height, width))
        right = np.clip(np.rint(right.astype(np.float64) + noise), 0, 255).astype(np.uint8)
    return left, right, disp


def stereo_unary_field(left: np.ndarray, right: np.ndarray, M: int, beta: float,
                       T_u: float):
    """(N, M) unaries and their analytic logs over right-image pixels."""
    if left.shape != right.shape:
        raise ValueError(f"image dimensions differ: left {left.shape}, right {right.shape}")
    h, w = right.shape
    L = left.astype(np.int64)
    R = right.astype(np.int64)
    energy = np.full((h, w, M), beta * T_u, dtype=np.float64)
    for x in range(min(M, w)):
        diff = np.abs(R[:, : w - x] - L[:, x:]).astype(np.float64)
        energy[:, : w - x, x] = beta * np.minimum(diff, T_u)
    flat = energy.reshape(-1, M)
    return np.exp(-flat), -flat


def quadratic_potential(M: int, alpha: float, cap: float):
    """exp(-alpha * min(d^2, cap)) in sparse form, floor taken from the table
    itself (``fbar = table[0, -1]``; SURVEY a8 pitfall: math.exp != np.exp)."""
    d = np.abs(np.arange(M)[:, None] - np.arange(M)[None, :]).astype(np.float64)
    table = np.exp(-alpha * np.minimum(d * d, cap))
    return sparse_from_dense(table, fbar=table[0, -1])


@dataclass(frozen=True)
class StereoConfig:
    name: str
    height: int
    width: int
    M: int
    potential: str          # "linear" | "quadratic"
    alpha: float
    T: float                # truncation (reference T; m = 2*ceil(T) - 1)
    iters: int
    domains: tuple
    sigma: float = 5.0
    beta: float = 0.1
    T_u: float = 255.0

    @property
    def n_directed(self) -> int:
        H, W = self.height, self.width
        return 2 * (H * (W - 1) + W * (H - 1))

    def build_potential(self):
        if self.potential == "linear":
            return truncated_linear_potential(self.M, self.alpha, self.T)
        return quadratic_potential(self.M, self.alpha, self.T)


# BASELINE.json configs (H x W; BASELINE writes W x H).  Reference T values
# follow SURVEY F3: BASELINE's band |d| <= T maps to reference |d| < T.
CONFIGS = {
    "C1": StereoConfig("C1", 48, 64, 16, "linear", 1.0, 2.0, 10, ("sum",)),
    "C2": StereoConfig("C2", 288, 384, 32, "linear", 0.5, 3.0, 50, ("sum", "max")),
    "C3": StereoConfig("C3", 768, 1024, 64, "quadratic", 0.2, 16.0, 100, ("max",),
                       sigma=10.0),
    "C4": StereoConfig("C4", 1536, 2048, 128, "linear", 0.5, 8.0, 100, ("sum",)),
}
for _T in (2, 5, 9, 17, 33):
    CONFIGS[f"C5_T{_T}"] = StereoConfig(f"C5_T{_T}", 1024, 1024, 256, "linear", 0.5,
                                        float(_T), 20, ("sum", "max"))


def build_config_model(cfg: StereoConfig, seed: int = 0, height: int | None = None,
                       width: int | None = None) -> GridMrf:
    """Seeded stereo grid model for a config (optionally at a reduced size)."""
    H = cfg.height if height is None else height
    W = cfg.width if width is None else width
    left, right, _ = noisy_stereo_pair(H, W, cfg.M, cfg.sigma, seed)
    unaries, log_unaries = stereo_unary_field(left, right, cfg.M, cfg.beta, cfg.T_u)
    return GridMrf(H, W, cfg.M, unaries, cfg.build_potential(), log_unaries=log_unaries)


def config_values(cfg: StereoConfig, domain: str, seed: int = 0, r0: int = 0,
                  rows: int | None = None) -> np.ndarray:
    """(rows*W, M) f64 unaries (sum) or analytic log unaries (max) of a row
    range.  A pixel's unary depends only on its own image row, so a strip
    is computed without the rest of the grid."""
    rows = cfg.height - r0 if rows is None else rows
    left, right, _ = noisy_stereo_pair(cfg.height, cfg.width, cfg.M, cfg.sigma, seed)
    u, lu = stereo_unary_field(left[r0:r0 + rows], right[r0:r0 + rows], cfg.M, cfg.beta, cfg.T_u)
    return u if domain == "sum" else lu


class StripModel:
    """Minimal model view for one strip of a config grid: geometry and the
    shared potential, no full-grid unary table (the engine takes the strip's
    values explicitly)."""

    def __init__(self, cfg: StereoConfig):
        self.M = cfg.M
        self.grid_shape = (cfg.height, cfg.width)
        self.shared_potential = cfg.build_potential()
        H, W = cfg.height, cfg.width
        self.n_edges = H * (W - 1) + W * (H - 1)
        self.n_nodes = H * W
