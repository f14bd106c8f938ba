"""Host-side planning: reference potential -> device kernel descriptor.

Mirrors ``_grid_setup`` / ``_oriented_arrays`` (reference bp.py:443-489):
orientation 0 is the stored potential (L->R and T->B passes), orientation 1
its transpose; the fast sum update uses ``col_residuals`` with floor
``fbar``, fast max-sum the log twin's ``col_values`` with floor ``ln fbar``,
the pruned update ``col_values`` without a floor, the standard update the
dense table.

Kernel choice:
* BAND  -- both orientations are Toeplitz bands: every stored entry of
  offset d = x_i - x_j carries the same weight and is present in every
  column where x_j + d is a label (the truncated linear / quadratic
  families).  Weights travel as kernel parameters; cost O((2R+1) M).
* ELL   -- any other CSC potential: per-column lists padded to m_max.
* DENSE -- the reference "standard" O(M^2) update (comparison kernel).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib as L

__all__ = ["PotentialPlan", "plan_potential", "toeplitz_band", "madds_per_update"]

MAX_BAND_R = L.SBP_MAX_R


@dataclass
class PotentialPlan:
    kind: int
    domain: str
    kernel: str
    floor_term: int
    M: int
    Ms: int
    fbar: tuple = (0.0, 0.0)
    R: int = 0
    band_w: np.ndarray | None = None        # (2, 2R+1) f64
    m_max: int = 0
    ell_idx: np.ndarray | None = None       # (2, m_max, Ms) int32
    ell_w: np.ndarray | None = None         # (2, m_max, Ms) f64
    dense_t: np.ndarray | None = None       # (2, Ms, Ms) f64, f(x_i=k, x_j=x) at [o, k, x]
    madds_per_update: int = 0
    # per-edge potentials (n_pot > 0): ell_idx / ell_w are (n_pot, 2, m_max, Ms)
    n_pot: int = 0
    fbar_all: np.ndarray | None = None      # (n_pot, 2)
    pid_h: np.ndarray | None = None         # (H*W,) int32, potential of edge (n, n+1)
    pid_v: np.ndarray | None = None         # (H*W,) int32, potential of edge (n, n+W)
    madds_per_sweep: int | None = None      # per-edge: the reference counter summed over edges
    accumulate: int = 0                     # SBP_ACC_F64: f64 sum-product (ELL kind)
    fbar64: tuple = (0.0, 0.0)
    device_arrays: list = field(default_factory=list)

    @property
    def kind_name(self) -> str:
        return {L.SBP_POT_BAND: "band", L.SBP_POT_ELL: "ell", L.SBP_POT_DENSE: "dense"}[self.kind]


def _is_sparse(p) -> bool:
    return hasattr(p, "col_indptr") and hasattr(p, "col_values")


def _dense_table(p) -> np.ndarray:
    return p.densify().table if _is_sparse(p) else np.asarray(p.table, dtype=np.float64)


def toeplitz_band(indptr, indices, weights, M: int, pad: float):
    """(R, w[2R+1]) when the CSC lists form a full Toeplitz band, else None.

    Offsets with no stored entry get ``pad`` (a stored-weight of exactly 0 in
    the sum domain, -inf in the max domain): both are exact no-ops.
    """
    indptr = np.asarray(indptr, dtype=np.int64)
    indices = np.asarray(indices, dtype=np.int64)
    weights = np.asarray(weights, dtype=np.float64)
    if indices.size == 0:
        return 0, np.array([pad])
    cols = np.repeat(np.arange(M, dtype=np.int64), np.diff(indptr))
    d = indices - cols
    R = int(np.abs(d).max())
    w = np.full(2 * R + 1, pad, dtype=np.float64)
    order = np.argsort(d, kind="stable")
    ds, ws = d[order], weights[order]
    uniq, start, count = np.unique(ds, return_index=True, return_counts=True)
    for dv, s0, n in zip(uniq, start, count):
        if n != M - abs(int(dv)):
            return None
        vals = ws[s0:s0 + n]
        if not (vals == vals[0]).all() or np.isnan(vals[0]):
            return None
        w[dv + R] = vals[0]
    return R, w


def madds_per_update(pot, kernel: str, M: int) -> int:
    """The reference kernel madd counter per directed update
    (numba_kernels.py:290-292, 313-315, 336-338)."""
    if kernel == "standard":
        return M * M
    nnz = int(pot.col_indptr[-1])
    return nnz + 2 * M if kernel == "fast" else nnz


def _ell(sp_list, Ms: int, pad: float):
    m_max = max(int(np.diff(np.asarray(sp.col_indptr)).max(initial=0)) for sp, _ in sp_list)
    m_max = max(m_max, 1)
    idx = np.zeros((2, m_max, Ms), dtype=np.int32)
    w = np.full((2, m_max, Ms), pad, dtype=np.float64)
    for o, (sp, wts) in enumerate(sp_list):
        indptr = np.asarray(sp.col_indptr, dtype=np.int64)
        lens = np.diff(indptr)
        cols = np.repeat(np.arange(len(lens)), lens)
        k = np.arange(indptr[-1]) - indptr[cols]
        idx[o, k, cols] = np.asarray(sp.col_indices)
        w[o, k, cols] = np.asarray(wts)
    return m_max, idx, w


def _oriented_lists(pot, domain: str, kernel: str, M: int):
    """[(indptr, indices, weights, fbar)] for orientations 0 and 1 (bp.py:443-463)."""
    pad = 0.0 if domain == "sum" else -np.inf
    use = pot.to_log() if domain == "max" else pot
    if kernel == "standard":
        table = _dense_table(use)
        out = []
        for t in (table, table.T):           # f_o(x_i = k, x_j = x) at [k][x]
            indptr = np.arange(M + 1, dtype=np.int64) * M
            indices = np.tile(np.arange(M, dtype=np.int64), M)
            out.append((indptr, indices, np.ascontiguousarray(t.T).ravel(), 0.0))
        return out, pad
    if not _is_sparse(use):
        raise TypeError(f"kernel={kernel!r} requires SparseTruncatedPotential, "
                        f"got {type(pot).__name__}")
    out = []
    for sp in (use, use.transpose()):
        if kernel == "fast":
            w = sp.col_residuals if domain == "sum" else sp.col_values
        else:
            w = sp.col_values
        out.append((np.asarray(sp.col_indptr), np.asarray(sp.col_indices), np.asarray(w),
                    float(sp.fbar)))
    return out, pad


def plan_per_edge(model, domain: str, kernel: str, M: int, Ms: int) -> PotentialPlan:
    """Per-edge (inhomogeneous) potentials -- the reference's generic engine
    (bp.py:506-584): unique potentials (by object identity, in edge order),
    both orientations each, ELL arrays stacked, one potential id per edge."""
    H, W = model.grid_shape
    uid: dict = {}
    unique = []
    pid_h = np.full(H * W, -1, dtype=np.int32)
    pid_v = np.full(H * W, -1, dtype=np.int32)
    from .model import canonical_edge_potentials, grid_edges
    edges = grid_edges(H, W)
    pots = canonical_edge_potentials(model)
    for (a, b), pot in zip(edges, pots):
        k = uid.setdefault(id(pot), len(unique))
        if k == len(unique):
            unique.append(pot)
        if b - a == 1 and W > 1:
            pid_h[a] = k
        else:
            pid_v[a] = k
    lists = []
    pad = 0.0
    for pot in unique:
        ol, pad = _oriented_lists(pot, domain, kernel, M)
        lists.append(ol)
    m_max = max(1, max(int(np.diff(l[0]).max(initial=0)) for ol in lists for l in ol))
    U = len(unique)
    idx = np.zeros((U, 2, m_max, Ms), dtype=np.int32)
    w = np.full((U, 2, m_max, Ms), pad, dtype=np.float64)
    fb = np.zeros((U, 2), dtype=np.float64)
    for u, ol in enumerate(lists):
        for o, (indptr, indices, wts, fbar) in enumerate(ol):
            lens = np.diff(indptr)
            cols = np.repeat(np.arange(len(lens)), lens)
            kk = np.arange(indptr[-1]) - indptr[cols]
            idx[u, o, kk, cols] = indices
            w[u, o, kk, cols] = wts
            fb[u, o] = fbar
    per_sweep = 0
    for pot in pots:
        per_sweep += 2 * (M * M if kernel == "standard" else madds_per_update(pot, kernel, M))
    kind = L.SBP_POT_DENSE if kernel == "standard" else L.SBP_POT_ELL
    return PotentialPlan(kind, L.SBP_SUM if domain == "sum" else L.SBP_MAX, kernel,
                         0 if kernel != "fast" else 1, M, Ms, (0.0, 0.0), m_max=m_max,
                         ell_idx=idx, ell_w=w, n_pot=U, fbar_all=fb, pid_h=pid_h, pid_v=pid_v,
                         madds_per_update=0, madds_per_sweep=per_sweep)


# effective band width above which sum-product accumulates in f64 (auto)
ACC64_MIN_EFFECTIVE_TAPS = 12.0


def effective_taps(pot) -> float:
    """Mean over columns of sum(residuals) / max(residual): how many stored
    entries carry weight comparable to the largest.  Truncated linear
    alpha=0.5 (every BASELINE config): ~4; alpha=0.1, T=33: ~19."""
    indptr = np.asarray(pot.col_indptr)
    res = np.abs(np.asarray(pot.col_residuals, dtype=np.float64))
    lens = np.diff(indptr)
    if res.size == 0:
        return 0.0
    cols = np.repeat(np.arange(len(lens)), lens)
    tot = np.bincount(cols, weights=res, minlength=len(lens))
    mx = np.zeros(len(lens))
    np.maximum.at(mx, cols, res)
    ok = mx > 0
    return float((tot[ok] / mx[ok]).mean()) if ok.any() else 0.0


def wants_f64(pot, domain: str, kernel: str, precision: str) -> bool:
    """Accumulation precision of a sum-product run:
    fp32 accumulation drifts past 1e-5 for weak smoothing over wide bands
    (5.1e-5 at alpha=0.1, T=33, M=256, 20 iterations), so those potentials --
    many comparable taps -- accumulate in f64 ("auto"); "f32" / "f64" force."""
    if domain != "sum" or kernel == "standard" or not _is_sparse(pot):
        return False
    if precision == "f64":
        return True
    if precision == "f32":
        return False
    return effective_taps(pot) > ACC64_MIN_EFFECTIVE_TAPS


def plan_potential(pot, domain: str, kernel: str, M: int, Ms: int,
                   allow_band: bool = True, precision: str = "auto") -> PotentialPlan:
    dom = L.SBP_SUM if domain == "sum" else L.SBP_MAX
    pad = 0.0 if domain == "sum" else -np.inf
    use = pot.to_log() if domain == "max" else pot
    if kernel == "standard":
        table = _dense_table(use)
        tabs = (table, table.T)     # orientation o: f_o(x_i = k, x_j = x) at [k][x]
        idx = np.zeros((2, M, Ms), dtype=np.int32)
        w = np.full((2, M, Ms), pad, dtype=np.float64)
        dense = np.full((2, Ms, Ms), pad, dtype=np.float64)
        for o in range(2):
            idx[o] = np.arange(M, dtype=np.int32)[:, None]
            w[o, :, :M] = tabs[o]
            dense[o, :M, :M] = tabs[o]
        return PotentialPlan(L.SBP_POT_DENSE, dom, kernel, 0, M, Ms, (0.0, 0.0), m_max=M,
                             ell_idx=idx, ell_w=w, dense_t=dense, madds_per_update=M * M)
    if not _is_sparse(use):
        raise TypeError(f"kernel={kernel!r} requires SparseTruncatedPotential, "
                        f"got {type(pot).__name__}")
    orients = (use, use.transpose())
    if kernel == "fast":
        weights = [(sp, sp.col_residuals if domain == "sum" else sp.col_values) for sp in orients]
        floor = 1
    else:  # pruned
        weights = [(sp, sp.col_values) for sp in orients]
        floor = 0
    fbar = (float(orients[0].fbar), float(orients[1].fbar))
    madds = madds_per_update(pot, kernel, M)
    if wants_f64(pot, domain, kernel, precision):
        m_max, idx, w = _ell(weights, Ms, pad)
        return PotentialPlan(L.SBP_POT_ELL, dom, kernel, floor, M, Ms, fbar, m_max=m_max,
                             ell_idx=idx, ell_w=w, madds_per_update=madds,
                             accumulate=L.SBP_ACC_F64, fbar64=fbar)
    if allow_band:
        bands = [toeplitz_band(sp.col_indptr, sp.col_indices, wt, M, pad) for sp, wt in weights]
        if all(b is not None for b in bands):
            R = max(b[0] for b in bands)
            # a band runs on the smallest compiled radius >= R below Ms; with
            # none compiled (e.g. Ms = 16, R = 9..15) the general ELL kernel
            # serves it (same arithmetic order, ascending x_i per column)
            if R <= MAX_BAND_R and (R == 0 or L.lib().sbp_band_radius(Ms, R) > 0):
                bw = np.full((2, 2 * R + 1), pad)
                for o, (r, wv) in enumerate(bands):
                    bw[o, R - r:R + r + 1] = wv
                return PotentialPlan(L.SBP_POT_BAND, dom, kernel, floor, M, Ms, fbar, R=R,
                                     band_w=bw, madds_per_update=madds)
    m_max, idx, w = _ell(weights, Ms, pad)
    return PotentialPlan(L.SBP_POT_ELL, dom, kernel, floor, M, Ms, fbar, m_max=m_max,
                         ell_idx=idx, ell_w=w, madds_per_update=madds)
