"""Host-side model types for the grid BP path (input contract of the engine).

These mirror the reference `sparsebp.mrf` data model closely enough that a
model built here and one built by the reference carry bit-identical arrays
(checked by tests/test_model.py against golden fixtures):

* ``SparseTruncatedPotential`` -- constant floor ``fbar`` plus per-column
  compatible entries in CSC form (reference ``mrf.py:77-201``).
* ``DensePotential`` -- full M x M table (``mrf.py:43-74``).
* ``truncated_linear_potential`` (``mrf.py:207-250``) and
  ``sparse_from_dense`` (``mrf.py:253-285``).
* ``GridMrf`` / ``build_grid_mrf`` -- a 4-connected grid with one shared
  potential (``mrf.py:288-456``).  Unlike the reference it never builds the
  Python edge sets of the topology check (``mrf.py:341-348``, ~60 s at
  2048x1536): the grid topology holds by construction and ``edges`` is
  materialised lazily in the reference's row-major order.

The engine (``engine.py``) accepts these objects or the reference's own
``sparsebp.MrfModel`` interchangeably (duck typing on ``M``, ``grid_shape``,
``unaries``, ``log_unaries``, ``edges``, ``potentials``).
"""

from __future__ import annotations

import math
from typing import Sequence

import numpy as np

__all__ = [
    "DensePotential",
    "SparseTruncatedPotential",
    "truncated_linear_potential",
    "sparse_from_dense",
    "GridMrf",
    "build_grid_mrf",
    "grid_edges",
    "MrfModel",
    "SweepSchedule",
]


def _frozen(a: np.ndarray) -> np.ndarray:
    a.setflags(write=False)
    return a


class DensePotential:
    """Pairwise potential as a full table; ``table[x_i, x_j] = f(x_i, x_j)``."""

    def __init__(self, table):
        t = np.array(table, dtype=np.float64)
        if t.ndim != 2 or t.shape[0] != t.shape[1]:
            raise ValueError(f"potential table must be square, got shape {t.shape}")
        if np.isnan(t).any():
            raise ValueError("potential table contains NaN")
        self.table = _frozen(t)
        self._log = None

    @property
    def M(self) -> int:
        return int(self.table.shape[0])

    def to_log(self) -> "DensePotential":
        if self._log is None:
            with np.errstate(divide="ignore"):
                self._log = DensePotential(np.log(self.table))
        return self._log

    def __repr__(self) -> str:
        return f"DensePotential(M={self.M})"


class SparseTruncatedPotential:
    """Floor ``fbar`` everywhere except the stored compatible entries.

    Column ``x_j`` owns ``col_indices[col_indptr[x_j]:col_indptr[x_j+1]]``
    (strictly increasing x_i) with values ``col_values`` and precomputed
    ``col_residuals = col_values - fbar`` (reference ``mrf.py:127-135``).
    """

    def __init__(self, M: int, fbar: float, col_indptr, col_indices, col_values):
        if M < 1:
            raise ValueError(f"label count must be positive, got {M}")
        fbar = float(fbar)
        if math.isnan(fbar):
            raise ValueError("fbar must not be NaN")
        indptr = np.asarray(col_indptr, dtype=np.int64)
        idx = np.asarray(col_indices, dtype=np.int64)
        vals = np.asarray(col_values, dtype=np.float64)
        if indptr.shape != (M + 1,) or indptr[0] != 0:
            raise ValueError("col_indptr must have length M+1 and start at 0")
        if indptr[-1] != idx.size or idx.size != vals.size:
            raise ValueError("index/value arrays inconsistent with col_indptr")
        if (np.diff(indptr) < 0).any():
            raise ValueError("col_indptr must be nondecreasing")
        if np.isnan(vals).any():
            raise ValueError("potential values contain NaN")
        if idx.size:
            if idx.min() < 0 or idx.max() >= M:
                raise ValueError(f"column references states outside [0, {M})")
            # strictly increasing within each column: every step inside a
            # column must be positive; steps across column starts are free
            step_ok = np.diff(idx) > 0
            starts = indptr[1:-1]
            interior = np.ones(idx.size - 1, dtype=bool)
            interior[starts[(starts > 0) & (starts < idx.size)] - 1] = False
            if not step_ok[interior].all():
                raise ValueError("column indices must be strictly increasing")
        self.M = int(M)
        self.fbar = fbar
        self.col_indptr = _frozen(indptr)
        self.col_indices = _frozen(idx)
        self.col_values = _frozen(vals)
        self.col_residuals = _frozen(vals - fbar)
        self.maxsum_safe = bool((vals >= fbar).all()) if vals.size else True
        self._log = None

    @property
    def nnz(self) -> int:
        return int(self.col_indptr[-1])

    @property
    def m(self) -> int:
        return int(np.diff(self.col_indptr).max()) if self.M else 0

    def neighborhood(self, xj: int):
        lo, hi = self.col_indptr[xj], self.col_indptr[xj + 1]
        return self.col_indices[lo:hi], self.col_values[lo:hi]

    def densify(self) -> DensePotential:
        t = np.full((self.M, self.M), self.fbar, dtype=np.float64)
        cols = np.repeat(np.arange(self.M), np.diff(self.col_indptr))
        t[self.col_indices, cols] = self.col_values
        return DensePotential(t)

    def transpose(self) -> "SparseTruncatedPotential":
        """Rows and columns swapped; new column x_i lists x_j ascending."""
        cols = np.repeat(np.arange(self.M, dtype=np.int64), np.diff(self.col_indptr))
        order = np.lexsort((cols, self.col_indices))
        counts = np.bincount(self.col_indices, minlength=self.M)
        indptr = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
        return SparseTruncatedPotential(self.M, self.fbar, indptr, cols[order],
                                        self.col_values[order])

    def to_log(self) -> "SparseTruncatedPotential":
        """ln-domain twin (reference ``mrf.py:177-195``); cached."""
        if self._log is None:
            if self.fbar < 0 or (self.col_values < 0).any():
                raise ValueError("cannot take log of a potential with negative entries")
            with np.errstate(divide="ignore"):
                self._log = SparseTruncatedPotential(
                    self.M, math.log(self.fbar) if self.fbar > 0 else -math.inf,
                    self.col_indptr, self.col_indices, np.log(self.col_values))
        return self._log

    def __repr__(self) -> str:
        return (f"SparseTruncatedPotential(M={self.M}, fbar={self.fbar:g}, m={self.m}, "
                f"maxsum_safe={self.maxsum_safe})")


def truncated_linear_potential(M: int, alpha: float, T: float) -> SparseTruncatedPotential:
    """f = exp(-alpha * min(|x_i - x_j|, T)), floor at |d| >= T.

    Values use ``math.exp`` per distance exactly as the reference does
    (``mrf.py:229-242``; ``np.exp`` can differ by one ulp), and the log twin
    is attached analytically (``mrf.py:247-249``).
    """
    if M < 1:
        raise ValueError(f"label count must be a positive integer, got {M!r}")
    if not alpha > 0:
        raise ValueError(f"alpha must be > 0, got {alpha}")
    if not T > 0:
        raise ValueError(f"T must be > 0, got {T}")
    fbar = math.exp(-alpha * T)
    val_of = {}
    idx, val, logv = [], [], []
    indptr = np.zeros(M + 1, dtype=np.int64)
    for xj in range(M):
        lo = max(0, xj - int(math.ceil(T)))
        for xi in range(lo, min(M, xj + int(math.ceil(T)) + 1)):
            d = abs(xi - xj)
            if not d < T:
                continue
            if d not in val_of:
                val_of[d] = math.exp(-alpha * d)
            if val_of[d] == fbar:
                continue
            idx.append(xi)
            val.append(val_of[d])
            logv.append(-alpha * d)
        indptr[xj + 1] = len(idx)
    idx_a = np.array(idx, dtype=np.int64)
    pot = SparseTruncatedPotential(M, fbar, indptr, idx_a, np.array(val, dtype=np.float64))
    pot._log = SparseTruncatedPotential(M, -alpha * T, indptr, idx_a,
                                        np.array(logv, dtype=np.float64))
    return pot


def sparse_from_dense(dense, fbar: float, tol: float = 0.0) -> SparseTruncatedPotential:
    """Keep entries with |v - fbar| > tol * max(|fbar|, 1) (``mrf.py:253-285``)."""
    if tol < 0:
        raise ValueError(f"tol must be >= 0, got {tol}")
    t = dense.table if isinstance(dense, DensePotential) else np.asarray(dense, np.float64)
    if t.ndim != 2 or t.shape[0] != t.shape[1]:
        raise ValueError(f"dense table must be square, got shape {t.shape}")
    M = t.shape[0]
    keep = np.abs(t - fbar) > tol * max(abs(fbar), 1.0)
    xj_of, xi_of = np.nonzero(keep.T)          # column-major walk: xj outer, xi ascending
    counts = np.bincount(xj_of, minlength=M)
    indptr = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
    return SparseTruncatedPotential(M, fbar, indptr, xi_of.astype(np.int64), t[xi_of, xj_of])


def grid_edges(height: int, width: int) -> np.ndarray:
    """(E, 2) edges in the reference's canonical order (``mrf.py:401-411``):
    node-major, each node emitting (n, n+1) then (n, n+W)."""
    n = np.arange(height * width, dtype=np.int64).reshape(height, width)
    right = np.full((height, width, 2), -1, dtype=np.int64)
    down = np.full((height, width, 2), -1, dtype=np.int64)
    right[:, :-1, 0], right[:, :-1, 1] = n[:, :-1], n[:, 1:]
    down[:-1, :, 0], down[:-1, :, 1] = n[:-1, :], n[1:, :]
    both = np.stack([right, down], axis=2).reshape(-1, 2)
    return both[both[:, 0] >= 0]


class _SharedPotentials(Sequence):
    """Read-only length-E view that repeats one shared potential object."""

    def __init__(self, pot, n: int):
        self._pot, self._n = pot, n

    def __len__(self) -> int:
        return self._n

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self._pot] * len(range(*i.indices(self._n)))
        if not -self._n <= i < self._n:
            raise IndexError(i)
        return self._pot

    def __iter__(self):
        return (self._pot for _ in range(self._n))


class GridMrf:
    """4-connected H x W grid MRF with one shared pairwise potential, or one
    potential per edge (a sequence in the reference edge order).

    Attribute surface matches the reference ``MrfModel`` for grid models
    (``M``, ``unaries``, ``log_unaries``, ``edges``, ``potentials``,
    ``grid_shape``, ``n_nodes``, ``n_edges``).  ``shared_potential`` lets the
    engine skip the identity scan over ``potentials``; it is None for
    per-edge potentials.
    """

    def __init__(self, height: int, width: int, M: int, unaries, potential,
                 log_unaries=None):
        if height < 1 or width < 1:
            raise ValueError(f"grid dimensions must be positive, got {height}x{width}")
        if M < 1:
            raise ValueError(f"label count must be a positive integer, got {M!r}")
        u = np.ascontiguousarray(unaries, dtype=np.float64)
        if u.shape != (height * width, M):
            raise ValueError(f"unaries must be ({height * width}, {M}), got {u.shape}")
        if not np.isfinite(u).all():
            raise ValueError("unary tables must be finite")
        if (u < 0).any():
            raise ValueError("unary tables must be nonnegative")
        if not (u > 0).any(axis=1).all():
            bad = int(np.flatnonzero(~(u > 0).any(axis=1))[0])
            raise ValueError(f"unary table of node {bad} has no positive entry")
        per_edge = None
        if isinstance(potential, (list, tuple)):
            per_edge = list(potential)
            n_edges = height * (width - 1) + width * (height - 1)
            if len(per_edge) != n_edges:
                raise ValueError(f"need one potential per edge ({n_edges}), got {len(per_edge)}")
            for p in per_edge:
                if p.M != M:
                    raise ValueError(f"potential label count {p.M} != model label count {M}")
        elif potential.M != M:
            raise ValueError(f"potential label count {potential.M} != model label count {M}")
        if log_unaries is not None:
            log_unaries = np.ascontiguousarray(log_unaries, dtype=np.float64)
            if log_unaries.shape != u.shape:
                raise ValueError("log_unaries shape must match unaries")
            log_unaries.setflags(write=False)
        self.M = int(M)
        self.grid_shape = (int(height), int(width))
        self.unaries = _frozen(u)
        self._log_unaries = log_unaries
        self.shared_potential = None if per_edge is not None else potential
        self._per_edge = per_edge
        self._edges = None

    @property
    def n_nodes(self) -> int:
        return self.unaries.shape[0]

    @property
    def n_edges(self) -> int:
        h, w = self.grid_shape
        return h * (w - 1) + w * (h - 1)

    @property
    def edges(self) -> np.ndarray:
        if self._edges is None:
            self._edges = _frozen(grid_edges(*self.grid_shape))
        return self._edges

    @property
    def potentials(self) -> Sequence:
        if self._per_edge is not None:
            return self._per_edge
        return _SharedPotentials(self.shared_potential, self.n_edges)

    @property
    def log_unaries(self) -> np.ndarray:
        if self._log_unaries is None:
            with np.errstate(divide="ignore"):
                lu = np.log(self.unaries)
            self._log_unaries = _frozen(lu)
        return self._log_unaries

    def __repr__(self) -> str:
        return f"GridMrf(M={self.M}, nodes={self.n_nodes}, edges={self.n_edges}, grid{self.grid_shape})"


def build_grid_mrf(height: int, width: int, M: int, unary_provider, pairwise,
                   log_unary_provider=None) -> GridMrf:
    """Grid model from (N, M) unary arrays (or per-pixel callbacks), mirroring
    the reference ``build_grid_mrf`` (``mrf.py:414-456``)."""

    def collect(p):
        if isinstance(p, np.ndarray):
            return p
        out = np.empty((height * width, M), dtype=np.float64)
        for r in range(height):
            for c in range(width):
                g = np.asarray(p(r, c), dtype=np.float64)
                if g.shape != (M,):
                    raise ValueError(f"unary vector at ({r}, {c}) has shape {g.shape}, want ({M},)")
                out[r * width + c] = g
        return out

    lu = collect(log_unary_provider) if log_unary_provider is not None else None
    return GridMrf(height, width, M, collect(unary_provider), pairwise, log_unaries=lu)


def _grid_edge_keys(height: int, width: int) -> np.ndarray:
    """Canonical grid edges as sorted keys a * N + b (a < b), in canonical order."""
    e = grid_edges(height, width)
    return e[:, 0] * (height * width) + e[:, 1]


class MrfModel(GridMrf):
    """The reference constructor ``MrfModel(M, unaries, edges, potentials,
    grid_shape=None, log_unaries=None)`` (``mrf.py:298-369``).

    Validation follows the reference (same checks, same messages), with the
    grid-topology check vectorised (the reference builds two Python edge sets,
    ``mrf.py:341-348``).  A grid model keeps the caller's edge list and
    potential list as given; internally it also holds them in the canonical
    grid order (``canonical_potentials``, ``edge_perm`` / ``edge_flip``) so the
    GPU engine runs on its fixed layout and ``MessageStore`` maps its rows back
    to the caller's edge ids (2e: a->b, 2e+1: b->a, bp.py:113-133).

    A model without ``grid_shape`` constructs (the reference's generic
    engine handles it), but the GPU path serves grid models only and raises
    ``NotImplementedError`` at ``run_sweeps``.
    """

    def __init__(self, M: int, unaries, edges, potentials, grid_shape=None, log_unaries=None):
        if not isinstance(M, (int, np.integer)) or M < 1:
            raise ValueError(f"label count must be a positive integer, got {M!r}")
        u = np.ascontiguousarray(unaries, dtype=np.float64)
        if u.ndim != 2 or u.shape[1] != M:
            raise ValueError(f"unaries must be (n_nodes, {M}), got {u.shape}")
        if not np.isfinite(u).all():
            raise ValueError("unary tables must be finite")
        if (u < 0).any():
            raise ValueError("unary tables must be nonnegative")
        if u.shape[0] == 0:
            raise ValueError("model needs at least one node")
        if not (u > 0).any(axis=1).all():
            bad = int(np.flatnonzero(~(u > 0).any(axis=1))[0])
            raise ValueError(f"unary table of node {bad} has no positive entry")
        n = u.shape[0]
        e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
        if e.size:
            if e.min() < 0 or e.max() >= n:
                raise ValueError("edge endpoint out of range")
            if (e[:, 0] == e[:, 1]).any():
                raise ValueError("self-edges are not allowed")
            canon = np.sort(e, axis=1)
            if len(np.unique(canon, axis=0)) != len(canon):
                raise ValueError("duplicate edges are not allowed")
        if hasattr(potentials, "M") and (hasattr(potentials, "col_indptr")
                                         or hasattr(potentials, "table")):
            shared = potentials
            pots = [potentials] * len(e)
        else:
            pots = list(potentials)
            shared = pots[0] if pots and all(p is pots[0] for p in pots) else None
        if len(pots) != len(e):
            raise ValueError(f"need one potential per edge ({len(e)}), got {len(pots)}")
        for p in pots:
            if p.M != M:
                raise ValueError(f"potential label count {p.M} != model label count {M}")
        lo, hi = np.minimum(e[:, 0], e[:, 1]), np.maximum(e[:, 0], e[:, 1])
        if grid_shape is not None:
            h, w = (int(v) for v in grid_shape)
            if h * w != n:
                raise ValueError(f"grid {h}x{w} does not match {n} nodes")
            want = _grid_edge_keys(h, w)
            keys = lo * n + hi
            order = np.argsort(keys, kind="stable")
            if len(keys) != len(want) or not np.array_equal(keys[order], np.sort(want)):
                raise ValueError("grid topology requires exactly the 4-connected neighbor edges")
            # canonical position of every model edge (want is already sorted:
            # node-major, (n, n+1) before (n, n+W))
            perm = np.empty(len(e), dtype=np.int64)
            perm[order] = np.arange(len(e))
            flip = (e[:, 0] > e[:, 1])
            identity = bool((perm == np.arange(len(e))).all() and not flip.any())
            if shared is not None:
                # one shared potential: the reference grid engine, whose
                # orientation is fixed by the pass direction (bp.py:466-489)
                canon_pot = shared
            else:
                # per-edge: the generic engine orients each potential by its
                # edge's (a, b) (bp.py:520-541); a reversed edge is the
                # canonical edge with the transposed potential
                canon_pot = [None] * len(e)
                tcache: dict = {}
                for k in range(len(e)):
                    p = pots[k]
                    if flip[k] and hasattr(p, "col_indptr"):
                        p = tcache.setdefault(id(p), p.transpose())
                    elif flip[k]:
                        p = tcache.setdefault(id(p), DensePotential(p.table.T))
                    canon_pot[perm[k]] = p
            super().__init__(h, w, M, u, canon_pot, log_unaries=log_unaries)
            self.edge_perm = None if identity else perm
            self.edge_flip = None if identity else flip
        else:
            if log_unaries is not None:
                log_unaries = np.ascontiguousarray(log_unaries, dtype=np.float64)
                if log_unaries.shape != u.shape:
                    raise ValueError("log_unaries shape must match unaries")
                log_unaries.setflags(write=False)
            self.M = int(M)
            self.grid_shape = None
            self.unaries = _frozen(u)
            self._log_unaries = log_unaries
            self.shared_potential = None
            self._per_edge = pots
            self.edge_perm = None
            self.edge_flip = None
        self._model_edges = _frozen(e)
        self._model_pots = pots

    @property
    def n_edges(self) -> int:
        return len(self._model_edges)

    @property
    def edges(self) -> np.ndarray:
        return self._model_edges

    @property
    def potentials(self) -> Sequence:
        return self._model_pots

    @property
    def canonical_potentials(self) -> Sequence:
        """Potentials in the canonical grid edge order (GridMrf semantics)."""
        return GridMrf.potentials.fget(self)

    def __repr__(self) -> str:
        topo = f"grid{self.grid_shape}" if self.grid_shape else "generic"
        return f"MrfModel(M={self.M}, nodes={self.n_nodes}, edges={self.n_edges}, {topo})"


class SweepSchedule:
    """Reference ``SweepSchedule`` (bp.py:190-211): ordered directional passes
    of directed-edge ids.  The GPU path runs the canonical grid schedule
    (``grid_canonical``) as in-place sequential sweeps; custom pass orders
    are not supported on the GPU and raise at ``run_sweeps``."""

    def __init__(self, passes, grid_canonical: bool = False):
        self.passes = [np.asarray(p, dtype=np.int64) for p in passes]
        self.grid_canonical = grid_canonical

    @classmethod
    def canonical(cls, model) -> "SweepSchedule":
        if model.grid_shape is not None:
            return cls(_grid_passes(model), grid_canonical=True)
        ne = model.n_edges
        forward = np.arange(ne, dtype=np.int64) * 2
        backward = np.arange(ne - 1, -1, -1, dtype=np.int64) * 2 + 1
        return cls([np.concatenate([forward, backward])])

    @property
    def n_updates_per_sweep(self) -> int:
        return sum(len(p) for p in self.passes)


def edge_mapping(model):
    """(perm, flip) of a grid model whose edge list is not the canonical one
    (model edge k is canonical edge perm[k], given as (b, a) where flip[k]),
    or None for the canonical order.  Works for this package's models
    (precomputed) and for any object with ``edges`` / ``grid_shape``, e.g. the
    reference's own ``MrfModel``."""
    if isinstance(model, GridMrf) and not isinstance(model, MrfModel):
        return None
    if hasattr(model, "edge_perm"):
        return None if model.edge_perm is None else (model.edge_perm, model.edge_flip)
    h, w = model.grid_shape
    e = np.asarray(model.edges, dtype=np.int64).reshape(-1, 2)
    n = h * w
    keys = np.minimum(e[:, 0], e[:, 1]) * n + np.maximum(e[:, 0], e[:, 1])
    want = _grid_edge_keys(h, w)
    if len(keys) == len(want) and np.array_equal(keys, want) and not (e[:, 0] > e[:, 1]).any():
        return None
    order = np.argsort(keys, kind="stable")
    perm = np.empty(len(e), dtype=np.int64)
    perm[order] = np.arange(len(e))
    return perm, e[:, 0] > e[:, 1]


def canonical_edge_potentials(model) -> list:
    """Per-edge potentials in the canonical grid edge order; a reversed edge
    (b, a) contributes its potential transposed (the generic engine orients a
    potential by its edge, bp.py:520-541)."""
    if hasattr(model, "canonical_potentials"):
        return list(model.canonical_potentials)
    pots = list(model.potentials)
    mp = edge_mapping(model)
    if mp is None:
        return pots
    perm, flip = mp
    out = [None] * len(pots)
    tcache: dict = {}
    for k, p in enumerate(pots):
        if flip[k]:
            p = tcache.setdefault(id(p), p.transpose() if hasattr(p, "col_indptr")
                                  else DensePotential(np.asarray(p.table).T))
        out[perm[k]] = p
    return out


def model_directed_ids(model, canon_ids: np.ndarray, mapping="auto") -> np.ndarray:
    """Canonical directed-edge ids -> ids in the model's own edge order."""
    mp = edge_mapping(model) if mapping == "auto" else mapping
    if mp is None:
        return canon_ids
    perm, flip = mp
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm))
    e = inv[canon_ids // 2]
    return 2 * e + ((canon_ids % 2) ^ flip[e].astype(np.int64))


def _grid_passes(model) -> list:
    """Directed-edge ids of the four canonical passes (bp.py:214-234), vectorised."""
    h, w = model.grid_shape
    n = np.arange(h * w, dtype=np.int64).reshape(h, w)
    ce = np.full((h, w, 2), -1, dtype=np.int64)      # canonical edge of (n, n+1) / (n, n+W)
    valid = np.zeros((h, w, 2), dtype=bool)
    valid[:, :-1, 0] = True
    valid[:-1, :, 1] = True
    ce[valid] = np.arange(int(valid.sum()))
    l2r = 2 * ce[:, :-1, 0].ravel()
    r2l = 2 * ce[:, ::-1, 0][:, 1:].ravel() + 1
    t2b = 2 * ce[:-1, :, 1].T.ravel()
    b2t = 2 * ce[::-1, :, 1][1:].T.ravel() + 1
    del n
    return [model_directed_ids(model, p) for p in (l2r, r2l, t2b, b2t)]
