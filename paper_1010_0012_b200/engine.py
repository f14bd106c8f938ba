"""GPU grid BP engine and the reference-shaped public API.

Drop-in surface of the reference ``sparsebp`` grid path (bp.py:620-744):

* ``run_sweeps(model, n_sweeps, kernel="fast", domain="sum", schedule=...,
  convergence_tol=None) -> MessageStore``
* ``compute_beliefs(model, store) -> BeliefTable``
* ``compute_max_marginals(model, store) -> ndarray (N, M)``
* ``map_labels(scores | BeliefTable | MessageStore) -> ndarray (N,) int64``

with the reference's exception types and attributes
(``DegenerateMessageError.edge``, ``DegenerateBeliefError.node``,
``UnsafePotentialError``) and validation (bp.py:411-433).

Schedules: ``schedule=None`` (or the reference's canonical
``SweepSchedule``) runs the reference's own in-place sequential sweep
(bp.py:630-633: L->R, R->L, T->B, B->T passes, each a set of independent
row/column chains) -- a true drop-in of the default.  ``schedule=
"synchronous"`` runs the Jacobi schedule of the benchmark -- all directed
messages of iteration t+1 from those of iteration t, fully parallel and
HBM-bound.  The two give different numbers; both are pinned to
the oracle.

Every device computation goes through libsbp.so (hand-written sm_100a
kernels, ``csrc/``); torch provides device memory, streams and events only.
"""

from __future__ import annotations

import os
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .model import edge_mapping, model_directed_ids
from .plan import PotentialPlan, plan_per_edge, plan_potential

__all__ = ["SYNCHRONOUS", "SEQUENTIAL", "DegenerateMessageError", "DegenerateBeliefError",
           "UnsafePotentialError", "SweepStats", "BeliefTable", "MessageStore", "GridEngine",
           "run_sweeps", "compute_beliefs", "compute_max_marginals", "map_labels"]

SYNCHRONOUS = "synchronous"
SEQUENTIAL = "sequential"
KERNELS = ("standard", "fast", "pruned")
DOMAINS = ("sum", "max")


class DegenerateMessageError(ValueError):
    """A message could not be normalised (reference bp.py:58-67)."""

    def __init__(self, msg: str, edge: tuple[int, int] | None = None):
        super().__init__(msg)
        self.edge = edge


class DegenerateBeliefError(ValueError):
    """A belief vector is zero everywhere (reference bp.py:70-75)."""

    def __init__(self, msg: str, node: int | None = None):
        super().__init__(msg)
        self.node = node


class UnsafePotentialError(ValueError):
    """Fast max-sum requires every stored value >= the floor (bp.py:78-79)."""


@dataclass
class SweepStats:
    """Reference bp.py:95-107; ``sweep_seconds`` are device times per iteration."""

    sweep_seconds: list = field(default_factory=list)
    madds: int = 0
    n_updates: int = 0
    sweeps_run: int = 0
    converged: bool = False

    @property
    def seconds_per_sweep(self) -> float:
        return sum(self.sweep_seconds) / max(len(self.sweep_seconds), 1)


@dataclass
class BeliefTable:
    """Reference bp.py:174-187 (beliefs sum to 1 per node, Z_i normalisers)."""

    beliefs: np.ndarray
    normalizers: np.ndarray
    labels: np.ndarray | None = None   # argmax computed on the device


# ---------------------------------------------------------------------------
# model introspection (reference MrfModel or this package's GridMrf)
# ---------------------------------------------------------------------------

def _shared_potential(model):
    """The potential shared by every edge, or None when edges carry their own
    (the reference then runs its generic engine, bp.py:652-654)."""
    pot = getattr(model, "shared_potential", None)
    if pot is not None:
        return pot
    pots = model.potentials
    if len(pots) == 0:
        return None
    first = pots[0]
    if any(p is not first for p in pots):
        return None
    return first


def _unique_potentials(model) -> list:
    """Reference bp.py:436-440 (identity-deduplicated, first-seen order)."""
    pot = getattr(model, "shared_potential", None)
    if pot is not None:
        return [pot]
    seen: dict = {}
    for p in model.potentials:
        seen.setdefault(id(p), p)
    return list(seen.values())


def _validate(model, kernel: str, domain: str, pot) -> None:
    """Reference ``_validate_run_args`` (bp.py:411-433) on the shared potential."""
    if kernel not in KERNELS:
        raise ValueError(f"kernel must be one of {KERNELS}, got {kernel!r}")
    if domain not in DOMAINS:
        raise ValueError(f"domain must be one of {DOMAINS}, got {domain!r}")
    if pot is None:
        return
    sparse = hasattr(pot, "col_indptr")
    if kernel in ("fast", "pruned") and not sparse:
        raise TypeError(f"kernel={kernel!r} requires SparseTruncatedPotential on every edge, "
                        f"found {type(pot).__name__}")
    if domain == "sum":
        if sparse:
            if pot.fbar < 0 or (np.asarray(pot.col_values) < 0).any():
                raise ValueError("sum-product potentials must be nonnegative (fbar >= 0)")
        elif (np.asarray(pot.table) < 0).any():
            raise ValueError("sum-product potentials must be nonnegative")
    if domain == "max" and kernel == "fast":
        lp = pot.to_log()
        if hasattr(lp, "maxsum_safe") and not lp.maxsum_safe:
            raise UnsafePotentialError(
                "fast max-sum requires values >= fbar on every edge potential")


def _edge_endpoints(H: int, W: int, d: int) -> tuple[int, int]:
    """Reference directed-edge id -> (i, j) (bp.py:154-156 over mrf.py:401-411)."""
    e = d // 2
    r = min(e // (2 * W - 1), H - 1)
    o = e - r * (2 * W - 1)
    if r < H - 1:
        if o < 2 * (W - 1):
            c, horiz = o // 2, o % 2 == 0
        else:
            c, horiz = W - 1, False
    else:
        c, horiz = o, True
    a = r * W + c
    b = a + (1 if horiz else W)
    return (a, b) if d % 2 == 0 else (b, a)


def _stream_handle(device=None) -> int:
    """The current torch stream of ``device`` (not of the current device: an
    engine on cuda:1 launches on cuda:1's stream whatever device is current)."""
    return torch.cuda.current_stream(device).cuda_stream


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


class GridEngine:
    """Device state of one grid (or one row strip of it) for one domain.

    Owns the padded f32 value table, two message buffers (ping-pong) and
    the error word; the potential plan's arrays live on the device too.
    """

    def __init__(self, model, domain: str = "sum", kernel: str = "fast", device=None,
                 r0: int = 0, rows: int | None = None, values: np.ndarray | None = None,
                 schedule: str = SYNCHRONOUS, precision: str | None = None,
                 defer_values: bool = False):
        if not torch.cuda.is_available():
            raise RuntimeError("the GPU grid engine needs a CUDA device (no CPU fallback)")
        self.lib = L.lib()
        self.model = model
        if model.grid_shape is None:
            raise NotImplementedError("GPU engine supports grid models only (grid_shape is None)")
        self.H, self.W = (int(v) for v in model.grid_shape)
        self.M = int(model.M)
        self.domain = domain
        self.kernel = kernel
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        if self.device.index is None:      # pin the device the engine was created on
            self.device = torch.device("cuda", torch.cuda.current_device())
        pot = _shared_potential(model) if model.n_edges else None
        for p in (_unique_potentials(model) if model.n_edges else []):
            _validate(model, kernel, domain, p)
        self.schedule = schedule
        if schedule == SEQUENTIAL and (r0 != 0 or (rows is not None and rows != self.H)):
            raise NotImplementedError("sequential sweeps run on the whole grid (no strips)")
        self.r0 = r0
        self.rows = self.H - r0 if rows is None else rows
        self.Ms = self.lib.sbp_padded_labels(self.M)
        if self.Ms > 256:
            raise NotImplementedError(f"M={self.M} > 256 labels is not supported on the GPU path")
        self.grid = L.SbpGrid(self.H, self.W, self.M, self.Ms, self.r0, self.rows,
                              self.device.index)
        self.dom = L.SBP_SUM if domain == "sum" else L.SBP_MAX
        self.plan: PotentialPlan | None = None
        # sum-product accumulation: "auto" (f64 for weak smoothing over wide
        # bands, plan.wants_f64), "f32" or "f64"; SBP_PRECISION overrides
        self.precision = precision or os.environ.get("SBP_PRECISION", "auto")
        if self.precision not in ("auto", "f32", "f64"):
            raise ValueError(f"precision must be 'auto', 'f32' or 'f64', got {self.precision!r}")
        if pot is not None:
            self.plan = plan_potential(pot, domain, kernel, self.M, self.Ms,
                                       precision=self.precision)
        elif model.n_edges:
            self.plan = plan_per_edge(model, domain, kernel, self.M, self.Ms)
        if self.plan is not None:
            self._pot_struct = self._make_pot_struct(self.plan)
        with torch.cuda.device(self.device):
            shape = (4, self.rows + 2, self.W, self.Ms)
            self.msgs = [torch.empty(shape, dtype=torch.float32, device=self.device),
                         torch.empty(shape, dtype=torch.float32, device=self.device)]
            self.err = torch.full((1,), -1, dtype=torch.int64, device=self.device)
            self.values = torch.empty((self.rows, self.W, self.Ms), dtype=torch.float32,
                                      device=self.device)
            if not defer_values:         # else run_streamed uploads them by row bands
                self.upload_values(values)
        for buf in self.msgs:
            self._init(buf, ghosts_only=True)
        # temporal blocking (sbp_iterate_fused): up to `fuse` synchronous
        # iterations per launch on a whole single-GPU grid; SBP_FUSE=1 turns
        # it off.  Lag (rows between levels) and rounds (pixel groups per
        # warp and work unit) are tuning knobs of the wavefront.
        self.fuse = _default_fuse(self.domain, self.Ms, self.plan)
        self.fuse_lag = int(os.environ.get("SBP_FUSE_LAG", "4"))
        self.fuse_rounds = int(os.environ.get("SBP_FUSE_ROUNDS", "2"))
        self._fused_ok: bool | None = None
        self._stamps: torch.Tensor | None = None
        self._epoch = 0
        self.reset()

    # -- setup -------------------------------------------------------------
    def _make_pot_struct(self, plan: PotentialPlan) -> L.SbpPotential:
        s = L.SbpPotential()
        s.kind, s.domain, s.floor_term = plan.kind, self.dom, plan.floor_term
        s.R, s.m_max = plan.R, plan.m_max
        s.fbar[0], s.fbar[1] = plan.fbar
        if plan.kind == L.SBP_POT_BAND:
            for o in range(2):
                for k, v in enumerate(plan.band_w[o]):
                    s.band_w[o][k] = float(v)
        else:
            idx = torch.from_numpy(np.ascontiguousarray(plan.ell_idx)).to(self.device)
            hi = np.ascontiguousarray(plan.ell_w, dtype=np.float32)
            w = torch.from_numpy(hi).to(self.device)
            plan.device_arrays = [idx, w]
            # orientation 1 directly follows orientation 0 ([.., 2, m_max, Ms])
            step = plan.m_max * self.Ms * 4
            s.ell_idx[0], s.ell_idx[1] = idx.data_ptr(), idx.data_ptr() + step
            s.ell_w[0], s.ell_w[1] = w.data_ptr(), w.data_ptr() + step
            if plan.accumulate == L.SBP_ACC_F64:
                # f64 weights as hi + lo f32 planes (exact to ~2^-48 relative)
                with np.errstate(invalid="ignore"):
                    lo = np.where(np.isfinite(plan.ell_w), plan.ell_w - hi.astype(np.float64), 0.0)
                wl = torch.from_numpy(np.ascontiguousarray(lo, dtype=np.float32)).to(self.device)
                plan.device_arrays.append(wl)
                s.accumulate = L.SBP_ACC_F64
                s.fbar64[0], s.fbar64[1] = plan.fbar64
                s.ell_w_lo[0], s.ell_w_lo[1] = wl.data_ptr(), wl.data_ptr() + step
            if plan.n_pot:
                fb = torch.from_numpy(np.ascontiguousarray(plan.fbar_all, dtype=np.float32)).to(
                    self.device)
                ph = torch.from_numpy(plan.pid_h).to(self.device)
                pv = torch.from_numpy(plan.pid_v).to(self.device)
                plan.device_arrays += [fb, ph, pv]
                s.n_pot = plan.n_pot
                s.fbar_all, s.pid_h, s.pid_v = fb.data_ptr(), ph.data_ptr(), pv.data_ptr()
            if plan.dense_t is not None:
                t = torch.from_numpy(np.ascontiguousarray(plan.dense_t, dtype=np.float32)).to(
                    self.device)
                plan.device_arrays.append(t)
                # a symmetric table passes ONE pointer for both orientations:
                # libsbp then runs sum-product on the tensor cores (sbp.h)
                sym = np.array_equal(plan.dense_t[0], plan.dense_t[1])
                for o in range(2):
                    s.dense_t[o] = t[0 if sym else o].data_ptr()
        return s

    def upload_stereo(self) -> None:
        """Image pair -> unary table on the device (sbp_stereo_values): the
        H2D traffic is the two uint8 images of this strip's rows."""
        left, right, beta, T_u = self.model.stereo_source
        sl = slice(self.r0, self.r0 + self.rows)
        dev = []
        for img in (left, right):
            t = torch.from_numpy(np.ascontiguousarray(img[sl]))
            dev.append(t.to(self.device, non_blocking=t.is_pinned()))
        L.check(self.lib.sbp_stereo_values(ctypes_ref(self.grid), self.dom, _ptr(dev[0]),
                                           _ptr(dev[1]), beta, T_u, _ptr(self.values),
                                           _stream_handle(self.device)))
        self._staging = dev

    def upload_values(self, values: np.ndarray | torch.Tensor | None = None) -> None:
        """Host f64 unaries (sum) / log unaries (max) -> padded f32 device table."""
        if values is None and getattr(self.model, "stereo_source", None) is not None:
            self.upload_stereo()
            return
        if values is None:
            src = self.model.unaries if self.domain == "sum" else self.model.log_unaries
            values = src[self.r0 * self.W:(self.r0 + self.rows) * self.W]
        if isinstance(values, torch.Tensor):
            dev = values.to(self.device, dtype=torch.float64)
        else:
            arr = np.ascontiguousarray(values, dtype=np.float64)
            with warnings.catch_warnings():   # read-only model arrays: never written
                warnings.simplefilter("ignore", UserWarning)
                host = torch.from_numpy(arr)
            dev = host.to(self.device, non_blocking=host.is_pinned())
        L.check(self.lib.sbp_load_values(ctypes_ref(self.grid), self.dom, _ptr(dev),
                                         _ptr(self.values), _stream_handle(self.device)))
        self._staging = dev   # keep alive until the stream consumed it

    def run_streamed(self, iters: int, values=None, bands: int = 8,
                     events: list | None = None) -> None:
        """``iters`` synchronous iterations from the reference initial messages,
        overlapped with the host->device upload of the f64 unary table.

        The table crosses PCIe in ``bands`` row bands on a copy stream (pinned
        host memory makes the copies asynchronous) and each band is converted
        to the padded f32 layout as it lands.  Iterations run as a row
        wavefront: iteration t covers the rows whose inputs exist, its
        frontier trailing iteration t-1's by one row (a row needs the
        previous iteration's messages from the row below).  Because
        iteration t+1 only ever writes rows that iteration t has finished,
        the ping-pong buffers stay race-free, and the arithmetic is that of
        ``step``: bit-identical results."""
        if self.plan is None or self.r0 != 0 or self.rows != self.H:
            raise NotImplementedError("streamed upload runs a whole single-GPU grid")
        H, W = self.H, self.W
        if values is None:
            values = self.model.unaries if self.domain == "sum" else self.model.log_unaries
        arr = np.ascontiguousarray(values, dtype=np.float64)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", UserWarning)
            host = torch.from_numpy(arr)
        pinned = host.is_pinned()
        cs = torch.cuda.current_stream(self.device)
        if getattr(self, "_copy_stream", None) is None:
            self._copy_stream = torch.cuda.Stream(device=self.device)
        copy = self._copy_stream
        copy.wait_stream(cs)
        bands = max(1, min(bands, H))
        step = -(-H // bands)
        frontier = [0] * iters
        self.err.fill_(-1)
        keep = []
        for b0 in range(0, H, step):
            nb = min(step, H - b0)
            ev = torch.cuda.Event()
            with torch.cuda.stream(copy):
                chunk = host[b0 * W:(b0 + nb) * W].to(self.device, non_blocking=pinned)
                ev.record(copy)
            cs.wait_event(ev)
            chunk.record_stream(cs)
            keep.append(chunk)
            g = L.SbpGrid(H, W, self.M, self.Ms, b0, nb, self.device.index)
            L.check(self.lib.sbp_load_values(ctypes_ref(g), self.dom, _ptr(chunk),
                                             _ptr(self.values) + b0 * W * self.Ms * 4,
                                             _stream_handle(self.device)))
            ready = b0 + nb
            for t in range(iters):
                if t == 0:
                    new = ready
                else:
                    new = frontier[t - 1] if frontier[t - 1] == H else frontier[t - 1] - 1
                if new <= frontier[t]:
                    break           # iteration t is stuck, so is every later one
                ev0 = None
                if events is not None:
                    ev0 = torch.cuda.Event(enable_timing=True)
                    ev0.record(cs)
                L.check(self.lib.sbp_iterate(
                    ctypes_ref(self.grid), ctypes_ref(self._pot_struct), _ptr(self.values),
                    _ptr(self.msgs[t % 2]), _ptr(self.msgs[(t + 1) % 2]), frontier[t] + 1,
                    new + 1, t, L.SBP_ITER_FIRST if t == 0 else 0, _ptr(self.err),
                    _stream_handle(self.device)))
                if events is not None:
                    ev1 = torch.cuda.Event(enable_timing=True)
                    ev1.record(cs)
                    events.append((ev0, ev1, (new - frontier[t]) / H))
                frontier[t] = new
        assert all(f == H for f in frontier)
        self._staging = keep
        self.cur = iters % 2
        self.iterations = iters
        self._init_valid = True

    @property
    def kernel_name(self) -> str:
        """The kernel instantiation this engine launches per iteration / sweep."""
        if self.plan is None:
            return "none"
        import ctypes
        buf = ctypes.create_string_buffer(128)
        mode = 1 if self.schedule == SEQUENTIAL else (2 if self._can_fuse() else 0)
        L.check(self.lib.sbp_plan_name(ctypes_ref(self.grid), ctypes_ref(self._pot_struct),
                                       mode, buf, 128))
        return buf.value.decode()

    def _init(self, buf: torch.Tensor, ghosts_only: bool) -> None:
        L.check(self.lib.sbp_init_msgs(ctypes_ref(self.grid), self.dom, 1 if ghosts_only else 0,
                                       _ptr(buf), _stream_handle(self.device)))

    def reset(self, full: bool = False) -> None:
        """Start a new run from the reference initial messages (bp.py:587-601).

        The ghost (border) slots of both buffers were set once at construction
        and are never written by the iteration kernels; the first iteration
        runs with SBP_ITER_FIRST and takes the uniform initial messages as
        constants, so no per-run initialisation traffic is needed.  ``full``
        materialises the initial messages in the current buffer (needed when
        they are read: the convergence test after iteration 1, or a read-out
        before any iteration).
        """
        self.err.fill_(-1)
        self.cur = 0
        self.iterations = 0
        self._init_valid = False
        if full or self.schedule == SEQUENTIAL:   # in-place sweeps read every slot
            self._init(self.msgs[0], ghosts_only=False)
            self._init_valid = True

    # -- iteration ---------------------------------------------------------
    @property
    def current(self) -> torch.Tensor:
        if self.iterations == 0 and not self._init_valid:
            self._init(self.msgs[self.cur], ghosts_only=False)
            self._init_valid = True
        return self.msgs[self.cur]

    def iterate_rows(self, lr_begin: int, lr_end: int, stream: int | None = None,
                     delta: torch.Tensor | None = None) -> None:
        """One synchronous iteration over local rows [lr_begin, lr_end) from the
        current buffer into the other one (does not flip buffers).  ``delta``
        (device float32 scalar): fused convergence test, max |new - old|."""
        if self.plan is None:
            return
        args = (ctypes_ref(self.grid), ctypes_ref(self._pot_struct), _ptr(self.values),
                _ptr(self.msgs[self.cur]), _ptr(self.msgs[1 - self.cur]), lr_begin, lr_end,
                self.iterations, L.SBP_ITER_FIRST if self.iterations == 0 else 0, _ptr(self.err))
        s = _stream_handle(self.device) if stream is None else stream
        if delta is None:
            L.check(self.lib.sbp_iterate(*args, s))
        else:
            L.check(self.lib.sbp_iterate_delta(*args, _ptr(delta), s))

    @property
    def fused_delta(self) -> bool:
        """Whether the convergence test can ride in the iteration kernels
        (all but the tiled dense comparison kernel of the synchronous schedule)."""
        if self.plan is None:
            return False
        tiled_dense = (self.plan.kind == L.SBP_POT_DENSE and self.Ms >= 32
                       and not self.plan.n_pot)
        return self.schedule == SEQUENTIAL or not tiled_dense

    def flip(self) -> None:
        self.cur = 1 - self.cur
        self.iterations += 1

    def _can_fuse(self) -> bool:
        return (self.fuse >= 2 and self._fused_ok is not False
                and self.schedule == SYNCHRONOUS and self.plan is not None
                and self.plan.kind == L.SBP_POT_BAND and self.Ms >= 32
                and self.r0 == 0 and self.rows == self.H)

    def iterate_fused(self, levels: int) -> bool:
        """`levels` synchronous iterations in one temporally blocked launch
        (bit-identical to `levels` iterate_rows + flip).  Returns False, with
        nothing launched, when no fused kernel exists for this plan."""
        if self._stamps is None:
            words = self.lib.sbp_fused_stamp_words(ctypes_ref(self.grid))
            L.check(min(words, 0))
            self._stamps = torch.zeros(words, dtype=torch.int32, device=self.device)
        self._epoch += 1
        rc = self.lib.sbp_iterate_fused(
            ctypes_ref(self.grid), ctypes_ref(self._pot_struct), _ptr(self.values),
            _ptr(self.msgs[self.cur]), _ptr(self.msgs[1 - self.cur]), levels, self.iterations,
            L.SBP_ITER_FIRST if self.iterations == 0 else 0, _ptr(self._stamps), self._epoch,
            self.fuse_lag, self.fuse_rounds, _ptr(self.err), _stream_handle(self.device))
        if rc == L.SBP_EUNSUPPORTED:
            self._fused_ok = False
            return False
        L.check(rc)
        self._fused_ok = True
        self.cur = (self.cur + levels) % 2
        self.iterations += levels
        return True

    def sweep(self, delta: torch.Tensor | None = None) -> None:
        """One canonical sequential sweep in place (reference ``_run_grid``)."""
        if self.plan is not None:
            args = (ctypes_ref(self.grid), ctypes_ref(self._pot_struct), _ptr(self.values),
                    _ptr(self.msgs[0]), self.iterations, _ptr(self.err))
            if delta is None:
                L.check(self.lib.sbp_sweep(*args, _stream_handle(self.device)))
            else:
                L.check(self.lib.sbp_sweep_delta(*args, _ptr(delta), _stream_handle(self.device)))
        self.iterations += 1

    def snapshot(self) -> None:
        """Keep a copy of the current messages (sequential convergence test)."""
        self.msgs[1].copy_(self.msgs[0])

    def step(self, n: int = 1, events: list | None = None,
             delta: torch.Tensor | None = None) -> None:
        """``n`` iterations (sweeps); ``delta``: fused convergence test of the
        last one (device float32 scalar, max-updated, zeroed by the caller)."""
        if self.schedule == SEQUENTIAL:
            for _ in range(n):
                ev0 = ev1 = None
                if events is not None:
                    ev0 = torch.cuda.Event(enable_timing=True)
                    ev0.record(torch.cuda.current_stream(self.device))
                self.sweep(delta)
                if events is not None:
                    ev1 = torch.cuda.Event(enable_timing=True)
                    ev1.record(torch.cuda.current_stream(self.device))
                    events.append((ev0, ev1, 1))
            return
        done = 0
        while done < n:
            k = min(self.fuse, n - done) if (self._can_fuse() and delta is None) else 1
            if events is not None:
                ev0 = torch.cuda.Event(enable_timing=True)
                ev0.record(torch.cuda.current_stream(self.device))
            if k < 2 or not self.iterate_fused(k):
                k = 1
                self.iterate_rows(1, self.rows + 1, delta=delta)
                self.flip()
            if events is not None:
                ev1 = torch.cuda.Event(enable_timing=True)
                ev1.record(torch.cuda.current_stream(self.device))
                events.append((ev0, ev1, k))
            done += k

    def max_abs_delta(self) -> float:
        out = torch.zeros(1, dtype=torch.float32, device=self.device)
        L.check(self.lib.sbp_max_abs_diff(ctypes_ref(self.grid), _ptr(self.msgs[0]),
                                          _ptr(self.msgs[1]), _ptr(out), _stream_handle(self.device)))
        return float(out.item())

    def error(self) -> tuple[int, int] | None:
        """(iteration, directed edge id) of the first degenerate message, or None."""
        key = int(self.err.item()) & 0xFFFFFFFFFFFFFFFF
        if key == L.SBP_ERR_NONE:
            return None
        return key >> 40, key & ((1 << 40) - 1)

    def raise_if_degenerate(self) -> None:
        e = self.error()
        if e is None:
            return
        it, d = e
        if self.schedule == SEQUENTIAL:
            # key: sweep << 40 | pass << 38 | line * line_len + position
            direction, idx = (d >> 38) & 3, d & ((1 << 38) - 1)
            H, W = self.H, self.W
            lines_len = W - 1 if direction <= 1 else H - 1
            line, pos = divmod(idx, lines_len)
            stride, step, origin = {0: (W, 1, 0), 1: (W, -1, W - 1), 2: (1, W, 0),
                                    3: (1, -W, (H - 1) * W)}[direction]
            src = line * stride + origin + pos * step
            raise DegenerateMessageError(
                f"degenerate message on edge {src}->{src + step} (pass direction {direction})",
                edge=(int(src), int(src + step)))
        i, j = _edge_endpoints(self.H, self.W, d)
        raise DegenerateMessageError(
            f"degenerate message on edge {i}->{j} (synchronous iteration {it})", edge=(i, j))

    # -- read-out ----------------------------------------------------------
    def beliefs_device(self, want_beliefs: bool = True, want_labels: bool = True):
        n = self.rows * self.W
        b = (torch.empty((n, self.M), dtype=torch.float32, device=self.device)
             if want_beliefs else None)
        z = (torch.empty(n, dtype=torch.float64, device=self.device)
             if want_beliefs and self.domain == "sum" else None)
        lab = torch.empty(n, dtype=torch.int32, device=self.device) if want_labels else None
        bad = torch.full((1,), -1, dtype=torch.int64, device=self.device)
        L.check(self.lib.sbp_beliefs(
            ctypes_ref(self.grid), self.dom, _ptr(self.values), _ptr(self.current),
            _ptr(b) if b is not None else None, _ptr(z) if z is not None else None,
            _ptr(lab) if lab is not None else None, _ptr(bad), _stream_handle(self.device)))
        return b, z, lab, bad

    def labels(self) -> torch.Tensor:
        _, _, lab, bad = self.beliefs_device(want_beliefs=False)
        self._check_bad(bad)
        return lab

    def _check_bad(self, bad: torch.Tensor) -> None:
        if self.domain != "sum":
            return
        v = int(bad.item()) & 0xFFFFFFFFFFFFFFFF
        if v != L.SBP_ERR_NONE:
            node = v + self.r0 * self.W
            raise DegenerateBeliefError(f"belief of node {node} is zero everywhere", node=node)

    def store_device(self) -> torch.Tensor:
        """(2E, M) f32 messages in reference directed-edge order."""
        E = self.H * (self.W - 1) + self.W * (self.H - 1)
        out = torch.empty((2 * E, self.M), dtype=torch.float32, device=self.device)
        L.check(self.lib.sbp_gather_store(ctypes_ref(self.grid), _ptr(self.current), _ptr(out),
                                          _stream_handle(self.device)))
        return out

    def msgs4(self) -> np.ndarray:
        """Reference-layout (4, N, M) f64 copy of the current messages."""
        cur = self.current[:, 1:self.rows + 1, :, :self.M]
        return cur.reshape(4, self.rows * self.W, self.M).double().cpu().numpy()


def _default_fuse(domain: str, Ms: int, plan) -> int:
    """Iterations per launch (SBP_FUSE overrides).  Temporal blocking halves
    HBM traffic but adds per-unit synchronisation; on B200 it only wins where
    the band is cheap and memory dominates (A/B, profiles/r01_ab_fused.md):
    sum-product, Ms >= 256, R <= 2 (C5 T=2: 1.37 vs 1.58 ms per iteration).
    Everywhere else (C4: 2.41-2.60 vs 2.32) one iteration per launch."""
    env = os.environ.get("SBP_FUSE")
    if env is not None:
        return int(env)
    if (domain == "sum" and Ms >= 256 and plan is not None
            and plan.kind == L.SBP_POT_BAND and plan.R <= 2):
        return 3
    return 1


def ctypes_ref(obj):
    import ctypes
    return ctypes.byref(obj)


class MessageStore:
    """Result of ``run_sweeps`` (reference bp.py:110-171).

    ``data`` -- the (2E, M) f64 array in directed-edge order -- is
    materialised lazily from the device (a gather kernel + one copy), since
    at 2048x1536 with M=128 it is 12.9 GB of host memory.
    """

    def __init__(self, model, domain: str, engine: GridEngine | None = None,
                 data: np.ndarray | None = None):
        if domain not in DOMAINS:
            raise ValueError(f"domain must be one of {DOMAINS}, got {domain!r}")
        self.model = model
        self.domain = domain
        self.engine = engine
        self._data = data
        self.stats: SweepStats | None = None
        # a model whose edge list is not in the canonical grid order (the
        # reference MrfModel accepts any order / orientation): device rows
        # are canonical and get permuted into the model's directed-edge ids
        self._mapping = (edge_mapping(model) if getattr(model, "grid_shape", None) is not None
                         else None)

    @property
    def n_directed(self) -> int:
        return 2 * int(self.model.n_edges)

    @property
    def data(self) -> np.ndarray:
        if self._data is None:
            if self.engine is None or self.engine.plan is None:
                fill = 1.0 / self.model.M if self.domain == "sum" else 0.0
                self._data = np.full((self.n_directed, self.model.M), fill, dtype=np.float64)
            else:
                canon = self.engine.store_device().double().cpu().numpy()
                if self._mapping is not None:
                    ids = model_directed_ids(self.model, np.arange(len(canon)), self._mapping)
                    out = np.empty_like(canon)
                    out[ids] = canon
                    canon = out
                self._data = canon
        return self._data

    def edge_id(self, i: int, j: int) -> int:
        d = self._canonical_edge_id(i, j)
        if self._mapping is None:
            return d
        return int(model_directed_ids(self.model, np.array([d]), self._mapping)[0])

    def _canonical_edge_id(self, i: int, j: int) -> int:
        H, W = self.model.grid_shape
        ri, ci = divmod(int(i), W)
        d = int(j) - int(i)
        if d == 1 and ci + 1 < W:
            e = ri * (2 * W - 1) + (2 * ci if ri < H - 1 else ci)
            return 2 * e
        if d == -1 and ci > 0:
            return self._canonical_edge_id(j, i) + 1
        if d == W and ri + 1 < H:
            e = ri * (2 * W - 1) + 2 * ci + (1 if ci + 1 < W else 0)
            return 2 * e
        if d == -W and ri > 0:
            return self._canonical_edge_id(j, i) + 1
        raise KeyError(f"no directed edge {i}->{j} in model")

    def vector(self, i: int, j: int) -> np.ndarray:
        return self.data[self.edge_id(i, j)]

    def endpoints(self, d: int) -> tuple[int, int]:
        if self._mapping is not None:
            a, b = self.model.edges[int(d) // 2]
            return (int(a), int(b)) if int(d) % 2 == 0 else (int(b), int(a))
        H, W = self.model.grid_shape
        return _edge_endpoints(H, W, int(d))

    def check_normalized(self, atol: float = 1e-6) -> None:
        """Domain invariant (bp.py:162-171) at fp32 tolerance."""
        if self.n_directed == 0:
            return
        if self.domain == "sum":
            sums = self.data.sum(axis=1)
            assert np.abs(sums - 1.0).max() <= atol, "sum-domain message does not sum to 1"
            assert (self.data >= 0).all(), "sum-domain message has negative entries"
        else:
            assert (self.data.max(axis=1) == 0.0).all(), "max-domain message max is not exactly 0"


STREAM_MIN_BYTES = 64 << 20   # smaller unary tables upload in one piece


def _schedule_mode(schedule) -> str:
    """None / the reference canonical SweepSchedule -> sequential (bp.py:647-648);
    "synchronous" -> Jacobi."""
    if schedule is None or schedule in (SEQUENTIAL, "canonical"):
        return SEQUENTIAL
    if schedule == SYNCHRONOUS:
        return SYNCHRONOUS
    if getattr(schedule, "grid_canonical", False):
        return SEQUENTIAL
    raise NotImplementedError(
        "custom SweepSchedule pass orders are not supported on the GPU; use None (the "
        "canonical sequential sweep) or 'synchronous'")


def run_sweeps(model, n_sweeps: int, kernel: str = "fast", domain: str = "sum",
               schedule=None, convergence_tol: float | None = None, device=None,
               engine: GridEngine | None = None, precision: str | None = None) -> MessageStore:
    """Run ``n_sweeps`` sweeps on the GPU (reference bp.py:620-703).

    ``schedule=None`` -- the reference's canonical in-place sequential sweep;
    ``schedule="synchronous"`` -- one Jacobi iteration per sweep (every
    directed edge once, from the previous iteration's messages only).
    """
    if getattr(model, "grid_shape", None) is None:
        raise NotImplementedError(
            "the GPU engine runs grid models (grid_shape set); the reference's generic "
            "edge-list engine (bp.py:506-584) is out of scope")
    mode = _schedule_mode(schedule)
    if n_sweeps < 0:
        raise ValueError(f"n_sweeps must be >= 0, got {n_sweeps}")
    for p in (_unique_potentials(model) if model.n_edges else []):
        _validate(model, kernel, domain, p)
    stats = SweepStats()
    if model.n_edges == 0 or n_sweeps == 0:
        store = MessageStore(model, domain, engine=None)
        store.stats = stats
        return store
    # host unary tables (not built on the device from an image pair) of a
    # single-GPU synchronous run stream in by row bands under the first
    # iterations instead of crossing PCIe before iteration 0
    streamed = (engine is None and mode == SYNCHRONOUS and convergence_tol is None
                and getattr(model, "stereo_source", None) is None
                and int(model.n_nodes) * int(model.M) * 8 >= STREAM_MIN_BYTES
                and os.environ.get("SBP_STREAM", "1") != "0")
    eng = engine if engine is not None else GridEngine(model, domain, kernel, device=device,
                                                       schedule=mode, precision=precision,
                                                       defer_values=streamed)
    if streamed and (eng.plan is None or eng._can_fuse()):
        eng.upload_values()         # the temporally blocked kernel runs whole grids
        streamed = False
    if engine is not None or convergence_tol is not None:
        eng.reset(full=convergence_tol is not None and not eng.fused_delta)
    per_iter = 2 * int(model.n_edges)
    events: list = []
    if streamed:
        cs = torch.cuda.current_stream(eng.device)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(cs)
        eng.run_streamed(n_sweeps)
        ev1.record(cs)
        events.append((ev0, ev1, n_sweeps))   # includes the overlapped upload
        stats.sweeps_run += n_sweeps
        stats.n_updates += per_iter * n_sweeps
    elif convergence_tol is None:
        # no per-sweep test: the engine may fuse iterations into one launch
        eng.step(n_sweeps, events=events)
        stats.sweeps_run += n_sweeps
        stats.n_updates += per_iter * n_sweeps
    else:
        # fused: the iteration kernels compare each message with the one it
        # replaces (no snapshot, no second pass); the tiled dense kernel keeps
        # the separate max |a - b| pass
        fused = eng.fused_delta
        delta = torch.zeros(1, dtype=torch.float32, device=eng.device)
        for _ in range(n_sweeps):
            if fused:
                delta.zero_()
                eng.step(1, events=events, delta=delta)
                d = float(delta.item())
            else:
                if mode == SEQUENTIAL:
                    eng.snapshot()
                eng.step(1, events=events)
                d = eng.max_abs_delta()
            stats.sweeps_run += 1
            stats.n_updates += per_iter
            if d < convergence_tol:
                stats.converged = True
                break
    torch.cuda.synchronize(eng.device)
    # per-sweep device seconds (a fused launch of k iterations counts k equal shares)
    stats.sweep_seconds = [a.elapsed_time(b) / 1e3 / k for a, b, k in events for _ in range(k)]
    if eng.plan.madds_per_sweep is not None:
        stats.madds = eng.plan.madds_per_sweep * stats.sweeps_run
    else:
        stats.madds = eng.plan.madds_per_update * stats.n_updates
    eng.raise_if_degenerate()
    store = MessageStore(model, domain, engine=eng)
    store.stats = stats
    return store


def _engine_of(store) -> GridEngine | None:
    return getattr(store, "engine", None)


def compute_beliefs(model, msgs: MessageStore) -> BeliefTable:
    """Normalised beliefs b_i = g_i * prod incoming / Z_i (bp.py:711-725)."""
    if msgs.domain != "sum":
        raise ValueError("compute_beliefs requires sum-product messages")
    eng = _engine_of(msgs)
    if eng is None or eng.plan is None:
        u = np.asarray(model.unaries, dtype=np.float64)
        if model.n_edges:
            raise TypeError("compute_beliefs needs a store produced by this engine")
        z = u.sum(axis=1)
        if not (z > 0).all():
            node = int(np.flatnonzero(~(z > 0))[0])
            raise DegenerateBeliefError(f"belief of node {node} is zero everywhere", node=node)
        return BeliefTable(u / z[:, None], z, labels=np.argmax(u / z[:, None], axis=1))
    b, z, lab, bad = eng.beliefs_device()
    eng._check_bad(bad)
    return BeliefTable(b.double().cpu().numpy(), z.cpu().numpy(),
                       labels=lab.long().cpu().numpy())


def compute_max_marginals(model, msgs: MessageStore) -> np.ndarray:
    """log g + sum of incoming messages, minus the row max (bp.py:728-738)."""
    if msgs.domain != "max":
        raise ValueError("compute_max_marginals requires max-sum messages")
    eng = _engine_of(msgs)
    if eng is None or eng.plan is None:
        lu = np.asarray(model.log_unaries, dtype=np.float64)
        if model.n_edges:
            raise TypeError("compute_max_marginals needs a store produced by this engine")
        return lu - lu.max(axis=1, keepdims=True)
    b, _, _, _ = eng.beliefs_device(want_labels=False)
    return b.double().cpu().numpy()


def map_labels(scores) -> np.ndarray:
    """Per-node argmax, lowest index on ties (bp.py:741-744).

    Accepts a BeliefTable, a score array, or -- as an extension -- a
    MessageStore from this engine, in which case only the labels leave the
    device.
    """
    if isinstance(scores, MessageStore):
        eng = _engine_of(scores)
        if eng is not None and eng.plan is not None:
            return eng.labels().cpu().numpy().astype(np.int64)
        arr = (compute_beliefs(scores.model, scores).beliefs if scores.domain == "sum"
               else compute_max_marginals(scores.model, scores))
        return np.argmax(arr, axis=1)
    if isinstance(scores, BeliefTable):
        if scores.labels is not None:
            return scores.labels
        return np.argmax(scores.beliefs, axis=1)
    return np.argmax(np.asarray(scores), axis=1)
