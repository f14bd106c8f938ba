"""Row-strip domain decomposition of the synchronous iteration (multi-GPU).

The image is split into horizontal strips, one per rank (GPU).  Under the
synchronous schedule a node's outgoing messages depend only on its own
incoming slots from the previous iteration, so each iteration needs exactly
one exchange per internal strip boundary:

* strip k computes the DOWN messages of its last row into slot 0 of its
  bottom halo row; they belong to slot 0 of the first row of strip k+1;
* strip k computes the UP messages of its first row into slot 3 of its top
  halo row; they belong to slot 3 of the last row of strip k-1.

Each halo is one contiguous W * Ms f32 row of the [slot][row][W][Ms]
layout.  Per iteration a rank computes its two boundary rows first, posts
the sends/receives (NCCL send/recv over NVLink via torch.distributed, or
gloo on CPU in the tests), computes the interior rows on a second stream
while the halos are in flight, then waits for both.  The receive targets
(slot 0 of the first row, slot 3 of the last row) are written by no local
kernel, so there is no race between the exchange and the interior update.
"""

from __future__ import annotations

from typing import Protocol

import numpy as np
import torch

__all__ = ["partition_rows", "Strip", "GpuStrip", "StripRunner", "run_rank"]


def partition_rows(H: int, parts: int) -> list[tuple[int, int]]:
    """Balanced contiguous row ranges (r0, rows); every strip gets >= 1 row."""
    if parts < 1 or parts > H:
        raise ValueError(f"cannot split {H} rows into {parts} strips")
    base, extra = divmod(H, parts)
    out, r0 = [], 0
    for k in range(parts):
        rows = base + (1 if k < extra else 0)
        out.append((r0, rows))
        r0 += rows
    return out


class Strip(Protocol):
    rows: int

    def compute(self, lr_begin: int, lr_end: int, stream=None) -> None: ...

    def flip(self) -> None: ...

    def next_buffer(self) -> torch.Tensor: ...   # [4][rows+2][W][Ms]


def halo_views(next_buf: torch.Tensor, rows: int) -> dict:
    """Send / receive row views of the buffer being written this iteration."""
    return {
        "send_down": next_buf[0, rows + 1],   # my last row's down messages
        "send_up": next_buf[3, 0],            # my first row's up messages
        "recv_above": next_buf[0, 1],         # from the strip above
        "recv_below": next_buf[3, rows],      # from the strip below
    }


class GpuStrip:
    """A strip backed by the CUDA engine (one GridEngine over rows r0..r0+rows)."""

    def __init__(self, model, r0: int, rows: int, domain: str = "sum", kernel: str = "fast",
                 device=None, values=None):
        from .engine import GridEngine
        self.engine = GridEngine(model, domain, kernel, device=device, r0=r0, rows=rows,
                                 values=values)
        self.rows = rows
        self.r0 = r0

    def compute(self, lr_begin: int, lr_end: int, stream=None) -> None:
        self.engine.iterate_rows(lr_begin, lr_end,
                                 stream=None if stream is None else stream.cuda_stream)

    def flip(self) -> None:
        self.engine.flip()

    def next_buffer(self) -> torch.Tensor:
        return self.engine.msgs[1 - self.engine.cur]

    def current_buffer(self) -> torch.Tensor:
        return self.engine.current


def _split_rows(rows: int):
    """(boundary row ranges, interior range) in local 1-based row numbers."""
    if rows <= 2:
        return [(1, rows + 1)], None
    return [(1, 2), (rows, rows + 1)], (2, rows)


class StripRunner:
    """All strips in one process (one device): the exchange is a device copy.

    Exercises exactly the halo bookkeeping of ``run_rank`` without needing
    several GPUs; used by the GPU parity tests.
    """

    def __init__(self, model, strips: list):
        self.model = model
        self.strips = strips

    @classmethod
    def local(cls, model, n: int, domain: str = "sum", kernel: str = "fast", device=None):
        H = model.grid_shape[0]
        strips = [GpuStrip(model, r0, rows, domain, kernel, device)
                  for r0, rows in partition_rows(H, n)]
        return cls(model, strips)

    def run(self, iters: int) -> None:
        for _ in range(iters):
            for s in self.strips:
                s.compute(1, s.rows + 1)
            for k in range(len(self.strips) - 1):
                up, down = self.strips[k], self.strips[k + 1]
                hu = halo_views(up.next_buffer(), up.rows)
                hd = halo_views(down.next_buffer(), down.rows)
                hd["recv_above"].copy_(hu["send_down"])
                hu["recv_below"].copy_(hd["send_up"])
            for s in self.strips:
                s.flip()

    def gather_msgs4(self) -> np.ndarray:
        parts = []
        M = self.model.M
        for s in self.strips:
            cur = s.current_buffer()[:, 1:s.rows + 1, :, :M]
            parts.append(cur.double().cpu().numpy())
        full = np.concatenate(parts, axis=1)
        return full.reshape(4, -1, M)


def run_rank(strip, iters: int, rank: int, world: int, group=None, overlap: bool = True,
             compute_stream=None, interior_stream=None, dist=None, timing: list | None = None) -> None:
    """Per-rank loop of the distributed strip decomposition.

    ``strip`` is this rank's strip (rank k owns strip k, top to bottom).
    With CUDA tensors the exchange is NCCL send/recv; with CPU tensors it is
    gloo.  When ``overlap`` is set and streams are given, the interior rows run
    on ``interior_stream`` while the halos travel.  ``dist`` defaults to
    ``torch.distributed`` (tests substitute an in-process transport).

    ``timing`` (CUDA only): a list that receives one ``IterEvents`` per
    iteration -- boundary rows, halo arrival, interior rows, end -- so the
    caller can split the iteration into compute / exchange / overlap.
    """
    if dist is None:
        import torch.distributed as dist

    boundary, interior = _split_rows(strip.rows)
    cuda = strip.next_buffer().is_cuda
    rec = timing is not None and cuda
    for _ in range(iters):
        if rec:
            ev = IterEvents()
            ev.start.record()
        for lo, hi in boundary:
            strip.compute(lo, hi)
        if rec:
            ev.boundary.record()
        ops = []
        h = halo_views(strip.next_buffer(), strip.rows)
        if rank + 1 < world:
            ops.append(dist.P2POp(dist.isend, h["send_down"], rank + 1, group))
            ops.append(dist.P2POp(dist.irecv, h["recv_below"], rank + 1, group))
        if rank > 0:
            ops.append(dist.P2POp(dist.isend, h["send_up"], rank - 1, group))
            ops.append(dist.P2POp(dist.irecv, h["recv_above"], rank - 1, group))
        reqs = dist.batch_isend_irecv(ops) if ops else []
        joined = True
        if interior is not None:
            if cuda and overlap and interior_stream is not None:
                interior_stream.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(interior_stream):
                    if rec:
                        ev.interior_start.record(interior_stream)
                    strip.compute(*interior, stream=interior_stream)
                    if rec:
                        ev.interior_end.record(interior_stream)
                joined = False
            else:
                strip.compute(*interior)
        for r in reqs:
            r.wait()
        if rec:
            ev.halo.record()          # the halos have landed (stream-ordered wait)
        if not joined:
            torch.cuda.current_stream().wait_stream(interior_stream)
        if rec:
            ev.end.record()
            timing.append(ev)
        strip.flip()


class IterEvents:
    """CUDA events of one strip iteration (see run_rank)."""

    def __init__(self):
        mk = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
        self.start, self.boundary, self.halo, self.end = mk(), mk(), mk(), mk()
        self.interior_start, self.interior_end = mk(), mk()

    def split(self) -> dict:
        """ms: boundary rows, exchange (boundary done -> halos landed),
        interior rows, whole iteration, and the exchange time NOT hidden
        behind the interior rows."""
        b = self.start.elapsed_time(self.boundary)
        x = self.boundary.elapsed_time(self.halo)
        try:
            i = self.interior_start.elapsed_time(self.interior_end)
        except RuntimeError:          # no interior rows (strips of <= 2 rows)
            i = 0.0
        t = self.start.elapsed_time(self.end)
        return {"boundary_ms": b, "exchange_ms": x, "interior_ms": i, "iteration_ms": t,
                "exposed_exchange_ms": max(0.0, t - b - i)}


def summarize_timing(timing: list) -> dict:
    """Median per-iteration split over a run's IterEvents (after a sync)."""
    rows = [e.split() for e in timing]
    if not rows:
        return {}
    return {k: float(np.median([r[k] for r in rows])) for k in rows[0]}
