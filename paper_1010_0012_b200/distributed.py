"""Multi-GPU public entry point: one row strip per rank (torchrun, NCCL).

    import torch.distributed as dist
    dist.init_process_group("nccl")
    eng = run_sweeps_strips(model, 100, domain="sum")      # every rank
    labels = gather_labels(eng)                            # rank 0: (N,) int64

The model is the same object on every rank (e.g. ``build_stereo_mrf`` of the
image pair, whose unaries are then built on each GPU from its own image
rows).  Iterations follow ``strips.run_rank``: boundary rows, NCCL halo
rows, interior rows on a second stream.  Synchronous schedule only (the
sequential schedule's chains span the whole grid).
"""

from __future__ import annotations

import numpy as np
import torch

from .strips import GpuStrip, partition_rows, run_rank

__all__ = ["run_sweeps_strips", "gather_labels"]


def run_sweeps_strips(model, n_sweeps: int, domain: str = "sum", kernel: str = "fast",
                      group=None, device=None, values=None, strip: GpuStrip | None = None):
    """Run ``n_sweeps`` synchronous iterations over this rank's strip; returns
    the strip's engine (``.labels()``, ``.beliefs_device()``, ``.msgs4()``)."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if strip is None:
        r0, rows = partition_rows(model.grid_shape[0], world)[rank]
        strip = GpuStrip(model, r0, rows, domain, kernel, device=device, values=values)
    eng = strip.engine
    eng.reset()
    cuda = torch.device(eng.device).type == "cuda"
    interior = torch.cuda.Stream(device=eng.device) if cuda else None
    if world == 1:
        eng.step(n_sweeps)
    else:
        run_rank(strip, n_sweeps, rank, world, group=group, interior_stream=interior)
    eng.raise_if_degenerate()
    eng.strip = strip
    return eng


def gather_labels(eng, group=None) -> np.ndarray | None:
    """MAP labels of every strip, concatenated on rank 0 (None elsewhere)."""
    import torch.distributed as dist
    lab = eng.labels()
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return lab.cpu().numpy().astype(np.int64)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    H, W = eng.H, eng.W
    lab = lab.to(torch.int32)
    parts = partition_rows(H, world)
    width = max(rows for _, rows in parts) * W
    buf = torch.full((width,), -1, dtype=torch.int32, device=lab.device)
    buf[:lab.numel()] = lab
    bufs = [torch.empty_like(buf) for _ in range(world)] if rank == 0 else None
    dist.gather(buf, bufs, dst=0, group=group)
    if rank != 0:
        return None
    return np.concatenate([b[:rows * W].cpu().numpy() for b, (_, rows) in zip(bufs, parts)]
                          ).astype(np.int64)

