"""Host cost of the multi-GPU strip loop (strips.run_rank) against its device
time, on one GPU: one rank's strip of C4 split over N ranks (rows H/N), the
real per-iteration sequence (boundary rows, P2P ops, interior rows on a
second stream, stream joins), with a null transport in place of NCCL so no
peer is needed.  Reports host enqueue microseconds per iteration and device
milliseconds per iteration (CUDA events).

    python tools/strip_host_cost.py [N ...]
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1010_0012_b200 import synth  # noqa: E402
from paper_1010_0012_b200.strips import GpuStrip, partition_rows, run_rank, summarize_timing  # noqa: E402


class _Req:
    def wait(self):
        pass


class NullDist:
    isend, irecv = "isend", "irecv"

    class P2POp:
        def __init__(self, op, tensor, peer, group=None):
            pass

    def batch_isend_irecv(self, ops):
        return [_Req() for _ in ops]


def main():
    cfg = synth.CONFIGS["C4"]
    model = synth.StripModel(cfg)
    for n in [int(a) for a in sys.argv[1:]] or [2, 4, 8]:
        rank = 1 if n > 2 else 0          # an interior strip: two halo rows
        r0, rows = partition_rows(cfg.height, n)[rank]
        values = synth.config_values(cfg, "sum", r0=r0, rows=rows)
        strip = GpuStrip(model, r0, rows, "sum", "fast", values=values)
        # the null transport delivers no halos: give the halo rows (and every
        # slot of both buffers) valid initial messages, else NaN garbage makes
        # every message degenerate and the error-word atomics dominate
        for b in strip.engine.msgs:
            strip.engine._init(b, ghosts_only=False)
        interior = torch.cuda.Stream()
        d = NullDist()
        run_rank(strip, 5, rank, n, interior_stream=interior, dist=d)
        torch.cuda.synchronize()
        iters = 200
        t0 = time.perf_counter()
        run_rank(strip, iters, rank, n, interior_stream=interior, dist=d)
        host = (time.perf_counter() - t0) / iters         # enqueue cost, no events
        torch.cuda.synchronize()
        timing = []
        run_rank(strip, iters, rank, n, interior_stream=interior, dist=d, timing=timing)
        torch.cuda.synchronize()
        dev = summarize_timing(timing)
        strip.engine.raise_if_degenerate()
        print(json.dumps({"n_gpus": n, "strip_rows": rows, "host_us_per_iteration": host * 1e6,
                          "device": dev, "kernel": strip.engine.kernel_name}), flush=True)
        del strip
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
