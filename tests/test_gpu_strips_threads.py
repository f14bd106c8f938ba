"""The CUDA branch of the multi-GPU strip loop (`strips.run_rank`: boundary
rows, halo send/recv, interior rows on a second stream, flip) with the ranks
as threads on one GPU and an in-process transport in place of NCCL.  Kernels
of different ranks never wait on one another (the transport blocks on the
host), so sharing one device is safe.  Result must equal the whole-grid run
bit for bit."""

import queue
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1010_0012_b200 as sbp  # noqa: E402
from paper_1010_0012_b200 import synth  # noqa: E402
from paper_1010_0012_b200.strips import (GpuStrip, partition_rows, run_rank,  # noqa: E402
                                         summarize_timing)

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


class _Req:
    def __init__(self, fn):
        self.fn = fn

    def wait(self):
        self.fn()


class FakeDist:
    """isend/irecv/batch_isend_irecv over host queues; copies on the caller's
    current CUDA stream, like NCCL's stream-ordered P2P."""

    def __init__(self):
        self.q = {}
        self.lock = threading.Lock()
        self.isend, self.irecv = "isend", "irecv"

    def _chan(self, src, dst):
        with self.lock:
            return self.q.setdefault((src, dst), queue.Queue())

    class P2POp:
        def __init__(self, op, tensor, peer, group=None):
            self.op, self.tensor, self.peer = op, tensor, peer

    def batch_isend_irecv(self, ops):
        me = threading.current_thread().rank
        reqs = []
        for op in ops:
            if op.op == "isend":
                torch.cuda.current_stream().synchronize()
                self._chan(me, op.peer).put(op.tensor.clone())
                reqs.append(_Req(lambda: None))
            else:
                ch = self._chan(op.peer, me)
                reqs.append(_Req(lambda ch=ch, t=op.tensor: t.copy_(ch.get(timeout=60))))
        return reqs


@pytest.mark.parametrize("world,domain,cfg_name,kernel", [
    (2, "sum", "C2", "fast"), (3, "max", "C2", "fast"),
    # kernel="standard" on the tensor cores: row sub-ranges with halo rows, the
    # boundary and interior launches on two streams (each allocates tensor memory)
    (2, "sum", "C4", "standard"), (3, "sum", "C5_T9", "standard")])
def test_threaded_ranks_match_whole_grid(world, domain, cfg_name, kernel):
    cfg = synth.CONFIGS[cfg_name]
    H, W, iters = 29, 48, 7
    model = synth.build_config_model(cfg, height=H, width=W)
    whole = sbp.run_sweeps(model, iters, kernel=kernel, domain=domain, schedule="synchronous")
    if kernel == "standard":
        assert whole.engine.kernel_name.startswith("dense_tc_kernel")
    full = whole.engine.msgs4()
    fake = FakeDist()
    parts = [None] * world
    splits = [None] * world
    errors = []

    def rank_main(rank):
        threading.current_thread().rank = rank
        try:
            r0, rows = partition_rows(H, world)[rank]
            strip = GpuStrip(model, r0, rows, domain, kernel)
            interior = torch.cuda.Stream()
            timing = []
            with torch.cuda.stream(torch.cuda.Stream()):
                run_rank(strip, iters, rank, world, interior_stream=interior, dist=fake,
                         timing=timing)
                torch.cuda.current_stream().synchronize()
            interior.synchronize()
            assert len(timing) == iters
            splits[rank] = summarize_timing(timing)
            parts[rank] = strip.current_buffer()[:, 1:rows + 1, :, :model.M].double().cpu().numpy()
        except Exception as exc:   # surfaced below
            errors.append(exc)

    threads = [threading.Thread(target=rank_main, args=(k,)) for k in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=120)
    assert not errors, errors
    got = np.concatenate(parts, axis=1).reshape(4, H * W, model.M)
    np.testing.assert_array_equal(got, full)
    for sp in splits:     # per-rank compute / exchange / overlap split (bench --gpus N)
        assert sp["iteration_ms"] > 0 and sp["boundary_ms"] > 0 and sp["interior_ms"] > 0
        assert sp["exposed_exchange_ms"] <= sp["iteration_ms"]


def test_run_sweeps_strips_single_rank():
    """The multi-GPU public entry point at world size 1 equals run_sweeps."""
    from paper_1010_0012_b200.distributed import gather_labels, run_sweeps_strips
    left, right, _ = synth.noisy_stereo_pair(30, 50, 16, 5.0, 4)
    model = sbp.build_stereo_mrf(left, right, sbp.StereoParams(M=16, T_b=2, beta=0.1, T_u=255))
    eng = run_sweeps_strips(model, 9)
    want = sbp.map_labels(sbp.run_sweeps(model, 9, schedule="synchronous"))
    np.testing.assert_array_equal(gather_labels(eng), want)
