"""Multi-rank row-strip decomposition on CPU (gloo, world_size 2 and 3).

The per-rank loop (`strips.run_rank`) is the one the GPU path uses; here each
rank's strip computes with the f64 oracle (test infrastructure) and the halo
rows travel over gloo.  The gathered result must equal the whole-grid oracle
run bit-for-bit: the decomposition changes no arithmetic.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1010_0012_b200 import synth
from paper_1010_0012_b200.strips import partition_rows, run_rank


class OracleStrip:
    def __init__(self, model, r0, rows, domain, kernel):
        H, W = model.grid_shape
        self.H, self.W, self.M = H, W, model.M
        self.r0, self.rows = r0, rows
        self.domain, self.kernel = domain, kernel
        vals = model.unaries if domain == "sum" else model.log_unaries
        self.values = np.ascontiguousarray(vals[r0 * W:(r0 + rows) * W])
        init = oracle.init_msgs(H, W, model.M, domain, r0, rows)
        self.bufs = [torch.from_numpy(init.copy()), torch.from_numpy(init.copy())]
        self.cur = 0
        self.ori = oracle.oriented_pots(model, domain, kernel)
        self.it = 0

    def compute(self, lo, hi, stream=None):
        bad = oracle.sync_iterate_local(self.H, self.W, self.M, self.r0, self.rows, lo, hi,
                                        self.domain, self.kernel, self.values,
                                        self.bufs[self.cur].numpy(),
                                        self.bufs[1 - self.cur].numpy(), self.ori)
        assert bad < 0

    def flip(self):
        self.cur = 1 - self.cur

    def next_buffer(self):
        return self.bufs[1 - self.cur]


def _worker(rank, world, port, H, W, iters, domain, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        model = synth.build_config_model(synth.CONFIGS["C2"], height=H, width=W)
        r0, rows = partition_rows(H, world)[rank]
        strip = OracleStrip(model, r0, rows, domain, "fast")
        run_rank(strip, iters, rank, world)
        cur = strip.bufs[strip.cur].numpy()[:, 1:rows + 1]
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), cur)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,domain", [(2, "sum"), (3, "max")])
def test_strips_match_whole_grid(tmp_path, world, domain):
    H, W, iters = 11, 17, 6
    mp.spawn(_worker, args=(world, _free_port(), H, W, iters, domain, str(tmp_path)),
             nprocs=world, join=True)
    parts = [np.load(tmp_path / f"rank{k}.npy") for k in range(world)]
    got = np.concatenate(parts, axis=1).reshape(4, H * W, -1)
    model = synth.build_config_model(synth.CONFIGS["C2"], height=H, width=W)
    want = oracle.sync_run(model, iters, domain, "fast", nthreads=1)
    np.testing.assert_array_equal(got, want)


def test_partition_rows():
    assert partition_rows(10, 3) == [(0, 4), (4, 3), (7, 3)]
    assert partition_rows(1536, 8) == [(192 * k, 192) for k in range(8)]
    with pytest.raises(ValueError):
        partition_rows(2, 3)
