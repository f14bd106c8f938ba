"""The public multi-GPU entry points (`distributed.run_sweeps_strips` and
`distributed.gather_labels`) across 2 and 3 CPU ranks over gloo.

Each rank's strip computes with the f64 oracle (test infrastructure; the GPU
strip is `strips.GpuStrip`, same interface); everything else is the product
code path: the balanced row partition, `run_rank`'s boundary / halo /
interior loop, and the padded label gather to rank 0.  The gathered labels
must equal the whole-grid run's labels exactly.
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
from paper_1010_0012_b200.distributed import gather_labels, run_sweeps_strips
from paper_1010_0012_b200.strips import partition_rows


def node_labels(values, msgs, domain):
    """Per-node argmax of g * prod incoming (sum) / log g + sum incoming (max);
    ghost slots hold the identity.  msgs: (4, n, M) in slot order."""
    if domain == "sum":
        b = values * msgs[0] * msgs[1] * msgs[2] * msgs[3]
    else:
        b = values + msgs[0] + msgs[1] + msgs[2] + msgs[3]
    return np.argmax(b, axis=1)


class OracleStripEngine:
    """A row strip computed by the f64 oracle, with the strip + engine surface
    run_sweeps_strips / gather_labels use (compute, flip, next_buffer,
    reset, labels, ...)."""

    def __init__(self, model, r0, rows, domain):
        H, W = model.grid_shape
        self.H, self.W, self.M = H, W, model.M
        self.r0, self.rows, self.domain = r0, rows, domain
        vals = model.unaries if domain == "sum" else model.log_unaries
        self.values = np.ascontiguousarray(vals[r0 * W:(r0 + rows) * W])
        self.init = oracle.init_msgs(H, W, model.M, domain, r0, rows)
        self.ori = oracle.oriented_pots(model, domain, "fast")
        self.device = torch.device("cpu")
        self.engine = self
        self.reset()

    # strip surface (strips.run_rank)
    def compute(self, lo, hi, stream=None):
        bad = oracle.sync_iterate_local(self.H, self.W, self.M, self.r0, self.rows, lo, hi,
                                        self.domain, "fast", self.values,
                                        self.bufs[self.cur].numpy(),
                                        self.bufs[1 - self.cur].numpy(), self.ori)
        assert bad < 0

    def flip(self):
        self.cur = 1 - self.cur

    def next_buffer(self):
        return self.bufs[1 - self.cur]

    # engine surface (distributed.py)
    def reset(self):
        self.bufs = [torch.from_numpy(self.init.copy()), torch.from_numpy(self.init.copy())]
        self.cur = 0

    def step(self, n):
        for _ in range(n):
            self.compute(1, self.rows + 1)
            self.flip()

    def raise_if_degenerate(self):
        pass

    def labels(self):
        cur = self.bufs[self.cur].numpy()[:, 1:self.rows + 1].reshape(4, -1, self.M)
        return torch.from_numpy(node_labels(self.values, cur, self.domain).astype(np.int32))


def _worker(rank, world, port, H, W, iters, domain, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        model = synth.build_config_model(synth.CONFIGS["C2"], height=H, width=W)
        r0, rows = partition_rows(H, world)[rank]
        strip = OracleStripEngine(model, r0, rows, domain)
        eng = run_sweeps_strips(model, iters, domain=domain, strip=strip)
        labels = gather_labels(eng)
        if rank == 0:
            np.save(os.path.join(out_dir, "labels.npy"), labels)
        else:
            assert labels is None
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,domain", [(2, "sum"), (3, "max")])
def test_run_sweeps_strips_and_gather_labels(tmp_path, world, domain):
    H, W, iters = 13, 17, 7          # 13 rows over 3 ranks: uneven strips (5, 4, 4)
    mp.spawn(_worker, args=(world, _free_port(), H, W, iters, domain, str(tmp_path)),
             nprocs=world, join=True)
    got = np.load(tmp_path / "labels.npy")
    model = synth.build_config_model(synth.CONFIGS["C2"], height=H, width=W)
    msgs4 = oracle.sync_run(model, iters, domain, "fast", nthreads=1)
    vals = model.unaries if domain == "sum" else model.log_unaries
    want = node_labels(np.asarray(vals), msgs4, domain)
    assert got.shape == (H * W,) and got.dtype == np.int64
    np.testing.assert_array_equal(got, want)
