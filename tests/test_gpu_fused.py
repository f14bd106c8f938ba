"""Temporally blocked iterations (sbp_iterate_fused): T synchronous iterations
in one persistent launch must give exactly the bits of T one-iteration
launches -- same arithmetic, only the order in time differs -- for every
level count, wavefront lag and work-unit size, including the first
iteration (initial messages as constants), ragged widths (partial last
segment) and a remainder launch when the iteration count is not a multiple
of T.  The unfused path is itself pinned to the oracle (test_gpu_parity)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import paper_1010_0012_b200 as sbp  # noqa: E402
from paper_1010_0012_b200 import synth  # noqa: E402
from paper_1010_0012_b200.engine import GridEngine  # noqa: E402

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _run(model, domain, iters, fuse, lag=3, rounds=1):
    eng = GridEngine(model, domain, "fast")
    eng.fuse, eng.fuse_lag, eng.fuse_rounds = fuse, lag, rounds
    eng.step(iters)
    torch.cuda.synchronize()
    return eng


CASES = [("C4", "sum", 40, 72), ("C3", "max", 37, 50), ("C5_T9", "sum", 20, 33),
         ("C5_T5", "max", 19, 24), ("C2", "sum", 29, 45), ("C2", "max", 29, 45)]


@pytest.mark.parametrize("name,domain,H,W", CASES)
@pytest.mark.parametrize("levels", [2, 3, 4])
def test_fused_equals_unfused_bitwise(name, domain, H, W, levels):
    model = synth.build_config_model(synth.CONFIGS[name], height=H, width=W)
    ref = _run(model, domain, 7, fuse=1)
    got = _run(model, domain, 7, fuse=levels)
    assert got._fused_ok, "the fused kernel did not run"
    assert got.kernel_name.startswith("band_fused_kernel")
    np.testing.assert_array_equal(got.msgs4(), ref.msgs4())
    np.testing.assert_array_equal(got.labels().cpu().numpy(), ref.labels().cpu().numpy())


@pytest.mark.parametrize("lag,rounds", [(2, 1), (2, 2), (5, 1), (4, 3)])
def test_fused_wavefront_shapes(lag, rounds):
    """Lag between levels and segment width change the schedule, not the bits;
    a wide ragged row (W = 301) has many segments and a partial last one."""
    model = synth.build_config_model(synth.CONFIGS["C4"], height=23, width=301)
    ref = _run(model, "sum", 6, fuse=1)
    got = _run(model, "sum", 6, fuse=3, lag=lag, rounds=rounds)
    assert got._fused_ok
    np.testing.assert_array_equal(got.msgs4(), ref.msgs4())


def test_fused_continues_from_previous_state():
    """Fused launches after unfused ones (and vice versa) on the same engine."""
    model = synth.build_config_model(synth.CONFIGS["C2"], height=31, width=40)
    ref = _run(model, "max", 9, fuse=1)
    eng = GridEngine(model, "max", "fast")
    eng.fuse = 1
    eng.step(2)
    eng.fuse = 4
    eng.step(5)
    eng.fuse = 1
    eng.step(1)
    eng.fuse = 2
    eng.step(1)
    np.testing.assert_array_equal(eng.msgs4(), ref.msgs4())


def test_run_sweeps_fuses_and_matches_oracle(monkeypatch):
    """With SBP_FUSE set the public API fuses iterations; results stay within
    the oracle tolerance and the per-sweep stats have one entry per sweep."""
    monkeypatch.setenv("SBP_FUSE", "3")
    model = synth.build_config_model(synth.CONFIGS["C4"], height=24, width=40)
    store = sbp.run_sweeps(model, 9, schedule="synchronous")
    assert store.engine._fused_ok
    assert store.stats.sweeps_run == 9 and len(store.stats.sweep_seconds) == 9
    ref = oracle.sync_run(model, 9, "sum", "fast")
    assert oracle.rel_deviation(store.data, oracle.store_data(model, ref), floor=1e-30) <= 1e-5


def test_fused_stamps_survive_many_launches():
    """Epoch stamps are never cleared: many launches on one engine stay exact."""
    model = synth.build_config_model(synth.CONFIGS["C3"], height=16, width=48)
    ref = _run(model, "max", 41, fuse=1)
    got = _run(model, "max", 41, fuse=2)
    assert got._epoch == 20   # 20 fused launches + one single iteration
    np.testing.assert_array_equal(got.msgs4(), ref.msgs4())
