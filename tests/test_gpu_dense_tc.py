"""The tensor-core dense sum-product kernel (dense_tc_kernel.cu: tcgen05,
3xTF32, tensor-memory accumulators; Ms = 128 on one CTA, Ms = 256 on a CTA
pair) against the f64 oracle's reference standard update
(numba_kernels.py:35-41) and against the SIMT dense kernel.

Tolerance: the north_star bar, 1e-5 relative (reference ``rel_deviation``).
3xTF32 carries ~2^-21 per product instead of fp32's 2^-24; measured 1.4e-6
(M = 128) to 4.5e-6 (M = 256) after 3..20 iterations.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import paper_1010_0012_b200 as sbp  # noqa: E402
from paper_1010_0012_b200 import _lib as L  # noqa: E402
from paper_1010_0012_b200 import synth  # noqa: E402

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

SYNC = "synchronous"
TOL = 1e-5


@pytest.fixture
def env(monkeypatch):
    def apply(values):
        for k, v in values.items():
            monkeypatch.setenv(k, v)
        L.lib().sbp_reload_config()
    yield apply
    monkeypatch.undo()
    L.lib().sbp_reload_config()


def _run(model, iters):
    store = sbp.run_sweeps(model, iters, kernel="standard", domain="sum", schedule=SYNC)
    return store, store.engine.kernel_name


# shapes: fewer nodes than one 24-node tile, a ragged last tile, one row, one column
@pytest.mark.parametrize("name", ["C4", "C5_T9", "C5_T33"])
@pytest.mark.parametrize("shape,iters", [((2, 3), 4), ((5, 7), 3), ((13, 21), 20), ((20, 36), 6),
                                         ((1, 50), 5), ((31, 1), 5)])
def test_tensor_core_dense_matches_oracle(name, shape, iters):
    model = synth.build_config_model(synth.CONFIGS[name], height=shape[0], width=shape[1])
    store, kname = _run(model, iters)
    assert kname.startswith("dense_tc_kernel"), kname
    ref = oracle.sync_run(model, iters, "sum", "standard")
    assert oracle.rel_deviation(store.data, oracle.store_data(model, ref), floor=1e-30) <= TOL
    bt = sbp.compute_beliefs(model, store)
    rb, _ = oracle.beliefs(model, ref)
    assert oracle.rel_deviation(bt.beliefs, rb, floor=1e-30) <= TOL
    gap = oracle.top2_gap(rb)
    decided = gap > 1e-5 * rb.max(axis=1)
    assert np.array_equal(sbp.map_labels(bt)[decided], oracle.map_labels(rb)[decided])


@pytest.mark.parametrize("M", [100, 128, 200, 255])
def test_padded_label_counts(M):
    """M < Ms: the table's pad rows / columns are zero, pad labels stay zero."""
    rng = np.random.default_rng(M)
    H, W = 9, 11
    un = rng.uniform(0.05, 1.0, size=(H * W, M))
    model = sbp.GridMrf(H, W, M, un, sbp.truncated_linear_potential(M, 0.3, 6.0))
    store, kname = _run(model, 5)
    assert kname.startswith("dense_tc_kernel"), kname
    ref = oracle.store_data(model, oracle.sync_run(model, 5, "sum", "standard"))
    assert oracle.rel_deviation(store.data, ref, floor=1e-30) <= TOL
    eng = store.engine
    assert float(eng.current[:, 1:eng.rows + 1, :, M:].abs().max()) == 0.0 if eng.Ms > M else True


@pytest.mark.parametrize("name", ["C4", "C5_T9"])
def test_deep_pipeline_per_cluster(name, env):
    """Few clusters, many tiles each: the producers' item counter lets warps run
    ahead of the MMA, which once aliased an mbarrier parity (a warp two uses of
    a slot ahead overwrote live operand rows).  Bits must not depend on the
    launch geometry, and must match the oracle."""
    model = synth.build_config_model(synth.CONFIGS[name], height=40, width=50)   # 84 tiles
    ref = oracle.store_data(model, oracle.sync_run(model, 3, "sum", "standard"))
    outs = []
    for cap in (None, "1", "2", "5"):
        env({"SBP_MAX_BLOCKS": cap} if cap else {})
        store, kname = _run(model, 3)
        assert kname.startswith("dense_tc_kernel"), kname
        outs.append(store.engine.msgs4())
        assert oracle.rel_deviation(store.data, ref, floor=1e-30) <= TOL, cap
    for o in outs[1:]:
        np.testing.assert_array_equal(outs[0], o)


def test_tensor_core_and_simt_dense_agree(env):
    model = synth.build_config_model(synth.CONFIGS["C5_T17"], height=12, width=19)
    a, ka = _run(model, 10)
    env({"SBP_DENSE_TC": "0"})
    b, kb = _run(model, 10)
    assert ka.startswith("dense_tc_kernel") and kb.startswith("dense_iter_kernel"), (ka, kb)
    assert oracle.rel_deviation(a.data, b.data, floor=1e-30) <= TOL


@pytest.mark.parametrize("name", ["C4", "C5_T9", "C5_T33"])
def test_bf16_correction_variant(name, env):
    """SBP_DENSE_TC=2 (opt-in): the two correction products of the split run in
    bf16 (kind::f16) into the same accumulator -- a third fewer MMAs; measured
    4.7e-6 (M = 128) / 5.7e-6 (M = 256) from the oracle, still inside the bar."""
    env({"SBP_DENSE_TC": "2"})
    model = synth.build_config_model(synth.CONFIGS[name], height=13, width=21)
    store, kname = _run(model, 20)
    assert kname.startswith("dense_tc_kernel") and "BF16" in kname, kname
    ref = oracle.store_data(model, oracle.sync_run(model, 20, "sum", "standard"))
    assert oracle.rel_deviation(store.data, ref, floor=1e-30) <= TOL


def test_asymmetric_table_keeps_the_simt_kernel():
    """One resident table serves both orientations only if it is symmetric."""
    M, H, W = 128, 6, 7
    rng = np.random.default_rng(3)
    d = sbp.truncated_linear_potential(M, 0.5, 5.0).densify().table.copy()
    d[3, 9] *= 0.5                                    # f(3, 9) != f(9, 3)
    pot = sbp.sparse_from_dense(d, fbar=float(d[0, -1]))
    model = sbp.GridMrf(H, W, M, rng.uniform(0.1, 1.0, size=(H * W, M)), pot)
    store, kname = _run(model, 4)
    assert kname.startswith("dense_iter_kernel"), kname
    ref = oracle.store_data(model, oracle.sync_run(model, 4, "sum", "standard"))
    assert oracle.rel_deviation(store.data, ref, floor=1e-30) <= TOL


def test_degenerate_message_reports_the_reference_edge(env):
    """A node whose unaries underflow in fp32 products sends messages that
    cannot be normalised: same DegenerateMessageError(edge=) as the SIMT kernel."""
    M, H, W = 128, 5, 6
    rng = np.random.default_rng(5)
    un = rng.uniform(0.1, 1.0, size=(H * W, M))
    un[2 * W + 3] = 1e-42        # times three 1/128 messages: 0 in fp32
    model = sbp.GridMrf(H, W, M, un, sbp.truncated_linear_potential(M, 0.5, 4.0))
    edges = []
    for tc in ("1", "0"):
        env({"SBP_DENSE_TC": tc})
        with pytest.raises(sbp.DegenerateMessageError) as ei:
            sbp.run_sweeps(model, 3, kernel="standard", domain="sum", schedule=SYNC)
        edges.append(ei.value.edge)
    assert edges[0] == edges[1]


def test_full_size_c5_iteration_budget():
    """C5 at BASELINE size (1024 x 1024, M = 256): messages stay normalised
    and the labels agree with the banded kernel's wherever both are decided
    (the full-size goldens pin the banded kernel, tests/test_gpu_fullsize.py)."""
    cfg = synth.CONFIGS["C5_T9"]
    from paper_1010_0012_b200.engine import GridEngine
    vals = synth.config_values(cfg, "sum")
    a = GridEngine(synth.StripModel(cfg), "sum", "standard", values=vals)
    assert a.kernel_name.startswith("dense_tc_kernel")
    a.step(cfg.iters)
    la = a.labels().cpu().numpy()
    cur = a.current[:, 2:a.rows, 1:-1]        # interior nodes: all four slots are real messages
    sums = cur.sum(dim=-1)
    assert float((sums - 1).abs().max()) < 1e-5
    del a, cur, sums
    torch.cuda.empty_cache()
    b = GridEngine(synth.StripModel(cfg), "sum", "fast", values=vals)
    b.step(cfg.iters)
    lb = b.labels().cpu().numpy()
    assert (la != lb).mean() < 1e-4     # near-ties only
