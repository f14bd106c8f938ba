"""GPU canonical sequential sweep (the reference's default schedule,
bp.py:620-703 with schedule=None) against the reference itself (golden
fixtures from ``sparsebp.run_sweeps``) and the bit-pinned oracle."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import paper_1010_0012_b200 as sbp  # noqa: E402
from golden_util import GOLDEN, load_case, manifest  # noqa: E402
from paper_1010_0012_b200 import synth  # noqa: E402
from test_gpu_parity import assert_labels, max_dev  # noqa: E402

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

MAN = manifest()
TOL = 1e-5


def check_seq(model, sweeps, domain, ref_store=None):
    if ref_store is None:
        ref_store = oracle.store_data(model, oracle.seq_run(model, sweeps, domain, "fast")[0])
    store = sbp.run_sweeps(model, sweeps, kernel="fast", domain=domain)   # default schedule
    assert store.engine.schedule == sbp.SEQUENTIAL
    if domain == "sum":
        assert oracle.rel_deviation(store.data, ref_store, floor=1e-30) <= TOL
    else:
        assert max_dev(store.data, ref_store) <= TOL
    return store


@pytest.mark.parametrize("domain", ["sum", "max"])
def test_golden_reference_run_sweeps(domain):
    name = f"seq_small_{domain}_fast"
    e = MAN["cases"][name]
    model, z = load_case(name)
    store = check_seq(model, e["sweeps"], domain, ref_store=z["store"])
    assert store.stats.madds == e["madds"]           # reference kernel madd counter
    assert store.stats.sweeps_run == e["sweeps"]
    scores = (sbp.compute_beliefs(model, store).beliefs if domain == "sum"
              else sbp.compute_max_marginals(model, store))
    assert_labels(sbp.map_labels(scores), z["scores"], domain)


@pytest.mark.parametrize("domain", ["sum", "max"])
def test_c1_sequential(domain):
    model = synth.build_config_model(synth.CONFIGS["C1"])
    check_seq(model, 10, domain)


@pytest.mark.parametrize("domain", ["sum", "max"])
def test_c2_sequential(domain):
    model = synth.build_config_model(synth.CONFIGS["C2"])
    check_seq(model, 8, domain)


@pytest.mark.parametrize("name,domain,sweeps", [("C3", "max", 10), ("C4", "sum", 10),
                                                ("C5_T33", "sum", 5), ("C5_T9", "max", 5)])
def test_reduced_configs_sequential(name, domain, sweeps):
    model = synth.build_config_model(synth.CONFIGS[name], height=20, width=44)
    check_seq(model, sweeps, domain)


def test_sequential_degenerate_edge_matches_reference():
    e = MAN["cases"]["seq_degenerate_band_sum"]
    model, _ = load_case("seq_degenerate_band_sum")
    with pytest.raises(sbp.DegenerateMessageError) as ei:
        sbp.run_sweeps(model, e["sweeps"])
    assert list(ei.value.edge) == e["degenerate_edge"]


def test_sequential_chains_single_row_and_column():
    for (H, W) in [(1, 9), (9, 1), (2, 2)]:
        rng = np.random.default_rng(H * 31 + W)
        g = rng.uniform(0.1, 1.0, size=(H * W, 4))
        model = sbp.GridMrf(H, W, 4, g, sbp.truncated_linear_potential(4, 1.0, 2.0))
        for domain in ("sum", "max"):
            check_seq(model, 4, domain)


def test_sequential_convergence_tol():
    model = synth.build_config_model(synth.CONFIGS["C1"], height=12, width=16)
    tol = 1e-4
    ref = sbp.run_sweeps(model, 100, convergence_tol=tol)
    # oracle: iterate until the max |delta| over a sweep < tol
    msgs, prev, n = None, None, 0
    for n in range(1, 101):
        msgs, _ = oracle.seq_run(model, n, "sum", "fast")
        if prev is not None and np.abs(msgs - prev).max() < tol:
            break
        prev = msgs
    assert ref.stats.converged
    assert abs(ref.stats.sweeps_run - n) <= 1



@pytest.mark.parametrize("name", sorted(n for n, e in MAN["cases"].items() if e["kind"] == "pe_seq"))
def test_per_edge_potentials_sequential(name):
    """The reference default schedule with per-edge potentials (its generic
    engine) -- the GPU runs it with the warp-per-chain ELL kernel."""
    e = MAN["cases"][name]
    model, z = load_case(name)
    store = sbp.run_sweeps(model, e["sweeps"], kernel=e["kernel"], domain=e["domain"])
    assert store.stats.madds == e["madds"]
    if e["domain"] == "sum":
        assert oracle.rel_deviation(store.data, z["store"], floor=1e-30) <= TOL
    else:
        assert max_dev(store.data, z["store"]) <= TOL


def test_general_shared_potential_sequential():
    """A shared non-band (ELL) potential in the default schedule."""
    name = "sync_random0_sum"
    model, _ = load_case(name)
    for domain in ("sum", "max"):
        check_seq(model, 4, domain)


@pytest.mark.parametrize("kernel,sweeps", [("standard", 3), ("pruned", 1)])
@pytest.mark.parametrize("domain", ["sum", "max"])
def test_sequential_other_kernels(kernel, sweeps, domain):
    """Dense ("standard", warp-per-chain ELL kernel) and pruned (band chain
    kernel without the floor term) in the reference default schedule."""
    model = synth.build_config_model(synth.CONFIGS["C1"], height=12, width=20)
    ref = oracle.store_data(model, oracle.seq_run(model, sweeps, domain, kernel)[0])
    store = sbp.run_sweeps(model, sweeps, kernel=kernel, domain=domain)
    if domain == "sum":
        assert oracle.rel_deviation(store.data, ref, floor=1e-30) <= TOL
    else:
        assert max_dev(store.data, ref) <= TOL
