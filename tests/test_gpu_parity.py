"""GPU parity: the sm_100a path (through libsbp.so) against the f64 oracle.

Tolerances (north_star: fp32 beliefs/messages within 1e-5 relative, MAP
labels identical except at exact ties):
* sum-product messages and beliefs: reference ``rel_deviation``
  (cli.py:35-40) <= 1e-5 over entries >= 1e-30 (fp32 cannot hold the f64
  tail below that);
* max-sum messages / scores (log domain): |gpu - ref| <= 1e-5 * max(1, |ref|);
* labels: equal wherever the f64 top-2 gap exceeds the fp32 tie band
  (sum: 1e-5 relative to the node's largest belief; max: 1e-4 absolute).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import paper_1010_0012_b200 as sbp  # noqa: E402
from golden_util import GOLDEN, load_case, manifest  # noqa: E402
from paper_1010_0012_b200 import synth  # noqa: E402

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

MAN = manifest()
SUM_TOL = 1e-5
MAX_TOL = 1e-5
SYNC = "synchronous"


def max_dev(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    both_inf = np.isneginf(a) & np.isneginf(b)
    d = np.where(both_inf, 0.0, np.abs(a - b) / np.maximum(1.0, np.abs(b)))
    return float(d.max()) if d.size else 0.0


def assert_labels(gpu_labels, ref_scores, domain):
    ref_labels = np.argmax(ref_scores, axis=1)
    gap = oracle.top2_gap(ref_scores)
    if domain == "sum":
        decided = gap > 1e-5 * ref_scores.max(axis=1)
    else:
        decided = gap > 1e-4
    bad = (gpu_labels != ref_labels) & decided
    assert not bad.any(), f"{bad.sum()} decided labels differ (of {decided.sum()})"
    return int((~decided).sum())


def check_run(model, iters, domain, kernel="fast", ref_msgs4=None):
    """Run GPU + oracle (unless given) and compare store, beliefs, labels."""
    if ref_msgs4 is None:
        ref_msgs4 = oracle.sync_run(model, iters, domain, kernel)
    store = sbp.run_sweeps(model, iters, kernel=kernel, domain=domain, schedule=SYNC)
    ref_store = oracle.store_data(model, ref_msgs4)
    if domain == "sum":
        assert oracle.rel_deviation(store.data, ref_store, floor=1e-30) <= SUM_TOL
        bt = sbp.compute_beliefs(model, store)
        rb, rz = oracle.beliefs(model, ref_msgs4)
        assert oracle.rel_deviation(bt.beliefs, rb, floor=1e-30) <= SUM_TOL
        assert oracle.rel_deviation(bt.normalizers, rz) <= 1e-4
        assert_labels(sbp.map_labels(bt), rb, "sum")
        np.testing.assert_array_equal(sbp.map_labels(store), sbp.map_labels(bt))
    else:
        assert max_dev(store.data, ref_store) <= MAX_TOL
        s = sbp.compute_max_marginals(model, store)
        rs = oracle.max_marginals(model, ref_msgs4)
        assert max_dev(s, rs) <= MAX_TOL
        assert_labels(sbp.map_labels(s), rs, "max")
        assert (store.data.max(axis=1) == 0.0).all()
    return store


SMALL = sorted(n for n, e in MAN["cases"].items() if e["kind"] == "sync" and "degenerate" not in e
               and (GOLDEN / f"{n}.npz").exists()
               and "msgs4" in np.load(GOLDEN / f"{n}.npz").files)


@pytest.mark.parametrize("name", SMALL)
def test_golden_small_cases(name):
    e = MAN["cases"][name]
    model, z = load_case(name)
    if model.n_edges == 0:
        pytest.skip("no edges")
    if e["kernel"] == "pruned":
        # the lossy Fig. 3 demo (out of scope): without the floor
        # messages decay geometrically, below fp32 range within a few
        # iterations; parity is checked over the first two
        check_run(model, 2, e["domain"], "pruned")
        return
    check_run(model, e["iters"], e["domain"], e["kernel"], ref_msgs4=z["msgs4"])


@pytest.mark.parametrize("domain", ["sum", "max"])
def test_c1(domain):
    model = synth.build_config_model(synth.CONFIGS["C1"])
    check_run(model, 10, domain)


@pytest.mark.parametrize("domain", ["sum", "max"])
def test_c2(domain):
    model = synth.build_config_model(synth.CONFIGS["C2"])
    check_run(model, 50, domain)


def test_c3_reduced_grid():
    cfg = synth.CONFIGS["C3"]
    model = synth.build_config_model(cfg, height=96, width=128)
    check_run(model, 100, "max")


@pytest.mark.parametrize("T", [2, 5, 9, 17, 33])
@pytest.mark.parametrize("domain", ["sum", "max"])
def test_c5_reduced_grid(T, domain):
    model = synth.build_config_model(synth.CONFIGS[f"C5_T{T}"], height=24, width=40)
    check_run(model, 20, domain)


def test_c4_reduced_grid():
    model = synth.build_config_model(synth.CONFIGS["C4"], height=48, width=160)
    check_run(model, 100, "sum")


@pytest.mark.parametrize("kernel,iters", [("standard", 10), ("pruned", 2)])
@pytest.mark.parametrize("domain", ["sum", "max"])
def test_other_kernels_c1(kernel, iters, domain):
    model = synth.build_config_model(synth.CONFIGS["C1"], height=24, width=32)
    check_run(model, iters, domain, kernel)


def test_fast_equals_standard_max_bitwise():
    """Reference claim (bp.py:325-333): fast max-sum == standard bitwise."""
    model = synth.build_config_model(synth.CONFIGS["C2"], height=40, width=56)
    a = sbp.run_sweeps(model, 15, kernel="fast", domain="max", schedule=SYNC).data
    b = sbp.run_sweeps(model, 15, kernel="standard", domain="max", schedule=SYNC).data
    np.testing.assert_array_equal(a, b)


def test_deterministic_and_store_layout():
    model = synth.build_config_model(synth.CONFIGS["C2"], height=64, width=96)
    s1 = sbp.run_sweeps(model, 7, schedule=SYNC)
    s2 = sbp.run_sweeps(model, 7, schedule=SYNC)
    np.testing.assert_array_equal(s1.data, s2.data)
    # gather order == reference _grid_store_to_messages over the msgs4 layout
    np.testing.assert_array_equal(s1.data, oracle.store_data(model, s1.engine.msgs4()))
    s1.check_normalized(atol=1e-5)


@pytest.mark.parametrize("name", ["sync_degenerate_sum", "sync_degenerate_band_sum"])
def test_degenerate_message_raises_with_edge(name):
    e = MAN["cases"][name]
    model, _ = load_case(name)
    with pytest.raises(sbp.DegenerateMessageError) as ei:
        sbp.run_sweeps(model, e["iters"], schedule=SYNC)
    ids = e["degenerate"]["directed_edge_ids"]
    store = sbp.MessageStore(model, "sum")
    assert store.edge_id(*ei.value.edge) == min(ids)


@pytest.mark.parametrize("name", sorted(n for n, e in MAN["cases"].items() if e["kind"] == "exact"))
def test_chain_exact_marginals(name):
    model, z = load_case(name)
    W = model.grid_shape[1]
    bt = sbp.compute_beliefs(model, sbp.run_sweeps(model, W + 1, schedule=SYNC))
    assert oracle.rel_deviation(bt.beliefs, z["marginals"]) <= SUM_TOL
    if MAN["cases"][name]["map_unique"]:
        s = sbp.compute_max_marginals(model, sbp.run_sweeps(model, W + 1, domain="max",
                                                            schedule=SYNC))
        np.testing.assert_array_equal(sbp.map_labels(s), z["map_config"])


def test_convergence_tol_matches_oracle():
    model = synth.build_config_model(synth.CONFIGS["C1"], height=16, width=20)
    tol = 1e-3
    _, st = oracle.sync_run(model, 200, "sum", "fast", convergence_tol=tol, return_stats=True)
    store = sbp.run_sweeps(model, 200, schedule=SYNC, convergence_tol=tol)
    assert store.stats.converged and st["converged"]
    assert abs(store.stats.sweeps_run - st["iterations"]) <= 1


def test_row_strips_with_halo_exchange_bitwise():
    """Two strips (the multi-GPU decomposition) on one device, halo rows
    copied between them each iteration, equal the whole-grid run bitwise."""
    from paper_1010_0012_b200.strips import StripRunner
    model = synth.build_config_model(synth.CONFIGS["C2"], height=37, width=50)
    full = sbp.run_sweeps(model, 9, schedule=SYNC).engine.msgs4()
    for n_strips in (2, 3):
        runner = StripRunner.local(model, n_strips, "sum", "fast")
        runner.run(9)
        np.testing.assert_array_equal(runner.gather_msgs4(), full)


@pytest.mark.slow
@pytest.mark.parametrize("name,domain,t", [("C4", "sum", 6), ("C3", "max", 8),
                                           ("C5_T33", "sum", 4), ("C5_T9", "max", 5)])
def test_full_size_light_cone(name, domain, t):
    """Full-size BASELINE grids: after t iterations a message depends only on
    the t-neighbourhood, so oracle runs on crops of radius t+1 pin the
    full-size GPU result at sampled nodes (borders, corners, random)."""
    cfg = synth.CONFIGS[name]
    model = synth.build_config_model(cfg)
    store = sbp.run_sweeps(model, t, domain=domain, schedule=SYNC)
    gpu = store.engine
    H, W = model.grid_shape
    rng = np.random.default_rng(1)
    pts = [(0, 0), (H - 1, W - 1), (0, W // 3), (H // 2, 0), (H // 2, W // 2)] + \
        [(int(rng.integers(0, H)), int(rng.integers(0, W))) for _ in range(3)]
    cur = gpu.current
    for (r, c) in pts:
        r0, r1 = max(0, r - t - 1), min(H, r + t + 2)
        c0, c1 = max(0, c - t - 1), min(W, c + t + 2)
        # crop borders that are real grid borders stay borders; interior crop
        # edges are > t away from (r, c), so they cannot influence it yet
        idx = (np.arange(r0, r1)[:, None] * W + np.arange(c0, c1)[None, :]).ravel()
        crop = sbp.GridMrf(r1 - r0, c1 - c0, model.M, model.unaries[idx], model.shared_potential,
                           log_unaries=model.log_unaries[idx])
        ref = oracle.sync_run(crop, t, domain, "fast")
        n_crop = (r - r0) * (c1 - c0) + (c - c0)
        got = cur[:, r + 1, c, :model.M].double().cpu().numpy()
        if domain == "sum":
            assert oracle.rel_deviation(got, ref[:, n_crop], floor=1e-30) <= SUM_TOL
        else:
            assert max_dev(got, ref[:, n_crop]) <= MAX_TOL


@pytest.mark.slow
def test_c4_full_size_invariants():
    model = synth.build_config_model(synth.CONFIGS["C4"])
    eng = sbp.GridEngine(model, "sum", "fast")
    eng.step(100)
    torch.cuda.synchronize()
    eng.raise_if_degenerate()
    cur = eng.current[:, 1:-1, :, :model.M]
    sums = cur.sum(dim=-1)
    H, W = model.grid_shape
    # real slots sum to 1; ghost slots stay exactly 1 per entry
    real = torch.ones_like(sums, dtype=torch.bool)
    real[0, 0, :] = False
    real[1, :, 0] = False
    real[2, :, W - 1] = False
    real[3, H - 1, :] = False
    assert (sums[real] - 1).abs().max().item() < 1e-5
    assert (cur[~real] == 1).all()
    lab = eng.labels()
    assert lab.shape == (H * W,) and int(lab.min()) >= 0 and int(lab.max()) < model.M


@pytest.mark.parametrize("name", ["C3", "C4", "C5_T9"])
@pytest.mark.parametrize("domain", ["sum", "max"])
def test_dense_tiled_kernel(name, domain):
    """The tiled dense comparison kernel (Ms >= 32) against the oracle's
    reference standard update."""
    model = synth.build_config_model(synth.CONFIGS[name], height=20, width=36)
    check_run(model, 6, domain, "standard")


def test_fast_equals_standard_max_bitwise_m256():
    model = synth.build_config_model(synth.CONFIGS["C5_T9"], height=12, width=20)
    a = sbp.run_sweeps(model, 8, kernel="fast", domain="max", schedule=SYNC).data
    b = sbp.run_sweeps(model, 8, kernel="standard", domain="max", schedule=SYNC).data
    np.testing.assert_array_equal(a, b)


def _run_subprocess(env_extra, name, domain, iters, out):
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, **env_extra)
    subprocess.run([sys.executable, str(root / "tools" / "dump_case.py"), name, domain,
                    str(iters), "24", "40", str(out)], check=True, env=env, cwd=str(root))
    return np.load(out)


@pytest.mark.parametrize("name,domain", [("C4", "sum"), ("C3", "max"), ("C5_T33", "sum")])
def test_rolled_and_unrolled_kernels_agree_bitwise(tmp_path, name, domain):
    """The rolled (one band copy) and unrolled kernels perform identical arithmetic."""
    # same lane width (VL=8) so both variants use the same reduction trees
    a = _run_subprocess({"SBP_ROLL_MIN_R": "1", "SBP_BAND_VL": "8", "SBP_STAGED": "0",
                         "SBP_TAP": "0"}, name, domain, 7, tmp_path / "a.npy")
    b = _run_subprocess({"SBP_ROLL_MIN_R": "99", "SBP_BAND_VL": "8", "SBP_STAGED": "0",
                         "SBP_TAP": "0"}, name, domain, 7, tmp_path / "b.npy")
    np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("domain", ["sum", "max"])
def test_device_stereo_unaries(domain):
    """build_stereo_mrf builds the unaries on the GPU from the image pair; they
    equal the reference-formula host table (f64 -> f32), and BP on them
    matches the oracle."""
    from paper_1010_0012_b200.engine import GridEngine
    left, right, _ = synth.noisy_stereo_pair(40, 72, 32, 5.0, 9)
    params = sbp.StereoParams(M=32, alpha=0.5, T_b=3.0, beta=0.1, T_u=255.0)
    model = sbp.build_stereo_mrf(left, right, params)
    eng = GridEngine(model, domain, "fast")
    host = model.unaries if domain == "sum" else model.log_unaries
    if domain == "max":
        host = host - host.max(axis=1, keepdims=True)
    got = eng.values[:, :, :32].reshape(-1, 32).double().cpu().numpy()
    want = host.astype(np.float32).astype(np.float64)
    ulps = np.abs(got - want) / np.maximum(np.spacing(np.abs(want).astype(np.float32)), 1e-45)
    assert ulps.max() <= 1.0          # f64 exp on the device vs numpy: <= 1 f32 ulp
    check_run(model, 12, domain)



@pytest.mark.parametrize("name,domain", [("C4", "sum"), ("C3", "max"), ("C5_T9", "sum")])
def test_staged_and_register_kernels_agree_bitwise(tmp_path, name, domain):
    """The TMA-staged variant only changes how inputs reach the registers."""
    a = _run_subprocess({"SBP_STAGED": "1", "SBP_BAND_VL": "8", "SBP_TAP": "0"}, name, domain,
                        7, tmp_path / "a.npy")
    b = _run_subprocess({"SBP_STAGED": "0", "SBP_BAND_VL": "8", "SBP_TAP": "0"}, name, domain,
                        7, tmp_path / "b.npy")
    np.testing.assert_array_equal(a, b)



@pytest.mark.parametrize("name", sorted(n for n, e in MAN["cases"].items() if e["kind"] == "pe_sync"))
def test_per_edge_potentials_synchronous(name):
    e = MAN["cases"][name]
    model, z = load_case(name)
    store = sbp.run_sweeps(model, e["iters"], kernel=e["kernel"], domain=e["domain"],
                           schedule=SYNC)
    if e["domain"] == "sum":
        assert oracle.rel_deviation(store.data, z["store"], floor=1e-30) <= SUM_TOL
    else:
        assert max_dev(store.data, z["store"]) <= MAX_TOL


@pytest.mark.parametrize("M,T", [(1, 1.0), (2, 1.5), (3, 2.0), (7, 2.0), (13, 3.0), (24, 4.0),
                                 (100, 5.0), (129, 3.0), (200, 9.0)])
@pytest.mark.parametrize("domain", ["sum", "max"])
def test_label_counts_and_padding(M, T, domain):
    """Odd and non-power-of-two M (padded label stride), M=1, band radius close
    to M: the padding must stay an exact no-op."""
    H, W = 7, max(M, 9) if M <= 16 else 11
    left, right, _ = synth.noisy_stereo_pair(H, max(W, M), M, 5.0, M)
    u, lu = synth.stereo_unary_field(left, right, M, 0.1, 255.0)
    model = sbp.GridMrf(H, max(W, M), M, u, sbp.truncated_linear_potential(M, 0.6, T),
                        log_unaries=lu)
    check_run(model, 6, domain)


@pytest.mark.parametrize("H,W", [(1, 2), (2, 1), (1, 40), (40, 1), (3, 3)])
def test_degenerate_shapes(H, W):
    u = np.random.default_rng(H * 100 + W).uniform(0.05, 1.0, size=(H * W, 16))
    model = sbp.GridMrf(H, W, 16, u, sbp.truncated_linear_potential(16, 1.0, 3.0))
    for domain in ("sum", "max"):
        check_run(model, 5, domain)


@pytest.mark.slow
def test_large_grid_64bit_offsets():
    """A grid whose message buffers exceed 2^31 floats (int64 offsets):
    4100 x 4100 nodes, M=32 -> 2.15e9 floats per buffer."""
    H = W = 4100
    M = 32
    rng = np.random.default_rng(0)
    cfg = synth.CONFIGS["C2"]
    values = rng.uniform(0.1, 1.0, size=(H * W, M))
    from paper_1010_0012_b200.engine import GridEngine
    model = synth.StripModel(cfg)
    model.grid_shape = (H, W)
    model.n_edges = H * (W - 1) + W * (H - 1)
    eng = GridEngine(model, "sum", "fast", values=values)
    eng.step(3)
    torch.cuda.synchronize()
    eng.raise_if_degenerate()
    # the last node's messages are normalised and finite
    last = eng.current[:, H, W - 1, :M]
    assert torch.isfinite(last).all()
    assert abs(float(last[0].sum()) - 1.0) < 1e-5 and abs(float(last[1].sum()) - 1.0) < 1e-5
    # and the bottom-right 12x12 corner matches the oracle on the corner crop
    # (after 3 iterations a message depends on the 3-neighbourhood only)
    r0, c0 = H - 12, W - 12
    idx = (np.arange(r0, H)[:, None] * W + np.arange(c0, W)[None, :]).ravel()
    crop = sbp.GridMrf(12, 12, M, values[idx], model.shared_potential)
    ref = oracle.sync_run(crop, 3, "sum", "fast")
    got = eng.current[:, H - 5 + 1, W - 5:W, :M].double().cpu().numpy()   # rows H-5.., local +1
    want = ref[:, (12 - 5) * 12 + 7: (12 - 5) * 12 + 12]
    assert oracle.rel_deviation(got, want, floor=1e-30) <= SUM_TOL


class RefLikeModel:
    """Attribute surface of the reference ``sparsebp.MrfModel`` (mrf.py:288-398):
    plain ``potentials`` list (one object repeated), ``edges`` array, lazy
    ``log_unaries`` -- no ``shared_potential`` shortcut."""

    def __init__(self, model):
        self.M = model.M
        self.unaries = np.asarray(model.unaries)
        self._lu = np.asarray(model.log_unaries)
        self.edges = np.asarray(model.edges)
        self.potentials = [model.shared_potential] * len(self.edges)
        self.grid_shape = model.grid_shape

    @property
    def log_unaries(self):
        return self._lu

    @property
    def n_nodes(self):
        return self.unaries.shape[0]

    @property
    def n_edges(self):
        return len(self.edges)


@pytest.mark.parametrize("schedule", [None, "synchronous"])
def test_reference_shaped_model_object(schedule):
    base = synth.build_config_model(synth.CONFIGS["C2"], height=18, width=30)
    ref_like = RefLikeModel(base)
    for domain in ("sum", "max"):
        a = sbp.run_sweeps(ref_like, 6, domain=domain, schedule=schedule).data
        b = sbp.run_sweeps(base, 6, domain=domain, schedule=schedule).data
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("name,domain,variant", [
    ("C5_T33", "sum", {"SBP_TAP_ROLLED": "1"}), ("C5_T33", "max", {"SBP_TAP_ROLLED": "1"}),
    ("C5_T17", "max", {"SBP_TAP_STAGED": "1"}), ("C5_T17", "sum", {"SBP_TAP_STAGED": "0"}),
    ("C5_T9", "max", {"SBP_TAP_STAGED": "0", "SBP_TAP_ROLLED": "0"}),
    ("C5_T33", "sum", {"SBP_TAP_STAGED": "2"}), ("C5_T33", "max", {"SBP_TAP_STAGED": "2"}),
    ("C5_T17", "sum", {"SBP_TAP_STAGED": "3"}), ("C5_T9", "max", {"SBP_TAP_STAGED": "3"}),
])
def test_tap_and_shuffle_kernels_agree_bitwise(tmp_path, name, domain, variant):
    """The shared-memory-tap kernels (tap_kernel.cuh) only change how a lane
    reads its neighbours' h values: same lane width => identical bits."""
    a = _run_subprocess({"SBP_TAP": "1", "SBP_TAP_VL": "8", **variant}, name, domain, 7,
                        tmp_path / "a.npy")
    b = _run_subprocess({"SBP_TAP": "0", "SBP_BAND_VL": "8", "SBP_STAGED": "0",
                         "SBP_ROLL_MIN_R": "99"}, name, domain, 7, tmp_path / "b.npy")
    np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("schedule", ["synchronous", "sequential"])
@pytest.mark.parametrize("domain", ["sum", "max"])
@pytest.mark.parametrize("pot_kind", ["band", "ell"])
def test_fused_convergence_delta_is_exact(schedule, domain, pot_kind):
    """The fused convergence test (sbp_iterate_delta / sbp_sweep_delta) equals
    max |new - old| over every message slot, computed explicitly."""
    from paper_1010_0012_b200.engine import GridEngine
    model = synth.build_config_model(synth.CONFIGS["C2"], height=30, width=44)
    if pot_kind == "ell":   # a non-Toeplitz potential plans as ELL
        d = model.shared_potential.densify().table.copy()
        d[3, 5] = 0.5 * (d[3, 5] + 1.0)         # still >= the floor: max-sum safe
        model = sbp.GridMrf(30, 44, model.M, model.unaries,
                            sbp.sparse_from_dense(d, fbar=model.shared_potential.fbar),
                            log_unaries=model.log_unaries)
    eng = GridEngine(model, domain, "fast", schedule=schedule)
    assert eng.fused_delta and eng.plan.kind_name == pot_kind
    eng.reset(full=True)
    delta = torch.zeros(1, dtype=torch.float32, device=eng.device)
    M = model.M
    for _ in range(4):
        prev = eng.current[:, 1:-1, :, :M].clone()      # real rows (no halo rows)
        delta.zero_()
        eng.step(1, delta=delta)
        diff = (eng.current[:, 1:-1, :, :M] - prev).abs()
        want = float(torch.nan_to_num(diff, nan=0.0).max())
        assert float(delta.item()) == want


def test_convergence_tol_sequential_matches_oracle():
    model = synth.build_config_model(synth.CONFIGS["C1"], height=16, width=20)
    tol = 1e-4
    store = sbp.run_sweeps(model, 100, convergence_tol=tol)      # reference default schedule
    assert store.stats.converged
    n = store.stats.sweeps_run
    # the reference's rule: the first sweep whose max change is below tol
    a, _ = oracle.seq_run(model, n - 1, "sum", "fast")
    b, _ = oracle.seq_run(model, n, "sum", "fast")
    assert np.abs(b - a).max() < tol * 1.01
    if n > 2:
        c, _ = oracle.seq_run(model, n - 2, "sum", "fast")
        assert np.abs(a - c).max() >= tol * 0.99


@pytest.mark.parametrize("domain", ["sum", "max"])
def test_streamed_upload_wavefront_is_bitwise(monkeypatch, domain):
    """Host unaries streamed in row bands under a row wavefront of iterations
    (GridEngine.run_streamed) give the same bits as upload-then-iterate."""
    from paper_1010_0012_b200 import engine as E
    model = synth.build_config_model(synth.CONFIGS["C2"], height=61, width=47)
    monkeypatch.setenv("SBP_STREAM", "0")
    want = sbp.run_sweeps(model, 23, domain=domain, schedule=SYNC).engine.msgs4()
    monkeypatch.setenv("SBP_STREAM", "1")
    monkeypatch.setattr(E, "STREAM_MIN_BYTES", 0)
    for bands in (1, 3, 8, 61):
        eng = E.GridEngine(model, domain, "fast", defer_values=True)
        eng.run_streamed(23, bands=bands)
        np.testing.assert_array_equal(eng.msgs4(), want)
    store = sbp.run_sweeps(model, 23, domain=domain, schedule=SYNC)
    np.testing.assert_array_equal(store.engine.msgs4(), want)


@pytest.mark.parametrize("M,T", [(16, 12.0), (32, 20.0)])
@pytest.mark.parametrize("domain", ["sum", "max"])
def test_uncompiled_band_radius_runs_on_ell(M, T, domain):
    left, right, _ = synth.noisy_stereo_pair(9, 40, M, 5.0, 4)
    u, lu = synth.stereo_unary_field(left, right, M, 0.1, 255.0)
    model = sbp.GridMrf(9, 40, M, u, sbp.truncated_linear_potential(M, 0.5, T), log_unaries=lu)
    check_run(model, 8, domain)
