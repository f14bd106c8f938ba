"""Pin the CPU oracle (and the host model layer) to the reference's own outputs.

Every expectation here was produced by the reference package itself
(tests/golden/make_golden.py); the oracle must reproduce the f64 results
bit-for-bit (sha256 of the arrays).  No GPU needed.
"""

import numpy as np
import pytest

import oracle
from golden_util import GOLDEN, load_case, manifest, sha, sha_raw
from paper_1010_0012_b200 import synth
from paper_1010_0012_b200.model import truncated_linear_potential

MAN = manifest()
CASES = MAN["cases"]


def _full_cases(kind):
    return sorted(n for n, e in CASES.items() if e["kind"] == kind
                  and (GOLDEN / f"{n}.npz").exists()
                  and "grid_shape" in np.load(GOLDEN / f"{n}.npz").files
                  and "degenerate" not in e
                  and "degenerate_edge" not in e)


@pytest.mark.parametrize("name", _full_cases("sync"))
def test_sync_oracle_bitwise(name):
    e = CASES[name]
    model, z = load_case(name)
    if model.n_edges == 0:
        msgs4 = oracle.local_to_msgs4(oracle.init_msgs(*model.grid_shape, model.M, e["domain"]))
    else:
        msgs4 = oracle.sync_run(model, e["iters"], e["domain"], e["kernel"], nthreads=2)
    assert sha(msgs4) == e["msgs4_sha"], name
    assert sha(oracle.store_data(model, msgs4)) == e["store_sha"]
    if e["domain"] == "sum":
        b, zs = oracle.beliefs(model, msgs4)
        assert sha(b) == e["beliefs_sha"]
        assert sha(zs) == e["normalizers_sha"]
    else:
        s = oracle.max_marginals(model, msgs4)
        assert sha(s) == e["scores_sha"]
        b = s
    assert sha_raw(oracle.map_labels(b).astype(np.int64)) == e["labels_sha"]


@pytest.mark.parametrize("name", _full_cases("seq"))
def test_seq_oracle_bitwise(name):
    e = CASES[name]
    model, z = load_case(name)
    msgs4, madds = oracle.seq_run(model, e["sweeps"], e["domain"], e["kernel"])
    assert sha(oracle.store_data(model, msgs4)) == e["store_sha"]
    assert madds == e["madds"]


def _config_model(name):
    cfg = synth.CONFIGS[name]
    model = synth.build_config_model(cfg, seed=0)
    u = MAN["unaries"][name]
    assert sha(model.unaries) == u["unaries"] and sha(model.log_unaries) == u["log_unaries"]
    return model


@pytest.mark.parametrize("name,kind", [("C1_sync_sum", "sync"), ("C1_sync_max", "sync"),
                                       ("C1_sync_sum_standard", "sync"),
                                       ("seq_C1_sum_fast", "seq"), ("seq_C1_max_fast", "seq")])
def test_c1_digests(name, kind):
    e = CASES[name]
    model = _config_model("C1")
    if kind == "sync":
        msgs4 = oracle.sync_run(model, e["iters"], e["domain"], e["kernel"])
        assert sha(msgs4) == e["msgs4_sha"]
    else:
        msgs4, madds = oracle.seq_run(model, e["sweeps"], e["domain"], e["kernel"])
        assert madds == e["madds"]
    assert sha(oracle.store_data(model, msgs4)) == e["store_sha"]
    scores = (oracle.beliefs(model, msgs4)[0] if e["domain"] == "sum"
              else oracle.max_marginals(model, msgs4))
    assert sha_raw(oracle.map_labels(scores).astype(np.int64)) == e["labels_sha"]


@pytest.mark.parametrize("name", ["C2_sync_sum", "C2_sync_max"])
def test_c2_digests(name):
    e = CASES[name]
    model = _config_model("C2")
    msgs4 = oracle.sync_run(model, e["iters"], e["domain"], e["kernel"])
    assert sha(msgs4) == e["msgs4_sha"]
    z = np.load(GOLDEN / f"{name}.npz")
    np.testing.assert_array_equal(msgs4[:, z["sample_nodes"]], z["sample_msgs"])


def test_degenerate_sync_and_seq():
    e = CASES["sync_degenerate_sum"]
    model, _ = load_case("sync_degenerate_sum")
    with pytest.raises(RuntimeError) as ei:
        oracle.sync_run(model, e["iters"], "sum", "fast")
    assert ei.value.directed_edge == min(e["degenerate"]["directed_edge_ids"])
    assert ei.value.iteration == e["degenerate"]["iteration"]
    e2 = CASES["seq_degenerate_sum"]
    with pytest.raises(RuntimeError) as ei:
        oracle.seq_run(model, e2["sweeps"], "sum", "fast")
    assert list(ei.value.edge) == e2["degenerate_edge"]


@pytest.mark.parametrize("name", sorted(n for n, e in CASES.items() if e["kind"] == "exact"))
def test_chain_exact(name):
    model, z = load_case(name)
    W = model.grid_shape[1]
    msgs4 = oracle.sync_run(model, W + 1, "sum", "fast")
    b, _ = oracle.beliefs(model, msgs4)
    assert oracle.rel_deviation(b, z["marginals"]) < 1e-9
    if CASES[name]["map_unique"]:
        s = oracle.max_marginals(model, oracle.sync_run(model, W + 1, "max", "fast"))
        np.testing.assert_array_equal(oracle.map_labels(s), z["map_config"])


def test_directed_edge_ids_match_reference_order():
    # reference ids: 2e / 2e+1 over mrf.py:401-411 edge order
    for H, W in [(1, 5), (4, 1), (3, 4), (5, 7)]:
        from paper_1010_0012_b200.model import grid_edges
        edges = grid_edges(H, W)
        ref = {}
        for e, (a, b) in enumerate(edges):
            ref[(int(a), int(b))] = 2 * e
            ref[(int(b), int(a))] = 2 * e + 1
        for r in range(H):
            for c in range(W):
                n = r * W + c
                for d, (ok, dst) in enumerate([(c + 1 < W, n + 1), (c > 0, n - 1),
                                               (r + 1 < H, n + W), (r > 0, n - W)]):
                    if ok:
                        assert oracle.directed_edge_id(H, W, r, c, d) == ref[(n, dst)]


@pytest.mark.parametrize("key", sorted(MAN["potentials"]))
def test_potentials_match_reference(key):
    e = MAN["potentials"][key]
    parts = key.split("_")
    M = int(parts[1][1:])
    alpha = float(parts[2][1:])
    if parts[0] == "linear":
        p = truncated_linear_potential(M, alpha, float(parts[3][1:]))
    else:
        p = synth.quadratic_potential(M, alpha, float(parts[3][3:]))
        assert p.to_log().maxsum_safe == e["maxsum_safe"]
    t = p.transpose()
    assert p.fbar == e["fbar"] and p.nnz == e["nnz"] and p.m == e["m"]
    assert sha_raw(p.col_indptr) == e["indptr"] and sha_raw(p.col_indices) == e["indices"]
    assert sha(p.col_values) == e["values"] and sha(p.col_residuals) == e["residuals"]
    assert sha_raw(t.col_indptr) == e["t_indptr"] and sha_raw(t.col_indices) == e["t_indices"]
    assert sha(t.col_values) == e["t_values"]
    assert p.to_log().fbar == e["log_fbar"] and sha(p.to_log().col_values) == e["log_values"]
    assert sha(p.densify().table) == e["dense"]


@pytest.mark.parametrize("key", sorted(MAN["random_dot_pair"]))
def test_random_dot_pair_matches_reference(key):
    dims, m, s = key.split("_")
    H, W = (int(v) for v in dims.split("x"))
    M, seed = int(m[1:]), int(s[1:])
    disp = synth.rect_disparity(H, W, M, np.random.default_rng(seed))
    left, right = synth.random_dot_pair(H, W, disp, seed=seed + 1)
    e = MAN["random_dot_pair"][key]
    assert sha_raw(disp) == e["disp"]
    assert sha_raw(left) == e["left"] and sha_raw(right) == e["right"]


@pytest.mark.parametrize("name,dims", [("small", (10, 14, 8, 5.0, 3)), ("C3", (768, 1024, 64, 10.0, 0))])
def test_unary_field_matches_reference(name, dims):
    H, W, M, sigma, seed = dims
    left, right, _ = synth.noisy_stereo_pair(H, W, M, sigma, seed)
    u, lu = synth.stereo_unary_field(left, right, M, 0.1, 255.0)
    e = MAN["unaries"][name]
    assert sha_raw(right) == e["right"]
    assert sha(u) == e["unaries"] and sha(lu) == e["log_unaries"]


@pytest.mark.parametrize("name", sorted(n for n, e in CASES.items()
                                        if e["kind"] in ("pe_sync", "pe_seq")))
def test_per_edge_potentials_bitwise(name):
    """Per-edge potentials: the reference generic engine (bp.py:506-584),
    synchronous composition and its own sequential run_sweeps."""
    e = CASES[name]
    model, z = load_case(name)
    if e["kind"] == "pe_sync":
        msgs4 = oracle.sync_run(model, e["iters"], e["domain"], e["kernel"], nthreads=2)
    else:
        msgs4, madds = oracle.seq_run(model, e["sweeps"], e["domain"], e["kernel"])
        assert madds == e["madds"]
    assert sha(oracle.store_data(model, msgs4)) == e["store_sha"]
