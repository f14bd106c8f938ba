"""Host-side logic that needs no GPU: C ABI exports, potential planning,
edge-id bookkeeping, API validation."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import oracle
import paper_1010_0012_b200 as sbp
from paper_1010_0012_b200 import _lib as L
from paper_1010_0012_b200 import engine, plan, synth
from paper_1010_0012_b200.model import (SparseTruncatedPotential, grid_edges,
                                        sparse_from_dense, truncated_linear_potential)

ROOT = Path(__file__).resolve().parents[1]


def test_library_exports_every_header_symbol():
    header = (ROOT / "include" / "sbp.h").read_text()
    declared = set(re.findall(r"SBP_API\s+[\w\s\*]*?\b(sbp_\w+)\s*\(", header))
    assert declared, "no declarations parsed"
    lib = ctypes.CDLL(str(L.LIB_PATH))
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(L.exported_symbols())
    # host-only entry points are callable without a GPU
    assert lib.sbp_version() == 1
    l = L.lib()
    assert [l.sbp_padded_labels(m) for m in (1, 8, 9, 16, 33, 128, 200, 256)] == \
        [8, 8, 16, 16, 64, 128, 256, 256]


def test_struct_layout_matches_header():
    # sbp_grid: 7 ints; sbp_potential: 5 ints, 2 floats, 2x65 floats, 6 pointers
    assert ctypes.sizeof(L.SbpGrid) == 28
    assert L.SbpPotential.fbar.offset == 20
    assert L.SbpPotential.band_w.offset == 28
    assert L.SbpPotential.ell_idx.offset == 28 + 2 * 65 * 4 + 4  # 8-byte pointer alignment


@pytest.mark.parametrize("name", sorted(synth.CONFIGS))
@pytest.mark.parametrize("domain", ["sum", "max"])
def test_config_potentials_plan_as_bands(name, domain):
    cfg = synth.CONFIGS[name]
    pot = cfg.build_potential()
    Ms = L.lib().sbp_padded_labels(cfg.M)
    pl = plan.plan_potential(pot, domain, "fast", cfg.M, Ms)
    assert pl.kind == L.SBP_POT_BAND
    assert 2 * pl.R + 1 == pot.m          # reference m = 2*ceil(T) - 1
    use = pot.to_log() if domain == "max" else pot
    dense = use.densify().table
    # every stored band weight reproduces the dense table
    for o, table in enumerate((dense, dense.T)):
        for d in range(-pl.R, pl.R + 1):
            xj = np.arange(max(0, -d), min(cfg.M, cfg.M - d))
            vals = table[xj + d, xj]
            expect = vals - use.fbar if domain == "sum" else vals
            assert np.all(expect == pl.band_w[o, d + pl.R])
    assert pl.madds_per_update == pot.nnz + 2 * cfg.M


def test_non_toeplitz_potential_plans_as_ell():
    rng = np.random.default_rng(0)
    M = 11
    table = rng.uniform(0.2, 1.0, size=(M, M))
    table[np.abs(np.subtract.outer(np.arange(M), np.arange(M))) > 2] = 0.1
    pot = sparse_from_dense(table, fbar=0.1)
    pl = plan.plan_potential(pot, "sum", "fast", M, 16)
    assert pl.kind == L.SBP_POT_ELL and pl.m_max == pot.m
    # ELL rows reproduce the CSC lists (orientation 0) and the transpose (1)
    for o, sp in enumerate((pot, pot.transpose())):
        for xj in range(M):
            lo, hi = sp.col_indptr[xj], sp.col_indptr[xj + 1]
            n = hi - lo
            np.testing.assert_array_equal(pl.ell_idx[o, :n, xj], sp.col_indices[lo:hi])
            np.testing.assert_array_equal(pl.ell_w[o, :n, xj], sp.col_residuals[lo:hi])
            assert (pl.ell_w[o, n:, xj] == 0).all()


def test_standard_plan_is_dense_table():
    pot = truncated_linear_potential(6, 1.0, 2.0)
    pl = plan.plan_potential(pot, "max", "standard", 6, 8)
    assert pl.kind == L.SBP_POT_DENSE and pl.m_max == 6
    t = pot.to_log().densify().table
    np.testing.assert_array_equal(pl.ell_w[0, :, :6], t)
    np.testing.assert_array_equal(pl.ell_w[1, :, :6], t.T)
    assert pl.madds_per_update == 36


def test_toeplitz_detection_rejects_holes():
    M = 8
    pot = truncated_linear_potential(M, 1.0, 3.0)
    # drop one entry of column 4: no longer a full band
    keep = np.ones(pot.nnz, dtype=bool)
    keep[pot.col_indptr[4]] = False
    cols = np.repeat(np.arange(M), np.diff(pot.col_indptr))
    indptr = np.concatenate(([0], np.cumsum(np.bincount(cols[keep], minlength=M))))
    holed = SparseTruncatedPotential(M, pot.fbar, indptr, pot.col_indices[keep],
                                     pot.col_values[keep])
    assert plan.toeplitz_band(holed.col_indptr, holed.col_indices, holed.col_residuals, M,
                              0.0) is None
    assert plan.plan_potential(holed, "sum", "fast", M, 8).kind == L.SBP_POT_ELL


@pytest.mark.parametrize("H,W", [(1, 1), (1, 6), (5, 1), (3, 4), (6, 5)])
def test_edge_bookkeeping(H, W):
    edges = grid_edges(H, W)
    model = sbp.GridMrf(H, W, 2, np.ones((H * W, 2)), truncated_linear_potential(2, 1.0, 1.5))
    store = engine.MessageStore(model, "sum")
    for e, (a, b) in enumerate(edges):
        assert engine._edge_endpoints(H, W, 2 * e) == (a, b)
        assert engine._edge_endpoints(H, W, 2 * e + 1) == (b, a)
        assert store.edge_id(a, b) == 2 * e and store.edge_id(b, a) == 2 * e + 1
    with pytest.raises(KeyError):
        store.edge_id(0, H * W + 5)


def test_grid_edges_reference_order():
    # mrf.py:401-411: node-major, (n, n+1) then (n, n+W)
    expect = []
    H, W = 3, 4
    for r in range(H):
        for c in range(W):
            n = r * W + c
            if c + 1 < W:
                expect.append((n, n + 1))
            if r + 1 < H:
                expect.append((n, n + W))
    assert [tuple(e) for e in grid_edges(H, W)] == expect


def test_run_sweeps_validation_without_gpu():
    model = synth.build_config_model(synth.CONFIGS["C1"], height=4, width=6)
    with pytest.raises(NotImplementedError):
        sbp.run_sweeps(model, 2, schedule=object())     # custom pass orders
    if not __import__("torch").cuda.is_available():
        with pytest.raises(RuntimeError):               # no CPU fallback
            sbp.run_sweeps(model, 2)
    with pytest.raises(ValueError):
        sbp.run_sweeps(model, 2, kernel="bogus", schedule="synchronous")
    with pytest.raises(ValueError):
        sbp.run_sweeps(model, -1, schedule="synchronous")
    pot = SparseTruncatedPotential(3, 0.5, np.array([0, 1, 1, 1]), np.array([0]),
                                   np.array([0.25]))      # value below floor
    m = sbp.GridMrf(1, 2, 3, np.ones((2, 3)), pot)
    with pytest.raises(sbp.UnsafePotentialError):
        sbp.run_sweeps(m, 1, domain="max", schedule="synchronous")
    # no edges / zero sweeps: uniform store, nothing launched
    one = sbp.GridMrf(1, 1, 3, np.array([[1.0, 2.0, 1.0]]), truncated_linear_potential(3, 1, 2))
    st = sbp.run_sweeps(one, 5, schedule="synchronous")
    assert st.data.shape == (0, 3) and st.stats.sweeps_run == 0
    bt = sbp.compute_beliefs(one, st)
    np.testing.assert_allclose(bt.beliefs, [[0.25, 0.5, 0.25]])
    st0 = sbp.run_sweeps(model, 0, schedule="synchronous")
    assert np.all(st0.data == 1.0 / model.M)


def test_oracle_is_not_imported_by_product():
    import subprocess
    import sys
    code = ("import sys, paper_1010_0012_b200 as p; import paper_1010_0012_b200.engine, "
            "paper_1010_0012_b200.plan, paper_1010_0012_b200.synth; "
            "assert 'oracle' not in sys.modules, 'product imported the oracle'")
    subprocess.run([sys.executable, "-c", code], check=True, cwd=str(ROOT))
    for f in (ROOT / "paper_1010_0012_b200").rglob("*.py"):
        src = f.read_text()
        assert "import oracle" not in src and "from oracle" not in src, f


def test_oracle_sync_matches_per_edge_composition():
    """Tiny model: the C oracle's synchronous iteration equals a direct
    restatement of the reference per-edge API (compute_h -> update -> normalize)."""
    model = synth.build_config_model(synth.CONFIGS["C1"], height=3, width=4)
    pot = model.shared_potential
    H, W, M = 3, 4, model.M
    msgs4 = oracle.local_to_msgs4(oracle.init_msgs(H, W, M, "sum"))
    out = oracle.sync_run(model, 1, "sum", "fast", nthreads=1)
    ori = [pot, pot.transpose()]
    for r in range(H):
        for c in range(W):
            n = r * W + c
            for d, (ok, dst, excl, ws, o) in enumerate(
                    [(c + 1 < W, n + 1, 2, 1, 0), (c > 0, n - 1, 1, 2, 1),
                     (r + 1 < H, n + W, 3, 0, 0), (r > 0, n - W, 0, 3, 1)]):
                if not ok:
                    continue
                h = model.unaries[n].copy()
                for k in range(4):
                    if k != excl:
                        h *= msgs4[k, n]
                sp = ori[o]
                S = 0.0
                for x in range(M):
                    S += h[x]
                res = np.empty(M)
                for xj in range(M):
                    acc = sp.fbar * S
                    for k in range(sp.col_indptr[xj], sp.col_indptr[xj + 1]):
                        acc += sp.col_residuals[k] * h[sp.col_indices[k]]
                    res[xj] = acc
                s = 0.0
                for x in range(M):
                    s += res[x]
                np.testing.assert_array_equal(out[ws, dst], res * (1.0 / s))


def _band_structs(cfg_name, domain):
    cfg = synth.CONFIGS[cfg_name]
    Ms = L.lib().sbp_padded_labels(cfg.M)
    pl = plan.plan_potential(cfg.build_potential(), domain, "fast", cfg.M, Ms)

    class _E:   # the fields _make_pot_struct reads for a band plan
        dom = L.SBP_SUM if domain == "sum" else L.SBP_MAX
    s = engine.GridEngine._make_pot_struct(_E(), pl)
    g = L.SbpGrid(cfg.height, cfg.width, cfg.M, Ms, 0, cfg.height, L.SBP_DEVICE_AUTO)
    return g, s, pl


def _plan_name(cfg_name, domain, sequential=False):
    L.lib().sbp_reload_config()      # the knobs are read once per process
    g, s, _ = _band_structs(cfg_name, domain)
    buf = ctypes.create_string_buffer(128)
    mode = {False: 0, True: 1}.get(sequential, sequential)
    L.check(L.lib().sbp_plan_name(ctypes.byref(g), ctypes.byref(s), mode, buf, 128))
    return buf.value.decode()


def test_fused_plan_names():
    # mode 2 = sbp_iterate_fused; label sets below 32 have no fused kernel and
    # report the one-iteration kernel
    assert _plan_name("C4", "sum", 2) == "band_fused_kernel<sum,VL=16,LP=8,R=7,rolled>"
    assert _plan_name("C3", "max", 2) == "band_fused_kernel<max,VL=8,LP=8,R=3>"
    assert _plan_name("C5_T2", "sum", 2) == "band_fused_kernel<sum,VL=16,LP=16,R=1>"
    assert _plan_name("C1", "sum", 2) == _plan_name("C1", "sum", 0)


def test_iterate_fused_validates_without_touching_the_device():
    g, s, _ = _band_structs("C4", "sum")
    lib = L.lib()
    words = lib.sbp_fused_stamp_words(ctypes.byref(g))
    assert words == 4 * g.rows * g.W
    p = ctypes.c_void_p(0x1000)   # never dereferenced: validation fails first

    def call(levels=2, epoch=1, lag=4, rounds=2, ptr=p, pot=s):
        return lib.sbp_iterate_fused(ctypes.byref(g), ctypes.byref(pot), ptr, ptr, ptr, levels,
                                     0, 0, ptr, epoch, lag, rounds, ptr, None)
    assert call(levels=0) == L.SBP_EINVAL
    assert call(levels=5) == L.SBP_EINVAL
    assert call(lag=1) == L.SBP_EINVAL
    assert call(rounds=0) == L.SBP_EINVAL
    assert call(epoch=0) == L.SBP_EINVAL
    assert call(ptr=None) == L.SBP_EINVAL
    ell = L.SbpPotential()
    ell.kind, ell.domain = L.SBP_POT_ELL, L.SBP_SUM
    assert call(pot=ell) == L.SBP_EUNSUPPORTED


def test_default_fusion_policy(monkeypatch):
    monkeypatch.delenv("SBP_FUSE", raising=False)
    for name, domain, want in [("C5_T2", "sum", 3), ("C5_T2", "max", 1), ("C4", "sum", 1),
                               ("C5_T9", "sum", 1)]:
        g, _, pl = _band_structs(name, domain)
        assert engine._default_fuse(domain, g.Ms, pl) == want, name
    monkeypatch.setenv("SBP_FUSE", "2")
    g, _, pl = _band_structs("C4", "sum")
    assert engine._default_fuse("sum", g.Ms, pl) == 2


@pytest.mark.parametrize("name,domain,expect", [
    ("C4", "sum", "band_iter_tap_kernel<sum,VL=16,LP=8,R=8>"),
    ("C3", "max", "band_iter_staged_kernel<max,VL=8,LP=8,R=3>"),
    ("C2", "sum", "band_iter_kernel<sum,VL=8,LP=4,R=2>"),
    ("C5_T5", "sum", "band_iter_staged_kernel<sum,VL=16,LP=16,R=4>"),
    ("C5_T9", "sum", "band_iter_tap_kernel<sum,VL=16,LP=16,R=8>"),
    ("C5_T9", "max", "band_iter_tap2_kernel<max,VL=8,LP=32,R=8>"),
    ("C5_T17", "sum", "band_iter_tap2_kernel<sum,VL=8,LP=32,R=16>"),
    ("C5_T17", "max", "band_iter_tap2_kernel<max,VL=8,LP=32,R=16>"),
    ("C5_T33", "sum", "band_iter_tap2_kernel<sum,VL=8,LP=32,R=32>"),
    ("C5_T33", "max", "band_iter_tap2_kernel<max,VL=8,LP=32,R=32,rolled>"),
])
def test_default_kernel_choice(name, domain, expect):
    # host-only: names the instantiation sbp_iterate would launch
    assert _plan_name(name, domain) == expect


def test_plan_name_reports_the_fallback(monkeypatch):
    # plain VL=16 is not compiled for R=16: the launch falls back to VL=8 and
    # the reported name must say so (it did not, once)
    monkeypatch.setenv("SBP_TAP", "0")
    monkeypatch.setenv("SBP_STAGED", "0")
    monkeypatch.setenv("SBP_BAND_VL", "16")
    assert _plan_name("C5_T17", "sum") == "band_iter_kernel<sum,VL=8,LP=32,R=16>"
    assert _plan_name("C4", "sum") == "band_iter_kernel<sum,VL=16,LP=8,R=7,rolled>"
    monkeypatch.setenv("SBP_BAND_VL", "8")
    assert _plan_name("C4", "sum") == "band_iter_kernel<sum,VL=8,LP=16,R=7,rolled>"
    monkeypatch.setenv("SBP_ROLL_MIN_R", "99")
    assert _plan_name("C4", "sum") == "band_iter_kernel<sum,VL=8,LP=16,R=7>"


@pytest.mark.parametrize("M,T", [(16, 10.0), (16, 12.0), (32, 18.0), (32, 30.0)])
def test_band_without_compiled_radius_plans_as_ell(M, T):
    """a Toeplitz band whose radius has no compiled kernel below Ms
    (Ms=16, R=9..15; Ms=32, R=17..31) must plan the general ELL kernel, not a
    band launch that fails with 'no band kernel'."""
    pot = truncated_linear_potential(M, 0.5, T)
    Ms = L.lib().sbp_padded_labels(M)
    R, _ = plan.toeplitz_band(pot.col_indptr, pot.col_indices, pot.col_residuals, M, 0.0)
    assert R > 8 and L.lib().sbp_band_radius(Ms, R) == 0
    pl = plan.plan_potential(pot, "sum", "fast", M, Ms)
    assert pl.kind == L.SBP_POT_ELL
    # a compiled radius still plans as a band
    assert plan.plan_potential(truncated_linear_potential(M, 0.5, 3.0), "sum", "fast", M,
                               Ms).kind == L.SBP_POT_BAND


def _dense_name(Ms, domain, same_pointer, env=None, monkeypatch=None):
    for k, v in (env or {}).items():
        monkeypatch.setenv(k, v)
    L.lib().sbp_reload_config()
    s = L.SbpPotential()
    s.kind = L.SBP_POT_DENSE
    s.domain = L.SBP_SUM if domain == "sum" else L.SBP_MAX
    s.dense_t[0] = 0x1000                      # never dereferenced by sbp_plan_name
    s.dense_t[1] = 0x1000 if same_pointer else 0x2000
    g = L.SbpGrid(64, 64, Ms, Ms, 0, 64, L.SBP_DEVICE_AUTO)
    buf = ctypes.create_string_buffer(128)
    L.check(L.lib().sbp_plan_name(ctypes.byref(g), ctypes.byref(s), 0, buf, 128))
    return buf.value.decode()


def test_dense_kernel_choice(monkeypatch):
    """Sum-product with ONE table pointer for both orientations (a symmetric
    table) runs on the tensor cores at Ms = 128 / 256; everything else keeps
    the tiled SIMT kernel (include/sbp.h, sbp_potential.dense_t)."""
    assert _dense_name(128, "sum", True) == "dense_tc_kernel<sum,Ms=128,3xTF32>"
    assert _dense_name(256, "sum", True) == "dense_tc_kernel<sum,Ms=256,3xTF32>"
    assert _dense_name(256, "sum", False) == "dense_iter_kernel<sum,Ms=256>"
    assert _dense_name(64, "sum", True) == "dense_iter_kernel<sum,Ms=64>"
    assert _dense_name(256, "max", True) == "dense_iter_kernel<max,Ms=256>"
    assert _dense_name(128, "sum", True, {"SBP_DENSE_TC": "0"}, monkeypatch) == \
        "dense_iter_kernel<sum,Ms=128>"
    monkeypatch.undo()
    L.lib().sbp_reload_config()
