"""GPU checks of the reference-facing surface.

* ``MrfModel`` with the reference signature and a permuted / partly reversed
  edge list: stores in the model's own directed-edge ids, equal to what the
  reference returns (tests/golden/make_golden_api.py);
* the C-ABI stub of INTEGRATION.md, executed verbatim;
* f64 accumulation for weak smoothing over wide bands: alpha=0.1,
  T=33, M=256, 20 iterations within 1e-5 of the oracle.
"""

import re
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import paper_1010_0012_b200 as sbp  # noqa: E402
from golden_util import GOLDEN  # noqa: E402
from paper_1010_0012_b200 import synth  # noqa: E402
from paper_1010_0012_b200.model import SparseTruncatedPotential  # noqa: E402

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = Path(__file__).resolve().parents[1]
Z = np.load(GOLDEN / "api_permuted_edges.npz")


def _models():
    H, W = (int(v) for v in Z["grid_shape"])
    u = Z["unaries"]
    M = u.shape[1]
    pot = SparseTruncatedPotential(M, float(Z["pot_fbar"]), Z["pot_indptr"], Z["pot_indices"],
                                   Z["pot_values"])
    pe, off = [], 0
    for k, indptr in enumerate(Z["pe_indptr"]):
        n = int(indptr[-1])
        pe.append(SparseTruncatedPotential(M, float(Z["pe_fbar"][k]), indptr,
                                           Z["pe_indices"][off:off + n], Z["pe_values"][off:off + n]))
        off += n
    return (sbp.MrfModel(M, u, Z["edges"], pot, grid_shape=(H, W)),
            sbp.MrfModel(M, u, Z["edges"], pe, grid_shape=(H, W)))


def _close(a, b, domain):
    if domain == "sum":
        assert oracle.rel_deviation(a, b, floor=1e-30) <= 1e-5
    else:
        assert np.abs(a - b).max() <= 1e-5 * max(1.0, np.abs(b).max())


@pytest.mark.parametrize("domain", ["sum", "max"])
def test_mrfmodel_permuted_edges_shared(domain):
    shared, _ = _models()
    got = sbp.run_sweeps(shared, 3, domain=domain).data          # reference default schedule
    _close(got, Z[f"store_shared_generic_{domain}"], domain)     # every edge, bp.py:113-133
    rows = np.repeat(~Z["reversed"], 2)                           # the reference grid engine
    _close(got[rows], Z[f"store_shared_{domain}"][rows], domain)  # agrees off reversed edges


@pytest.mark.parametrize("domain", ["sum", "max"])
def test_mrfmodel_permuted_edges_per_edge(domain):
    key = f"store_per_edge_{domain}"
    if key not in Z.files:
        pytest.skip("no fixture")
    _, per_edge = _models()
    got = sbp.run_sweeps(per_edge, 3, domain=domain).data
    _close(got, Z[key], domain)


def _integration_blocks():
    text = (ROOT / "INTEGRATION.md").read_text()
    sec = text[text.index("## 2."):text.index("## 3.")]
    return re.findall(r"```python\n(.*?)```", sec, flags=re.S)


def test_integration_stub_runs_verbatim(monkeypatch):
    monkeypatch.chdir(ROOT)
    ns: dict = {}
    for block in _integration_blocks():
        exec(compile(block, "INTEGRATION.md", "exec"), ns)
    cfg = synth.CONFIGS["C2"]
    model = synth.build_config_model(cfg, height=30, width=44)
    pot = model.shared_potential
    from paper_1010_0012_b200.plan import toeplitz_band
    R, w0 = toeplitz_band(pot.col_indptr, pot.col_indices, pot.col_residuals, model.M, 0.0)
    t = pot.transpose()
    _, w1 = toeplitz_band(t.col_indptr, t.col_indices, t.col_residuals, model.M, 0.0)
    want = sbp.run_sweeps(model, 9, schedule="synchronous").engine.current
    got = ns["run_grid_gpu"](model, 9, [w0, w1], pot.fbar, R)
    torch.testing.assert_close(got[:, 1:-1], want[:, 1:-1], rtol=0, atol=0)
    got_f = ns["run_grid_gpu_fused"](model, 9, [w0, w1], pot.fbar, R)
    torch.testing.assert_close(got_f[:, 1:-1], want[:, 1:-1], rtol=0, atol=0)
    # the dense binding (tensor cores at M = 128): same bits as kernel="standard"
    m128 = synth.build_config_model(synth.CONFIGS["C4"], height=9, width=14)
    want_d = sbp.run_sweeps(m128, 4, kernel="standard", schedule="synchronous").engine
    assert want_d.kernel_name.startswith("dense_tc_kernel")
    got_d = ns["run_grid_gpu_dense"](m128, 4, m128.shared_potential.densify().table)
    torch.testing.assert_close(got_d[:, 1:-1], want_d.current[:, 1:-1], rtol=0, atol=0)


@pytest.mark.parametrize("schedule", ["synchronous", None])
def test_weak_smoothing_wide_band_f64_accumulation(schedule):
    """alpha=0.1, T=33, M=256 (fp32 accumulation drifts to 5.1e-5
    after 20 iterations).  precision='auto' picks f64 accumulation here."""
    M, H, W = 256, 20, 40
    left, right, _ = synth.noisy_stereo_pair(H, W, M, 5.0, 3)
    u, lu = synth.stereo_unary_field(left, right, M, 0.1, 255.0)
    model = sbp.GridMrf(H, W, M, u, sbp.truncated_linear_potential(M, 0.1, 33.0), log_unaries=lu)
    store = sbp.run_sweeps(model, 20, schedule=schedule)
    assert "f64" in store.engine.kernel_name
    if schedule == "synchronous":
        ref = oracle.sync_run(model, 20, "sum", "fast")
        ref_store = oracle.store_data(model, ref)
        rb, _ = oracle.beliefs(model, ref)
    else:
        ref, _ = oracle.seq_run(model, 20, "sum", "fast")
        ref_store = oracle.store_data(model, ref)
        rb, _ = oracle.beliefs(model, ref)
    dev = oracle.rel_deviation(store.data, ref_store, floor=1e-30)
    assert dev <= 1e-5, dev
    bt = sbp.compute_beliefs(model, store)
    assert oracle.rel_deviation(bt.beliefs, rb, floor=1e-30) <= 1e-5


def test_precision_auto_keeps_baseline_configs_on_bands():
    """Every BASELINE config keeps its f32 band kernel (C4's time unchanged)."""
    from paper_1010_0012_b200.plan import effective_taps
    for name, cfg in synth.CONFIGS.items():
        assert effective_taps(cfg.build_potential()) < 12, name
    model = synth.build_config_model(synth.CONFIGS["C4"], height=8, width=16)
    eng = sbp.GridEngine(model, "sum", "fast")
    assert eng.kernel_name.startswith("band_iter")
