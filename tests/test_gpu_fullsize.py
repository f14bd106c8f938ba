"""Full-size parity on every BASELINE config at its iteration count.

The GPU path at the BASELINE grid sizes (C3 768x1024 max-sum 100 it, C4
1536x2048 sum-product 100 it, C5 1024x1024 M=256 for every band width in both
domains 20 it, and C4 in the reference's sequential schedule for 50 sweeps)
against fixtures computed by the reference's own compiled update bodies at
the same size (``tests/golden/make_golden_full.py``, reference
numba_kernels.py:44-90,194-271 composed as in bp.py:587-744).

Checked per case (north_star tolerances, as in test_gpu_parity.py):
* MAP labels at every node of the grid, except nodes whose f64 top-2 gap is
  inside the fp32 tie band (sum: 1e-5 of the node's largest belief; max:
  1e-4 absolute) -- those are listed with their gaps in the fixture;
* the four incoming messages of sampled nodes: sum ``rel_deviation`` <= 1e-5
  (entries >= 1e-30), max |gpu - ref| <= 1e-5 * max(1, |ref|);
* beliefs / max-marginals of the sampled nodes to the same tolerances, and
  the sum-product normalisers Z to 1e-4 relative;
* the label histogram (a size-independent checksum of the whole label map).
"""

import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from golden_util import GOLDEN  # noqa: E402
from paper_1010_0012_b200 import synth  # noqa: E402
from paper_1010_0012_b200.engine import SEQUENTIAL, SYNCHRONOUS, GridEngine  # noqa: E402

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

FULL = GOLDEN / "full"
MAN = json.loads((FULL / "manifest_full.json").read_text()) if (FULL / "manifest_full.json").exists() \
    else {"cases": {}}
SUM_TOL = 1e-5
MAX_TOL = 1e-5


def max_dev(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    both_inf = np.isneginf(a) & np.isneginf(b)
    d = np.where(both_inf, 0.0, np.abs(a - b) / np.maximum(1.0, np.abs(b)))
    return float(d.max()) if d.size else 0.0


_engines: dict = {}


def _engine(cfg_name, domain, schedule, kernel="fast"):
    """One engine per (config, domain, schedule, kernel); the unary table is
    built on the host in f64 by the reference formula (stereo.py:82-99) and loaded."""
    key = (cfg_name, domain, schedule, kernel)
    if key not in _engines:
        _engines.clear()
        torch.cuda.empty_cache()
        cfg = synth.CONFIGS[cfg_name]
        _engines[key] = GridEngine(synth.StripModel(cfg), domain, kernel,
                                   values=synth.config_values(cfg, domain), schedule=schedule)
    return _engines[key]


@pytest.mark.parametrize("name", sorted(MAN["cases"]))
def test_full_size_against_reference(name):
    _check_case(name, "fast")


@pytest.mark.parametrize("name", [n for n in ("C4_sync_sum", "C5_T9_sync_sum", "C5_T33_sync_sum")
                                  if n in MAN["cases"]])
def test_full_size_tensor_core_dense(name):
    """kernel="standard" at full size: the dense update on the tensor cores
    (3xTF32) against the same reference fixtures -- the O(M^2) and the O(mM)
    updates are the same function (numba_kernels.py:35-54)."""
    eng = _check_case(name, "standard")
    assert eng.kernel_name.startswith("dense_tc_kernel"), eng.kernel_name


def _check_case(name, kernel):
    e = MAN["cases"][name]
    z = np.load(FULL / f"{name}.npz")
    dom = e["domain"]
    eng = _engine(e["config"], dom, SEQUENTIAL if e["schedule"] == "seq" else SYNCHRONOUS, kernel)
    eng.reset()
    eng.step(e["iters"])
    torch.cuda.synchronize()
    eng.raise_if_degenerate()
    H, W = e["grid"]
    M = e["M"]

    # labels everywhere except inside the fp32 tie band
    labels = eng.labels().cpu().numpy().astype(np.int64)
    ref_labels = z["labels"].astype(np.int64)
    near, gap, rowmax = z["near_nodes"], z["near_gap"], z["near_rowmax"]
    band = 1e-5 * rowmax if dom == "sum" else np.full(len(near), 1e-4)
    tied = near[gap <= band]
    decided = np.ones(H * W, dtype=bool)
    decided[tied] = False
    bad = (labels != ref_labels) & decided
    assert not bad.any(), f"{int(bad.sum())} decided labels differ (of {int(decided.sum())})"
    hist = np.bincount(ref_labels, minlength=M)
    assert hist.tolist() == e["label_hist"]

    # sampled nodes: incoming messages and beliefs / max-marginals
    nodes = z["sample_nodes"]
    r, c = nodes // W, nodes % W
    cur = eng.current
    got = cur[:, torch.as_tensor(r + 1, device=cur.device), torch.as_tensor(c, device=cur.device),
              :M].double().cpu().numpy()
    want = z["sample_msgs"]
    b, zz, _, _ = eng.beliefs_device(want_labels=False)
    gb = b[torch.as_tensor(nodes, device=b.device)].double().cpu().numpy()
    if dom == "sum":
        assert oracle.rel_deviation(got, want, floor=1e-30) <= SUM_TOL
        assert oracle.rel_deviation(gb, z["sample_scores"], floor=1e-30) <= SUM_TOL
        gz = zz[torch.as_tensor(nodes, device=zz.device)].cpu().numpy()
        assert oracle.rel_deviation(gz, z["sample_normalizers"]) <= 1e-4
    else:
        assert max_dev(got, want) <= MAX_TOL
        assert max_dev(gb, z["sample_scores"]) <= MAX_TOL
    return eng
