"""Full-size parity report: every BASELINE config at its grid size and
iteration count against the reference-computed fixtures of tests/golden/full
(the checks of tests/test_gpu_fullsize.py, with the measured numbers printed).

    python tools/fullsize_report.py > profiles/r02_fullsize_parity.jsonl
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1010_0012_b200 import synth  # noqa: E402
from paper_1010_0012_b200.engine import SEQUENTIAL, SYNCHRONOUS, GridEngine  # noqa: E402

FULL = ROOT / "tests" / "golden" / "full"
MAN = json.loads((FULL / "manifest_full.json").read_text())


def max_dev(a, b):
    d = np.where(np.isneginf(a) & np.isneginf(b), 0.0, np.abs(a - b) / np.maximum(1.0, np.abs(b)))
    return float(d.max())


eng = None
key = None
for name in sorted(MAN["cases"]):
    e = MAN["cases"][name]
    z = np.load(FULL / f"{name}.npz")
    dom = e["domain"]
    sched = SEQUENTIAL if e["schedule"] == "seq" else SYNCHRONOUS
    if key != (e["config"], dom, sched):
        eng = None
        torch.cuda.empty_cache()
        cfg = synth.CONFIGS[e["config"]]
        eng = GridEngine(synth.StripModel(cfg), dom, "fast", values=synth.config_values(cfg, dom),
                         schedule=sched)
        key = (e["config"], dom, sched)
    eng.reset()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    eng.step(e["iters"])
    ev1.record()
    torch.cuda.synchronize()
    eng.raise_if_degenerate()
    H, W = e["grid"]
    M = e["M"]
    labels = eng.labels().cpu().numpy().astype(np.int64)
    ref = z["labels"].astype(np.int64)
    near, gap, rowmax = z["near_nodes"], z["near_gap"], z["near_rowmax"]
    band = 1e-5 * rowmax if dom == "sum" else np.full(len(near), 1e-4)
    tied = near[gap <= band]
    decided = np.ones(H * W, dtype=bool)
    decided[tied] = False
    diff = labels != ref
    nodes = z["sample_nodes"]
    r, c = nodes // W, nodes % W
    cur = eng.current
    got = cur[:, torch.as_tensor(r + 1, device=cur.device), torch.as_tensor(c, device=cur.device),
              :M].double().cpu().numpy()
    b, zz, _, _ = eng.beliefs_device(want_labels=False)
    gb = b[torch.as_tensor(nodes, device=b.device)].double().cpu().numpy()
    out = {"case": name, "config": e["config"], "domain": dom, "schedule": e["schedule"],
           "grid": [H, W], "M": M, "iterations": e["iters"], "kernel": eng.kernel_name,
           "gpu_ms": ev0.elapsed_time(ev1), "nodes": H * W,
           "label_mismatch_decided": int((diff & decided).sum()),
           "label_mismatch_all": int(diff.sum()), "tie_band_nodes": int(len(tied)),
           "sampled_nodes": int(len(nodes))}
    if dom == "sum":
        out["msg_rel_dev"] = oracle.rel_deviation(got, z["sample_msgs"], floor=1e-30)
        out["belief_rel_dev"] = oracle.rel_deviation(gb, z["sample_scores"], floor=1e-30)
    else:
        out["msg_dev"] = max_dev(got, z["sample_msgs"])
        out["score_dev"] = max_dev(gb, z["sample_scores"])
    print(json.dumps(out), flush=True)
