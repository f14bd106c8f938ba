"""Parity report: GPU (fp32) vs the bit-pinned f64 oracle on every BASELINE
config.  C1 and C2 run at full size; C3, C4 and C5 on reduced grids with the
config's M, potential, iteration count and noise (the oracle is a CPU
program); full-size C3/C4/C5 are covered by the light-cone tests.

    python tools/parity_report.py > profiles/r01_parity.jsonl
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import oracle  # noqa: E402
import paper_1010_0012_b200 as sbp  # noqa: E402
from paper_1010_0012_b200 import synth  # noqa: E402

CASES = [("C1", "sum", None), ("C1", "max", None), ("C2", "sum", None), ("C2", "max", None),
         ("C3", "max", (96, 128)), ("C4", "sum", (48, 160))] + \
        [(f"C5_T{T}", d, (24, 40)) for T in (2, 5, 9, 17, 33) for d in ("sum", "max")]


def max_abs_rel(a, b):
    both = np.isneginf(a) & np.isneginf(b)
    d = np.where(both, 0.0, np.abs(a - b))
    return float(d.max()), float((d / np.maximum(1.0, np.abs(b))).max())


for schedule in ("synchronous", "sequential"):
    for name, domain, size in CASES:
        cfg = synth.CONFIGS[name]
        H, W = size if size else (cfg.height, cfg.width)
        model = synth.build_config_model(cfg, height=H, width=W)
        iters = cfg.iters if schedule == "synchronous" else min(cfg.iters, 10)
        if schedule == "synchronous":
            ref4 = oracle.sync_run(model, iters, domain, "fast")
            store = sbp.run_sweeps(model, iters, domain=domain, schedule="synchronous")
        else:
            ref4, _ = oracle.seq_run(model, iters, domain, "fast")
            store = sbp.run_sweeps(model, iters, domain=domain)
        ref = oracle.store_data(model, ref4)
        row = {"config": name, "domain": domain, "schedule": schedule, "grid": [H, W],
               "M": cfg.M, "iterations": iters, "kernel": store.engine.kernel_name}
        if domain == "sum":
            row["message_rel_dev"] = oracle.rel_deviation(store.data, ref, floor=1e-30)
            bt = sbp.compute_beliefs(model, store)
            rb, _ = oracle.beliefs(model, ref4)
            row["belief_rel_dev"] = oracle.rel_deviation(bt.beliefs, rb, floor=1e-30)
            scores, ref_scores = bt.beliefs, rb
            gap = oracle.top2_gap(rb)
            decided = gap > 1e-5 * rb.max(axis=1)
        else:
            row["message_abs_dev"], row["message_dev_rel1"] = max_abs_rel(store.data, ref)
            s = sbp.compute_max_marginals(model, store)
            rs = oracle.max_marginals(model, ref4)
            row["score_abs_dev"], row["score_dev_rel1"] = max_abs_rel(s, rs)
            scores, ref_scores = s, rs
            decided = oracle.top2_gap(rs) > 1e-4
        lab = sbp.map_labels(scores)
        ref_lab = np.argmax(ref_scores, axis=1)
        row["nodes"] = int(lab.size)
        row["label_mismatch_decided"] = int(((lab != ref_lab) & decided).sum())
        row["label_mismatch_all"] = int((lab != ref_lab).sum())
        row["near_ties_excluded"] = int((~decided).sum())
        mism = lab != ref_lab
        # f64 top-2 gap at the nodes whose labels differ: ~1e-15 means an
        # exact tie of the real-valued scores (sums of multiples of 0.1)
        row["max_gap_at_mismatch"] = float(oracle.top2_gap(ref_scores)[mism].max()) if mism.any() else 0.0
        print(json.dumps(row), flush=True)
