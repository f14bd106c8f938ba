"""Tensor-core dense kernel against the f64 oracle (small grids), with the SIMT
dense kernel beside it:  python tools/tc_check.py [config ...]"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
import paper_1010_0012_b200 as sbp  # noqa: E402
from paper_1010_0012_b200 import _lib, synth  # noqa: E402

names = sys.argv[1:] or ["C4", "C5_T9", "C5_T33"]
for name in names:
    for (H, W), iters in (((5, 7), 3), ((20, 36), 6), ((13, 21), 20)):
        model = synth.build_config_model(synth.CONFIGS[name], height=H, width=W)
        ref = oracle.store_data(model, oracle.sync_run(model, iters, "sum", "standard"))
        for tc in ("1", "0"):
            os.environ["SBP_DENSE_TC"] = tc
            _lib.lib().sbp_reload_config()
            store = sbp.run_sweeps(model, iters, kernel="standard", domain="sum", schedule="synchronous")
            dev = oracle.rel_deviation(store.data, ref, floor=1e-30)
            sums = store.data.sum(axis=1)
            print(f"{name} {H}x{W} it={iters} {store.engine.kernel_name}: rel dev {dev:.3e}, "
                  f"max |sum-1| {np.abs(sums - 1).max():.2e}", flush=True)
