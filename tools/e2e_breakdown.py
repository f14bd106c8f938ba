"""Where the end-to-end C4 time goes: pinned H2D of the f64 unaries, engine
setup, value conversion, 100 synchronous iterations, labels + D2H."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1010_0012_b200 as sbp  # noqa: E402
from paper_1010_0012_b200 import synth  # noqa: E402
from paper_1010_0012_b200.engine import GridEngine  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
vals = synth.config_values(cfg, "sum")
pinned = torch.empty(vals.shape, dtype=torch.float64, pin_memory=True)
pinned.numpy()[...] = vals
model = sbp.GridMrf(cfg.height, cfg.width, cfg.M, pinned.numpy(), cfg.build_potential())
out = {}
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev = pinned.to("cuda", non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    eng = GridEngine(model, "sum", "fast", values=dev)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    eng.step(cfg.iters)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    lab = eng.labels().cpu().numpy()
    t4 = time.perf_counter()
    del eng
    out = {"h2d_ms": (t1 - t0) * 1e3, "h2d_GBps": pinned.numel() * 8 / (t1 - t0) / 1e9,
           "engine_setup_ms": (t2 - t1) * 1e3, "iterations_ms": (t3 - t2) * 1e3,
           "labels_d2h_ms": (t4 - t3) * 1e3}
print(json.dumps(out))
