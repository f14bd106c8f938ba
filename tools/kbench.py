"""Kernel-level timing of one config: ms per synchronous iteration and the
achieved fraction of the HBM roofline (algorithmic bytes / time).

    python tools/kbench.py C4 sum [iters]
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1010_0012_b200 import synth  # noqa: E402
from paper_1010_0012_b200.engine import GridEngine  # noqa: E402

name, domain = sys.argv[1], sys.argv[2]
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
kernel = sys.argv[4] if len(sys.argv) > 4 else "fast"
cfg = synth.CONFIGS[name]
model = synth.StripModel(cfg)
eng = GridEngine(model, domain, kernel, values=synth.config_values(cfg, domain))
eng.step(3)
torch.cuda.synchronize()
evs = []
eng.step(iters, events=evs)
torch.cuda.synchronize()
ms = [a.elapsed_time(b) / k for a, b, k in evs]
steady = sorted(ms)[len(ms) // 2]
H, W, M = cfg.height, cfg.width, cfg.M
B = 4 * M * (H * W + 2 * cfg.n_directed)
pot = model.shared_potential
F = cfg.n_directed * 2 * (pot.nnz + 2 * M) if kernel != "standard" else cfg.n_directed * 2 * M * M
peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
print(json.dumps({"config": name, "domain": domain, "kernel": kernel, "kernel_name": eng.kernel_name, "plan": eng.plan.kind_name,
                  "R": eng.plan.R, "median_ms": steady, "min_ms": min(ms),
                  "GBps": B / steady / 1e6, "hbm_frac": B / steady / 1e6 / peak,
                  "TFLOPs": F / steady / 1e9, "updates_per_s": cfg.n_directed / steady * 1e3}))
