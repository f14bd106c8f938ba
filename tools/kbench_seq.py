"""Device time of one canonical sequential sweep (4 chained passes).

    python tools/kbench_seq.py C4 sum [sweeps]
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1010_0012_b200 import synth  # noqa: E402
from paper_1010_0012_b200.engine import SEQUENTIAL, GridEngine  # noqa: E402

name, domain = sys.argv[1], sys.argv[2]
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = synth.CONFIGS[name]
model = synth.StripModel(cfg)
eng = GridEngine(model, domain, "fast", values=synth.config_values(cfg, domain),
                 schedule=SEQUENTIAL)
eng.step(1)
torch.cuda.synchronize()
evs = []
eng.step(sweeps, events=evs)
torch.cuda.synchronize()
ms = sorted(a.elapsed_time(b) for a, b, _ in evs)[len(evs) // 2]
H, W, M = cfg.height, cfg.width, cfg.M
N = H * W
# per sweep: every directed message written once; per update the unary and two
# other incoming vectors are read (the chained one stays in registers)
B = 4 * M * cfg.n_directed * 4
print(json.dumps({"config": name, "domain": domain, "schedule": "sequential",
                  "ms_per_sweep": ms, "updates_per_s": cfg.n_directed / ms * 1e3,
                  "GBps_min_traffic": B / ms / 1e6}))
