"""Launch-bound small configs (C1, C2): wall time of run_sweeps on a
device-resident model vs the summed kernel time."""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1010_0012_b200 as sbp  # noqa: E402
from paper_1010_0012_b200 import synth  # noqa: E402
from paper_1010_0012_b200.engine import GridEngine  # noqa: E402

for name, domain in (("C1", "sum"), ("C2", "sum"), ("C2", "max")):
    cfg = synth.CONFIGS[name]
    model = synth.build_config_model(cfg)
    for schedule in ("synchronous", None):
        eng = GridEngine(model, domain, "fast",
                         schedule="sequential" if schedule is None else "synchronous")
        sbp.run_sweeps(model, cfg.iters, domain=domain, schedule=schedule, engine=eng)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = 20
        for _ in range(reps):
            st = sbp.run_sweeps(model, cfg.iters, domain=domain, schedule=schedule, engine=eng)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / reps
        dev = sum(st.stats.sweep_seconds)
        print(json.dumps({"config": name, "domain": domain, "schedule": schedule or "sequential",
                          "iters": cfg.iters, "wall_ms": wall * 1e3, "device_ms": dev * 1e3,
                          "updates_per_s_wall": cfg.n_directed * cfg.iters / wall}))
