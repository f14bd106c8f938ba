"""Bitwise fingerprint of a GPU run: sha256 of the message buffer and labels
after N synchronous iterations (or sequential sweeps) of a config model,
with whatever build (SBP_LIB) and kernel variant (SBP_* env) is selected.
Different builds / variants of the same arithmetic must print the same hash.

    python tools/lib_hash.py C3 max 20 [H W] [sequential]
"""
import hashlib
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1010_0012_b200 import synth  # noqa: E402
from paper_1010_0012_b200.engine import GridEngine  # noqa: E402

name, domain, iters = sys.argv[1], sys.argv[2], int(sys.argv[3])
cfg = synth.CONFIGS[name]
if len(sys.argv) > 5:
    model = synth.build_config_model(cfg, height=int(sys.argv[4]), width=int(sys.argv[5]))
    eng = GridEngine(model, domain, "fast",
                     schedule="sequential" if sys.argv[-1] == "sequential" else "synchronous")
else:
    model = synth.StripModel(cfg)
    eng = GridEngine(model, domain, "fast", values=synth.config_values(cfg, domain))
eng.step(iters)
torch.cuda.synchronize()
h = hashlib.sha256()
h.update(eng.current.cpu().numpy().tobytes())
h.update(eng.labels().cpu().numpy().tobytes())
print(json.dumps({"config": name, "domain": domain, "iters": iters, "kernel": eng.kernel_name,
                  "sha": h.hexdigest()[:16]}))
