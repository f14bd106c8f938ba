"""Debug helper: run one reduced config on the GPU and save its messages."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1010_0012_b200 as sbp  # noqa: E402
from paper_1010_0012_b200 import synth  # noqa: E402

name, domain, iters, H, W, out = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), \
    int(sys.argv[5]), sys.argv[6]
model = synth.build_config_model(synth.CONFIGS[name], height=H, width=W)
store = sbp.run_sweeps(model, iters, domain=domain, schedule="synchronous")
np.save(out, store.engine.msgs4())
