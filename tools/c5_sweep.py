"""BASELINE config 5: banded O(mM) vs dense O(M^2) kernels on the 1024x1024,
M=256 grid for every band width, both domains.  Per kernel: median device
time of one synchronous iteration (CUDA events, after warm-up), directed
updates/s, fraction of the HBM roofline (algorithmic bytes) and of the
measured FP32 FFMA peak (algorithmic flops), and the dense/banded speed-up.

    python tools/c5_sweep.py [iters] > profiles/c5_sweep.json
"""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1010_0012_b200 import synth  # noqa: E402
from paper_1010_0012_b200.engine import GridEngine  # noqa: E402

FFMA_TFLOPS = 70.74   # tools/microbench.cu on B200 (profiles/r01_microbench.txt)
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 8
peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
rows = []
for T in (2, 5, 9, 17, 33):
    cfg = synth.CONFIGS[f"C5_T{T}"]
    model = synth.StripModel(cfg)
    pot = model.shared_potential
    H, W, M = cfg.height, cfg.width, cfg.M
    E = cfg.n_directed
    B = 4 * M * (H * W + 2 * E)
    for domain in ("sum", "max"):
        vals = synth.config_values(cfg, domain)
        res = {"T": T, "m_ref": pot.m, "nnz": pot.nnz, "domain": domain}
        for kernel in ("fast", "standard"):
            eng = GridEngine(model, domain, kernel, values=vals)
            eng.step(2)
            torch.cuda.synchronize()
            evs = []
            eng.step(iters, events=evs)
            torch.cuda.synchronize()
            ms = sorted(a.elapsed_time(b) / k for a, b, k in evs[1:] or evs)[len(evs[1:] or evs) // 2]
            F = E * 2 * ((pot.nnz + 2 * M) if kernel == "fast" else M * M)
            res[kernel] = {"ms_per_iter": ms, "updates_per_s": E / ms * 1e3,
                           "hbm_frac": B / ms / 1e6 / peak,
                           "fp32_frac": F / ms / 1e9 / FFMA_TFLOPS,
                           "plan": eng.plan.kind_name}
            del eng
            torch.cuda.empty_cache()
        res["speedup_dense_over_band"] = res["standard"]["ms_per_iter"] / res["fast"]["ms_per_iter"]
        rows.append(res)
        print(json.dumps(res), flush=True)
