"""Small runs of every kernel family for compute-sanitizer (memcheck,
racecheck, synccheck): register / TMA-staged / rolled / shared-memory-tap /
temporally blocked band kernels, the sequential chain kernel, ELL (f32 and
f64 accumulation), the dense comparison kernel, the fused convergence test,
beliefs / gather.  Each case runs in this process with its kernel-variant
environment applied through sbp_reload_config.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1010_0012_b200 as sbp  # noqa: E402
from paper_1010_0012_b200 import _lib as L  # noqa: E402
from paper_1010_0012_b200 import synth  # noqa: E402

CASES = [
    # (config, domain, schedule, env, kernel, extra)
    ("C1", "sum", "synchronous", {}, "fast", None),                       # register VL=8
    ("C3", "max", "synchronous", {}, "fast", None),                       # TMA-staged
    ("C4", "sum", "synchronous", {}, "fast", None),                       # rolled VL=16
    ("C5_T9", "sum", "synchronous", {"SBP_TAP": "1"}, "fast", None),      # tap VL=16
    ("C5_T17", "max", "synchronous", {"SBP_TAP": "1", "SBP_TAP_STAGED": "1"}, "fast", None),
    ("C5_T33", "max", "synchronous", {"SBP_TAP": "1", "SBP_TAP_ROLLED": "1"}, "fast", None),
    ("C5_T2", "sum", "synchronous", {"SBP_FUSE": "3"}, "fast", None),     # temporal blocking
    ("C4", "sum", None, {}, "fast", None),                                # sequential chain
    ("C2", "max", None, {}, "fast", None),
    ("C3", "sum", "synchronous", {}, "standard", None),                   # dense tiled
    ("C1", "sum", "synchronous", {}, "standard", None),                   # dense via ELL (Ms<32)
    ("C2", "sum", "synchronous", {}, "fast", "ell"),                      # general CSC
    ("C2", "sum", "synchronous", {"SBP_PRECISION": "f64"}, "fast", "ell"),  # f64 accumulation
    ("C2", "sum", "synchronous", {}, "fast", "delta"),                    # fused convergence
    ("C2", "max", None, {}, "fast", "delta"),
]


def model_for(name, extra):
    H, W = (12, 20) if synth.CONFIGS[name].M >= 128 else (14, 23)
    m = synth.build_config_model(synth.CONFIGS[name], height=H, width=W)
    if extra == "ell":
        d = m.shared_potential.densify().table.copy()
        d[2, 4] = 0.5 * (d[2, 4] + 1.0)
        m = sbp.GridMrf(H, W, m.M, m.unaries, sbp.sparse_from_dense(d, fbar=m.shared_potential.fbar),
                        log_unaries=m.log_unaries)
    return m


def main():
    only = sys.argv[1:]
    for i, (name, dom, sched, env, kernel, extra) in enumerate(CASES):
        if only and str(i) not in only:
            continue
        saved = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        L.lib().sbp_reload_config()
        try:
            model = model_for(name, extra)
            tol = 1e-12 if extra == "delta" else None
            store = sbp.run_sweeps(model, 3, kernel=kernel, domain=dom, schedule=sched,
                                   convergence_tol=tol)
            data = store.data
            if dom == "sum":
                sbp.compute_beliefs(model, store)
            else:
                sbp.compute_max_marginals(model, store)
            sbp.map_labels(store)
            torch.cuda.synchronize()
            print(f"case {i} {name} {dom} {sched} {env} {kernel} {extra}: "
                  f"{store.engine.kernel_name} ok {np.isfinite(data).mean():.3f}", flush=True)
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
            L.lib().sbp_reload_config()


if __name__ == "__main__":
    main()
