# Soak of the tensor-core dense kernel: repeated test runs, full-size C5 / C4 with several launch geometries (bits must
# not change), long runs (sums stay 1).
OUT=gpurun_out/soak.txt; rm -f $OUT
for rep in 1 2 3; do
  timeout 900 python -m pytest tests/test_gpu_dense_tc.py tests/test_gpu_guards.py -m gpu -q --timeout 600 -p no:cacheprovider 2>&1 | tail -1 >> $OUT
done
python - >> $OUT 2>&1 <<'EOF'
import os, sys, hashlib
import torch
sys.path.insert(0, ".")
from paper_1010_0012_b200 import _lib as L, synth
from paper_1010_0012_b200.engine import GridEngine
for name, iters in (("C5_T9", 20), ("C4", 10)):
    cfg = synth.CONFIGS[name]
    vals = synth.config_values(cfg, "sum")
    hashes = []
    for cap in (None, "1", "9", "37", "74"):
        if cap is None: os.environ.pop("SBP_MAX_BLOCKS", None)
        else: os.environ["SBP_MAX_BLOCKS"] = cap
        L.lib().sbp_reload_config()
        eng = GridEngine(synth.StripModel(cfg), "sum", "standard", values=vals)
        n = iters if cap in (None, "37", "74") else 2
        eng.step(n)
        torch.cuda.synchronize()
        eng.raise_if_degenerate()
        cur = eng.current[:, 2:eng.rows, 1:-1]
        dev = float((cur.sum(dim=-1) - 1).abs().max())
        h = hashlib.sha256(eng.current.cpu().numpy().tobytes()).hexdigest()[:12]
        hashes.append((cap, n, h))
        print(name, eng.kernel_name, "cap", cap, "iters", n, "max|sum-1|", dev, "sha", h, flush=True)
        del eng, cur
        torch.cuda.empty_cache()
    full = {h for c, n, h in hashes if n == iters}
    short = {h for c, n, h in hashes if n == 2}
    print(name, "geometry-independent bits:", len(full) == 1 and len(short) == 1)
os.environ.pop("SBP_MAX_BLOCKS", None); L.lib().sbp_reload_config()
cfg = synth.CONFIGS["C5_T33"]
eng = GridEngine(synth.StripModel(cfg), "sum", "standard", values=synth.config_values(cfg, "sum"))
eng.step(300); torch.cuda.synchronize(); eng.raise_if_degenerate()
cur = eng.current[:, 2:eng.rows, 1:-1]
print("C5_T33 300 iterations max|sum-1|", float((cur.sum(dim=-1) - 1).abs().max()))
EOF
cat $OUT
