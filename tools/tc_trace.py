"""Pipeline timeline of the tensor-core dense kernel (debug build with
-DSBP_TC_TRACE): cycles between events of cluster 0's first tiles.
    make -C paper_1010_0012_b200/csrc EXTRA=-DSBP_TC_TRACE   (after touching dense_tc_kernel.cu)
    python tools/tc_trace.py C4"""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1010_0012_b200 import _lib, synth  # noqa: E402
from paper_1010_0012_b200.engine import GridEngine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = synth.CONFIGS[name]
model = synth.StripModel(cfg)
eng = GridEngine(model, "sum", "standard", values=synth.config_values(cfg, "sum"))
eng.step(3)
torch.cuda.synchronize()
lib = _lib.lib()
T, E = 48, 16
buf = (ctypes.c_longlong * (T * E))()
rc = lib.sbp_debug_tc_trace(buf, T * E)
t = np.array(buf, dtype=np.int64).reshape(T, E)
names = ["E.accf", "E.done", "M.accfree", "M.full0", "M.iss0", "M.full1", "M.iss1", "P.start", "P.prod",
         "P.empty0", "P.arr0", "P.empty1", "P.arr1"]
t0 = t[8, 7]
print(name, eng.kernel_name, "rc", rc)
print("tile " + " ".join(f"{n:>9}" for n in names))
for i in range(8, 28):
    print(f"{i:4d} " + " ".join(f"{int(t[i, k] - t0):9d}" for k in range(13)))
d = np.diff(t[8:40, 1])
print("cycles per tile (epilogue done to done): median", int(np.median(d)))
for a, b, lab in [(7, 8, "P start->products"), (8, 9, "P products->empty0"), (9, 10, "P empty0->arrive0"),
                  (10, 11, "P arrive0->empty1"), (11, 12, "P empty1->arrive1"), (3, 4, "M full0->issued0"),
                  (4, 5, "M issued0->full1"), (5, 6, "M full1->issued1"), (6, 0, "M issued1->E accf"),
                  (0, 1, "E accf->done"), (12, 5, "P arrive1->M full1")]:
    print(f"{lab:24s} median {int(np.median(t[8:40, b] - t[8:40, a]))}")
