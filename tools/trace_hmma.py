"""Per-layer timeline of the warp-MMA kernel (csrc/cell_hmma.cu), CTA 0 thread 0, clock64:
[start, phase-A GEMM done, gate + skip epilogue done, pops/prefetch done, barrier passed,
phase B done, barrier passed]. python tools/trace_hmma.py [config]"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1611_09482_b200 import CellGenerator, Sampler, _lib, build_cell_model, configs  # noqa: E402

spec = configs.by_name(sys.argv[1] if len(sys.argv) > 1 else "cfg5")
L = spec.cell.total_layers
gen = CellGenerator(build_cell_model(spec.cell), spec.batch, kernel="simt")
tr = torch.zeros(((L + 2) * 8,), dtype=torch.int64, device="cuda")
_lib.check(gen._lib.fw_debug_trace(gen._h, C.c_void_p(tr.data_ptr())))
x = torch.full((1, spec.batch), 128, dtype=torch.int32, device="cuda")
gen.generate(x, 3, Sampler(0))
torch.cuda.synchronize()
t = tr.view(L + 2, 8).cpu().numpy().astype(np.int64)
print("layer period  gemmA   epiA   pops   bar1 phaseB   bar2   next")
per = []
for l in range(L):
    d = [t[l, k] - t[l, k - 1] for k in range(1, 7)] + [(t[l + 1, 0] if l + 1 < L else t[l, 6]) - t[l, 6]]
    pd = t[l, 0] - t[l - 1, 0] if l else 0
    if l > 1:
        per.append(pd)
    if l < 12 or l == L - 1:
        print(f"{l:5d} {pd:6d} " + " ".join(f"{v:6d}" for v in d))
print("median period", np.median(per), "median phases", np.median(np.diff(t[2:L, :7], axis=1), axis=0).tolist())
