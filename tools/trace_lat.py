"""Phase timeline of the small-batch cluster kernel (csrc/cell_lat.cu), CTA 0, step 1 of a
launch, %globaltimer ns: per phase [start, exchange seen, dil GEMV, res/skip GEMV, pop
value stored, CTA barrier passed, sends issued, ring push issued]; phases 0..L-1 = layers, L = top skip + ReLU(s), L+1 = head1, L+2 = head2,
L+3 = selection.

    python tools/trace_lat.py [config] [cluster]
"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1611_09482_b200 import CellGenerator, Sampler, _lib, build_cell_model, configs  # noqa: E402

spec = configs.by_name(sys.argv[1] if len(sys.argv) > 1 else "cfg1")
if len(sys.argv) > 2:
    os.environ["FW_SIMT_CLUSTER"] = sys.argv[2]
L = spec.cell.total_layers
gen = CellGenerator(build_cell_model(spec.cell), 1, kernel="simt")
tr = torch.zeros(((L + 4) * 8,), dtype=torch.int64, device="cuda")
_lib.check(gen._lib.fw_debug_trace(gen._h, C.c_void_p(tr.data_ptr())))
x = torch.full((1, 1), 128, dtype=torch.int32, device="cuda")
gen.generate(x, 4, Sampler(0))
torch.cuda.synchronize()
t = tr.view(L + 4, 8).cpu().numpy()
t0 = t[0, 0]
print("phase   start   wait    dil  res/s    pop   sync  sends   push  (ns; start from phase-0 start, then deltas)")
for p in range(L + 4):
    row = t[p] - t0
    d = [t[p, k] - t[p, k - 1] if t[p, k] and t[p, k - 1] else 0 for k in range(1, 8)]
    name = p if p < L else ["skip", "head1", "head2", "select"][p - L]
    print(f"{str(name):>6} {row[0]:7d} " + " ".join(f"{v:6d}" for v in d))
print(f"step: {t[L + 3, 2] - t0} ns")
print('raw', t.tolist())
