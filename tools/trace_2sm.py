"""Cross-CTA timeline of the 2-SM chain (pair 0, globaltimer ns): per layer, each CTA's
x_full seen / x_t arrive / z0 arrive / acc0 seen, relative to rank 0's x_full seen.
    FW_CHAIN_2SM=1 python tools/trace_2sm.py"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
os.environ.setdefault("FW_CHAIN_2SM", "1")
from paper_1611_09482_b200 import CellGenerator, Sampler, _lib, build_cell_model, configs  # noqa: E402

spec = configs.cfg4()
m = build_cell_model(spec.cell)
B = int(sys.argv[1]) if len(sys.argv) > 1 else spec.batch
gen = CellGenerator(m, B, kernel="tcgen05")
L = spec.cell.total_layers
tr = torch.zeros((L + 1, 48), dtype=torch.int64, device="cuda")
_lib.check(gen._lib.fw_debug_trace(gen._h, C.c_void_p(tr.data_ptr())))
primer = torch.full((1, B), 128, dtype=torch.int32, device="cuda")
gen.generate(primer, 3, Sampler(spec.sampler, configs.NOISE_SEED))
torch.cuda.synchronize()
t = tr.cpu().numpy().astype(np.int64)
print("layer  q:xfull   xt  g:z0 acc0 | mma:xd   xt B0rdy   z0   (ns vs rank 0 x_full seen) | period")
for l in range(L):
    ref = t[l, 40]
    print(f"{l:5d} " + " ".join(f"{t[l, 40 + k] - ref:5d}" for k in range(4)) + " | " +
          " ".join(f"{t[l, 44 + k] - ref:5d}" for k in range(4)) + " | relay xt seen/fwd, mma xd issued: " +
          " ".join(f"{t[l, 32 + k] - ref:5d}" for k in range(7)) + f" | {t[l, 40] - t[l - 1, 40] if l else 0}")
