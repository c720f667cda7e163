"""Run cfg4 teacher-forced step by step on the tcgen05 and SIMT paths; diff the HBM queues."""
import ctypes as C
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1611_09482_b200 import CellGenerator, Sampler, _lib, build_cell_model, configs

spec = configs.cfg4()
m = build_cell_model(spec.cell)
B, R = spec.batch, 128
dil = spec.cell.dilations()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cls = np.random.default_rng(0).integers(0, 256, (n, B)).astype(np.int32)
gens = {k: CellGenerator(m, B, kernel=k) for k in ("tcgen05", "simt")}
qb = gens["simt"].queue_bytes
bufs = {k: torch.empty(qb // 4, dtype=torch.float32, device="cuda") for k in gens}
off = np.concatenate([[0], np.cumsum(dil)]) * B * R
for step in range(n):
    for k, g in gens.items():
        g.generate(torch.as_tensor(cls[step:step + 1], device="cuda"), 1, Sampler(0))
        _lib.check(g._lib.fw_debug_copy(g._h, 0, C.c_void_p(bufs[k].data_ptr()), qb, _lib.stream_ptr()))
    torch.cuda.synchronize()
    a, b = bufs["tcgen05"].cpu().numpy(), bufs["simt"].cpu().numpy()
    for l, d in enumerate(dil):
        slot = step % d
        seg = slice(off[l] + slot * B * R, off[l] + (slot + 1) * B * R)
        diff = np.abs(a[seg] - b[seg]).reshape(B // 128, 32, 128, 4)  # tile, chunk, row, 4
        worst = diff.max(axis=(1, 2, 3))
        if worst.max() > 0.05:
            print(f"step {step} layer {l} (d={d}, slot {slot}): bad tiles {np.nonzero(worst > 0.05)[0].tolist()[:10]} "
                  f"max {worst.max():.3g}; ref |x| {np.abs(b[seg]).mean():.3g}")
            break
    else:
        print(f"step {step}: pushed slots agree (max {max(np.abs(a - b).max(), 0):.3g})")
