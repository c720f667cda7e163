"""Lockstep tcgen05 vs SIMT runs (logits requested); after each step report queue/logit deviations
per tile and row so a race can be localised."""
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
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cls = np.random.default_rng(0).integers(0, 256, (n, B)).astype(np.int32)
gens = {k: CellGenerator(m, B, kernel=k) for k in ("tcgen05", "simt")}
qb = gens["simt"].queue_bytes
bufs = {k: torch.empty(qb // 4, dtype=torch.float32, device="cuda") for k in gens}
off = np.concatenate([[0], np.cumsum(dil)]) * B * R
for step in range(n):
    lg = {}
    for k, g in gens.items():
        _, l = g.generate(torch.as_tensor(cls[step:step + 1], device="cuda"), 1, Sampler(0), n_logit_steps=1)
        _lib.check(g._lib.fw_debug_copy(g._h, 0, C.c_void_p(bufs[k].data_ptr()), qb, _lib.stream_ptr()))
        torch.cuda.synchronize()
        lg[k] = l.cpu().numpy()[0]
    a, b = bufs["tcgen05"].cpu().numpy(), bufs["simt"].cpu().numpy()
    msg = []
    for li, d in enumerate(dil):
        seg = slice(off[li] + (step % d) * B * R, off[li] + (step % d + 1) * B * R)
        diff = np.abs(a[seg] - b[seg]).reshape(B // 128, 32, 128, 4).max(axis=(1, 3))  # tile, row
        if diff.max() > 0.05:
            t, r = np.nonzero(diff > 0.05)
            msg.append(f"push layer {li}: tiles {np.unique(t).tolist()[:6]} rows {np.unique(r).tolist()[:8]}..{len(np.unique(r))}")
            break
    dl = np.abs(lg["tcgen05"] - lg["simt"]).max(axis=1)
    bad = np.nonzero(dl > 0.02)[0]
    msg.append(f"logits: {len(bad)} bad, tiles {np.unique(bad // 128).tolist()[:6]}, rows {np.unique(bad % 128).tolist()[:40]}")
    print(f"step {step}: " + " | ".join(msg))
