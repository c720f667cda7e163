"""Per-step stage check of the tcgen05 path (teacher-forced cfg4, lockstep with SIMT):
queue pushes vs SIMT, z stash vs the fp64 oracle, logits vs SIMT. Prints the first stage
that disagrees for each step, with tile/row detail."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import cell as oc  # noqa: E402
from paper_1611_09482_b200 import CellGenerator, Sampler, _lib, build_cell_model, configs  # noqa: E402

spec = configs.cfg4()
m = build_cell_model(spec.cell)
B, R, L = spec.batch, 128, spec.cell.total_layers
dil = spec.cell.dilations()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cls = np.random.default_rng(0).integers(0, 256, (n, B)).astype(np.int32)
gens = {k: CellGenerator(m, B, kernel=k) for k in ("tcgen05", "simt")}
qb = gens["simt"].queue_bytes
qbuf = {k: torch.empty(qb // 4, dtype=torch.float32, device="cuda") for k in gens}
zb = L * 128 * B * 2
zbuf = torch.empty(zb // 2, dtype=torch.float16, device="cuda")
off = np.concatenate([[0], np.cumsum(dil)]) * B * R
o = oc.CellOracle(m, exact=False)


def unswizzle(img):
    t = img.reshape(B // 128, L * 2, 16, 8, 8, 8)
    out = np.empty((B // 128, L * 2, 128, 64), dtype=np.float32)
    for r8 in range(8):
        for p in range(8):
            out[:, :, r8::8, p * 8:(p + 1) * 8] = t[:, :, :, r8, p ^ r8, :]
    return out.transpose(0, 2, 1, 3).reshape(B, L, 128)


def desc(mask2d):  # (tiles, rows) bool -> short text
    t, r = np.nonzero(mask2d)
    return f"tiles {np.unique(t).tolist()[:4]} rows {np.unique(r).tolist()[:10]} ({len(r)})"


for step in range(n):
    lg = {}
    for k, g in gens.items():
        _, l = g.generate(torch.as_tensor(cls[step:step + 1], device="cuda"), 1, Sampler(0),
                          n_logit_steps=1)
        _lib.check(g._lib.fw_debug_copy(g._h, 0, C.c_void_p(qbuf[k].data_ptr()), qb,
                                        _lib.stream_ptr()))
        if k == "tcgen05":
            _lib.check(g._lib.fw_debug_copy(g._h, 1, C.c_void_p(zbuf.data_ptr()), zb,
                                            _lib.stream_ptr()))
        torch.cuda.synchronize()
        lg[k] = l.cpu().numpy()[0]
    a, b = qbuf["tcgen05"].cpu().numpy(), qbuf["simt"].cpu().numpy()
    msgs = []
    for li, d in enumerate(dil):
        seg = slice(off[li] + (step % d) * B * R, off[li] + (step % d + 1) * B * R)
        diff = np.abs(a[seg] - b[seg]).reshape(B // 128, 32, 128, 4).max(axis=(1, 3))
        if diff.max() > 0.05:
            msgs.append(f"push L{li}: {desc(diff > 0.05)}")
            break
    # z stash vs oracle (teacher-forced history, all streams)
    z = unswizzle(zbuf.cpu().numpy())
    T = step + 1
    x = o.E[cls[:T]]
    for li in range(L):
        d = dil[li]
        xp = np.zeros_like(x)
        if d < T:
            xp[d:] = x[:-d]
        zz = o.layer(li, x.reshape(-1, R), xp.reshape(-1, R)).reshape(T, B, 128)
        dz = np.abs(z[:, li] - zz[-1]).max(axis=1).reshape(B // 128, 128)
        if dz.max() > 0.02:
            msgs.append(f"zstash L{li}: {desc(dz > 0.02)}")
            break
        if li + 1 < L:
            x = x + o.res(li, zz.reshape(-1, 128)).reshape(T, B, R)
    dl = np.abs(lg["tcgen05"] - lg["simt"]).max(axis=1).reshape(B // 128, 128)
    if dl.max() > 0.02:
        msgs.append(f"logits: {desc(dl > 0.02)}")
    print(f"step {step}: " + (" | ".join(msgs) if msgs else "ok"), flush=True)
