"""Decode the tcgen05 z stash (fp16 SW128 images) after each teacher-forced step and compare
with the fp64 oracle's z for a few streams."""
import ctypes as C
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import cell as oc
from paper_1611_09482_b200 import CellGenerator, Sampler, _lib, build_cell_model, configs

spec = configs.cfg4()
m = build_cell_model(spec.cell)
B, L = spec.batch, spec.cell.total_layers
n = 4
cls = np.random.default_rng(0).integers(0, 256, (n, B)).astype(np.int32)
g = CellGenerator(m, B, kernel="tcgen05")
zb = L * 128 * B * 2
buf = torch.empty(zb // 2, dtype=torch.float16, device="cuda")
o = oc.CellOracle(m, exact=False)

def unswizzle(img):  # [ntile][L*2][128 rows][64] fp16 image -> [B][L*128]
    t = img.reshape(B // 128, L * 2, 16, 8, 8, 8)  # tile, chunk, row/8, row%8, piece, 8 halves
    out = np.empty((B // 128, L * 2, 128, 64), dtype=np.float32)
    for r8 in range(8):
        for p in range(8):
            out[:, :, r8::8, p * 8:(p + 1) * 8] = t[:, :, :, r8, p ^ r8, :]
    return out.transpose(0, 2, 1, 3).reshape(B, L * 128)

streams = [0, 1, 1408, 4095]
for step in range(n):
    g.generate(torch.as_tensor(cls[step:step + 1], device="cuda"), 1, Sampler(0))
    _lib.check(g._lib.fw_debug_copy(g._h, 1, C.c_void_p(buf.data_ptr()), zb, _lib.stream_ptr()))
    torch.cuda.synchronize()
    z = unswizzle(buf.cpu().numpy())
    for s in streams:
        # oracle z of every layer at this step, teacher-forced history of stream s
        hist = cls[: step + 1, s]
        x = o.E[hist]
        zs = []
        for l in range(L):
            d = o.dil[l]
            xp = np.zeros_like(x)
            xp[d:] = x[:-d] if d < len(x) else 0
            zz = o.layer(l, x, xp)
            zs.append(zz[-1])
            if l + 1 < L:
                x = x + o.res(l, zz)
        ref = np.concatenate(zs)
        dev = np.abs(z[s] - ref).reshape(L, 128).max(axis=1)
        worst = int(np.argmax(dev))
        print(f"step {step} stream {s}: max z dev {dev.max():.4g} at layer {worst}; "
              f"layers > 0.01: {np.nonzero(dev > 0.01)[0].tolist()[:12]}")

print("--- skip GEMM check: ReLU(sum_l W_skip_l z_l) from the GPU z stash vs the GPU s image")
S = spec.cell.skip_channels
Wcat = np.concatenate([np.asarray(lw.skip_w, np.float64) for lw in m.layers], axis=1)  # (S, L*128)
sb = torch.empty(B * S, dtype=torch.float16, device="cuda")
g2 = CellGenerator(m, B, kernel="tcgen05")
for step in range(n):
    g2.generate(torch.as_tensor(cls[step:step + 1], device="cuda"), 1, Sampler(0))
    _lib.check(g2._lib.fw_debug_copy(g2._h, 1, C.c_void_p(buf.data_ptr()), zb, _lib.stream_ptr()))
    _lib.check(g2._lib.fw_debug_copy(g2._h, 2, C.c_void_p(sb.data_ptr()), B * S * 2, _lib.stream_ptr()))
    torch.cuda.synchronize()
    z = unswizzle(buf.cpu().numpy()).astype(np.float64)
    simg = sb.cpu().numpy().reshape(B // 128, S // 64, 16, 8, 8, 8)
    s_gpu = np.empty((B // 128, S // 64, 128, 64), dtype=np.float32)
    for r8 in range(8):
        for p in range(8):
            s_gpu[:, :, r8::8, p * 8:(p + 1) * 8] = simg[:, :, :, r8, p ^ r8, :]
    s_gpu = s_gpu.transpose(0, 2, 1, 3).reshape(B, S)
    s_ref = np.maximum(z @ Wcat.T, 0)
    dev = np.abs(s_gpu - s_ref).max(axis=1)
    print(f"step {step}: skip max dev {dev.max():.4g}; bad streams {int((dev > 0.05).sum())}; "
          f"bad tiles {np.unique(np.nonzero(dev > 0.05)[0] // 128).tolist()[:12]}")

print("--- head checks from the GPU's own s image")
H, A = spec.cell.H, spec.cell.classes
W1 = np.asarray(m.head1_w, np.float64); W2 = np.asarray(m.head2_w, np.float64)
hb = torch.empty(B * H, dtype=torch.float16, device="cuda")
g3 = CellGenerator(m, B, kernel="tcgen05")
def unimg(t16, N):
    t = t16.reshape(B // 128, N // 64, 16, 8, 8, 8)
    o_ = np.empty((B // 128, N // 64, 128, 64), dtype=np.float32)
    for r8 in range(8):
        for p in range(8):
            o_[:, :, r8::8, p * 8:(p + 1) * 8] = t[:, :, :, r8, p ^ r8, :]
    return o_.transpose(0, 2, 1, 3).reshape(B, N).astype(np.float64)
for step in range(n):
    _, lgt = g3.generate(torch.as_tensor(cls[step:step + 1], device="cuda"), 1, Sampler(0), n_logit_steps=1)
    _lib.check(g3._lib.fw_debug_copy(g3._h, 2, C.c_void_p(sb.data_ptr()), B * S * 2, _lib.stream_ptr()))
    _lib.check(g3._lib.fw_debug_copy(g3._h, 3, C.c_void_p(hb.data_ptr()), B * H * 2, _lib.stream_ptr()))
    torch.cuda.synchronize()
    s_gpu = unimg(sb.cpu().numpy(), S)
    h_gpu = unimg(hb.cpu().numpy(), H)
    h_ref = np.maximum(s_gpu @ W1.T, 0)
    lg_ref = h_gpu @ W2.T
    dh = np.abs(h_gpu - h_ref).max(axis=1)
    dl = np.abs(lgt.cpu().numpy()[0] - lg_ref).max(axis=1)
    print(f"step {step}: head1 max dev {dh.max():.4g} (bad tiles {np.unique(np.nonzero(dh > 0.05)[0] // 128).tolist()[:8]}); "
          f"head2 max dev {dl.max():.4g} (bad tiles {np.unique(np.nonzero(dl > 0.05)[0] // 128).tolist()[:8]})")
