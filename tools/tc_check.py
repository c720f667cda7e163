"""tcgen05 path vs the CPU oracle for one shape: python tools/tc_check.py L S H [B] [T] [mode]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import cell as oc  # noqa: E402
from paper_1611_09482_b200 import CellGenerator, Sampler, build_cell_model  # noqa: E402
from paper_1611_09482_b200.cell import CellConfig  # noqa: E402

L, S, H = (int(v) for v in sys.argv[1:4])
B = int(sys.argv[4]) if len(sys.argv) > 4 else 256
T = int(sys.argv[5]) if len(sys.argv) > 5 else 3
mode = int(sys.argv[6]) if len(sys.argv) > 6 else 0
nb = L // 10 if L > 10 else 1
m = build_cell_model(CellConfig(nb, L // nb, 128, 128, S, head_channels=H, weight_dtype="bf16",
                                bias="fan_in", init_seed=5))
g = CellGenerator(m, B, kernel="tcgen05")
cls = np.random.default_rng(2).integers(0, 256, (T, B))
_, lg = g.generate(torch.as_tensor(cls, dtype=torch.int32, device="cuda"), T, Sampler(mode, 7),
                   n_logit_steps=T)
lg = lg.cpu().numpy()
o = oc.CellOracle(m, exact=False)
bad = []
streams = range(B) if B <= 512 else (0, 63, 64, 127, 128, B - 1)
worst = 0.0
for s in streams:
    ref = o.forward_full(cls[:, s])
    dev = np.abs(lg[:, s] - ref).max(axis=1)
    worst = max(worst, float(dev.max()))
    if dev.max() > 0.02:
        bad.append((s, [int(i) for i in np.nonzero(dev > 0.02)[0]]))
print(f"L={L} S={S} H={H} B={B} T={T}: worst {worst:.3g}, bad streams {len(bad)}: {bad[:12]}")
