"""tcgen05 path vs the CPU oracle for one shape: python tools/tc_check.py L S H [B] [T]"""
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
nb = L // 10 if L > 10 else 1
m = build_cell_model(CellConfig(nb, L // nb, 128, 128, S, head_channels=H, weight_dtype="bf16",
                                bias="fan_in", init_seed=5))
g = CellGenerator(m, B, kernel="tcgen05")
cls = np.random.default_rng(2).integers(0, 256, (T, B))
_, lg = g.generate(torch.as_tensor(cls, dtype=torch.int32, device="cuda"), T, Sampler(0),
                   n_logit_steps=T)
lg = lg.cpu().numpy()
o = oc.CellOracle(m, exact=False)
for s in (0, 63, 64, 127, 128, B - 1):
    ref = o.forward_full(cls[:, s])
    print(f"L={L} S={S} H={H} stream {s}: max dev {float(np.abs(lg[:, s] - ref).max()):.3g}")
