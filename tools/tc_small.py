"""Small tcgen05 run for compute-sanitizer / debugging: python tools/tc_small.py [layers] [streams] [steps]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1611_09482_b200 import CellGenerator, Sampler, build_cell_model  # noqa: E402
from paper_1611_09482_b200.cell import CellConfig  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 2
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
T = int(sys.argv[3]) if len(sys.argv) > 3 else 2
m = build_cell_model(CellConfig(1, L, 128, 128, 256, weight_dtype="bf16", bias="fan_in", init_seed=5))
g = CellGenerator(m, B, kernel="tcgen05")
cls = np.random.default_rng(2).integers(0, 256, (T, B))
out, lg = g.generate(torch.as_tensor(cls, dtype=torch.int32, device="cuda"), T, Sampler(0), n_logit_steps=T)
torch.cuda.synchronize()
print("ok", float(lg.abs().max()))
