"""Step time of the cfg4 shape at 1-4 blocks of 10 layers (tcgen05, 4,096 streams): the
intercept of the linear fit is the per-step cost outside the layer chain (tail + step start).
python tools/tail_fit.py [steps]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1611_09482_b200 import CellGenerator, Sampler, build_cell_model, configs  # noqa: E402
from paper_1611_09482_b200.cell import CellConfig  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 200
pts = []
for blocks in (1, 2, 3, 4):
    m = build_cell_model(CellConfig(blocks, 10, 128, 128, 512, weight_dtype="bf16"))
    gen = CellGenerator(m, 4096, kernel="tcgen05")
    primer = torch.full((1, 4096), 128, dtype=torch.int32, device="cuda")
    s = Sampler(configs.SAMPLE_GUMBEL, configs.NOISE_SEED)
    gen.generate(primer, 10, s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    gen.generate(primer, T, s)
    e1.record()
    torch.cuda.synchronize()
    us = 1e3 * e0.elapsed_time(e1) / T
    pts.append((10 * blocks, us))
    gen.close()
L = np.array([p[0] for p in pts], float)
y = np.array([p[1] for p in pts])
slope, icpt = np.polyfit(L, y, 1)
print(json.dumps({"points_us": pts, "us_per_layer": slope, "intercept_us": icpt}))
