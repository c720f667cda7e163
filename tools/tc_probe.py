"""Probe one tcgen05 configuration (run under `timeout`): python tools/tc_probe.py L S H B bias"""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1611_09482_b200 import CellGenerator, Sampler, build_cell_model
from paper_1611_09482_b200.cell import CellConfig
L, S, H, B, bias = (int(a) for a in sys.argv[1:6])
cfg = CellConfig(1, L, 128, 128, S, head_channels=H, weight_dtype="bf16",
                 bias="fan_in" if bias else "zero", init_seed=7)
m = build_cell_model(cfg)
gen = CellGenerator(m, B, kernel="tcgen05")
t0 = time.time()
out, lg = gen.generate(torch.full((1, B), 5, dtype=torch.int32, device="cuda"), 4, Sampler(0), n_logit_steps=4)
torch.cuda.synchronize()
print("ok", sys.argv[1:], f"{time.time()-t0:.2f}s", out[:, :4].cpu().numpy().tolist(), flush=True)
