"""Split vs unsplit tcgen05 kernel, 600 teacher-forced steps, repeated; prints where they
differ by more than the bf16 tolerance. python tools/race_split2.py [batch] [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1611_09482_b200 import CellGenerator, Sampler, build_cell_model, configs  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
n = 600
m = build_cell_model(configs.cfg4().cell)
cls = torch.as_tensor(np.random.default_rng(B).integers(0, 256, (n, B)), dtype=torch.int32, device="cuda")


def run(split):
    os.environ["FW_CHAIN_SPLIT"] = "1" if split else "0"
    g = CellGenerator(m, B, kernel="tcgen05")
    _, lg = g.generate(cls, n, Sampler(0), n_logit_steps=n)
    torch.cuda.synchronize()
    g.close()
    return lg


ref = run(False)
for r in range(reps):
    for split in (True, False):
        lg = run(split)
        d = (lg - ref).abs().amax(dim=2)
        bad = torch.nonzero(d > 2e-2)
        first = bad[:8].tolist()
        print(f"rep {r} split={split}: max {float(d.max()):.3g}, rows > 2e-2: {bad.shape[0]}, first {first}",
              flush=True)
