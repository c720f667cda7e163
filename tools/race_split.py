"""Determinism check of the tcgen05 kernel (split or not): the same teacher-forced run
repeated; any difference between repetitions is a race.
    FW_CHAIN_SPLIT=0|1 python tools/race_split.py [batch] [steps] [reps]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1611_09482_b200 import CellGenerator, Sampler, build_cell_model, configs  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
n = int(sys.argv[2]) if len(sys.argv) > 2 else 300
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 8
m = build_cell_model(configs.cfg4().cell)
cls = torch.as_tensor(np.random.default_rng(B).integers(0, 256, (n, B)), dtype=torch.int32, device="cuda")
ref = None
for r in range(reps):
    g = CellGenerator(m, B, kernel="tcgen05")
    _, lg = g.generate(cls, n, Sampler(0), n_logit_steps=n)
    torch.cuda.synchronize()
    g.close()
    if ref is None:
        ref = lg
        continue
    d = (lg - ref).abs()
    bad = torch.nonzero(d.amax(dim=2) > 0)
    print(f"rep {r}: max diff {float(d.max()):.3g}, differing (step, stream) rows {bad.shape[0]}",
          bad[:6].tolist(), flush=True)
