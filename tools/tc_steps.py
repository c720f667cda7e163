"""tcgen05 vs SIMT logits with one generate call per step (host-synchronised) vs one call."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1611_09482_b200 import CellGenerator, Sampler, build_cell_model, configs

spec = configs.cfg4()
m = build_cell_model(spec.cell)
n = 6
cls = np.random.default_rng(0).integers(0, 256, (n, spec.batch)).astype(np.int32)
out = {}
for k in ("tcgen05", "simt"):
    for mode in ("stepwise", "single"):
        g = CellGenerator(m, spec.batch, kernel=k)
        if mode == "single":
            _, lg = g.generate(torch.as_tensor(cls, device="cuda"), n, Sampler(0), n_logit_steps=n)
            lg = lg.cpu().numpy()
        else:
            rows = []
            for s in range(n):
                _, l1 = g.generate(torch.as_tensor(cls[s:s + 1], device="cuda"), 1, Sampler(0), n_logit_steps=1)
                torch.cuda.synchronize()
                rows.append(l1.cpu().numpy()[0])
            lg = np.stack(rows)
        out[(k, mode)] = lg
        g.close()
for mode in ("stepwise", "single"):
    d = np.abs(out[("tcgen05", mode)] - out[("simt", "single")]).max(axis=(1, 2))
    print(mode, np.round(d, 4).tolist())
print("simt stepwise vs single", np.abs(out[("simt", "stepwise")] - out[("simt", "single")]).max())
