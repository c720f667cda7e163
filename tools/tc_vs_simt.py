"""Teacher-forced cfg4 logits, tcgen05 vs SIMT kernel, per (step, stream): locate outliers."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1611_09482_b200 import CellGenerator, Sampler, build_cell_model, configs

spec = configs.cfg4()
m = build_cell_model(spec.cell)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
cls = np.random.default_rng(0).integers(0, 256, (n, spec.batch)).astype(np.int32)
inp = torch.as_tensor(cls, device="cuda")
res = {}
for k in ("tcgen05", "simt"):
    g = CellGenerator(m, spec.batch, kernel=k)
    _, lg = g.generate(inp, n, Sampler(0), n_logit_steps=n)
    res[k] = lg.cpu().numpy()
    g.close()
d = np.abs(res["tcgen05"] - res["simt"]).max(axis=2)  # (n, B)
print("per-step max:", np.round(d.max(axis=1), 4).tolist())
bad = np.argwhere(d > 0.02)
print("bad count", len(bad), "of", d.size)
if len(bad):
    tiles = np.unique(bad[:, 1] // 128)
    rows = np.unique(bad[:, 1] % 128)
    print("bad tiles", tiles.tolist()[:40])
    print("bad rows", rows.tolist()[:64])
    print("first bad (step, stream)", bad[:20].tolist())
