"""Isolate the skip contribution of single layers: zero every W_skip except layer k and compare
tcgen05 vs SIMT logits (steps 0..n-1, teacher-forced)."""
import dataclasses
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1611_09482_b200 import CellGenerator, Sampler, build_cell_model, configs
from paper_1611_09482_b200.cell import CellModel

spec = configs.cfg4()
base = build_cell_model(spec.cell)
n = 4
cls = np.random.default_rng(0).integers(0, 256, (n, spec.batch)).astype(np.int32)
for k in [int(a) for a in sys.argv[1:]] or [0, 1, 9, 10, 38, 39]:
    layers = tuple(dataclasses.replace(lw, skip_w=lw.skip_w * (1.0 if i == k else 0.0))
                   for i, lw in enumerate(base.layers))
    m = CellModel(base.config, base.embed, layers, base.head1_w, base.head1_b, base.head2_w, base.head2_b)
    lg = {}
    for kern in ("tcgen05", "simt"):
        g = CellGenerator(m, spec.batch, kernel=kern)
        _, l = g.generate(torch.as_tensor(cls, device="cuda"), n, Sampler(0), n_logit_steps=n)
        lg[kern] = l.cpu().numpy()
        g.close()
    d = np.abs(lg["tcgen05"] - lg["simt"]).max(axis=(2))
    bad = [int((d[s] > 0.02).sum()) for s in range(n)]
    print(f"layer {k}: per-step max {np.round(d.max(axis=1), 4).tolist()} bad streams {bad}")
