"""Determinism of the tcgen05 step kernel: one teacher-forced run repeated `reps` times,
each compared with the first; prints the (step, stream) rows whose logits differ.
    [FW_CHAIN_SPLIT=0|1] python tools/race_tc.py batch steps reps"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1611_09482_b200 import CellGenerator, Sampler, build_cell_model, configs  # noqa: E402

B, n, reps = (int(v) for v in sys.argv[1:4])
m = build_cell_model(configs.cfg4().cell)
cls = torch.as_tensor(np.random.default_rng(B).integers(0, 256, (n, B)), dtype=torch.int32, device="cuda")
ref = None
bad_total = 0
for r in range(reps):
    g = CellGenerator(m, B, kernel="tcgen05")
    out, lg = g.generate(cls, n, Sampler(0), n_logit_steps=n)
    torch.cuda.synchronize()
    g.close()
    if ref is None:
        ref = (out, lg)
        continue
    d = (lg - ref[1]).abs().amax(dim=2)
    bad = torch.nonzero(d > 0)
    bad_total += int(bad.shape[0] > 0)
    steps = sorted(set(bad[:, 0].tolist()))[:10]
    streams = bad[:, 1]
    print(f"rep {r}: rows differing {bad.shape[0]}, max {float(d.max()):.3g}, steps {steps}, "
          f"streams {int(streams.min()) if bad.shape[0] else -1}..{int(streams.max()) if bad.shape[0] else -1}",
          flush=True)
print(f"B={B}: {bad_total} of {reps - 1} repetitions differ")
