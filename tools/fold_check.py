"""An opt-in tcgen05 chain variant vs the default chain on the cfg4 shape: teacher-forced
logits of every stream, a few streams against the fp64 oracle, and repeated-run determinism.

python tools/fold_check.py BATCH STEPS [REPEATS] [ENV]    (ENV: FW_CHAIN_FOLD | FW_CHAIN_2SM)
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

from cellcheck import check_streams  # noqa: E402
from oracle import cell as oc  # noqa: E402
from paper_1611_09482_b200 import CellGenerator, Sampler, build_cell_model, configs  # noqa: E402

B = int(sys.argv[1])
n = int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
ENV = sys.argv[4] if len(sys.argv) > 4 else "FW_CHAIN_FOLD"
VAL = sys.argv[5] if len(sys.argv) > 5 else "1"
m = build_cell_model(configs.cfg4().cell)
cls = torch.as_tensor(np.random.default_rng(B + 3).integers(0, 256, (n, B)), dtype=torch.int32,
                      device="cuda")


def run(fold):
    os.environ[ENV] = fold
    gen = CellGenerator(m, B, kernel="tcgen05")
    t = time.time()
    out, lg = gen.generate(cls, n, Sampler(0), n_logit_steps=n)
    torch.cuda.synchronize()
    dt = time.time() - t
    gen.close()
    return out, lg, dt


out_f, lg_f, dt = run(VAL)
print(f"fold run done in {dt:.2f}s", flush=True)
for r in range(reps - 1):
    _, lg2, _ = run(VAL)
    same = bool(torch.equal(lg2, lg_f))
    print(f"repeat {r}: bit-identical {same}", flush=True)
out_r, lg_r, _ = run("0")
dev = max(float((lg_f[t:t + 100] - lg_r[t:t + 100]).abs().max()) for t in range(0, n, 100))
print("per-step max |diff| (first 12):", [round(float((lg_f[t] - lg_r[t]).abs().max()), 4) for t in range(min(n, 12))], flush=True)
print(f"fold vs round-2 chain: max |logit diff| {dev:.4g}", flush=True)
streams = [0, 1, 127, 128, B - 1]
report = []
check_streams(oc.CellOracle(m, exact=False), cls[:, streams].cpu().numpy(),
              out_f[:, streams].cpu().numpy(), lg_f[:, streams].cpu().numpy(), range(len(streams)),
              0, 0, 1.0, 4e-2, report=report, gids=streams)
print("fold vs oracle max dev", report[-1][1], flush=True)
report = []
check_streams(oc.CellOracle(m, exact=False), cls[:, streams].cpu().numpy(),
              out_r[:, streams].cpu().numpy(), lg_r[:, streams].cpu().numpy(), range(len(streams)),
              0, 0, 1.0, 4e-2, report=report, gids=streams)
print("round-2 vs oracle max dev", report[-1][1], flush=True)
