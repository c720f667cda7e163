"""Per-step generation latency vs depth on the GPU, fast (queues) vs naive (recompute the
receptive field every step): SURVEY §8(d) config 2 (1 block, L = 2..14, R = D = 128,
S = 256, A = 256, fp32, one stream) and the paper's Fig. 7 comparison.

    python tools/depth_sweep.py [--steps 1000] [--naive-steps 50]

fast: one fw_cell_generate call of `steps` steps (device loop), per-step = total / steps.
naive: NaiveCellGenerator primed with a full receptive field, so every step recomputes the
whole window (its steady-state cost). Times with CUDA events.
"""

import argparse
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1611_09482_b200 import CellGenerator, NaiveCellGenerator, Sampler, build_cell_model, configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--naive-steps", type=int, default=50)
    args = ap.parse_args()
    rows = []
    for L in configs.CFG2_LAYERS:
        spec = configs.cfg2(L)
        m = build_cell_model(spec.cell)
        rf = spec.cell.receptive_field()
        gen = CellGenerator(m, 1)
        x = torch.full((1, 1), 128, dtype=torch.int32, device="cuda")
        gen.generate(x, 10, Sampler(0))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gen.generate(x, args.steps, Sampler(0))
        e1.record()
        torch.cuda.synchronize()
        fast_us = e0.elapsed_time(e1) * 1e3 / args.steps
        ng = NaiveCellGenerator(m, 1)
        hist = torch.as_tensor(np.random.default_rng(L).integers(0, 256, (rf + args.naive_steps, 1)),
                               dtype=torch.int32, device="cuda")
        ng.logits(hist[:rf])
        torch.cuda.synchronize()
        e0.record()
        for k in range(args.naive_steps):
            ng.logits(hist[: rf + k + 1])
        e1.record()
        torch.cuda.synchronize()
        naive_us = e0.elapsed_time(e1) * 1e3 / args.naive_steps
        rows.append({"L": L, "receptive_field": rf, "kernel": gen.kernel,
                     "gpu_fast_us_per_step": fast_us, "gpu_naive_us_per_step": naive_us,
                     "naive_over_fast": naive_us / fast_us})
        print(json.dumps(rows[-1]), flush=True)


if __name__ == "__main__":
    main()
