"""Prefill (fw_cell_prefill, time-parallel) vs teacher-forced stepping on a BASELINE config.

    python tools/bench_prefill.py [--config cfg4] [--T 256]

Times with CUDA events (after one warm-up of each): the full-sequence forward with and
without logits, and fw_cell_generate over the same T inputs (teacher forced).
"""

import argparse
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1611_09482_b200 import CellGenerator, Sampler, build_cell_model, configs  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--T", type=int, default=256)
    ap.add_argument("--mode", default="", help="gemm | steps (FW_PREFILL_MODE); default: auto")
    args = ap.parse_args()
    if args.mode:
        import os

        os.environ["FW_PREFILL_MODE"] = args.mode
    spec = configs.by_name(args.config)
    m = build_cell_model(spec.cell)
    B, T = spec.batch, args.T
    x = torch.as_tensor(np.random.default_rng(1).integers(0, 256, (T, B)), dtype=torch.int32,
                        device="cuda")
    gen = CellGenerator(m, B)
    out = torch.empty((T, B), dtype=torch.int32, device="cuda")
    lg = torch.empty((T, B, 256), dtype=torch.float32, device="cuda")
    res = {"config": spec.name, "kernel": gen.kernel, "streams": B, "T": T,
           "mode": args.mode or "auto"}
    res["prefill_ms"] = timed(lambda: gen.prefill(x))
    res["prefill_logits_ms"] = timed(lambda: gen.prefill(x, want_logits=True, logits=lg))
    res["stepped_ms"] = timed(lambda: gen.generate(x, T, Sampler(0), out=out))
    for k in ("prefill_ms", "prefill_logits_ms", "stepped_ms"):
        res[k.replace("_ms", "_samples_per_s")] = B * T / (res[k] * 1e-3)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
