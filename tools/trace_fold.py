"""Per-layer timeline of the folded chain (CTA 0, clock64 cycles; chain_fold.cuh FT slots).

    python tools/trace_fold.py [--batch 4096] [--steps 3]

Each row: the layer's slots relative to the gate seeing acc_full (slot 8), and the period
(slot 8 minus the previous layer's slot 8).
"""

import argparse
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1611_09482_b200 import CellGenerator, Sampler, _lib, build_cell_model, configs  # noqa: E402

NAMES = {0: "m_accfr", 1: "m_pop", 2: "m_xt", 3: "m_zown", 4: "m_zpeer", 5: "m_accful", 6: "m_xful",
         8: "g_acc", 9: "g_ld", 10: "g_math", 11: "g_imgw", 12: "g_zown", 13: "g_sendw", 14: "g_sent",
         16: "x_xful", 17: "x_xt", 20: "p_zown", 21: "p_rel", 24: "pr_lay", 25: "pr_pop"}
SLOTS = 48


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--batch", type=int, default=4096)
    args = ap.parse_args()
    spec = configs.cfg4()
    m = build_cell_model(spec.cell)
    gen = CellGenerator(m, args.batch, kernel="tcgen05")
    L = spec.cell.total_layers
    tr = torch.zeros((L + 1, SLOTS), dtype=torch.int64, device="cuda")
    _lib.check(gen._lib.fw_debug_trace(gen._h, C.c_void_p(tr.data_ptr())))
    primer = torch.full((1, args.batch), 128, dtype=torch.int32, device="cuda")
    gen.generate(primer, args.steps, Sampler(spec.sampler, configs.NOISE_SEED))
    torch.cuda.synchronize()
    t = tr.cpu().numpy().astype(np.int64)
    keys = sorted(NAMES)
    print("layer  period " + " ".join(f"{NAMES[k]:>8s}" for k in keys))
    periods = []
    for l in range(L):
        ref = t[l, 8]
        per = ref - t[l - 1, 8] if l > 0 else 0
        if l > 1:
            periods.append(per)
        cells = [f"{(t[l, k] - ref) if t[l, k] else 0:8d}" for k in keys]
        print(f"{l:5d} {per:7d} " + " ".join(cells))
    print(f"median period (layers 2..): {np.median(periods):.0f} cycles")
    tg = t[L, :8]
    print("step timeline (ns) slots 0..7:", (tg - tg[0]).tolist())
    gen.close()


if __name__ == "__main__":
    main()
