"""Per-layer phase timeline of the tcgen05 chain kernel (CTA 0, clock64 cycles).

    python tools/trace_chain.py [--config cfg4] [--steps 3]

Slots (csrc/cell_tc.cu TraceSlot): MMA warp -- x_{t-d} half 0 issued, xt_ready
seen, acc0 committed, acc1 committed, z0 seen, z1 seen, x_full committed, cycles
spent waiting on weights, whether half 0 was issued during the previous layer;
gate thread (warp 2 lane 0) -- layer start, x_full seen, xt arrive, acc0 seen,
z0 arrive, acc1 seen, z1 arrive; queue thread -- xd arrive, next slot loads
issued; producer stage A0/A1/B/C issued.
"""

import argparse
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1611_09482_b200 import CellGenerator, Sampler, _lib, build_cell_model, configs  # noqa: E402

NAMES = ["mma_xd", "mma_xt", "mma_acc0", "mma_acc1", "mma_z0", "mma_z1", "mma_xful", "mma_wwai",
         "epi_a", "epi_xful", "epi_xt", "epi_acc0", "epi_z0", "epi_acc1", "epi_z1", "h0_early",
         "q_xd", "q_load", "prod_a0", "prod_a1", "prod_b", "prod_c", "g0_ld", "g0_math",
         "q_xdfree", "q_xqfull", "g1_ld", "g1_math", "q_bar", "q_rel", "q_stash", "q_end",
         "c_xt0", "c_xd1", "c_xt1", "c_resz0", "c_xd0e", "c_resz1"]
RAW = {7, 15}  # counts / flags, not timestamps
SLOTS = 48  # kTraceSlots


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--batch", type=int, default=0)
    args = ap.parse_args()
    spec = configs.by_name(args.config)
    m = build_cell_model(spec.cell)
    B = args.batch or spec.batch
    gen = CellGenerator(m, B, kernel="tcgen05")
    L = spec.cell.total_layers
    tr = torch.zeros((L + 1, SLOTS), dtype=torch.int64, device="cuda")
    _lib.check(gen._lib.fw_debug_trace(gen._h, C.c_void_p(tr.data_ptr())))
    primer = torch.full((1, B), 128, dtype=torch.int32, device="cuda")
    gen.generate(primer, args.steps, Sampler(spec.sampler, configs.NOISE_SEED))
    torch.cuda.synchronize()
    t = tr.cpu().numpy().astype(np.int64)
    base = t[0, 8]  # epi_a of layer 0
    print("cycles relative to layer-0 epi_a; per-layer deltas vs that layer's epi_a")
    print("layer " + " ".join(f"{n[:8]:>8s}" for n in NAMES))
    for l in range(L):
        row = t[l].copy()
        ref = row[8]
        cells = []
        for i, v in enumerate(row[:len(NAMES)]):
            if i in RAW:
                cells.append(f"{v:8d}")
            elif v == 0:
                cells.append(f"{'-':>8s}")
            else:
                cells.append(f"{v - ref:8d}")
        print(f"{l:5d} " + " ".join(cells) + f"   (start {ref - base})")
    g = t[L]
    if g[0]:
        names = ["chain start", "chain last layer", "skip: last z seen", "s published",
                 "head1 published", "head2 acc seen", "selection done", "skip acc committed",
                 "h1 mma: tmem free", "h1 first stage", "h1 acc committed",
                 "h2 mma: tmem free", "h2 first stage", "h2 acc committed", "epi: skip acc seen",
                 "epi: h1 acc seen", "chain: cls seen", "prev step selection done",
                 "chain: layer-0 xt ready", "chain: cls loaded", "chain: embedding loaded",
                 "sel: cc0 done", "sel: cc1 done", "sel: cc2 done", "sel: epilogue done", "sel: bar", "sel: loop done", "sel: exchange done", "sel: start", "sel: first tmem ld"]
        print("step timeline (global ns, last step): " + ", ".join(
            f"{n} {(g[i] - g[0]) / 1e3:.2f} us" for i, n in enumerate(names) if g[i]))
    t = t[:L]
    per_layer = np.diff(t[:, 8])
    print(f"mean cycles/layer {per_layer.mean():.0f}; total {t[-1, 8] - base}; "
          f"weight-wait cycles total {t[:, 7].sum()}")


if __name__ == "__main__":
    main()
