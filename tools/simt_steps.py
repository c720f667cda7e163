"""Per-step time of the SIMT kernels on a config (device loop, CUDA events):
python tools/simt_steps.py cfg5 [steps] -- prints one JSON line per kernel variant
(FW_SIMT_STAGED=1 weight-staged, =0 the __ldg kernel)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1611_09482_b200 import CellGenerator, Sampler, build_cell_model, configs  # noqa: E402


def main():
    spec = configs.by_name(sys.argv[1] if len(sys.argv) > 1 else "cfg5")
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    m = build_cell_model(spec.cell)
    bts = os.environ.get("BTS", "1,2,4,8").split(",")
    variants = [(f"staged_bt{b}", "1", b) for b in bts if b] + \
        ([("ldg", "0", None)] if os.environ.get("LDG", "1") == "1" else [])
    mc = "is%s_st%s" % (os.environ.get("FW_SIMT_ISSUERS", "4"), os.environ.get("FW_SIMT_STAGES", "3"))
    for name, staged, bt in variants:
        name = f"{name}_{mc}" if staged == "1" else name
        os.environ["FW_SIMT_STAGED"] = staged
        if bt:
            os.environ["FW_SIMT_BT"] = bt
        else:
            os.environ.pop("FW_SIMT_BT", None)
        gen = CellGenerator(m, spec.batch, kernel="simt")
        primer = torch.full((1, spec.batch), 128, dtype=torch.int32, device="cuda")
        s = Sampler(spec.sampler, configs.NOISE_SEED)
        gen.generate(primer, 5, s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        out, _ = gen.generate(primer, T, s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(json.dumps({"config": spec.name, "variant": name, "streams": spec.batch, "T": T,
                          "us_per_step": 1e3 * ms / T,
                          "samples_per_s": spec.batch * T / (ms * 1e-3),
                          "checksum": int(out.sum().item())}), flush=True)
        gen.close()


if __name__ == "__main__":
    main()
