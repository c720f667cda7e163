"""Max |logit| deviation of a GPU kernel vs the fp64 oracle (teacher-forced on its own history)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from oracle import cell as oc
from paper_1611_09482_b200 import CellGenerator, Sampler, build_cell_model, configs
from cellcheck import histories

kernel = sys.argv[1] if len(sys.argv) > 1 else "tcgen05"
spec = configs.cfg4()
m = build_cell_model(spec.cell)
gen = CellGenerator(m, spec.batch, kernel=kernel)
n = 32
primer = torch.full((1, spec.batch), 128, dtype=torch.int32, device="cuda")
out, lg = gen.generate(primer, n, Sampler(2, configs.NOISE_SEED), n_logit_steps=n)
out, lg = out.cpu().numpy(), lg.cpu().numpy()
o = oc.CellOracle(m, exact=False)
hist = histories(np.full((1, spec.batch), 128), out)
devs = []
for s in range(0, spec.batch, 257):
    ref = o.forward_full(hist[:, s])
    devs.append(np.max(np.abs(lg[:, s] - ref)))
print(f"{kernel}: max logit dev over {len(devs)} streams x {n} steps: {max(devs):.4g} (median {np.median(devs):.4g}); |logits| ~ {np.abs(lg).mean():.3g}")
