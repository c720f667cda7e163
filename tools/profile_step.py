"""One generate call of STEPS steps after a warm-up call -- the target of the committed ncu
captures: ncu -k regex:step_kernel -s 1 -c 1 ... python tools/profile_step.py [steps] [config] [batch]
(cfg4: the tcgen05 step kernel; fp32 configs: the SIMT kernel auto-selected for the batch)"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1611_09482_b200 import CellGenerator, Sampler, build_cell_model, configs  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
spec = configs.by_name(sys.argv[2] if len(sys.argv) > 2 else "cfg4")
batch = int(sys.argv[3]) if len(sys.argv) > 3 else spec.batch
gen = CellGenerator(build_cell_model(spec.cell), batch,
                    kernel="tcgen05" if spec.cell.weight_dtype == "bf16" else "simt")
primer = torch.full((1, batch), spec.primer_class, dtype=torch.int32, device="cuda")
gen.generate(primer, steps, Sampler(spec.sampler, configs.NOISE_SEED))  # warm-up launch
torch.cuda.synchronize()
torch.cuda.profiler.start()  # range for ncu --replay-mode (app-)range --profile-from-start off
gen.generate(primer, steps, Sampler(spec.sampler, configs.NOISE_SEED))  # profiled launch
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"profiled: {steps} steps of {spec.name} in one launch")
