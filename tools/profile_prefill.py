"""One fw_cell_prefill call (time-parallel forward with logits) after a warm-up call -- the
target of the prefill launch list: python tools/profile_prefill.py [config] [T] [batch]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1611_09482_b200 import CellGenerator, build_cell_model, configs  # noqa: E402

spec = configs.by_name(sys.argv[1] if len(sys.argv) > 1 else "cfg5")
T = int(sys.argv[2]) if len(sys.argv) > 2 else 64
batch = int(sys.argv[3]) if len(sys.argv) > 3 else spec.batch
gen = CellGenerator(build_cell_model(spec.cell), batch)
x = torch.randint(0, spec.cell.classes, (T, batch), dtype=torch.int32, device="cuda")
gen.prefill(x, want_logits=True)
gen.reset()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
gen.prefill(x, want_logits=True)
ev[1].record()
torch.cuda.synchronize()
print(f"prefill {spec.name} T={T} B={batch} kernel={gen.kernel}: {ev[0].elapsed_time(ev[1]):.3f} ms")
