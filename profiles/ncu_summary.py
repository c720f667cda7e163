"""Per-workload ncu summary (bench.py reads `<workload>/<kernel family>` entries):

    python profiles/ncu_summary.py OUT.json TAG REPORT WORKLOAD FAMILY STREAMS STEPS [note]

Adds (or replaces) one entry: the kernel's duration, DRAM bytes, tensor-pipe activity and
L2->SM bytes per launch and per step (the report holds ONE launch running STEPS steps)."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

out, tag, rep, workload, fam, streams, steps = sys.argv[1:8]
note = sys.argv[8] if len(sys.argv) > 8 else ""
streams, steps = int(streams), int(steps)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
ix = {h: i for i, h in enumerate(hdr)}
scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6,
         "Gbyte": 1e9}


def val(r, m):
    v = r[ix[m]].replace(",", "")
    return float(v) * scale.get(units[ix[m]], 1.0)


r = rows[2]
k = {"kernel": r[ix["Kernel Name"]].split("(")[0], "report": Path(rep).name,
     "duration_us": val(r, "gpu__time_duration.sum"),
     "dram_read": val(r, "dram__bytes_read.sum"), "dram_write": val(r, "dram__bytes_write.sum"),
     "l2_to_sm_bytes": val(r, "l1tex__m_xbar2l1tex_read_bytes.sum"),
     "tensor_active_pct": val(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
     "sm_clock_ghz": val(r, "sm__cycles_elapsed.avg.per_second") / 1e9
     if units[ix["sm__cycles_elapsed.avg.per_second"]] == "hz" else val(r, "sm__cycles_elapsed.avg.per_second"),
     "grid": val(r, "launch__grid_size"), "registers": val(r, "launch__registers_per_thread"),
     "inst_executed": val(r, "smsp__inst_executed.sum")}
entry = {"streams": streams, "steps_per_launch": steps, "kernels": [k["kernel"]],
         "dram_bytes_per_step": (k["dram_read"] + k["dram_write"]) / steps,
         "l2_to_sm_bytes_per_step": k["l2_to_sm_bytes"] / steps,
         "duration_us_per_step_profiled": k["duration_us"] / steps, "detail": k, "note": note}
p = Path(out)
d = json.loads(p.read_text()) if p.exists() else {"round": tag}
d[f"{workload}/{fam}"] = entry
p.write_text(json.dumps(d, indent=1) + "\n")
print(json.dumps(entry, indent=1))
