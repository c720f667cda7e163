"""Write profiles/ncu_summary_<tag>.json from an ncu --set full report (+ launch list).

    python profiles/make_summary.py r01b gpurun_out/prof_r01_step.ncu-rep \
        gpurun_out/launches_r01_v2.csv [steps_per_launch]

Per kernel: duration, DRAM bytes read/written, tensor-pipe activity, L2/L1 throughput.
Also the per-step DRAM traffic of the cfg4 tcgen05 step (sum over its 4 kernels), which
bench.py reports as roofline.traffic.
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

tag, rep = sys.argv[1], sys.argv[2]
launch_csv = sys.argv[3] if len(sys.argv) > 3 else None
steps_per_launch = int(sys.argv[4]) if len(sys.argv) > 4 else 1
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
ix = {h: i for i, h in enumerate(hdr)}
keys = {"duration_us": "gpu__time_duration.sum", "dram_read": "dram__bytes_read.sum",
        "dram_write": "dram__bytes_write.sum",
        "tensor_active_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l2_throughput_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1_throughput_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second", "grid": "launch__grid_size",
        "registers": "launch__registers_per_thread"}
scale = {"us": 1.0, "ns": 1e-3, "ms": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6,
         "Gbyte": 1e9, "%": 1.0, "Ghz": 1.0, "Mhz": 1e-3, "": 1.0, "register/thread": 1.0}
kernels = []
for r in rows[2:]:
    k = {"kernel": r[ix["Kernel Name"]].split("(")[0]}
    if "step_kernel" in k["kernel"]:
        k["steps_per_launch"] = steps_per_launch
    for name, metric in keys.items():
        if metric in ix:
            v = r[ix[metric]].replace(",", "")
            try:
                k[name] = float(v) * scale.get(units[ix[metric]], 1.0)
            except ValueError:
                k[name] = None
    kernels.append(k)
out = {"round": tag, "report": Path(rep).name, "kernels": kernels}
persist = [k for k in kernels if "step_kernel" in k["kernel"]]
if persist:
    k = persist[0]
    n = k["steps_per_launch"]
    out["cfg4_large_batch/tcgen05"] = {
        "dram_bytes_per_step": ((k["dram_read"] or 0) + (k["dram_write"] or 0)) / n,
        "kernels": [k["kernel"]], "steps_per_launch": n,
        "duration_us_per_step_cold": (k["duration_us"] or 0) / n,
        "note": "ncu --set full of one persistent launch (all steps' work); per-step = / steps"}
step = [k for k in kernels if "chain_kernel" in k["kernel"] or "gemm_kernel" in k["kernel"]]
if step and not persist:
    # one chain + skip + head1 + head2 launch = one cfg4 step (the capture order)
    first = next(i for i, k in enumerate(step) if "chain_kernel" in k["kernel"])
    one = step[first:first + 4]
    dram = sum((k["dram_read"] or 0) + (k["dram_write"] or 0) for k in one)
    out["cfg4_large_batch/tcgen05"] = {
        "dram_bytes_per_step": dram, "kernels": [k["kernel"] for k in one],
        "duration_us_cold": sum(k["duration_us"] or 0 for k in one),
        "note": "ncu --set full, serialised cold-cache replays: compare shares, not absolutes"}
if launch_csv:
    text = Path(launch_csv).read_text().splitlines()
    start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
    agg = {}
    for r in csv.DictReader(io.StringIO("\n".join(text[start:]))):
        if r["Metric Name"] == "gpu__time_duration.sum":
            name = r["Kernel Name"].split("(")[0].replace("void ", "")
            agg.setdefault(name, []).append(float(r["Metric Value"]) / 1e3)
    tot = sum(sum(v) for v in agg.values())
    out["launch_list"] = {k: {"n": len(v), "mean_us": sum(v) / len(v), "share": sum(v) / tot}
                          for k, v in agg.items()}
dst = Path(__file__).parent / f"ncu_summary_{tag}.json"
dst.write_text(json.dumps(out, indent=1))
print(dst)
print(json.dumps(out.get("cfg4_large_batch/tcgen05"), indent=1))
