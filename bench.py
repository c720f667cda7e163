#!/usr/bin/env python
"""Benchmark of the cached generation step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--kernel auto]
    python bench.py --impl reference ...      # the reference arm (CPU, host cores)

A "step" is one generation step of every stream of the workload (embed ->
all layers -> head -> selection -> re-embed), i.e. `batch` samples. Default
workload: BASELINE config 4 (4 blocks x 10 layers, R=128, 2D=256, S=512,
bf16 weights, 4,096 streams, Gumbel sampling) -- the config the samples/s
scaling metric is quoted on. Under torchrun the 4,096 streams are split over
the ranks (strong scaling, 512/GPU at 8 as BASELINE states; --weak runs the
config's streams on every GPU instead); noise is keyed by global stream id so
the generated sequences do not depend on N. Queue slots: fp32 on the SIMT
path; fp16 on the tcgen05 path (the MMA operand the tensor cores consume --
the line states both byte counts).

Prints one JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                  "source": "fallback (B200_PROFILING.md)"}
REPEATS = 3  # timed K-step runs; the line reports their median


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        d["source"] = "measured (MEASURED_PEAKS.json)"
        return d
    return dict(PEAKS_FALLBACK)


def fp32_peak():
    """Measured FP32 FFMA peak (tools/fp32_peak.cu on a B200, profiles/fp32_peak_*.json), else
    the nominal 148 x 128 x 2 x 1.965 GHz."""
    for f in sorted((ROOT / "profiles").glob("fp32_peak_*.json"), reverse=True):
        try:
            d = json.loads(f.read_text())
            return d["fp32_tflops"] * 1e12, f"measured ({f.relative_to(ROOT)}: FFMA microbenchmark)"
        except (ValueError, KeyError):
            continue
    return 148 * 128 * 2 * 1.965e9, "computed 148x128x2x1.965GHz (not measured)"


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def host_info():
    cores = len(os.sched_getaffinity(0))
    model = "unknown"
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return cores, model


# ---- clocks sampled during the timed region ------------------------------------------
REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 3:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.05)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        for r in self.rows:
            try:
                bits = int(r[2], 16)
            except ValueError:
                continue
            for b, name in REASON_BITS.items():
                if bits & b:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


# ---- workload accounting --------------------------------------------------------------
def step_accounting(cell, batch, queue_elem_bytes=4):
    """Algorithmic FLOPs and bytes of one step: every layer's
    dilated + residual + skip projections and the two head layers for every stream, the
    weights once, one ring slot read + one written per layer per stream (fp32 slots on the
    SIMT path, fp16 operand slots on the tcgen05 path), the embedding row and class io."""
    wbytes = 2 if cell.weight_dtype == "bf16" else 4
    flops = 2 * cell.macs_per_sample() * batch
    weight_bytes = cell.weight_count() * wbytes
    R, N = cell.residual_channels, cell.total_layers
    queue_bytes = batch * N * 2 * R * queue_elem_bytes
    io_bytes = batch * (R * 4 + 8)  # embedding row + class in/out
    return flops, weight_bytes + queue_bytes + io_bytes, queue_bytes


def simt_kernel_name(cell, batch):
    """The fp32 kernel the library selects (cell_simt.cu launch_cell_simt): one cluster per
    stream while the clusters fit the SMs (2 CTAs per stream up to 74 streams), then the
    warp-MMA kernel for the fp32 configs' shape (R = D = 64, S = H = A = 256), else the
    weight-staged kernel."""
    if batch * 2 <= 148:
        return "cell_lat_kernel"
    if (cell.residual_channels, cell.dilation_channels, cell.skip_channels, cell.H,
            cell.classes) == (64, 64, 256, 256, 256) and os.environ.get("FW_SIMT_HMMA") != "0":
        return "cell_hmma_kernel"
    return "cell_staged_kernel"


def traffic_per_launch(workload, kernel, batch):
    """DRAM bytes per step of the dominant kernel from the newest committed ncu summary of
    this exact workload, kernel family and per-GPU batch (never another config's)."""
    key = f"{workload}/{kernel}"
    for f in sorted((ROOT / "profiles").glob("ncu_summary_*.json"), reverse=True):
        try:
            d = json.loads(f.read_text())
        except ValueError:
            continue
        e = d.get(key)
        if not isinstance(e, dict) or e.get("dram_bytes_per_step") is None:
            continue
        if int(e.get("streams", -1)) != batch:
            continue
        return e["dram_bytes_per_step"], f.name
    return None, None


def workload_config(spec, total_batch, B, world, gen_queue_bytes=None):
    """The config dict both arms print (the workload, not the implementation)."""
    cell = spec.cell
    q32 = total_batch * cell.queue_slots() * cell.residual_channels * 4
    return {"workload": spec.name, "streams": total_batch, "streams_per_gpu": B,
            "layers": cell.total_layers, "residual": cell.residual_channels,
            "dilation": cell.dilation_channels, "skip": cell.skip_channels,
            "head": cell.H, "classes": cell.classes, "weights": cell.weight_dtype,
            "sampler": {0: "argmax", 1: "inverse-cdf", 2: "gumbel"}[spec.sampler],
            "parallelism": f"streams sharded x{world}",
            "l2": (f"queues {q32 / 1e9:.1f} GB (fp32) >> L2 (126 MB); each step touches "
                   "fresh slots of every layer's ring (no flush needed)") if q32 > 126e6 else
                  (f"queues {q32 / 1e6:.0f} MB (fp32) fit in L2: steady-state generation "
                   "keeps them resident, as a deployment would (no flush)")}


# ---- CPU baselines -------------------------------------------------------------------------
def _blas_threads():
    from threadpoolctl import threadpool_info

    return max([i.get("num_threads", 1) for i in threadpool_info()] or [1])


def oracle_port_timing(spec, model, total_batch, warmup, steps, max_seconds):
    """The cell oracle port (oracle/cell.py CachedCell, fp64, BLAS on all host threads) over
    the FULL batch of the workload: ``warmup`` untimed steps, then up to ``steps`` timed
    steps (stopping early after ``max_seconds``, at least 2). Returns (samples/s, steps
    timed, seconds)."""
    from oracle import cell as oc

    o = oc.CellOracle(model, exact=False)
    st = oc.CachedCell(o, total_batch)
    cls = np.full(total_batch, spec.primer_class)
    sid = np.arange(total_batch)
    for _ in range(max(1, warmup)):
        lg = st.step(cls)
        cls = oc.select(spec.sampler, lg, 2016, sid, st.t - 1)
    n = 0
    t0 = time.perf_counter()
    while True:
        lg = st.step(cls)
        cls = oc.select(spec.sampler, lg, 2016, sid, st.t - 1)
        n += 1
        el = time.perf_counter() - t0
        if n >= steps or (el >= max_seconds and n >= 2):
            break
    return total_batch * n / el, n, el


# shape proxies of the unmodified reference (plain tanh stack): blocks x L,
# hidden channels = the residual width
PROXY = {"cfg1_toy": (1, 10, 32), "cfg3_wavenet": (5, 10, 64), "cfg4_large_batch": (4, 10, 128),
         "cfg5_deep": (8, 12, 64)}


def _ref_worker(job):
    """One session of the unmodified reference (streamconv from baseline/_ref), timed by the
    reference's own runners (streamconv/bench.py:100-117)."""
    mode, blocks, L, C, steps = job
    from streamconv import ModelConfig, build_model
    from streamconv import bench as sb

    m = build_model(ModelConfig(blocks, L, hidden_channels=C, activation="tanh", init_seed=0))
    run = sb._timed_run_fast if mode == "fast" else sb._timed_run_naive
    run(m, 5)  # warm-up
    return run(m, steps) / steps


def reference_proxy_timing(spec):
    """The unmodified reference's CPU fast path on the workload's shape proxy, one session
    per host core (spawned processes), each 5 warm-up + 200 timed steps; plus its naive path
    for the depth-sweep proxies at L <= 12. Unavailable if baseline/_ref is not installed."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "streamconv").exists():
        return {"unavailable": "baseline/_ref not installed (see DESIGN.md)"}
    if spec.name in PROXY:
        blocks, L, C = PROXY[spec.name]
    elif spec.name.startswith("cfg2_L"):
        blocks, L, C = 1, spec.cell.layers_per_block, 128
    else:
        return {"unavailable": f"no proxy for {spec.name}"}
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/fw_numba_cache")
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import multiprocessing as mp

    cores, cpu = host_info()
    t0 = time.perf_counter()
    _ref_worker(("fast", blocks, L, C, 5))  # JIT compile once: the children load numba's cache
    jobs = [("fast", blocks, L, C, 200)] * cores
    # spawn, not fork: the parent may hold a CUDA context and library threads
    with mp.get_context("spawn").Pool(cores) as pool:
        per_step = pool.map(_ref_worker, jobs)
    out = {"kind": "reference (unmodified streamconv, baseline/_ref)",
           "proxy": f"ModelConfig({blocks}, {L}, hidden_channels={C}, activation='tanh', "
                    "init_seed=0): plain tanh stack, batch 1 per session",
           "fast_us_per_step": 1e6 * statistics.mean(per_step),
           "fast_samples_per_s_all_cores": sum(1.0 / s for s in per_step),
           "sessions": cores, "cores": cores, "cpu": cpu,
           "timing": "reference streamconv.bench._timed_run_fast (perf_counter), 5 warm-up + "
                     "200 timed steps per session, one session per core (spawned processes)"}
    if spec.name.startswith("cfg2_L") and L <= 12:
        out["naive_us_per_step"] = 1e6 * _ref_worker(("naive", blocks, L, C, 20))
    out["seconds"] = time.perf_counter() - t0
    return out


def cpu_baseline(spec, model, total_batch, max_seconds=20.0):
    cores, cpu = host_info()
    v, n, el = oracle_port_timing(spec, model, total_batch, 1, 10_000, max_seconds)
    return {"value": v, "unit": "samples/s", "cores": _blas_threads(), "kind": "port",
            "sample": f"oracle/cell.py CachedCell fp64 (BLAS), all {total_batch} streams of "
                      f"{spec.name} x {n} steps, {el:.1f} s",
            "host_cores": cores, "cpu": cpu,
            "reference_proxy": reference_proxy_timing(spec)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--kernel", default="auto", choices=["auto", "simt", "tcgen05"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=0, help="override total streams")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--sampler", type=int, default=-1, help="override the config's selection rule")
    ap.add_argument("--weak", action="store_true",
                    help="run the config's streams on every GPU instead of splitting them over "
                         "the GPUs (BASELINE cfg4: 4,096 total, 512 per GPU at 8)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    from paper_1611_09482_b200 import configs
    from paper_1611_09482_b200.cell import build_cell_model

    spec = configs.by_name(args.config)
    if args.sampler >= 0:
        import dataclasses

        spec = dataclasses.replace(spec, sampler=args.sampler)
    rank, world, local = dist_env()
    total_batch = (args.batch or spec.batch) * (world if args.weak else 1)
    metric = "generated samples/sec (batch x steps / s)"
    scaling = "weak" if args.weak else "strong"

    if args.impl == "reference":
        # the reference arm: the CPU path on the host cores, rank 0 only
        if rank != 0:
            return
        from paper_1611_09482_b200.distributed import shard_streams

        model = build_cell_model(spec.cell)
        B = shard_streams(total_batch, world, 0).count
        v, n, el = oracle_port_timing(spec, model, total_batch, args.warmup, args.steps,
                                      max_seconds=150.0)
        cores, cpu = host_info()
        cb = {"value": v, "unit": "samples/s", "cores": _blas_threads(), "kind": "port",
              "sample": f"oracle/cell.py CachedCell fp64 (BLAS), all {total_batch} streams x "
                        f"{n} steps after {args.warmup} warm-up steps, {el:.1f} s",
              "host_cores": cores, "cpu": cpu,
              "reference_proxy": reference_proxy_timing(spec)}
        line = {"impl": "reference", "metric": metric, "value": v, "unit": "samples/s",
                "n_gpus": world, "steps": n, "warmup": args.warmup,
                "ms_per_step": 1e3 * total_batch / v, "higher_is_better": True,
                "scaling": scaling, "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded N(0,1/fan_in) weights, primer class 128, "
                        "counter-hash Gumbel noise)",
                "config": workload_config(spec, total_batch, B, world),
                "note": "reference arm = the CPU port of the cell (oracle/cell.py): the "
                        "reference (pure Python/numba, plain stacks only) has no gated cell; "
                        "its own fast path on the shape proxy is in cpu_baseline."
                        "reference_proxy (DESIGN.md §6)",
                "cpu_baseline": cb,
                "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch

    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)

    from paper_1611_09482_b200 import CellGenerator, Sampler
    from paper_1611_09482_b200.distributed import gather_sequences, shard_streams

    shard = shard_streams(total_batch, world, rank)
    B, offset = shard.count, shard.offset
    model = build_cell_model(spec.cell)
    gen = CellGenerator(model, B, kernel=args.kernel)
    sampler = Sampler(spec.sampler, configs.NOISE_SEED, offset)
    primer = torch.full((1, B), spec.primer_class, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x):
        if world > 1:
            t = torch.tensor([x], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            return float(t.item())
        return x

    # warm-up
    gen.generate(primer, args.warmup, sampler)
    torch.cuda.synchronize()

    # device-timed K steps, inputs resident in HBM (REPEATS runs, median)
    out = torch.empty((args.steps, B), dtype=torch.int32, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    runs_ms = []
    with ClockSampler(dev.index) as clk:
        for _ in range(REPEATS):
            gen.reset()
            barrier()
            torch.cuda.synchronize()
            e0.record(stream)
            gen.generate(primer, args.steps, sampler, out=out, check_inputs=False)
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
            runs_ms.append(max_over_ranks(e0.elapsed_time(e1)))
    ms = statistics.median(runs_ms)
    launches = gen.last_launch_count

    # end-to-end through the public host-buffer API (copies inside the timed region), plus
    # the final gather of the generated sequences when N > 1 (the only collective)
    host_in = torch.full((1, B), spec.primer_class, dtype=torch.int32).pin_memory().numpy()
    host_out = torch.empty((args.steps, B), dtype=torch.int32).pin_memory().numpy()
    # warm the host path at the timed size (the library's device staging buffer grows to
    # the largest call it has seen; a first call at a new size allocates)
    gen.reset()
    gen.generate_host(host_in, args.steps, sampler, out=host_out)
    gather_buf = torch.empty((args.steps, B), dtype=torch.int32, device=dev) if world > 1 else None
    e2e_runs = []
    full = None
    for _ in range(REPEATS):
        gen.reset()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        gen.generate_host(host_in, args.steps, sampler, out=host_out)
        if world > 1:
            gather_buf.copy_(torch.from_numpy(host_out), non_blocking=True)
            full = gather_sequences(gather_buf, shard, total_batch).cpu()
        e2e_runs.append(max_over_ranks(time.perf_counter() - t0))
    e2e_s = statistics.median(e2e_runs)
    same = bool(np.array_equal(host_out, out.cpu().numpy()))
    if world > 1:
        assert full.shape == (args.steps, total_batch)

    # dominant-kernel time per step, CUDA events on the launching stream (separate pass so
    # the timed region above carries no extra events)
    gen.reset()
    gen.set_kernel_timing(True)
    nk = min(args.steps, 100)
    gen.generate(primer, nk, sampler)
    torch.cuda.synchronize()
    k_ms, _, k_steps = gen.kernel_times()
    gen.set_kernel_timing(False)
    kernel_s_per_step = k_ms / 1e3 / max(k_steps, 1)

    if rank == 0:
        peaks = load_peaks()
        tc = gen.kernel == "tcgen05"
        qeb = 2 if tc else 4
        flops, bytes_step, qbytes = step_accounting(spec.cell, B, qeb)
        _, bytes_fp32q, qbytes32 = step_accounting(spec.cell, B, 4)
        s_per_step = ms / 1e3 / args.steps
        value = total_batch * args.steps / (ms / 1e3)
        hbm = peaks["hbm_gbs"] * 1e9
        if spec.cell.weight_dtype == "bf16":
            # burst: the timed region is a few ms of one kernel, not a seconds-long power-
            # capped run (the sustained figure is reported beside it)
            comp_peak = peaks["bf16_tflops"] * 1e12
            peak_src = peaks["source"] + ", bf16 dense burst"
        else:
            comp_peak, peak_src = fp32_peak()
        t_flop, t_byte = flops / comp_peak, bytes_step / hbm
        k_s = kernel_s_per_step
        if t_flop >= t_byte:
            roof = {"bound": "tensor" if spec.cell.weight_dtype == "bf16" else "fp32",
                    "achieved": flops / k_s / 1e12, "peak": comp_peak / 1e12, "unit": "TFLOP/s"}
        else:
            roof = {"bound": "hbm", "achieved": bytes_step / k_s / 1e9, "peak": hbm / 1e9,
                    "unit": "GB/s"}
        roof["frac"] = roof["achieved"] / roof["peak"]
        kname = "step_kernel" if tc else simt_kernel_name(spec.cell, B)
        kfam = "tcgen05" if tc else {"cell_lat_kernel": "simt", "cell_hmma_kernel": "hmma",
                                     "cell_staged_kernel": "simt"}[kname]
        traffic, tsrc = traffic_per_launch(spec.name, kfam, B)
        roof["traffic"] = traffic
        roof["kernel"] = ("step_kernel (persistent: chain + skip sum + heads + selection, one "
                          "cooperative launch per generate call, per-step share)" if tc
                          else f"{kname} (persistent fp32 kernel, one launch per generate call, "
                          "per-step share" + ("; its products run on the tensor cores as mma.sync "
                          "with a 3-term fp16 split, reported against the FP32 peak of the fp32 "
                          "model's FLOPs)" if kname == "cell_hmma_kernel" else ")"))
        roof["algorithmic_per_step"] = {
            "flop": flops, "bytes": bytes_step,
            "queue_bytes": qbytes, "queue_slot_dtype": "fp16" if tc else "fp32",
            "bytes_with_fp32_queues": bytes_fp32q, "queue_bytes_fp32": qbytes32}
        roof["kernel_us_per_step"] = 1e6 * k_s
        roof["kernel_share_of_step"] = k_s / s_per_step
        roof["step_roofline_us"] = 1e6 * max(t_flop, t_byte)
        roof["step_roofline_frac"] = max(t_flop, t_byte) / s_per_step
        roof["peak_source"] = peak_src
        if spec.cell.weight_dtype == "bf16":
            sus = peaks.get("bf16_tflops_sustained")
            if sus:
                roof["frac_vs_sustained_peak"] = flops / k_s / (sus * 1e12)
        roof["traffic_source"] = (f"profiles/{tsrc} (ncu --set full, {spec.name}, {kfam}, "
                                  f"{B} streams)" if tsrc else
                                  f"no ncu capture of {spec.name}/{kfam} at {B} streams")
        line = {
            "metric": metric, "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": ("bf16 weights, fp16 MMA operands (fp16 queue slots), fp32 accumulation"
                      if tc else ("bf16 weights, fp32 arithmetic" if spec.cell.weight_dtype ==
                                  "bf16" else "f32")),
            "data": "synthetic (seeded N(0,1/fan_in) weights, primer class 128, "
                    "counter-hash Gumbel noise)",
            "config": workload_config(spec, total_batch, B, world),
            "kernel": gen.kernel,
            "timed_runs_ms": runs_ms,
            "roofline": roof,
            "e2e": {"value": total_batch * args.steps / e2e_s, "unit": "samples/s",
                    "h2d_bytes_per_step": B * 4 / args.steps, "d2h_bytes_per_step": B * 4,
                    "api": "CellGenerator.generate_host -> fw_cell_generate_host"
                           + (" + all_gather of the sequences (NCCL)" if world > 1 else ""),
                    "runs_s": e2e_runs, "matches_device_run": same},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(spec, model, total_batch, args.cpu_seconds)
        print(json.dumps(line), flush=True)
    gen.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
