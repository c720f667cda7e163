"""Command line: SURVEY §8(f) rank 4 -- the reference's entry points (``cli.py:236-302``) on
the GPU, for both model kinds.

    python -m paper_1611_09482_b200 init-model --layers 4 --out m.txt     (plain, as the reference)
    python -m paper_1611_09482_b200 init-cell --layers 10 --residual 32 --skip 128 --out c.txt
    python -m paper_1611_09482_b200 generate --model m.txt --steps 100 --mode fast --out y.txt
    python -m paper_1611_09482_b200 verify --model m.txt            (or --random-grid)
    python -m paper_1611_09482_b200 bench --layers-to 8 --out sweep.csv

Plain documents generate float samples (one per line, as the reference writes them), cell
documents class ids. ``generate --mode naive`` is the cache-free generator (recompute the
receptive field every step). ``verify`` cross-checks the implementations against each other
-- plain: the device step loop, per-step calls and the naive generator (bit-exact, default
tolerance 0 as in the reference); cell: step-kernel logits, the time-parallel full-sequence
forward and the naive generator (tolerance of the weight dtype). ``bench`` writes the
reference's CSV columns (``bench.py:52-70``). Exit codes: 0 success, 1 verification
failure, 2 usage error (ValueError / OSError), as the reference.
"""

from __future__ import annotations

import argparse
import sys
import time

import numpy as np

from .cell import CellConfig, CellModel, build_cell_model
from .model import ACTIVATIONS, Model, ModelConfig, build_model, count_macs, receptive_field
from .model_io import load_any, save_cell_model, save_model

CELL_TOL = {"f32": 1e-4, "bf16": 2e-2}


def _write_lines(path: str, values, fmt) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        for v in values:
            fh.write(fmt(v) + "\n")


def _read_numbers(path: str, cast):
    out = []
    with open(path, encoding="utf-8") as fh:
        for ln, line in enumerate(fh, start=1):
            line = line.strip()
            if not line:
                continue
            try:
                v = cast(line)
            except ValueError:
                raise ValueError(f"{path}:{ln}: not a number: {line!r}") from None
            if not np.isfinite(v):
                raise ValueError(f"{path}:{ln}: non-finite sample")
            out.append(v)
    return out


# ---- init ----------------------------------------------------------------------------------
def cmd_init_model(a) -> int:
    cfg = ModelConfig(blocks=a.blocks, layers_per_block=a.layers, filter_width=a.width,
                      dilation_base=a.base, hidden_channels=a.channels,
                      activation=a.activation, init_seed=a.seed)
    save_model(build_model(cfg), a.out)
    print(f"receptive field: {receptive_field(cfg)}")
    print("queue capacities: " + " ".join(str((cfg.filter_width - 1) * d) for d in cfg.dilations()))
    return 0


def cmd_init_cell(a) -> int:
    cfg = CellConfig(blocks=a.blocks, layers_per_block=a.layers, residual_channels=a.residual,
                     dilation_channels=a.dilation or a.residual, skip_channels=a.skip,
                     classes=a.classes, head_channels=a.head, dilation_base=a.base,
                     weight_dtype=a.dtype, init=a.init, bias=a.bias, init_seed=a.seed)
    save_cell_model(build_cell_model(cfg), a.out)
    print(f"receptive field: {cfg.receptive_field()}")
    print(f"ring slots per stream: {cfg.queue_slots()}")
    return 0


# ---- generate --------------------------------------------------------------------------------
def cmd_generate(a) -> int:
    model = load_any(a.model)
    t0 = time.perf_counter()
    if isinstance(model, CellModel):
        from .generate import Sampler, cell_fast_generate
        from .naive import cell_naive_generate

        primer = _read_numbers(a.primer, int) if a.primer else []
        if a.mode == "fast":
            out = cell_fast_generate(model, primer, a.steps,
                                     sampler=Sampler(a.sampler, a.seed))[0]
        else:
            if a.sampler != 0:
                raise ValueError("the naive cell generator is greedy (--sampler 0)")
            out = cell_naive_generate(model, primer, a.steps)[0]
        _write_lines(a.out, out, lambda v: str(int(v)))
        macs = model.config.macs_per_sample()
    else:
        from .fast import fast_generate
        from .naive import plain_naive_generate

        primer = _read_numbers(a.primer, float) if a.primer else []
        gen = fast_generate if a.mode == "fast" else plain_naive_generate
        out = gen(model, primer, a.steps).scalars()
        _write_lines(a.out, out, lambda v: repr(float(v)))
        macs = count_macs(model.config, a.mode).multiply_accumulates
    elapsed = time.perf_counter() - t0
    rate = a.steps / elapsed if elapsed > 0 else float("inf")
    print(f"{a.mode}: {a.steps} samples, {rate:.1f} samples/s, {macs} MACs/step", file=sys.stderr)
    return 0


# ---- verify ---------------------------------------------------------------------------------
def verification_grid(seed: int = 7) -> list[ModelConfig]:
    """The reference's seeded verification grid (cli.py:138-157): 144 plain architectures."""
    cfgs = []
    for blocks in (1, 2, 3):
        for layers in range(1, 7):
            for width in (2, 3):
                for channels in (1, 4):
                    for act in ("linear", "tanh"):
                        cfgs.append(ModelConfig(blocks=blocks, layers_per_block=layers,
                                                filter_width=width, dilation_base=2,
                                                hidden_channels=channels, activation=act,
                                                init_seed=seed + len(cfgs)))
    return cfgs


def _max_dev(a, b) -> float:
    return float(np.max(np.abs(np.asarray(a, dtype=np.float64) - np.asarray(b, dtype=np.float64)),
                        initial=0.0))


def verify_plain(model: Model, steps: int) -> list[tuple[str, float]]:
    import ctypes as C

    import torch

    from . import _lib
    from .fast import fast_generate, fast_step, init_state
    from .naive import plain_naive_generate, plain_naive_step

    rng = np.random.default_rng([model.config.init_seed, 0xA5])
    x = rng.uniform(-1.0, 1.0, steps)
    st = init_state(model)
    xin = torch.as_tensor(x.reshape(-1, 1), device=st._dev)
    yout = torch.empty((steps, 1), dtype=torch.float64, device=st._dev)
    _lib.check(st._lib.fw_plain_generate(st._h, C.c_void_p(xin.data_ptr()), steps, steps,
                                         C.c_void_p(yout.data_ptr()), _lib.stream_ptr()))
    loop = yout[:, 0].cpu().numpy()
    st.reset()
    stepped = np.array([fast_step(st, v, model) for v in x])
    naive = np.array([plain_naive_step(model, x[: i + 1], st) for i in range(steps)])
    st.close()
    free_fast = fast_generate(model, x[:1], steps).scalars()
    free_naive = plain_naive_generate(model, x[:1], steps).scalars()
    return [("teacher-forced device loop vs per-step calls", _max_dev(loop, stepped)),
            ("teacher-forced fast vs naive", _max_dev(loop, naive)),
            ("free-run fast vs naive", _max_dev(free_fast, free_naive))]


def verify_cell(model: CellModel, steps: int) -> list[tuple[str, float]]:
    import torch

    from .generate import CellGenerator, Sampler, cell_fast_generate
    from .naive import NaiveCellGenerator, cell_naive_generate

    A = model.config.classes
    x = np.random.default_rng([model.config.init_seed, 0xA5]).integers(0, A, (steps, 1))
    xt = torch.as_tensor(x, dtype=torch.int32, device="cuda")
    g = CellGenerator(model, 1)
    _, lg = g.generate(xt, steps, Sampler(0), n_logit_steps=steps)
    fast = lg[:, 0].cpu().numpy()
    g.reset()
    full = g.prefill(xt, want_logits=True)[:, 0].cpu().numpy()
    g.close()
    ng = NaiveCellGenerator(model, 1)
    naive = np.stack([ng.logits(xt[: i + 1])[0].cpu().numpy() for i in range(steps)])
    ng.close()
    a = cell_fast_generate(model, x[:1, 0], steps)
    b = cell_naive_generate(model, x[:1, 0], steps)
    return [("teacher-forced step kernel vs full-sequence forward", _max_dev(fast, full)),
            ("teacher-forced step kernel vs naive", _max_dev(fast, naive)),
            ("free-run fast vs naive (fraction of differing samples)",
             float(np.mean(a != b)))]


def cmd_verify(a) -> int:
    if a.random_grid:
        models = [(f"grid {i}", build_model(c)) for i, c in enumerate(verification_grid())]
    else:
        models = [(a.model, load_any(a.model))]
    worst = 0.0
    failed = False
    for name, m in models:
        if isinstance(m, CellModel):
            tol = CELL_TOL[m.config.weight_dtype] if a.tol is None else a.tol
            rows = verify_cell(m, a.steps)
        else:
            tol = 0.0 if a.tol is None else a.tol
            rows = verify_plain(m, a.steps)
        for label, dev in rows:
            worst = max(worst, dev)
            bad = dev > tol
            failed |= bad
            if bad or not a.random_grid:
                print(f"{name}: {label}: {dev:.3e}{'  FAIL' if bad else ''}")
    print(f"{len(models)} model(s), max deviation {worst:.3e}: {'FAIL' if failed else 'ok'}")
    return 1 if failed else 0


# ---- bench -----------------------------------------------------------------------------------
def cmd_bench(a) -> int:
    from .benchmark import default_grid, emit_records, run_benchmark

    grid = default_grid(a.layers_from, a.layers_to, a.blocks, a.width, a.base, a.channels)
    emit_records(run_benchmark(grid, a.steps, a.repeats, a.warmup, time_budget_s=a.budget_s),
                 a.out)
    return 0


def build_parser() -> argparse.ArgumentParser:
    p0 = argparse.ArgumentParser(prog="paper_1611_09482_b200",
                                 description="B200 queue-cached generation for stacks of "
                                             "dilated causal convolutions (Fast WaveNet).")
    sub = p0.add_subparsers(dest="command", required=True)

    p = sub.add_parser("init-model", help="build a seeded plain model and save it")
    p.add_argument("--layers", type=int, required=True, help="layers per block")
    p.add_argument("--blocks", type=int, default=1)
    p.add_argument("--width", type=int, default=2, help="filter taps per layer")
    p.add_argument("--base", type=int, default=2, help="dilation growth base")
    p.add_argument("--channels", type=int, default=1, help="hidden channels")
    p.add_argument("--activation", choices=ACTIVATIONS, default="tanh")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out", required=True)
    p.set_defaults(func=cmd_init_model)

    p = sub.add_parser("init-cell", help="build a seeded gated-cell model and save it")
    p.add_argument("--layers", type=int, required=True, help="layers per block")
    p.add_argument("--blocks", type=int, default=1)
    p.add_argument("--residual", type=int, default=32)
    p.add_argument("--dilation", type=int, default=None, help="default: --residual")
    p.add_argument("--skip", type=int, default=128)
    p.add_argument("--head", type=int, default=None, help="default: --skip")
    p.add_argument("--classes", type=int, default=256)
    p.add_argument("--base", type=int, default=2)
    p.add_argument("--dtype", choices=("f32", "bf16"), default="f32")
    p.add_argument("--init", default="fan_in")
    p.add_argument("--bias", choices=("zero", "fan_in"), default="zero")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out", required=True)
    p.set_defaults(func=cmd_init_cell)

    p = sub.add_parser("generate", help="free-run a generator, one sample per line")
    p.add_argument("--model", required=True)
    p.add_argument("--steps", type=int, required=True)
    p.add_argument("--mode", choices=("fast", "naive"), required=True)
    p.add_argument("--primer", help="optional primer file (samples, or classes for a cell)")
    p.add_argument("--sampler", type=int, default=0,
                   help="cell models: 0 argmax, 1 inverse CDF, 2 Gumbel-max")
    p.add_argument("--seed", type=int, default=0, help="cell models: noise seed")
    p.add_argument("--out", required=True)
    p.set_defaults(func=cmd_generate)

    p = sub.add_parser("verify", help="cross-check the generators against each other")
    g = p.add_mutually_exclusive_group(required=True)
    g.add_argument("--model", help="verify one saved model")
    g.add_argument("--random-grid", action="store_true",
                   help="verify the seeded grid of plain architectures")
    p.add_argument("--steps", type=int, default=64)
    p.add_argument("--tol", type=float, default=None,
                   help="max tolerated deviation (default: exact for plain models, the "
                        "weight dtype's tolerance for cell models)")
    p.set_defaults(func=cmd_verify)

    p = sub.add_parser("bench", help="layer-sweep timing experiment (plain models), CSV output")
    p.add_argument("--layers-from", type=int, default=1)
    p.add_argument("--layers-to", type=int, default=10)
    p.add_argument("--blocks", type=int, default=2)
    p.add_argument("--width", type=int, default=2)
    p.add_argument("--base", type=int, default=2)
    p.add_argument("--channels", type=int, default=16)
    p.add_argument("--steps", type=int, default=64)
    p.add_argument("--repeats", type=int, default=100)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--budget-s", type=float, default=None,
                   help="per config x mode wall-clock budget in seconds")
    p.add_argument("--out", required=True)
    p.set_defaults(func=cmd_bench)
    return p0


def main(argv: list[str] | None = None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
