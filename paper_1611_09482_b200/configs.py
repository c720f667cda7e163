"""The five BASELINE.json configurations as cell configs plus run parameters.

Choices BASELINE leaves open are fixed here and recorded in
DESIGN.md: head hidden H = S; tanh on the first gate half; zero biases for
every config (cfg1 says so explicitly); embedding fan-in = A; the top layer's
residual projection is skipped (it has no consumer); sampling noise is the
counter hash of ``paper_1611_09482_b200.noise`` keyed by
(seed, global stream, step, class) with the seeds below.
"""

from __future__ import annotations

from dataclasses import dataclass

from .cell import CellConfig

SAMPLE_ARGMAX = 0
SAMPLE_INVCDF = 1
SAMPLE_GUMBEL = 2

NOISE_SEED = 2016  # shared seed of the uniform / Gumbel noise hash (cfg2-cfg4)
TEACHER_SEED = 1  # cfg1 teacher-forced class sequence: default_rng(1).integers(0, 256, 2000)
WALK_SEED = 5  # cfg5 random walk: default_rng(5), +-1 steps from 128, clipped to [0, 255]


@dataclass(frozen=True)
class RunSpec:
    name: str
    cell: CellConfig
    batch: int
    steps: int
    sampler: int
    primer_class: int = 128
    teacher: str | None = None  # None | "uniform" | "walk"
    compare_steps: int = 0  # teacher-forced logits compared on this many steps


def cfg1() -> RunSpec:
    return RunSpec("cfg1_toy", CellConfig(1, 10, 32, 32, 128, init="normal:0.1"),
                   batch=1, steps=2000, sampler=SAMPLE_ARGMAX, teacher="uniform",
                   compare_steps=2000)


def cfg2(layers: int) -> RunSpec:
    return RunSpec(f"cfg2_L{layers}", CellConfig(1, layers, 128, 128, 256),
                   batch=1, steps=1000, sampler=SAMPLE_INVCDF)


def cfg3() -> RunSpec:
    return RunSpec("cfg3_wavenet", CellConfig(5, 10, 64, 64, 256),
                   batch=64, steps=16000, sampler=SAMPLE_GUMBEL)


def cfg4() -> RunSpec:
    return RunSpec("cfg4_large_batch", CellConfig(4, 10, 128, 128, 512, weight_dtype="bf16"),
                   batch=4096, steps=24000, sampler=SAMPLE_GUMBEL)


def cfg5() -> RunSpec:
    return RunSpec("cfg5_deep", CellConfig(8, 12, 64, 64, 256),
                   batch=1024, steps=48000, sampler=SAMPLE_ARGMAX, teacher="walk",
                   compare_steps=2000)


CFG2_LAYERS = (2, 4, 6, 8, 10, 12, 14)


def all_specs() -> list[RunSpec]:
    return [cfg1(), *[cfg2(L) for L in CFG2_LAYERS], cfg3(), cfg4(), cfg5()]


def by_name(name: str) -> RunSpec:
    for s in all_specs():
        if s.name == name or s.name.split("_")[0] == name:
            return s
    raise ValueError(f"unknown config {name!r}")
