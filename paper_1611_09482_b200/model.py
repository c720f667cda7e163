"""Plain-mode model: the reference's own dilated causal conv stack.

This restates the data contract of ``streamconv.model`` (reference
``pkg/src/streamconv/model.py:36-192``) so a caller of the reference can hand
the same objects to the GPU path:

* ``ModelConfig`` -- validation rules of ``model.py:48-64``; dilation schedule
  ``r**i`` restarting per block (``model.py:70-76``); scalar ends
  (``model.py:78-84``); receptive field closed form (``model.py:87-95``).
* ``LayerWeights`` -- ``taps`` has shape ``(w, out, in)``, ``taps[0]`` reads the
  current step and ``taps[k]`` reads ``k * dilation`` steps back
  (``model.py:98-129``).
* ``build_model`` -- ``np.random.default_rng(init_seed)``, uniform [-0.5, 0.5],
  per layer the taps are drawn before the bias (``model.py:177-192``), so an
  identical config gives bit-identical float64 weights to the reference.
  ``tests/golden/plain_*.npz`` pins this against weights the reference built.

The model text format (``model.py:195-306``) is read and written byte-compatibly by
``model_io.py``.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np

ACTIVATIONS = ("linear", "tanh")
_ACT_CODE = {"linear": 0, "tanh": 1}


def activation_code(name: str) -> int:
    """Integer code of an activation, as the reference kernel uses it (kernel.py:18-27)."""
    try:
        return _ACT_CODE[name]
    except KeyError:
        raise ValueError(f"unknown activation {name!r}") from None


@dataclass(frozen=True)
class MacCount:
    """Exact per-sample cost (reference counters.py:8-30)."""

    multiply_accumulates: int
    node_evaluations: int

    def __post_init__(self) -> None:
        if self.multiply_accumulates < 0 or self.node_evaluations < 0:
            raise ValueError("counts must be non-negative")

    def __add__(self, other: "MacCount") -> "MacCount":
        return MacCount(self.multiply_accumulates + other.multiply_accumulates,
                        self.node_evaluations + other.node_evaluations)


@dataclass(frozen=True)
class ModelConfig:
    """Architecture hyperparameters of the plain stack (reference model.py:36-95)."""

    blocks: int
    layers_per_block: int
    filter_width: int = 2
    dilation_base: int = 2
    hidden_channels: int = 1
    activation: str = "tanh"
    init_seed: int = 0

    def __post_init__(self) -> None:
        checks = (
            (self.blocks >= 1, "blocks must be a positive integer"),
            (self.layers_per_block >= 1, "layers_per_block must be a positive integer"),
            (self.filter_width >= 2, "filter_width must be at least 2"),
            (self.dilation_base >= 2, "dilation_base must be at least 2"),
            (self.hidden_channels >= 1, "hidden_channels must be a positive integer"),
            (self.activation in ACTIVATIONS,
             f"activation must be one of {ACTIVATIONS}, got {self.activation!r}"),
            (0 <= self.init_seed < 2**64, "init_seed must fit in an unsigned 64-bit integer"),
        )
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)

    @property
    def total_layers(self) -> int:
        return self.blocks * self.layers_per_block

    def dilations(self) -> tuple[int, ...]:
        per_block = [self.dilation_base**i for i in range(self.layers_per_block)]
        return tuple(per_block * self.blocks)

    def channel_dims(self) -> tuple[tuple[int, int], ...]:
        n, c = self.total_layers, self.hidden_channels
        return tuple((1 if l == 0 else c, 1 if l == n - 1 else c) for l in range(n))


def receptive_field(config: ModelConfig) -> int:
    """1 + blocks * (w - 1) * (r**L - 1) / (r - 1)  (reference model.py:87-95)."""
    r, w = config.dilation_base, config.filter_width
    return 1 + config.blocks * ((w - 1) * (r**config.layers_per_block - 1) // (r - 1))


@dataclass(frozen=True, eq=False)
class LayerWeights:
    """One layer's taps ``(w, out, in)`` (tap 0 = current) and bias ``(out,)``."""

    taps: np.ndarray
    bias: np.ndarray

    def __post_init__(self) -> None:
        if self.taps.ndim != 3:
            raise ValueError("taps must have shape (filter_width, out, in)")
        if self.taps.shape[0] < 2:
            raise ValueError("a layer needs at least two taps")
        if self.bias.ndim != 1 or self.bias.shape[0] != self.taps.shape[1]:
            raise ValueError("bias length must match the tap out dimension")
        if not (np.isfinite(self.taps).all() and np.isfinite(self.bias).all()):
            raise ValueError("layer weights must be finite")

    @property
    def filter_width(self) -> int:
        return self.taps.shape[0]

    @property
    def out_channels(self) -> int:
        return self.taps.shape[1]

    @property
    def in_channels(self) -> int:
        return self.taps.shape[2]


@dataclass(frozen=True, eq=False)
class Model:
    """Immutable config + weights; shareable across sessions (reference model.py:132-161)."""

    config: ModelConfig
    layers: tuple[LayerWeights, ...]

    def __post_init__(self) -> None:
        dims = self.config.channel_dims()
        if len(self.layers) != len(dims):
            raise ValueError(f"config declares {len(dims)} layers, got {len(self.layers)}")
        for l, (lw, (c_in, c_out)) in enumerate(zip(self.layers, dims)):
            if lw.filter_width != self.config.filter_width:
                raise ValueError(f"layer {l}: tap count mismatch")
            if (lw.in_channels, lw.out_channels) != (c_in, c_out):
                raise ValueError(f"layer {l}: expected {c_in}x{c_out} channels, "
                                 f"got {lw.in_channels}x{lw.out_channels}")

    def equals(self, other: "Model") -> bool:
        if self.config != other.config:
            return False
        return all(np.array_equal(a.taps, b.taps) and np.array_equal(a.bias, b.bias)
                   for a, b in zip(self.layers, other.layers))


def build_model(config: ModelConfig) -> Model:
    """Seeded uniform[-0.5, 0.5] weights in the reference's draw order (model.py:177-192)."""
    if config.dilation_base < config.filter_width:
        warnings.warn(
            f"dilation_base {config.dilation_base} is smaller than filter_width "
            f"{config.filter_width}; space grows past the (w-1)*r**L bound",
            UserWarning, stacklevel=2)
    rng = np.random.default_rng(config.init_seed)
    layers = []
    for c_in, c_out in config.channel_dims():
        taps = rng.uniform(-0.5, 0.5, size=(config.filter_width, c_out, c_in))
        bias = rng.uniform(-0.5, 0.5, size=c_out)
        taps.setflags(write=False)
        bias.setflags(write=False)
        layers.append(LayerWeights(taps=taps, bias=bias))
    return Model(config=config, layers=tuple(layers))


def demand_offsets(config: ModelConfig) -> list[set[int]]:
    """Time offsets (steps back from the output) at which each layer is evaluated by the
    cache-free generator: the top layer at 0, and layer l-1 wherever layer l's taps read it,
    o + k * d_l for k < w (the reference's demand plan, naive.py:27-110)."""
    w, dil = config.filter_width, config.dilations()
    dem = [set() for _ in dil]
    dem[-1] = {0}
    for l in range(len(dil) - 1, 0, -1):
        dem[l - 1] = {o + k * dil[l] for o in dem[l] for k in range(w)}
    return dem


def count_macs(config: ModelConfig, mode: str = "fast") -> MacCount:
    """Per-sample cost: sum of w * in * out over the layer evaluations of one step --
    once per layer on the fast path, once per demanded offset on the naive path (reference
    bench.py:30-43)."""
    w = config.filter_width
    dims = config.channel_dims()
    if mode == "fast":
        return MacCount(sum(w * ci * co for ci, co in dims), config.total_layers)
    if mode == "naive":
        dem = demand_offsets(config)
        return MacCount(sum(len(o) * w * ci * co for o, (ci, co) in zip(dem, dims)),
                        sum(len(o) for o in dem))
    raise ValueError(f"unknown mode {mode!r}")
