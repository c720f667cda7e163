"""Gated WaveNet cell model: the north-star generation cell.

The reference stops at a plain conv stack; the cell below keeps its
conventions and adds the gate, residual/skip projections, output head, and
class embedding that ``BASELINE.json`` names:

* every dilated layer is a reference ``LayerWeights``-style tap tensor
  ``(2, 2D, R)``, tap 0 = current step, tap 1 = ``dilation`` steps back
  (reference ``model.py:98-129``); dilation ``2**i`` restarting per block
  (``model.py:70-76``);
* ``a = W0 x_l[t] + W1 x_l[t-d] + b``; ``z = tanh(a[:D]) * sigmoid(a[D:])``
  (tanh on the first half -- a builder choice);
* ``x_{l+1} = x_l + W_res z + b_res`` (skipped for the top layer: it has no
  consumer), ``s += W_skip z + b_skip``;
* ``logits = W_h2 relu(W_h1 relu(s) + b_h1) + b_h2``; head hidden ``H = S``;
* ``x_0[t] = E[c_t]`` with ``E`` of shape ``(A, R)``.

Queue ``l`` caches the layer input ``x_l[t]`` exactly as the reference caches
each layer's fresh input (``fast.py:192``).

Weights are drawn from ``np.random.default_rng(seed)`` in a fixed order
(embedding, then per layer dil taps, dil bias, res W, res b, skip W, skip b,
then head1 W, b, head2 W, b), following the reference's fixed-draw-order
idiom (``model.py:177-192``). They are stored as float32 values (already
rounded to bf16 when ``weight_dtype == "bf16"``) and upcast to float64 by the
oracle, so weight quantisation is never charged as kernel error
(SURVEY App. A.5).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def round_to_bf16(x: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16 (ties to even), returned as float32."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    rounded = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    out = rounded.astype(np.uint32).view(np.float32).reshape(a.shape)
    return np.where(np.isfinite(a), out, a)


@dataclass(frozen=True)
class CellConfig:
    """Architecture + initialisation of a gated cell stack."""

    blocks: int
    layers_per_block: int
    residual_channels: int
    dilation_channels: int
    skip_channels: int
    classes: int = 256
    head_channels: int | None = None  # None -> skip_channels (H = S)
    dilation_base: int = 2
    weight_dtype: str = "f32"  # "f32" or "bf16"
    init: str = "fan_in"  # "fan_in": N(0, 1/fan_in); "normal:<std>": N(0, std^2)
    bias: str = "zero"  # "zero" or "fan_in" (tests exercise non-zero biases)
    init_seed: int = 0
    filter_width: int = field(default=2, init=False)

    def __post_init__(self) -> None:
        for name in ("blocks", "layers_per_block", "residual_channels",
                     "dilation_channels", "skip_channels", "classes"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be a positive integer")
        if self.head_channels is not None and self.head_channels < 1:
            raise ValueError("head_channels must be a positive integer")
        if self.dilation_base < 2:
            raise ValueError("dilation_base must be at least 2")
        if self.weight_dtype not in ("f32", "bf16"):
            raise ValueError("weight_dtype must be 'f32' or 'bf16'")
        if not (self.init == "fan_in" or self.init.startswith("normal:")):
            raise ValueError("init must be 'fan_in' or 'normal:<std>'")
        if self.bias not in ("zero", "fan_in"):
            raise ValueError("bias must be 'zero' or 'fan_in'")
        if not 0 <= self.init_seed < 2**64:
            raise ValueError("init_seed must fit in an unsigned 64-bit integer")
        if self.dilation_base ** (self.layers_per_block - 1) >= 2**30:
            raise ValueError("dilation_base**(layers_per_block-1) must be below 2**30")

    @property
    def total_layers(self) -> int:
        return self.blocks * self.layers_per_block

    @property
    def H(self) -> int:
        return self.skip_channels if self.head_channels is None else self.head_channels

    def dilations(self) -> tuple[int, ...]:
        return tuple([self.dilation_base**i for i in range(self.layers_per_block)] * self.blocks)

    def receptive_field(self) -> int:
        return 1 + sum(self.dilations())

    def queue_slots(self) -> int:
        """Ring slots per stream over all layers: sum of (w-1)*d_l (reference fast.py:39-44)."""
        return sum(self.dilations())

    def macs_per_sample(self) -> int:
        """MACs of one cached step for one stream (top residual skipped)."""
        n, R, D, S, H, A = (self.total_layers, self.residual_channels, self.dilation_channels,
                            self.skip_channels, self.H, self.classes)
        return n * (2 * 2 * D * R + S * D) + (n - 1) * R * D + S * H + H * A

    def weight_count(self) -> int:
        n, R, D, S, H, A = (self.total_layers, self.residual_channels, self.dilation_channels,
                            self.skip_channels, self.H, self.classes)
        per_layer = 2 * 2 * D * R + 2 * D + R * D + R + S * D + S
        return A * R + n * per_layer + H * S + H + A * H + A


@dataclass(frozen=True, eq=False)
class CellLayer:
    dil_taps: np.ndarray  # (2, 2D, R)
    dil_bias: np.ndarray  # (2D,)
    res_w: np.ndarray  # (R, D)
    res_b: np.ndarray  # (R,)
    skip_w: np.ndarray  # (S, D)
    skip_b: np.ndarray  # (S,)


@dataclass(frozen=True, eq=False)
class CellModel:
    """Immutable cell weights (float32 storage, bf16-representable for bf16 configs)."""

    config: CellConfig
    embed: np.ndarray  # (A, R)
    layers: tuple[CellLayer, ...]
    head1_w: np.ndarray  # (H, S)
    head1_b: np.ndarray  # (H,)
    head2_w: np.ndarray  # (A, H)
    head2_b: np.ndarray  # (A,)

    def __post_init__(self) -> None:
        c = self.config
        R, D, S, H, A = (c.residual_channels, c.dilation_channels, c.skip_channels, c.H, c.classes)
        expect = {"embed": (A, R), "head1_w": (H, S), "head1_b": (H,), "head2_w": (A, H),
                  "head2_b": (A,)}
        for name, shape in expect.items():
            if getattr(self, name).shape != shape:
                raise ValueError(f"{name} must have shape {shape}")
        if len(self.layers) != c.total_layers:
            raise ValueError(f"config declares {c.total_layers} layers, got {len(self.layers)}")
        lshape = {"dil_taps": (2, 2 * D, R), "dil_bias": (2 * D,), "res_w": (R, D),
                  "res_b": (R,), "skip_w": (S, D), "skip_b": (S,)}
        for l, lw in enumerate(self.layers):
            for name, shape in lshape.items():
                if getattr(lw, name).shape != shape:
                    raise ValueError(f"layer {l}: {name} must have shape {shape}")

    def packed(self) -> dict[str, np.ndarray]:
        """Contiguous float32 arrays in the C-ABI order of include/fastwavenet.h."""
        L = self.layers
        f = lambda xs: np.ascontiguousarray(np.stack(xs), dtype=np.float32)
        return {
            "embed": np.ascontiguousarray(self.embed, dtype=np.float32),
            "dil_w": f([lw.dil_taps for lw in L]),
            "dil_b": f([lw.dil_bias for lw in L]),
            "res_w": f([lw.res_w for lw in L]),
            "res_b": f([lw.res_b for lw in L]),
            "skip_w": f([lw.skip_w for lw in L]),
            "skip_b": f([lw.skip_b for lw in L]),
            "head1_w": np.ascontiguousarray(self.head1_w, dtype=np.float32),
            "head1_b": np.ascontiguousarray(self.head1_b, dtype=np.float32),
            "head2_w": np.ascontiguousarray(self.head2_w, dtype=np.float32),
            "head2_b": np.ascontiguousarray(self.head2_b, dtype=np.float32),
        }


def build_cell_model(config: CellConfig) -> CellModel:
    """Seeded weights in a fixed draw order; see module docstring."""
    rng = np.random.default_rng(config.init_seed)
    R, D, S, H, A = (config.residual_channels, config.dilation_channels, config.skip_channels,
                     config.H, config.classes)

    def std_for(fan_in: int) -> float:
        if config.init == "fan_in":
            return 1.0 / np.sqrt(fan_in)
        return float(config.init.split(":", 1)[1])

    def draw(shape, fan_in):
        w = (rng.standard_normal(size=shape) * std_for(fan_in)).astype(np.float32)
        if config.weight_dtype == "bf16":
            w = round_to_bf16(w)
        w.setflags(write=False)
        return w

    def bias(n, fan_in):
        if config.bias == "zero":
            b = np.zeros(n, dtype=np.float32)
        else:
            b = (rng.standard_normal(size=n) / np.sqrt(fan_in)).astype(np.float32)
            if config.weight_dtype == "bf16":
                b = round_to_bf16(b)
        b.setflags(write=False)
        return b

    embed = draw((A, R), A)  # a 1x1 conv over the one-hot input: fan_in = A
    layers = []
    for _ in range(config.total_layers):
        dil_taps = draw((2, 2 * D, R), 2 * R)
        dil_bias = bias(2 * D, 2 * R)
        res_w = draw((R, D), D)
        res_b = bias(R, D)
        skip_w = draw((S, D), D)
        skip_b = bias(S, D)
        layers.append(CellLayer(dil_taps, dil_bias, res_w, res_b, skip_w, skip_b))
    head1_w = draw((H, S), S)
    head1_b = bias(H, S)
    head2_w = draw((A, H), H)
    head2_b = bias(A, H)
    return CellModel(config, embed, tuple(layers), head1_w, head1_b, head2_w, head2_b)
