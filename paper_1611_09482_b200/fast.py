"""GPU drop-in for the reference's queue-cached generator (plain mode).

Same names, argument meaning and error behaviour as
``streamconv.fast`` (reference ``pkg/src/streamconv/fast.py:98-252``); the
state lives in HBM behind a libfastwavenet handle and every step runs in the
fp64 plain-mode kernel (csrc/plain_f64.cu) in the reference's pinned
accumulation order.

* ``init_state(model)``            -> fast.py:122-128 (zero-filled queues)
* ``fast_step(state, x, model)``   -> fast.py:216-224
* ``fast_generate(model, primer, steps)`` -> fast.py:227-252 (one launch)
* ``pop_phase`` / ``compute_step`` / ``push_phase`` -> fast.py:131-213, with
  the same phase-misuse ``QueueStateError``s (raised by the C ABI).

Extension over the reference: ``init_state(model, batch=B)`` steps B
independent streams in lockstep (``fast_step`` then takes and returns arrays).
"""

from __future__ import annotations

import weakref

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import QueueStateError
from .model import MacCount, Model, activation_code, count_macs


@dataclass(frozen=True, eq=False)
class SampleSequence:
    """A stretch of channel-vector samples (reference oracle.py:20-62)."""

    values: np.ndarray
    start_index: int = 0

    def __post_init__(self) -> None:
        arr = np.array(self.values, dtype=np.float64, copy=True)
        if arr.ndim != 2:
            raise ValueError("values must have shape (timesteps, channels)")
        if not np.isfinite(arr).all():
            raise ValueError("sample values must be finite")
        arr.setflags(write=False)
        object.__setattr__(self, "values", arr)

    @classmethod
    def from_scalars(cls, samples, start_index: int = 0) -> "SampleSequence":
        arr = np.asarray(list(samples) if not isinstance(samples, np.ndarray) else samples,
                         dtype=np.float64)
        if arr.ndim != 1:
            raise ValueError("scalar samples must be 1-D")
        return cls(values=arr.reshape(-1, 1), start_index=start_index)

    def scalars(self) -> np.ndarray:
        if self.channels != 1:
            raise ValueError("sequence is not scalar-channel")
        return self.values[:, 0]

    @property
    def channels(self) -> int:
        return self.values.shape[1]

    def __len__(self) -> int:
        return self.values.shape[0]


def scalar_primer(primer) -> np.ndarray:
    """Empty primer -> [0.0] (reference oracle.py:65-81)."""
    if isinstance(primer, SampleSequence):
        seed = primer.scalars()
    else:
        seed = np.asarray(primer, dtype=np.float64)
        if seed.ndim != 1:
            raise ValueError("primer must be a 1-D scalar sequence")
        if not np.isfinite(seed).all():
            raise ValueError("primer samples must be finite")
    return np.zeros(1) if seed.shape[0] == 0 else seed


@dataclass(frozen=True)
class RecurrentInputs:
    """Per layer, the w-1 cached values its taps k = 1..w-1 read (fast.py:91-95)."""

    per_layer: tuple[tuple[np.ndarray, ...], ...]


class QueueView:
    """Capacity/length view of one HBM ring queue (ConvQueue's observable shape)."""

    def __init__(self, state: "GenerationState", layer: int, capacity: int, channels: int):
        self._state, self._layer = state, layer
        self.capacity, self.channels = capacity, channels

    def __len__(self) -> int:
        return self.capacity - 1 if self._state._popped else self.capacity


class GenerationState:
    """One GPU session: a handle owning HBM queues plus the step counter."""

    def __init__(self, model: Model, batch: int = 1, device: int | None = None):
        import torch

        cfg = model.config
        self.config = cfg
        self.batch = int(batch)
        self.device = torch.cuda.current_device() if device is None else int(device)
        lib = _lib.load()
        taps = np.ascontiguousarray(np.concatenate([lw.taps.ravel() for lw in model.layers]))
        bias = np.ascontiguousarray(np.concatenate([lw.bias.ravel() for lw in model.layers]))
        desc = _lib.FwPlainDesc(cfg.blocks, cfg.layers_per_block, cfg.filter_width,
                                cfg.dilation_base, cfg.hidden_channels,
                                activation_code(cfg.activation),
                                taps.ctypes.data, bias.ctypes.data)
        h = C.c_void_p()
        _lib.check(lib.fw_plain_create(C.byref(desc), self.batch, self.device, C.byref(h)))
        self._h = h
        self._lib = lib
        self._popped = False
        w = cfg.filter_width
        self.queues = tuple(QueueView(self, l, (w - 1) * d, ci) for l, (d, (ci, _)) in
                            enumerate(zip(cfg.dilations(), cfg.channel_dims())))
        self.macs_last_step: MacCount | None = None
        self._dev = torch.device("cuda", self.device)

    @property
    def step_index(self) -> int:
        v = C.c_int64()
        _lib.check(self._lib.fw_step_index(self._h, C.byref(v)))
        return v.value

    def cached_scalar_count(self) -> int:
        """Scalars held across all queues, per stream (fast.py:117-119)."""
        return sum(q.capacity * q.channels for q in self.queues)

    def reset(self) -> None:
        _lib.check(self._lib.fw_reset(self._h, _lib.stream_ptr()))
        self._popped = False

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.fw_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def init_state(model: Model, batch: int = 1, device: int | None = None) -> GenerationState:
    """Fresh session: every queue zero-filled to capacity (fast.py:122-128)."""
    return GenerationState(model, batch, device)


def _check_model(state: GenerationState, model: Model) -> None:
    if state.config is not model.config and state.config != model.config:
        raise ValueError("state was initialized for a different architecture")


def fast_step(state: GenerationState, input, model: Model):
    """Pop, compute, push on the GPU; returns the output sample(s)."""
    import torch

    _check_model(state, model)
    scalar = np.ndim(input) == 0
    x = torch.as_tensor(np.asarray(input, dtype=np.float64).reshape(state.batch),
                        device=state._dev)
    y = torch.empty(state.batch, dtype=torch.float64, device=state._dev)
    _lib.check(state._lib.fw_plain_step(state._h, C.c_void_p(x.data_ptr()),
                                        C.c_void_p(y.data_ptr()), _lib.stream_ptr()))
    state.macs_last_step = count_macs(state.config)
    out = y.cpu().numpy()
    return float(out[0]) if scalar else out


def fast_generate(model: Model, primer: SampleSequence | Sequence[float], steps: int,
                  device: int | None = None) -> SampleSequence:
    """Free-run with queue caching, all steps in one launch (fast.py:227-252)."""
    import torch

    if steps < 0:
        raise ValueError("steps must be non-negative")
    seed = scalar_primer(primer)
    start = seed.shape[0]
    if steps == 0:
        return SampleSequence.from_scalars([], start_index=start)
    state = init_state(model, 1, device)
    n = start - 1 + steps
    xin = torch.as_tensor(seed.reshape(-1, 1), device=state._dev)
    out = torch.empty((n, 1), dtype=torch.float64, device=state._dev)
    _lib.check(state._lib.fw_plain_generate(state._h, C.c_void_p(xin.data_ptr()), start, n,
                                            C.c_void_p(out.data_ptr()), _lib.stream_ptr()))
    res = out[start - 1:, 0].cpu().numpy()
    state.close()
    return SampleSequence.from_scalars(res, start_index=start)


def pop_phase(state: GenerationState) -> RecurrentInputs:
    """Read each layer's w-1 tap values and discard the oldest (fast.py:131-147)."""
    import torch

    cfg = state.config
    w = cfg.filter_width
    rows = sum((w - 1) * ci for ci, _ in cfg.channel_dims())
    rec = torch.empty((rows, state.batch), dtype=torch.float64, device=state._dev)
    _lib.check(state._lib.fw_plain_pop(state._h, C.c_void_p(rec.data_ptr()), _lib.stream_ptr()))
    state._popped = True
    host = rec.cpu().numpy()
    per_layer, r = [], 0
    for ci, _ in cfg.channel_dims():
        taps = []
        for _k in range(1, w):
            v = host[r:r + ci]
            taps.append(v[:, 0].copy() if state.batch == 1 else v.T.copy())
            r += ci
        per_layer.append(tuple(taps))
    return RecurrentInputs(per_layer=tuple(per_layer))


def compute_step(model: Model, input, rec: RecurrentInputs, device: int | None = None):
    """One bottom-to-top evaluation from explicit tap values (fast.py:157-197).

    Returns (output sample, per-layer fresh inputs to cache, MacCount); the
    queues are not touched.
    """
    import torch

    cfg = model.config
    w = cfg.filter_width
    if len(rec.per_layer) != cfg.total_layers:
        raise ValueError(f"recurrent inputs cover {len(rec.per_layer)} layers, "
                         f"model has {cfg.total_layers}")
    dims = cfg.channel_dims()
    cols = []
    batch = None
    for layer_rec, (ci, _) in zip(rec.per_layer, dims):
        if len(layer_rec) != w - 1:
            raise ValueError("recurrent inputs must hold w-1 values per layer")
        for v in layer_rec:
            v = np.asarray(v, dtype=np.float64)
            if v.shape[-1] != ci:
                raise ValueError("recurrent input channel mismatch")
            v2 = v.reshape(-1, ci)
            batch = v2.shape[0] if batch is None else batch
            cols.append(v2.T)
    host_rec = np.ascontiguousarray(np.concatenate(cols, axis=0))
    scalar = np.ndim(input) == 0
    state = _scratch_state(model, batch, device)
    dev = state._dev
    x = torch.as_tensor(np.asarray(input, dtype=np.float64).reshape(batch), device=dev)
    r = torch.as_tensor(host_rec, device=dev)
    y = torch.empty(batch, dtype=torch.float64, device=dev)
    srows = sum(ci for ci, _ in dims)
    states = torch.empty((srows, batch), dtype=torch.float64, device=dev)
    _lib.check(state._lib.fw_plain_compute(state._h, C.c_void_p(x.data_ptr()),
                                           C.c_void_p(r.data_ptr()), C.c_void_p(y.data_ptr()),
                                           C.c_void_p(states.data_ptr()), _lib.stream_ptr()))
    sh = states.cpu().numpy()
    new_states, r0 = [], 0
    for ci, _ in dims:
        v = sh[r0:r0 + ci]
        new_states.append(v[:, 0].copy() if scalar else v.T.copy())
        r0 += ci
    out = y.cpu().numpy()
    return (float(out[0]) if scalar else out), new_states, count_macs(cfg)


_SCRATCH: dict = {}


def _scratch_state(model: Model, batch: int, device) -> GenerationState:
    """A device handle for compute_step's stateless evaluation, cached for the last model.
    The cache holds a weak reference to the model and only hits for that very object: an
    id() alone can be reused by a new model after the old one is collected."""
    key = (id(model), batch, device)
    hit = _SCRATCH.get(key)
    if hit is not None and hit[0]() is model:
        return hit[1]
    st = GenerationState(model, batch, device)
    _SCRATCH.clear()
    _SCRATCH[key] = (weakref.ref(model), st)
    return st


def push_phase(state: GenerationState, new_states: Sequence[np.ndarray]) -> None:
    """Cache each layer's fresh input and advance the step (fast.py:200-213)."""
    import torch

    cfg = state.config
    if len(new_states) != len(state.queues):
        raise ValueError("one new state per layer required")
    cols = []
    for v, (ci, _) in zip(new_states, cfg.channel_dims()):
        v = np.asarray(v, dtype=np.float64).reshape(-1, ci)
        if v.shape[0] != state.batch:
            raise ValueError("new state batch mismatch")
        cols.append(v.T)
    host = torch.as_tensor(np.ascontiguousarray(np.concatenate(cols, axis=0)), device=state._dev)
    _lib.check(state._lib.fw_plain_push(state._h, C.c_void_p(host.data_ptr()), _lib.stream_ptr()))
    state._popped = False


__all__ = [
    "GenerationState", "QueueStateError", "RecurrentInputs", "SampleSequence", "compute_step",
    "fast_generate", "fast_step", "init_state", "pop_phase", "push_phase", "scalar_primer",
]
