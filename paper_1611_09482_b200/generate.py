"""GPU generation with the gated cell: the north-star hot path.

``CellGenerator`` owns one libfastwavenet handle (HBM ring queues for
``batch`` streams plus repacked weights) and exposes the reference's
generation contract for the cell:

* ``init_cell_state(model, batch)``  -- ``init_state`` (fast.py:122-128)
* ``CellGenerator.step``             -- ``fast_step`` over all streams (fast.py:216-224)
* ``CellGenerator.generate``         -- the device-side step loop of
  ``fast_generate`` (fast.py:227-252) with teacher/primer inputs
* ``cell_fast_generate(model, primer, steps, batch, sampler)`` -- the
  reference's ``fast_generate`` semantics for class streams: primer[:-1] is
  stepped with outputs discarded, out[0] = step(primer[-1]), then feedback.

All compute runs in the CUDA kernels behind the C ABI; there is no CPU path.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .cell import CellModel
from .configs import SAMPLE_ARGMAX

KERNELS = {"auto": _lib.FW_KERNEL_AUTO, "simt": _lib.FW_KERNEL_SIMT,
           "tcgen05": _lib.FW_KERNEL_TCGEN05}


@dataclass(frozen=True)
class Sampler:
    """Selection rule: mode FW_SAMPLE_* (0 argmax, 1 inverse CDF, 2 Gumbel-max)."""

    mode: int = SAMPLE_ARGMAX
    seed: int = 0
    stream_offset: int = 0

    def c(self) -> _lib.FwSampler:
        return _lib.FwSampler(int(self.mode), int(self.seed) & 0xFFFFFFFF, int(self.stream_offset))


class CellGenerator:
    def __init__(self, model: CellModel, batch: int, device: int | None = None,
                 kernel: str = "auto"):
        import torch

        if kernel not in KERNELS:
            raise ValueError(f"kernel must be one of {tuple(KERNELS)}")
        self.model = model
        cfg = model.config
        self.config = cfg
        self.batch = int(batch)
        self.device = torch.cuda.current_device() if device is None else int(device)
        self._dev = torch.device("cuda", self.device)
        self._lib = _lib.load()
        pk = model.packed()
        self._keep = pk  # host arrays must outlive the create call only; kept for clarity
        dil = np.ascontiguousarray(cfg.dilations(), dtype=np.int32)
        ptr = lambda a: a.ctypes.data
        desc = _lib.FwCellDesc(
            cfg.total_layers, dil.ctypes.data_as(C.POINTER(C.c_int32)), cfg.residual_channels,
            cfg.dilation_channels, cfg.skip_channels, cfg.H, cfg.classes,
            _lib.FW_DTYPE_BF16 if cfg.weight_dtype == "bf16" else _lib.FW_DTYPE_F32,
            ptr(pk["embed"]), ptr(pk["dil_w"]), ptr(pk["dil_b"]), ptr(pk["res_w"]),
            ptr(pk["res_b"]), ptr(pk["skip_w"]), ptr(pk["skip_b"]), ptr(pk["head1_w"]),
            ptr(pk["head1_b"]), ptr(pk["head2_w"]), ptr(pk["head2_b"]))
        h = C.c_void_p()
        _lib.check(self._lib.fw_cell_create(C.byref(desc), self.batch, self.device,
                                            KERNELS[kernel], C.byref(h)))
        self._h = h

    # ---- state --------------------------------------------------------------------
    @property
    def step_index(self) -> int:
        v = C.c_int64()
        _lib.check(self._lib.fw_step_index(self._h, C.byref(v)))
        return v.value

    @property
    def queue_bytes(self) -> int:
        v = C.c_int64()
        _lib.check(self._lib.fw_queue_bytes(self._h, C.byref(v)))
        return v.value

    @property
    def kernel(self) -> str:
        v = C.c_int32()
        _lib.check(self._lib.fw_kernel_kind(self._h, C.byref(v)))
        return {1: "simt", 2: "tcgen05"}[v.value]

    @property
    def last_launch_count(self) -> int:
        v = C.c_int64()
        _lib.check(self._lib.fw_last_launch_count(self._h, C.byref(v)))
        return v.value

    def set_kernel_timing(self, enable: bool) -> None:
        """Record CUDA events around each step's dominant kernel on later generate calls."""
        _lib.check(self._lib.fw_debug_timing(self._h, 1 if enable else 0))

    def kernel_times(self) -> tuple[float, float, int]:
        """(dominant-kernel ms, whole-step ms, steps) of the last timed generate call."""
        a, b, n = C.c_double(), C.c_double(), C.c_int64()
        _lib.check(self._lib.fw_debug_timing_read(self._h, C.byref(a), C.byref(b), C.byref(n)))
        return a.value, b.value, n.value

    def reset(self, stream=None) -> None:
        _lib.check(self._lib.fw_reset(self._h, _lib.stream_ptr(stream)))

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.fw_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- compute ------------------------------------------------------------------
    def _i32(self, x):
        import torch

        t = torch.as_tensor(x, device=self._dev)
        if t.dtype != torch.int32:
            t = t.to(torch.int32)
        return t.contiguous()

    def _check_classes(self, t) -> None:
        """Input class ids must lie in [0, classes): the kernels index the embedding table
        with them (out-of-range ids are clamped on the device, never read out of bounds, but
        they are a caller error -- ValueError, as the reference's shape/arity checks)."""
        if t.numel() == 0:
            return
        lo, hi = (int(v) for v in t.aminmax())
        if lo < 0 or hi >= self.config.classes:
            raise ValueError(f"input class ids must lie in [0, {self.config.classes}), "
                             f"got [{lo}, {hi}]")

    def step(self, classes, sampler: Sampler = Sampler(), want_logits: bool = False,
             stream=None):
        """One cached step of every stream: returns (classes_out [B], logits [B, A] | None)."""
        import torch

        x = self._i32(classes).reshape(self.batch)
        self._check_classes(x)
        out = torch.empty(self.batch, dtype=torch.int32, device=self._dev)
        lg = (torch.empty((self.batch, self.config.classes), dtype=torch.float32, device=self._dev)
              if want_logits else None)
        s = sampler.c()
        _lib.check(self._lib.fw_cell_step(self._h, C.c_void_p(x.data_ptr()),
                                          C.c_void_p(out.data_ptr()),
                                          C.c_void_p(lg.data_ptr() if lg is not None else 0),
                                          C.byref(s), _lib.stream_ptr(stream)))
        return out, lg

    def generate(self, inputs, n_steps: int, sampler: Sampler = Sampler(),
                 n_logit_steps: int = 0, out=None, logits=None, stream=None,
                 check_inputs: bool = True):
        """Device-side step loop; inputs (n_inputs, B) int32 on the GPU.

        Returns (classes (n_steps, B) int32, logits (n_logit_steps, B, A) | None).
        ``check_inputs=False`` skips the class-range check (a device reduction and a host
        sync) for inputs the caller has already validated.
        """
        import torch

        x = self._i32(inputs)
        if x.dim() != 2 or x.shape[1] != self.batch:
            raise ValueError("inputs must have shape (n_inputs, batch)")
        if check_inputs:
            self._check_classes(x)
        if out is None:
            out = torch.empty((n_steps, self.batch), dtype=torch.int32, device=self._dev)
        if n_logit_steps and logits is None:
            logits = torch.empty((n_logit_steps, self.batch, self.config.classes),
                                 dtype=torch.float32, device=self._dev)
        s = sampler.c()
        _lib.check(self._lib.fw_cell_generate(
            self._h, C.c_void_p(x.data_ptr()), int(x.shape[0]), int(n_steps),
            C.c_void_p(out.data_ptr()), C.c_void_p(logits.data_ptr() if n_logit_steps else 0),
            int(n_logit_steps), C.byref(s), _lib.stream_ptr(stream)))
        return out, (logits if n_logit_steps else None)

    def prefill(self, inputs, want_logits: bool = False, logits=None, stream=None):
        """Full-sequence forward over given inputs (T, B) int32 on the GPU
        (fw_cell_prefill): the queues and the step counter end where T teacher-forced
        steps would leave them, computed time-parallel. Returns the logits (T, B, A) of
        every step when asked for, else None."""
        import torch

        x = self._i32(inputs)
        if x.dim() != 2 or x.shape[1] != self.batch:
            raise ValueError("inputs must have shape (T, batch)")
        self._check_classes(x)
        T = int(x.shape[0])
        if want_logits and logits is None:
            logits = torch.empty((T, self.batch, self.config.classes), dtype=torch.float32,
                                 device=self._dev)
        _lib.check(self._lib.fw_cell_prefill(
            self._h, C.c_void_p(x.data_ptr()), T,
            C.c_void_p(logits.data_ptr() if want_logits else 0), _lib.stream_ptr(stream)))
        return logits if want_logits else None

    def select(self, logits, step: int, sampler: Sampler = Sampler(), out=None, stream=None):
        """The selection rule alone (fw_cell_select) over logits (n, B, A) or (B, A) fp32 on
        the GPU: row (i, b) is stream b at step ``step + i``. Returns int32 classes of the
        leading shape."""
        import torch

        lg = torch.as_tensor(logits, device=self._dev)
        if lg.dtype != torch.float32 or lg.shape[-1] != self.config.classes or \
                lg.shape[-2] != self.batch:
            raise ValueError("logits must be float32 of shape (..., batch, classes)")
        lg = lg.contiguous()
        lead = lg.shape[:-1]
        if out is None:
            out = torch.empty(lead, dtype=torch.int32, device=self._dev)
        s = sampler.c()
        _lib.check(self._lib.fw_cell_select(
            self._h, C.c_void_p(lg.data_ptr()), int(lg.numel() // self.config.classes),
            int(step), C.byref(s), C.c_void_p(out.data_ptr()), _lib.stream_ptr(stream)))
        return out

    def generate_host(self, inputs: np.ndarray, n_steps: int, sampler: Sampler = Sampler(),
                      out: np.ndarray | None = None, stream=None) -> np.ndarray:
        """Host in, host out: the end-to-end C-ABI entry (fw_cell_generate_host)."""
        x = np.ascontiguousarray(inputs, dtype=np.int32)
        if x.ndim != 2 or x.shape[1] != self.batch:
            raise ValueError("inputs must have shape (n_inputs, batch)")
        if x.size and (x.min() < 0 or x.max() >= self.config.classes):
            raise ValueError(f"input class ids must lie in [0, {self.config.classes})")
        if out is None:
            out = np.empty((n_steps, self.batch), dtype=np.int32)
        s = sampler.c()
        _lib.check(self._lib.fw_cell_generate_host(
            self._h, C.c_void_p(x.ctypes.data), int(x.shape[0]), int(n_steps),
            C.c_void_p(out.ctypes.data), C.byref(s), _lib.stream_ptr(stream)))
        return out


def init_cell_state(model: CellModel, batch: int = 1, device: int | None = None,
                    kernel: str = "auto") -> CellGenerator:
    return CellGenerator(model, batch, device, kernel)


PREFILL_MIN_PRIMER = 64  # primers at least this long run their phase time-parallel


def cell_fast_generate(model: CellModel, primer, steps: int, batch: int | None = None,
                       sampler: Sampler = Sampler(), device: int | None = None,
                       kernel: str = "auto", prefill_primer: bool = True) -> np.ndarray:
    """fast_generate for class streams; returns generated classes (B, steps).

    ``primer`` is (P,) shared by all streams or (B, P); an empty primer is the
    single class 0 (the reference's empty-primer rule, oracle.py:65-81, with the
    zero sample as class 0). The reference steps primer[:-1] with the outputs
    discarded (fast.py:244-245); from PREFILL_MIN_PRIMER samples on (and with
    ``prefill_primer``) that phase is the time-parallel full-sequence forward
    (fw_cell_prefill), which leaves the same state.
    """
    if steps < 0:
        raise ValueError("steps must be non-negative")
    p = np.asarray(primer, dtype=np.int64)
    if p.ndim == 1:
        B = 1 if batch is None else int(batch)
        p = np.broadcast_to(p, (B, p.shape[0]))
    B = p.shape[0]
    if p.shape[1] == 0:
        p = np.zeros((B, 1), dtype=np.int64)
    if ((p < 0) | (p >= model.config.classes)).any():
        raise ValueError("primer classes out of range")
    if steps == 0:
        return np.zeros((B, 0), dtype=np.int32)
    P = p.shape[1]
    gen = CellGenerator(model, B, device, kernel)
    if prefill_primer and P - 1 >= PREFILL_MIN_PRIMER:
        import torch

        gen.prefill(torch.as_tensor(np.array(p[:, :-1].T, dtype=np.int32), dtype=torch.int32,
                                    device=gen._dev))
        out = gen.generate_host(np.ascontiguousarray(p[:, -1:].T), steps, sampler)
        gen.close()
        return np.ascontiguousarray(out.T)
    out = gen.generate_host(np.ascontiguousarray(p.T), P - 1 + steps, sampler)
    gen.close()
    return np.ascontiguousarray(out[P - 1:].T)
