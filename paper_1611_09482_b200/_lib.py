"""ctypes binding of libfastwavenet.so (include/fastwavenet.h).

The product path has no CPU fallback: if the library is missing this module
raises on first use, and every compute call goes through the CUDA kernels.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libfastwavenet.so"

FW_OK, FW_ERR_INVALID, FW_ERR_STATE, FW_ERR_CUDA, FW_ERR_UNSUPPORTED = 0, 1, 2, 3, 4
FW_DTYPE_F32, FW_DTYPE_BF16 = 0, 1
FW_KERNEL_AUTO, FW_KERNEL_SIMT, FW_KERNEL_TCGEN05 = 0, 1, 2

# Every symbol include/fastwavenet.h declares (checked by tests/test_capi_symbols.py).
EXPORTS = (
    "fw_cell_create", "fw_cell_step", "fw_cell_generate", "fw_cell_generate_host",
    "fw_cell_prefill", "fw_cell_select", "fw_plain_create", "fw_plain_naive", "fw_plain_step", "fw_plain_generate", "fw_plain_pop",
    "fw_plain_compute", "fw_plain_push", "fw_reset", "fw_step_index", "fw_queue_bytes",
    "fw_kernel_kind", "fw_last_launch_count", "fw_destroy", "fw_last_error", "fw_version",
    "fw_debug_trace", "fw_debug_copy", "fw_debug_timing", "fw_debug_timing_read",
)


class QueueStateError(RuntimeError):
    """A convolution queue was popped or pushed out of turn (reference fast.py:25-26)."""


class FwCellDesc(C.Structure):
    _fields_ = [
        ("n_layers", C.c_int32), ("dilations", C.POINTER(C.c_int32)),
        ("residual_channels", C.c_int32), ("dilation_channels", C.c_int32),
        ("skip_channels", C.c_int32), ("head_channels", C.c_int32), ("classes", C.c_int32),
        ("weight_dtype", C.c_int32),
        ("embed", C.c_void_p), ("dil_w", C.c_void_p), ("dil_b", C.c_void_p),
        ("res_w", C.c_void_p), ("res_b", C.c_void_p), ("skip_w", C.c_void_p),
        ("skip_b", C.c_void_p), ("head1_w", C.c_void_p), ("head1_b", C.c_void_p),
        ("head2_w", C.c_void_p), ("head2_b", C.c_void_p),
    ]


class FwSampler(C.Structure):
    _fields_ = [("mode", C.c_int32), ("seed", C.c_uint32), ("stream_offset", C.c_int64)]


class FwPlainDesc(C.Structure):
    _fields_ = [
        ("blocks", C.c_int32), ("layers_per_block", C.c_int32), ("filter_width", C.c_int32),
        ("dilation_base", C.c_int32), ("hidden_channels", C.c_int32), ("activation", C.c_int32),
        ("taps", C.c_void_p), ("bias", C.c_void_p),
    ]


_lib = None


def load(path: Path | None = None) -> C.CDLL:
    """Load (once) and type the library; raises if it is absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"{p} is missing: the CUDA extension is not built "
            "(run `python -m paper_1611_09482_b200.build`). There is no CPU fallback.")
    lib = C.CDLL(str(p))
    H = C.c_void_p
    P = C.c_void_p
    sig = {
        "fw_cell_create": (C.c_int, [C.POINTER(FwCellDesc), C.c_int32, C.c_int32, C.c_int32,
                                     C.POINTER(H)]),
        "fw_cell_step": (C.c_int, [H, P, P, P, C.POINTER(FwSampler), P]),
        "fw_cell_generate": (C.c_int, [H, P, C.c_int32, C.c_int32, P, P, C.c_int32,
                                       C.POINTER(FwSampler), P]),
        "fw_cell_generate_host": (C.c_int, [H, P, C.c_int32, C.c_int32, P,
                                            C.POINTER(FwSampler), P]),
        "fw_cell_prefill": (C.c_int, [H, P, C.c_int32, P, P]),
        "fw_cell_select": (C.c_int, [H, P, C.c_int64, C.c_int64, C.POINTER(FwSampler), P, P]),
        "fw_plain_create": (C.c_int, [C.POINTER(FwPlainDesc), C.c_int32, C.c_int32, C.POINTER(H)]),
        "fw_plain_step": (C.c_int, [H, P, P, P]),
        "fw_plain_naive": (C.c_int, [H, P, C.c_int32, P, P]),
        "fw_plain_generate": (C.c_int, [H, P, C.c_int32, C.c_int32, P, P]),
        "fw_plain_pop": (C.c_int, [H, P, P]),
        "fw_plain_compute": (C.c_int, [H, P, P, P, P, P]),
        "fw_plain_push": (C.c_int, [H, P, P]),
        "fw_reset": (C.c_int, [H, P]),
        "fw_step_index": (C.c_int, [H, C.POINTER(C.c_int64)]),
        "fw_queue_bytes": (C.c_int, [H, C.POINTER(C.c_int64)]),
        "fw_kernel_kind": (C.c_int, [H, C.POINTER(C.c_int32)]),
        "fw_last_launch_count": (C.c_int, [H, C.POINTER(C.c_int64)]),
        "fw_destroy": (C.c_int, [H]),
        "fw_debug_trace": (C.c_int, [H, P]),
        "fw_debug_copy": (C.c_int, [H, C.c_int32, P, C.c_int64, P]),
        "fw_debug_timing": (C.c_int, [H, C.c_int32]),
        "fw_debug_timing_read": (C.c_int, [H, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                           C.POINTER(C.c_int64)]),
        "fw_last_error": (C.c_char_p, []),
        "fw_version": (C.c_int32, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def check(rc: int) -> None:
    """Map a C-ABI return code to the reference's exception types."""
    if rc == FW_OK:
        return
    msg = load().fw_last_error().decode(errors="replace")
    if rc == FW_ERR_INVALID:
        raise ValueError(msg)
    if rc == FW_ERR_STATE:
        raise QueueStateError(msg)
    raise RuntimeError(f"libfastwavenet error {rc}: {msg}")


def stream_ptr(stream=None) -> C.c_void_p:
    """cudaStream_t of a torch stream (default: torch's current stream)."""
    import torch

    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)
