"""Cache-free ("naive") generation of the cell on the GPU: SURVEY §8(f) rank 2.

The reference's naive path (``naive.py:27-110``) recomputes every step's output from the
raw input history through the demand plan of its receptive field, carrying no queues
between steps; the paper's Fig. 7 compares it with the queue-cached fast path. Here a
naive step is one time-parallel forward (``fw_cell_prefill``) over the step's window of
the history -- the last ``receptive_field`` inputs, or the whole history from a zeroed
state while it is shorter (the causal zero padding of ``oracle.py:84-123``). Only the last
row's logits are used: the cone of the output at t lies inside the window, so nothing
computed from before the window reaches it. The work per step therefore grows with the
receptive field (2^L for one block) instead of staying at L layers, which is the
comparison the paper draws.
"""

from __future__ import annotations

import numpy as np

from .cell import CellModel
from .generate import CellGenerator


class NaiveCellGenerator:
    """Per-step recomputation over the receptive field (greedy argmax feedback)."""

    def __init__(self, model: CellModel, batch: int, device: int | None = None,
                 kernel: str = "auto"):
        self.model = model
        self.batch = batch
        self.rf = model.config.receptive_field()
        self._gen = CellGenerator(model, batch, device, kernel)

    @property
    def kernel(self) -> str:
        return self._gen.kernel

    def close(self) -> None:
        self._gen.close()

    def logits(self, history):
        """Logits (B, A) of the step aligned with history[-1]; history (n, B) int32 on the GPU,
        n >= 1."""
        n = int(history.shape[0])
        if n < 1:
            raise ValueError("the history must hold at least one input")
        if n < self.rf:
            self._gen.reset()  # the window starts at t = 0: zero state before it
            window = history
        else:
            window = history[n - self.rf:]
        return self._gen.prefill(window, want_logits=True)[-1]

    def generate(self, primer, steps: int):
        """fast_generate's feedback rule (primer[:-1] conditions, then argmax feedback),
        every step recomputed from the history. primer (P, B) or (P,); returns (steps, B)."""
        import torch

        p = torch.as_tensor(np.array(primer, dtype=np.int32), device=self._gen._dev)
        if p.dim() == 1:
            p = p[:, None].expand(-1, self.batch)
        if p.shape[0] == 0:
            p = torch.zeros((1, self.batch), dtype=torch.int32, device=self._gen._dev)
        hist = torch.empty((p.shape[0] + steps, self.batch), dtype=torch.int32,
                           device=self._gen._dev)
        hist[:p.shape[0]] = p
        n = p.shape[0]
        for _ in range(steps):
            lg = self.logits(hist[:n])
            self._gen.select(lg, n - 1, out=hist[n])  # argmax, on the device (fw_cell_select)
            n += 1
        return hist[p.shape[0]:]


def cell_naive_generate(model: CellModel, primer, steps: int, batch: int | None = None,
                        device: int | None = None, kernel: str = "auto") -> np.ndarray:
    """The naive counterpart of ``cell_fast_generate`` (greedy): returns (B, steps)."""
    if steps < 0:
        raise ValueError("steps must be non-negative")
    p = np.asarray(primer, dtype=np.int64)
    if p.ndim == 1:
        B = 1 if batch is None else int(batch)
        p = np.broadcast_to(p, (B, p.shape[0]))
    B = p.shape[0]
    if ((p < 0) | (p >= model.config.classes)).any():
        raise ValueError("primer classes out of range")
    if steps == 0:
        return np.zeros((B, 0), dtype=np.int32)
    g = NaiveCellGenerator(model, B, device, kernel)
    out = g.generate(np.ascontiguousarray(p.T), steps).cpu().numpy()
    g.close()
    return np.ascontiguousarray(out.T)


# ---- plain mode (the reference's own stack) --------------------------------------------------
def plain_naive_step(model, history, state=None) -> float:
    """The reference's naive_step output (naive.py:27-110) for history[-1], recomputed
    cache-free on the GPU (fw_plain_naive): every node of the demand plan of its receptive
    field, layer by layer, each in the pinned order of the cached path -- so the result
    equals the queue-cached output bit for bit. `state` (a GenerationState of this model)
    lends its handle; its queues are not touched."""
    import ctypes as C

    import torch

    from . import _lib
    from .fast import init_state

    h = np.asarray(history, dtype=np.float64).ravel()
    if h.size == 0:
        raise ValueError("the history must hold at least one sample")
    own = state is None
    st = init_state(model, 1) if own else state
    x = torch.as_tensor(h.reshape(-1, 1), device=st._dev)
    y = torch.empty(1, dtype=torch.float64, device=st._dev)
    _lib.check(st._lib.fw_plain_naive(st._h, C.c_void_p(x.data_ptr()), int(h.size),
                                      C.c_void_p(y.data_ptr()), _lib.stream_ptr()))
    out = float(y.item())
    if own:
        st.close()
    return out


def plain_naive_generate(model, primer, steps: int):
    """The reference's naive_generate: fast_generate's feedback rule with every output
    recomputed from the history (cache-free, the demand plan on the GPU)."""
    from .fast import SampleSequence, init_state, scalar_primer

    if steps < 0:
        raise ValueError("steps must be non-negative")
    seed = scalar_primer(primer)
    hist = list(seed)
    st = init_state(model, 1)
    out = []
    for _ in range(steps):
        y = plain_naive_step(model, hist, st)
        out.append(y)
        hist.append(y)
    st.close()
    return SampleSequence.from_scalars(out, start_index=len(seed))


def naive_step(model, history):
    """The reference's ``naive_step(model, history) -> (sample, MacCount)``: the sample that
    extends the history by one, computed cache-free on the GPU, and its exact cost."""
    from .model import count_macs

    return plain_naive_step(model, history), count_macs(model.config, "naive")


naive_generate = plain_naive_generate  # the reference's name (naive.py:113)
