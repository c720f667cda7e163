"""CPU restatement of the reference's plain-mode evaluation paths (float64).

TEST INFRASTRUCTURE ONLY: used by tests/ and bench.py's baseline legs as the
checker; the product path never imports it.

Restates, in pinned accumulation order:
* ``eval_nodes``   -- reference ``pkg/src/streamconv/kernel.py:30-56``: taps in
  ascending k, input channels ascending, separate multiply and add (no FMA),
  bias after the taps, activation last; gather index -1 is causal zero padding
  (the term is skipped, not added as zero).
* ``forward_full`` -- ``oracle.py:84-123``: time-parallel dilated causal conv.
* ``CachedStack``  -- ``fast.py:29-224``: per-layer ring queues of capacity
  (w-1)*d, zero-initialised; tap k reads the entry from t - k*d, the layer
  *input* is pushed (``fast.py:192``). Ring slots follow SURVEY App. A.2:
  tap k reads slot (t - k*d) mod cap and the push writes slot t mod cap,
  which is ``ConvQueue.peek((w-1-k)*d)`` followed by ``pop``/``push``.
* ``fast_generate`` -- ``fast.py:227-252`` with ``scalar_primer``
  (``oracle.py:65-81``): an empty primer is [0.0]; primer[:-1] is stepped
  with outputs discarded; feedback of the output sample.
* ``naive_step`` -- ``naive.py:27-110``: demand-driven recompute.

Vectorisation runs over nodes (rows) only, so every element sees exactly the
reference's operation sequence; tanh is libm's (``math.tanh``), as numba's is.
Pinned by tests/golden/plain_reference.npz, produced by the unmodified
reference (oracle/make_golden.py).
"""

from __future__ import annotations

import math
from functools import lru_cache

import numpy as np

_tanh = np.frompyfunc(math.tanh, 1, 1)


def libm_tanh(x: np.ndarray) -> np.ndarray:
    return _tanh(np.asarray(x, dtype=np.float64)).astype(np.float64)


def eval_nodes(taps: np.ndarray, bias: np.ndarray, act: int, prev: np.ndarray,
               gather: np.ndarray) -> np.ndarray:
    """out[i, o] = act(sum_k sum_c taps[k, o, c] * prev[gather[i, k], c] + bias[o])."""
    w, oc, ic = taps.shape
    n = gather.shape[0]
    acc = np.zeros((n, oc), dtype=np.float64)
    for k in range(w):
        g = gather[:, k]
        valid = (g >= 0)[:, None]
        src = prev[np.maximum(g, 0)]
        for c in range(ic):
            acc = np.where(valid, acc + taps[k, :, c][None, :] * src[:, c:c + 1], acc)
    acc = acc + bias[None, :]
    if act == 1:
        acc = libm_tanh(acc)
    return acc


def _act(model) -> int:
    return 1 if model.config.activation == "tanh" else 0


def forward_full(model, xs: np.ndarray) -> np.ndarray:
    """Whole stack over a whole scalar sequence (reference oracle.py:115-123)."""
    seq = np.asarray(xs, dtype=np.float64).reshape(-1, 1)
    n = seq.shape[0]
    for layer, d in zip(model.layers, model.config.dilations()):
        w = layer.taps.shape[0]
        gather = np.arange(n)[:, None] - d * np.arange(w)[None, :]
        gather[gather < 0] = -1
        seq = eval_nodes(layer.taps, layer.bias, _act(model), seq, gather)
    return seq[:, 0]


class CachedStack:
    """Queue-cached stepping of B independent scalar streams (reference fast.py)."""

    def __init__(self, model, batch: int = 1):
        cfg = model.config
        self.model = model
        self.batch = batch
        self.w = cfg.filter_width
        self.dil = cfg.dilations()
        self.queues = [np.zeros(((self.w - 1) * d, batch, ci), dtype=np.float64)
                       for d, (ci, _) in zip(self.dil, cfg.channel_dims())]
        self.t = 0

    def step(self, x: np.ndarray) -> np.ndarray:
        h = np.asarray(x, dtype=np.float64).reshape(self.batch, 1)
        gather = np.arange(self.w, dtype=np.int64)[None, :].repeat(self.batch, 0)
        gather = gather * self.batch + np.arange(self.batch)[:, None]
        act = _act(self.model)
        for q, d, layer in zip(self.queues, self.dil, self.model.layers):
            cap = q.shape[0]
            prev = np.empty((self.w, self.batch, q.shape[2]))
            prev[0] = h
            for k in range(1, self.w):
                prev[k] = q[(self.t - k * d) % cap]
            q[self.t % cap] = h  # cache the layer input (fast.py:192)
            h = eval_nodes(layer.taps, layer.bias, act, prev.reshape(-1, prev.shape[2]), gather)
        self.t += 1
        return h[:, 0]


def scalar_primer(primer) -> np.ndarray:
    seed = np.asarray(primer, dtype=np.float64)
    if seed.ndim != 1:
        raise ValueError("primer must be a 1-D scalar sequence")
    return np.zeros(1) if seed.shape[0] == 0 else seed


def fast_generate(model, primer, steps: int) -> np.ndarray:
    seed = scalar_primer(primer)
    if steps == 0:
        return np.zeros(0)
    st = CachedStack(model, 1)
    for x in seed[:-1]:
        st.step(np.array([x]))
    out = np.empty(steps)
    y = st.step(np.array([seed[-1]]))[0]
    out[0] = y
    for i in range(1, steps):
        y = st.step(np.array([y]))[0]
        out[i] = y
    return out


@lru_cache(maxsize=None)
def demand_plan(dilations: tuple[int, ...], w: int):
    """Per-layer demanded back-offsets and gathers (reference naive.py:27-61)."""
    n_layers = len(dilations)
    demanded = [None] * n_layers
    need = {0}
    for l in reversed(range(n_layers)):
        demanded[l] = np.array(sorted(need), dtype=np.int64)
        need = {o + k * dilations[l] for o in need for k in range(w)}
    inputs = np.array(sorted(need), dtype=np.int64)
    gathers = []
    for l in range(n_layers):
        below = inputs if l == 0 else demanded[l - 1]
        pos = {int(o): i for i, o in enumerate(below)}
        gathers.append(np.array([[pos[int(o) + k * dilations[l]] for k in range(w)]
                                 for o in demanded[l]], dtype=np.int64))
    return tuple(demanded), inputs, tuple(gathers)


def naive_step(model, history: np.ndarray) -> float:
    """Cache-free recompute of the sample aligned with history[-1] (naive.py:64-110)."""
    hist = np.asarray(history, dtype=np.float64)
    if hist.shape[0] == 0:
        hist = np.zeros(1)
    t = hist.shape[0] - 1
    cfg = model.config
    demanded, inputs, gathers = demand_plan(cfg.dilations(), cfg.filter_width)
    n_in = int(np.searchsorted(inputs, t, side="right"))
    prev = hist[t - inputs[:n_in]].reshape(-1, 1)
    n_below = n_in
    for l, layer in enumerate(model.layers):
        m = int(np.searchsorted(demanded[l], t, side="right"))
        g = gathers[l][:m]
        g = np.where(g < n_below, g, -1)
        prev = eval_nodes(layer.taps, layer.bias, _act(model), prev, g)
        n_below = m
    return float(prev[0, 0])


def naive_generate(model, primer, steps: int) -> np.ndarray:
    seed = scalar_primer(primer)
    buf = np.concatenate([seed, np.zeros(steps)])
    n0 = seed.shape[0]
    for i in range(steps):
        buf[n0 + i] = naive_step(model, buf[: n0 + i])
    return buf[n0:]
