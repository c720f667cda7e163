"""CPU oracle of the gated cell, float64.

TEST INFRASTRUCTURE ONLY: the checker for tests/, __graft_entry__.smoke()
and bench.py's baseline legs. The product path never imports it.

The reference has no gated cell (its SPEC.md:11,314 put gate/skip/head out of
scope), so this is new code that follows the reference's conventions:

* one pinned-order node kernel shared by every evaluation path, as the
  reference's ``eval_nodes`` (kernel.py:30-56): per output, tap 0 (current)
  over input channels ascending, then tap 1 (d back) the same way, separate
  multiply/add, bias after the taps, nonlinearity last; a tap landing before
  time zero is skipped (causal zero padding, oracle.py:105-109);
* three paths, as the reference has (cli.py:102-135): time-parallel
  ``forward_full`` (oracle.py:84-123), queue-cached ``CachedCell``
  (fast.py:29-252; the layer input is what is cached, fast.py:192), and the
  demand-driven ``naive_logits`` (naive.py:27-110; the cell's demand sets equal
  the plain stack's). They are bit-identical in float64,
  checked by tests/test_oracle_cell.py the way test_fast.py:217-241 checks
  the reference's paths;
* weights are the model's float32 (bf16-representable for bf16 configs)
  values upcast to float64.

``exact=False`` swaps the pinned-order loops for BLAS matmuls (same math,
different rounding order, ~1e-15 relative) so large configs check quickly.

Parity of this cell arithmetic is unpinned by the reference: it
is pinned by the 3-way self-equivalence, constructed-weight golden cases in
tests/, and -- for the queue machinery it shares with plain mode -- by the
reference's own outputs through oracle/plain.py.
"""

from __future__ import annotations

import numpy as np

from . import noise as _noise
from .plain import demand_plan


class CellOracle:
    """Float64 view of a CellModel plus the pinned-order primitives."""

    def __init__(self, model, exact: bool = True):
        c = model.config
        self.cfg = c
        self.exact = exact
        f64 = lambda a: np.asarray(a, dtype=np.float64)
        self.E = f64(model.embed)
        self.W0 = [f64(lw.dil_taps[0]) for lw in model.layers]
        self.W1 = [f64(lw.dil_taps[1]) for lw in model.layers]
        self.bd = [f64(lw.dil_bias) for lw in model.layers]
        self.Wr = [f64(lw.res_w) for lw in model.layers]
        self.br = [f64(lw.res_b) for lw in model.layers]
        self.Ws = [f64(lw.skip_w) for lw in model.layers]
        self.bs = [f64(lw.skip_b) for lw in model.layers]
        self.H1, self.b1 = f64(model.head1_w), f64(model.head1_b)
        self.H2, self.b2 = f64(model.head2_w), f64(model.head2_b)
        self.D = c.dilation_channels
        self.L = c.total_layers
        self.dil = c.dilations()

    # ---- pinned-order primitives -------------------------------------------------
    def _acc(self, acc: np.ndarray, W: np.ndarray, X: np.ndarray, valid=None) -> np.ndarray:
        """acc[n, o] += sum_c W[o, c] * X[n, c], c ascending, one rounding per op."""
        if not self.exact:
            upd = X @ W.T
            return acc + upd if valid is None else np.where(valid, acc + upd, acc)
        for c in range(W.shape[1]):
            nxt = acc + W[None, :, c] * X[:, c:c + 1]
            acc = nxt if valid is None else np.where(valid, nxt, acc)
        return acc

    def lin(self, W, b, X):
        return self._acc(np.zeros((X.shape[0], W.shape[0])), W, X) + b[None, :]

    def gate(self, a: np.ndarray) -> np.ndarray:
        D = self.D
        return np.tanh(a[:, :D]) * (1.0 / (1.0 + np.exp(-a[:, D:])))

    def layer(self, l: int, x_cur: np.ndarray, x_past: np.ndarray, past_valid=None):
        """Returns (z, residual update) of layer l for rows x_cur / x_past."""
        acc = self._acc(np.zeros((x_cur.shape[0], 2 * self.D)), self.W0[l], x_cur)
        acc = self._acc(acc, self.W1[l], x_past, past_valid)
        z = self.gate(acc + self.bd[l][None, :])
        return z

    def res(self, l, z):
        return self.lin(self.Wr[l], self.br[l], z)

    def skip(self, l, z):
        return self.lin(self.Ws[l], self.bs[l], z)

    def head(self, s: np.ndarray) -> np.ndarray:
        h = np.maximum(self.lin(self.H1, self.b1, np.maximum(s, 0.0)), 0.0)
        return self.lin(self.H2, self.b2, h)

    # ---- path 1: time-parallel forward over one stream ----------------------------
    def forward_full(self, classes: np.ndarray) -> np.ndarray:
        """Logits (T, A) for one stream driven by the class sequence (teacher-forced)."""
        classes = np.asarray(classes, dtype=np.int64)
        T = classes.shape[0]
        x = self.E[classes]
        s = np.zeros((T, self.cfg.skip_channels))
        for l in range(self.L):
            d = self.dil[l]
            idx = np.arange(T) - d
            valid = (idx >= 0)[:, None]
            x_past = x[np.maximum(idx, 0)]
            z = self.layer(l, x, x_past, valid)
            s = s + self.skip(l, z)
            if l + 1 < self.L:
                x = x + self.res(l, z)
        return self.head(s)

    # ---- path 3: demand-driven recompute of one output ----------------------------
    def naive_logits(self, history: np.ndarray) -> np.ndarray:
        """Logits of the step aligned with history[-1], recomputed from raw classes."""
        hist = np.asarray(history, dtype=np.int64)
        t = hist.shape[0] - 1
        demanded, inputs, gathers = demand_plan(self.dil, 2)
        n_in = int(np.searchsorted(inputs, t, side="right"))
        x = self.E[hist[t - inputs[:n_in]]]  # rows at offsets inputs[:n_in]
        s = None
        for l in range(self.L):
            m = int(np.searchsorted(demanded[l], t, side="right"))
            g = gathers[l][:m]
            cur = x[g[:, 0]]  # offset o: always computed when o itself is
            past_ok = g[:, 1] < x.shape[0]
            past = x[np.where(past_ok, g[:, 1], 0)]
            z = self.layer(l, cur, past, past_ok[:, None])
            sk = self.skip(l, z[:1])
            s = (np.zeros_like(sk) if s is None else s) + sk
            if l + 1 < self.L:
                x = cur + self.res(l, z)
        return self.head(s)[0]


class CachedCell:
    """Path 2: queue-cached stepping of B streams (reference fast.py:29-252)."""

    def __init__(self, oracle: CellOracle, batch: int):
        self.o = oracle
        self.batch = batch
        R = oracle.cfg.residual_channels
        self.queues = [np.zeros((d, batch, R)) for d in oracle.dil]  # (w-1)*d slots
        self.t = 0

    def step(self, classes: np.ndarray) -> np.ndarray:
        """Consume one class per stream, return logits (B, A)."""
        o = self.o
        x = o.E[np.asarray(classes, dtype=np.int64)]
        s = np.zeros((self.batch, o.cfg.skip_channels))
        for l in range(o.L):
            q = self.queues[l]
            slot = self.t % q.shape[0]
            x_past = q[slot].copy()  # pop phase: the entry from t - d (fast.py:131-147)
            q[slot] = x  # push phase: cache the layer input (fast.py:192, 200-213)
            z = o.layer(l, x, x_past)
            s = s + o.skip(l, z)
            if l + 1 < o.L:
                x = x + o.res(l, z)
        self.t += 1
        return o.head(s)


# ---- selection rules -----------------------------------------------
def select_argmax(logits: np.ndarray) -> np.ndarray:
    return np.argmax(logits, axis=-1)  # first max on ties


def select_gumbel(logits, seed, streams, step):
    g = _noise.gumbel(seed, streams, step, logits.shape[-1])
    return np.argmax(logits + g, axis=-1)


def select_invcdf(logits, seed, streams, step):
    """Smallest i with cumsum(exp(l - max))_i > u * total (sequential cumsum)."""
    u = _noise.step_uniform(seed, streams, step)
    e = np.exp(logits - logits.max(axis=-1, keepdims=True))
    cs = np.cumsum(e, axis=-1)
    thr = u * cs[:, -1]
    idx = (cs > thr[:, None]).argmax(axis=-1)
    none = ~(cs > thr[:, None]).any(axis=-1)
    return np.where(none, logits.shape[-1] - 1, idx)


def select(mode: int, logits, seed, streams, step):
    if mode == 0:
        return select_argmax(logits)
    if mode == 1:
        return select_invcdf(logits, seed, streams, step)
    if mode == 2:
        return select_gumbel(logits, seed, streams, step)
    raise ValueError(f"unknown sampler {mode}")


def selection_margin(mode: int, logits, seed, streams, step, a, b) -> np.ndarray:
    """How far choice ``a`` (oracle) is ahead of choice ``b`` in the rule's own score."""
    rows = np.arange(logits.shape[0])
    if mode == 0:
        score = logits
    elif mode == 2:
        score = logits + _noise.gumbel(seed, streams, step, logits.shape[-1])
    else:  # inverse CDF: distance of the threshold to the nearer cumsum boundary
        u = _noise.step_uniform(seed, streams, step)
        e = np.exp(logits - logits.max(axis=-1, keepdims=True))
        cs = np.cumsum(e, axis=-1)
        thr = u * cs[:, -1]
        lo, hi = np.minimum(a, b), np.maximum(a, b)
        out = np.empty(len(rows))
        for r in rows:
            seg = cs[r, lo[r]:max(hi[r], lo[r] + 1)]
            out[r] = np.min(np.abs(seg - thr[r])) / cs[r, -1]
        return out
    return score[rows, a] - score[rows, b]


def generate(oracle: CellOracle, inputs: np.ndarray, n_steps: int, sampler: int,
             seed: int = 0, stream_offset: int = 0, t0: int = 0):
    """Mirror of fw_cell_generate: inputs (n_inputs, B) teacher classes, then feedback.

    Returns (choices (n_steps, B), logits (n_steps, B, A)).
    """
    inputs = np.asarray(inputs, dtype=np.int64)
    B = inputs.shape[1]
    st = CachedCell(oracle, B)
    st.t = 0
    streams = np.arange(B) + stream_offset
    out = np.zeros((n_steps, B), dtype=np.int64)
    logits_all = np.zeros((n_steps, B, oracle.cfg.classes))
    cur = inputs[0]
    for i in range(n_steps):
        if i < inputs.shape[0]:
            cur = inputs[i]
        lg = st.step(cur)
        logits_all[i] = lg
        out[i] = select(sampler, lg, seed, streams, t0 + i)
        cur = out[i]
    return out, logits_all
