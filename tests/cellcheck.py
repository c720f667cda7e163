"""Shared checker for GPU cell runs (test helper, uses the CPU oracle)."""

from __future__ import annotations

import numpy as np

from oracle import cell as oc


def histories(inputs: np.ndarray, choices: np.ndarray) -> np.ndarray:
    """Per-step input classes the GPU consumed: teacher rows, then its own choices."""
    n_in = inputs.shape[0]
    n = choices.shape[0]
    hist = np.empty((n,) + choices.shape[1:], dtype=np.int64)
    hist[:min(n, n_in)] = inputs[:n]
    if n > n_in:
        hist[n_in:] = choices[n_in - 1:n - 1]
    return hist


def check_streams(oracle: oc.CellOracle, inputs, choices, logits, streams, mode, seed,
                  logit_tol, tie_tol, stream_offset=0, t0=0, report=None, gids=None):
    """Compare GPU logits/choices of ``streams`` against the oracle run on the
    GPU's own input history (teacher-forced on it), SURVEY section 7.

    ``inputs``/``choices``/``logits`` are indexed [step, column]; ``gids`` maps a column to
    the global stream id that keys its noise (default: column + stream_offset), so callers
    can pass a column subset of a large batch.

    Returns the number of near-tie choice mismatches (logged, allowed)."""
    hist = histories(np.asarray(inputs), np.asarray(choices))
    ties = 0
    worst = 0.0
    for s in streams:
        ref = oracle.forward_full(hist[:, s])  # (n, A)
        if logits is not None:
            n_l = logits.shape[0]
            dev = np.max(np.abs(logits[:, s].astype(np.float64) - ref[:n_l]))
            worst = max(worst, dev)
            assert dev <= logit_tol, f"stream {s}: logits max-abs {dev:.3g} > {logit_tol}"
        gsid = np.array([gids[s] if gids is not None else s + stream_offset])
        for i in range(choices.shape[0]):
            want = oc.select(mode, ref[i:i + 1], seed, gsid, t0 + i)[0]
            got = int(choices[i, s])
            if want != got:
                margin = float(oc.selection_margin(mode, ref[i:i + 1], seed, gsid, t0 + i,
                                                   np.array([want]), np.array([got]))[0])
                assert margin <= tie_tol, (
                    f"stream {s} step {i}: GPU chose {got}, oracle {want}, margin {margin:.3g}")
                ties += 1
                if report is not None:
                    report.append((s, i, got, want, margin))
    if report is not None:
        report.append(("max_logit_dev", worst))
    return ties
