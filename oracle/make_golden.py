"""Generate tests/golden/plain_reference.npz from the UNMODIFIED reference.

Run here (where /root/reference exists), never on the GPU box:

    python oracle/make_golden.py

The reference package is copied to /tmp and imported with NUMBA_CACHE_DIR in
/tmp (running it in place writes numba caches into /root/reference, SURVEY.md
section 0 item 4). Nothing from the reference is copied into this repo: only
its numerical outputs on seeded inputs are stored.

Contents, per case key ``<name>/...``:
* ``config``   (blocks, layers_per_block, filter_width, dilation_base,
  hidden_channels, act_code, init_seed)
* ``weights``  all taps then bias per layer, flattened float64 (pins build_model)
* ``xs``       teacher-forced inputs (seeded uniform[-1, 1])
* ``tf``       reference fast_step outputs on xs (== forward_full, bit-exact)
* ``primer`` / ``free``  reference fast_generate(primer, steps) outputs
* ``naive``    reference naive_generate on the same primer (small configs)
* ``caps``     queue capacities of init_state
"""

from __future__ import annotations

import os
import shutil
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parents[1] / "tests" / "golden" / "plain_reference.npz"


def import_reference():
    dst = Path("/tmp/refpkg_golden")
    if dst.exists():
        shutil.rmtree(dst)
    shutil.copytree(REF, dst)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
    sys.path.insert(0, str(dst / "src"))
    import streamconv  # noqa: E402

    return streamconv


def grid(sc):
    """The reference's own verification grid (cli.py:138-157), every config."""
    return sc.cli.verification_grid()


def main() -> None:
    sc = import_reference()
    import streamconv.cli  # noqa: F401

    out: dict[str, np.ndarray] = {}
    cases = []
    for i, cfg in enumerate(grid(sc)):
        cases.append((f"grid{i:03d}", cfg, 40, 24, cfg.total_layers <= 12))
    # BASELINE shape-proxies, short runs.
    for name, blocks, layers, ch in (("proxy_cfg1", 1, 10, 32), ("proxy_cfg2_L6", 1, 6, 128),
                                     ("proxy_cfg3", 5, 10, 64)):
        cfg = sc.ModelConfig(blocks=blocks, layers_per_block=layers, hidden_channels=ch,
                             activation="tanh", init_seed=0)
        cases.append((name, cfg, 24, 12, False))
    for name, cfg, n_tf, n_free, do_naive in cases:
        model = sc.build_model(cfg)
        rng = np.random.default_rng([cfg.init_seed, 0xA5])
        xs = rng.uniform(-1.0, 1.0, n_tf)
        state = sc.init_state(model)
        tf = np.array([sc.fast_step(state, x, model) for x in xs])
        full = sc.forward_full(model, sc.SampleSequence.from_scalars(xs)).scalars()
        assert np.array_equal(tf, full)
        primer = xs[: 1 + (cfg.init_seed % 5)]
        free = sc.fast_generate(model, primer, n_free).scalars()
        act = 1 if cfg.activation == "tanh" else 0
        out[f"{name}/config"] = np.array([cfg.blocks, cfg.layers_per_block, cfg.filter_width,
                                          cfg.dilation_base, cfg.hidden_channels, act,
                                          cfg.init_seed], dtype=np.int64)
        w = np.concatenate([np.concatenate([lw.taps.ravel(), lw.bias.ravel()])
                            for lw in model.layers])
        if w.size <= 20000:
            out[f"{name}/weights"] = w
        else:
            out[f"{name}/weights_sum"] = np.array([w.sum(), np.abs(w).sum(), w[::97].sum()])
        out[f"{name}/xs"] = xs
        out[f"{name}/tf"] = tf
        out[f"{name}/primer"] = primer
        out[f"{name}/free"] = free
        out[f"{name}/caps"] = np.array([q.capacity for q in sc.init_state(model).queues])
        if do_naive:
            out[f"{name}/naive"] = sc.naive_generate(model, primer, n_free).scalars()
    # Delay-line golden model (reference tests/conftest.py:35-57 construction, rebuilt here).
    for layers in (1, 3, 4):
        cfg = sc.ModelConfig(blocks=1, layers_per_block=layers, filter_width=2,
                             dilation_base=2, hidden_channels=1, activation="linear")
        lws = []
        for l in range(cfg.total_layers):
            taps = np.zeros((2, 1, 1))
            taps[1 if l == cfg.total_layers - 1 else 0, 0, 0] = 1.0
            lws.append(sc.LayerWeights(taps=taps, bias=np.zeros(1)))
        model = sc.Model(config=cfg, layers=tuple(lws))
        delay = 2 ** (layers - 1)
        xs = np.random.default_rng(6).uniform(-1.0, 1.0, 3 * delay + 5)
        st = sc.init_state(model)
        out[f"delay{layers}/xs"] = xs
        out[f"delay{layers}/tf"] = np.array([sc.fast_step(st, x, model) for x in xs])
    OUT.parent.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(cases)} configs)")


if __name__ == "__main__":
    main()
