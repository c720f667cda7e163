"""Pin the plain-mode oracle (oracle/plain.py) against the unmodified reference.

tests/golden/plain_reference.npz holds outputs of the reference package run
from a /tmp copy (oracle/make_golden.py): its full 144-config verification
grid (cli.py:138-157), three BASELINE shape-proxies and the delay-line models
(conftest.py:35-57). Every comparison is bit-exact, as the reference's own
tests are (test_fast.py:217-241).
"""

from pathlib import Path

import numpy as np
import pytest

from oracle import plain
from paper_1611_09482_b200.model import LayerWeights, Model, ModelConfig, build_model, receptive_field

GOLDEN = Path(__file__).parent / "golden" / "plain_reference.npz"
G = np.load(GOLDEN)
NAMES = sorted({k.split("/")[0] for k in G.files if not k.startswith("delay")})


def model_of(name):
    c = G[f"{name}/config"]
    cfg = ModelConfig(int(c[0]), int(c[1]), int(c[2]), int(c[3]), int(c[4]),
                      "tanh" if c[5] else "linear", int(c[6]))
    return build_model(cfg)


def flat_weights(m):
    return np.concatenate([np.concatenate([lw.taps.ravel(), lw.bias.ravel()]) for lw in m.layers])


def test_golden_covers_reference_grid():
    assert sum(n.startswith("grid") for n in NAMES) == 144


@pytest.mark.parametrize("name", NAMES)
def test_build_model_matches_reference_weights(name):
    m = model_of(name)
    w = flat_weights(m)
    if f"{name}/weights" in G.files:
        assert np.array_equal(w, G[f"{name}/weights"])
    else:
        ref = G[f"{name}/weights_sum"]
        assert np.array_equal(np.array([w.sum(), np.abs(w).sum(), w[::97].sum()]), ref)


@pytest.mark.parametrize("name", NAMES)
def test_oracle_paths_match_reference_bit_exact(name):
    m = model_of(name)
    xs = G[f"{name}/xs"]
    assert np.array_equal(plain.forward_full(m, xs), G[f"{name}/tf"])
    st = plain.CachedStack(m, 1)
    assert np.array_equal(np.array([st.step(np.array([x]))[0] for x in xs]), G[f"{name}/tf"])
    free = G[f"{name}/free"]
    assert np.array_equal(plain.fast_generate(m, G[f"{name}/primer"], len(free)), free)
    if f"{name}/naive" in G.files:
        assert np.array_equal(plain.naive_generate(m, G[f"{name}/primer"], len(free)),
                              G[f"{name}/naive"])


@pytest.mark.parametrize("name", NAMES[:40])
def test_queue_capacities_match_reference(name):
    m = model_of(name)
    cfg = m.config
    caps = [(cfg.filter_width - 1) * d for d in cfg.dilations()]
    assert caps == G[f"{name}/caps"].tolist()


@pytest.mark.parametrize("layers", [1, 3, 4])
def test_delay_line_golden(layers):
    cfg = ModelConfig(1, layers, 2, 2, 1, "linear", 0)
    lws = []
    for l in range(layers):
        taps = np.zeros((2, 1, 1))
        taps[1 if l == layers - 1 else 0, 0, 0] = 1.0
        lws.append(LayerWeights(taps, np.zeros(1)))
    m = Model(cfg, tuple(lws))
    xs = G[f"delay{layers}/xs"]
    out = plain.forward_full(m, xs)
    assert np.array_equal(out, G[f"delay{layers}/tf"])
    d = 2 ** (layers - 1)
    assert np.array_equal(out[:d], np.zeros(d)) and np.array_equal(out[d:], xs[:-d])


def test_model_validation_mirrors_reference():
    with pytest.raises(ValueError, match="blocks"):
        ModelConfig(0, 1)
    with pytest.raises(ValueError, match="filter_width"):
        ModelConfig(1, 1, filter_width=1)
    with pytest.raises(ValueError, match="activation"):
        ModelConfig(1, 1, activation="relu")
    assert receptive_field(ModelConfig(1, 10)) == 1024
    assert receptive_field(ModelConfig(2, 3, filter_width=3, dilation_base=4)) == 1 + 2 * 2 * 21
    with pytest.raises(ValueError, match="finite"):
        LayerWeights(np.full((2, 1, 1), np.nan), np.zeros(1))


def test_libm_tanh_restatement():
    """oracle/libm_tanh.py (the algorithm csrc/libm_tanh.cuh ports to the device) equals the
    host libm's tanh -- the one the reference's numba kernel calls -- bit for bit, on every
    branch: tiny, |x| < 0.5 ln2 / 2 (k = 0), the k = -1 reduction, |x| >= 1, |x| >= 22."""
    import math

    from oracle.libm_tanh import tanh

    rng = np.random.default_rng(7)
    xs = 10.0 ** rng.uniform(-20, 1.6, 20_000) * rng.choice([-1.0, 1.0], 20_000)
    xs = np.concatenate([xs, [0.0, -0.0, 5e-324, 22.0, -22.0, 21.999999, 1.0, -1.0,
                              0.17328679513998632, 0.5198603854199589]])
    bad = [x for x in xs if tanh(float(x)) != math.tanh(float(x))]
    assert not bad, bad[:5]
