"""GPU plain mode (fp64 kernel) against the reference's own outputs.

Golden outputs come from the unmodified reference (tests/golden/
plain_reference.npz). Every stack must match bit-exactly: the same pinned
order, no FMA contraction (__dmul_rn/__dadd_rn), and the host libm's tanh
restated on the device (csrc/libm_tanh.cuh: glibc's fdlibm-derived
tanh/expm1 with its fused multiply-adds), so even the chaotic free run of the
50-layer tanh proxy reproduces the reference's samples bit for bit.
"""

from pathlib import Path

import numpy as np
import pytest

from paper_1611_09482_b200 import (
    QueueStateError, compute_step, fast_generate, fast_step, init_state, pop_phase, push_phase)
from paper_1611_09482_b200.model import LayerWeights, Model, ModelConfig, build_model

pytestmark = pytest.mark.gpu

G = np.load(Path(__file__).parent / "golden" / "plain_reference.npz")
NAMES = sorted({k.split("/")[0] for k in G.files if not k.startswith("delay")})


def model_of(name):
    c = G[f"{name}/config"]
    return build_model(ModelConfig(int(c[0]), int(c[1]), int(c[2]), int(c[3]), int(c[4]),
                                   "tanh" if c[5] else "linear", int(c[6])))


def assert_match(got, want, tanh=False, layers=1):
    """Bit-exact, linear and tanh stacks alike (SPEC.md:306's 1e-12 fallback unused)."""
    assert np.array_equal(got, want), (np.max(np.abs(np.asarray(got) - want)), layers)


@pytest.mark.parametrize("name", NAMES)
def test_teacher_forced_and_free_run_match_reference(cuda, name):
    m = model_of(name)
    tanh = m.config.activation == "tanh"
    xs = G[f"{name}/xs"]
    st = init_state(m)
    got = np.array([fast_step(st, float(x), m) for x in xs])
    L = m.config.total_layers
    assert_match(got, G[f"{name}/tf"], tanh, L)
    assert st.step_index == len(xs)
    free = G[f"{name}/free"]
    primer = G[f"{name}/primer"]
    out = fast_generate(m, primer, len(free))
    assert out.start_index == len(primer)
    assert_match(out.scalars(), free, tanh, L)


def test_device_tanh_is_libm_tanh(cuda):
    """The device tanh (libm_tanh.cuh) through a one-layer identity stack: tanh(x) of the
    stack's input equals the host libm's math.tanh bit for bit over 2e5 arguments spanning
    1e-12 .. 40 in magnitude (every branch of fdlibm's tanh/expm1)."""
    import math

    lw = LayerWeights(np.array([[[1.0]], [[0.0]]]), np.zeros(1))
    m = Model(ModelConfig(1, 1, 2, 2, 1, "tanh", 0), (lw,))
    rng = np.random.default_rng(5)
    xs = 10.0 ** rng.uniform(-12, 1.6, 200_000) * rng.choice([-1.0, 1.0], 200_000)
    xs = np.concatenate([xs, [0.0, -0.0, 22.0, -22.0, 0.17328679513998632, 1.0, -1.0]])
    st = init_state(m, batch=xs.size)
    got = fast_step(st, xs, m)
    want = np.array([math.tanh(x) for x in xs])
    assert np.array_equal(got, want), int(np.sum(got != want))


@pytest.mark.parametrize("layers", [1, 3, 4])
def test_delay_line_exact(cuda, layers):
    cfg = ModelConfig(1, layers, 2, 2, 1, "linear", 0)
    lws = []
    for l in range(layers):
        taps = np.zeros((2, 1, 1))
        taps[1 if l == layers - 1 else 0, 0, 0] = 1.0
        lws.append(LayerWeights(taps, np.zeros(1)))
    m = Model(cfg, tuple(lws))
    xs = G[f"delay{layers}/xs"]
    st = init_state(m)
    got = np.array([fast_step(st, float(x), m) for x in xs])
    assert np.array_equal(got, G[f"delay{layers}/tf"])


def test_batched_streams_are_independent(cuda):
    m = model_of("grid100")
    xs = np.random.default_rng(3).uniform(-1, 1, (12, 5))
    st = init_state(m, batch=5)
    got = np.stack([fast_step(st, x, m) for x in xs])
    for b in range(5):
        st1 = init_state(m)
        one = np.array([fast_step(st1, float(x), m) for x in xs[:, b]])
        assert np.array_equal(got[:, b], one)


def test_phase_api_and_errors(cuda):
    m = build_model(ModelConfig(1, 4, hidden_channels=1, activation="tanh", init_seed=7))
    st = init_state(m)
    assert [q.capacity for q in st.queues] == [1, 2, 4, 8]
    assert st.cached_scalar_count() == 15
    rec = pop_phase(st)
    assert len(rec.per_layer) == 4 and all(np.array_equal(r[0], np.zeros(1)) for r in rec.per_layer)
    with pytest.raises(QueueStateError):
        pop_phase(st)
    y, new_states, macs = compute_step(m, 0.3, rec)
    assert macs.multiply_accumulates == 8 and macs.node_evaluations == 4
    push_phase(st, new_states)
    assert st.step_index == 1
    with pytest.raises(QueueStateError):
        push_phase(st, new_states)
    # the pushed value is the layer input: the next pop of layer 0 at t=1 reads t-1 = 0.3
    st2 = init_state(m)
    y_ref = fast_step(st2, 0.3, m)
    assert y == y_ref or abs(y - y_ref) < 1e-15
    rec2 = pop_phase(st)
    assert rec2.per_layer[0][0][0] == 0.3
    assert np.array_equal(rec2.per_layer[1][0], np.zeros(1))  # layer 1 has d=2


def test_foreign_state_rejected(cuda):
    m = model_of("grid000")
    other = build_model(ModelConfig(blocks=2, layers_per_block=2, init_seed=1))
    with pytest.raises(ValueError, match="architecture"):
        fast_step(init_state(other), 0.0, m)


def test_generate_zero_steps_is_empty(cuda):
    m = model_of("grid000")
    assert len(fast_generate(m, [0.5], 0)) == 0
    with pytest.raises(ValueError):
        fast_generate(m, [0.5], -1)


NAIVE_NAMES = sorted(n for n in NAMES if f"{n}/naive" in G.files)


@pytest.mark.parametrize("name", NAIVE_NAMES)
def test_gpu_naive_matches_reference_naive_generate(cuda, name):
    """The GPU demand-plan generator (fw_plain_naive) against the
    unmodified reference's naive_generate on the same primer (golden vectors): bit-exact for
    linear stacks, tanh within CUDA-vs-glibc ulps; and against the GPU cached path on the
    same history: bit-exact for every stack (same kernel arithmetic)."""
    from paper_1611_09482_b200 import naive_generate, naive_step

    m = model_of(name)
    tanh = m.config.activation == "tanh"
    primer = G[f"{name}/primer"]
    want = G[f"{name}/naive"]
    got = naive_generate(m, primer, len(want))
    assert got.start_index == len(primer)
    assert_match(got.scalars(), want, tanh, m.config.total_layers)
    fast = fast_generate(m, primer, len(want)).scalars()
    assert np.array_equal(got.scalars(), fast)
    y, macs = naive_step(m, primer)
    assert y == fast[0] and macs.node_evaluations >= m.config.total_layers
