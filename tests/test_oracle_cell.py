"""The gated-cell oracle: 3-way fp64 self-equivalence plus constructed cases.

The reference has no gated cell, so these tests are the pin for the cell
arithmetic: the time-parallel forward, the queue-cached step and
the demand-driven recompute must agree bit-exactly (the reference's own
parity method, test_fast.py:217-241 / test_naive.py:59-81), and constructed
weights must give hand-computable results.
"""

import numpy as np
import pytest

from oracle import cell as oc
from oracle import noise
from paper_1611_09482_b200.cell import CellConfig, CellLayer, CellModel, build_cell_model, round_to_bf16
from paper_1611_09482_b200 import configs

SMALL = [
    CellConfig(1, 4, 4, 3, 5, classes=7, bias="fan_in", init_seed=3),
    CellConfig(2, 3, 8, 8, 16, classes=16, bias="fan_in", init_seed=1),
    CellConfig(1, 5, 6, 4, 8, classes=11, dilation_base=3, bias="fan_in", init_seed=9),
    CellConfig(1, 10, 32, 32, 128, init="normal:0.1"),
    CellConfig(2, 2, 8, 8, 8, classes=8, weight_dtype="bf16", bias="fan_in", init_seed=4),
]


@pytest.mark.parametrize("cfg", SMALL, ids=lambda c: f"L{c.total_layers}R{c.residual_channels}")
def test_three_paths_bit_exact(cfg):
    m = build_cell_model(cfg)
    o = oc.CellOracle(m)
    T = 3 * max(cfg.dilations()) + 5 if cfg.total_layers < 10 else 24
    cls = np.random.default_rng(cfg.init_seed + 11).integers(0, cfg.classes, T)
    full = o.forward_full(cls)
    st = oc.CachedCell(o, 1)
    cached = np.stack([st.step(cls[i:i + 1])[0] for i in range(T)])
    naive = np.stack([o.naive_logits(cls[:i + 1]) for i in range(T)])
    assert np.array_equal(full, cached)
    assert np.array_equal(full, naive)


def test_batched_cached_step_equals_per_stream():
    cfg = SMALL[1]
    o = oc.CellOracle(build_cell_model(cfg))
    B, T = 5, 20
    cls = np.random.default_rng(2).integers(0, cfg.classes, (T, B))
    st = oc.CachedCell(o, B)
    batched = np.stack([st.step(cls[i]) for i in range(T)])
    for b in range(B):
        assert np.array_equal(batched[:, b], o.forward_full(cls[:, b]))


def test_blas_mode_close_to_pinned():
    cfg = SMALL[3]
    m = build_cell_model(cfg)
    cls = np.random.default_rng(1).integers(0, 256, 64)
    a = oc.CellOracle(m).forward_full(cls)
    b = oc.CellOracle(m, exact=False).forward_full(cls)
    assert np.max(np.abs(a - b)) < 1e-12


def _zero_model(cfg, b2):
    R, D, S, H, A = (cfg.residual_channels, cfg.dilation_channels, cfg.skip_channels, cfg.H,
                     cfg.classes)
    z = lambda *s: np.zeros(s, dtype=np.float32)
    layers = tuple(CellLayer(z(2, 2 * D, R), z(2 * D), z(R, D), z(R), z(S, D), z(S))
                   for _ in range(cfg.total_layers))
    return CellModel(cfg, z(A, R), layers, z(H, S), z(H), z(A, H), b2.astype(np.float32))


def test_zero_weights_give_head_bias():
    cfg = CellConfig(1, 3, 4, 4, 4, classes=6)
    b2 = np.arange(6, dtype=np.float32) * 0.5 - 1
    o = oc.CellOracle(_zero_model(cfg, b2))
    lg = o.forward_full(np.array([0, 3, 5, 1]))
    assert np.array_equal(lg, np.tile(b2.astype(np.float64), (4, 1)))


def test_gate_and_skip_hand_computed():
    """One layer, R=D=S=H=1, A=2: logits are computable in closed form."""
    cfg = CellConfig(1, 1, 1, 1, 1, classes=2, head_channels=1)
    f = lambda *v: np.array(v, dtype=np.float32)
    dil = np.zeros((2, 2, 1), dtype=np.float32)
    dil[0, :, 0] = [0.5, 0.25]  # tap 0 (current) -> tanh half, sigmoid half
    dil[1, :, 0] = [-1.0, 2.0]  # tap 1 (d = 1 back)
    layer = CellLayer(dil, f(0.0, 0.0), np.zeros((1, 1), np.float32), f(0.0), f(1.0).reshape(1, 1), f(0.0))
    m = CellModel(cfg, f(1.0, -2.0).reshape(2, 1), (layer,), f(1.0).reshape(1, 1), f(0.0),
                  f(1.0, -1.0).reshape(2, 1), f(0.0, 0.0))
    lg = oc.CellOracle(m).forward_full(np.array([0, 1]))
    # t=0: x=1, past=0: a=(0.5, 0.25); t=1: x=-2, past=1: a=(-1-1, -0.5+2)
    z0 = np.tanh(0.5) / (1 + np.exp(-0.25))
    z1 = np.tanh(-2.0) / (1 + np.exp(-1.5))
    for t, zz in enumerate((z0, z1)):
        h = max(max(zz, 0.0), 0.0)
        assert np.allclose(lg[t], [h, -h], rtol=0, atol=1e-15)


def test_noise_hash_golden_values():
    """Pins the counter hash shared with csrc/internal.h (mix32 chain)."""
    h = noise.hash_bits(2016, np.array([0, 1, 4095]), np.array([0, 7, 23999]),
                        np.array([0, 255, 0xFFFFFFFF]))
    assert h.tolist() == [197887118, 3960416316, 4080196203]
    assert noise.uniform(0, 3, 5, 7) == 0.7776133716106415
    g = noise.gumbel(2016, np.array([0]), 0, 4)
    assert np.allclose(g, [[-1.1241184, 3.20122546, -0.96208715, -0.19697924]], atol=1e-8)


def test_selection_rules():
    lg = np.array([[0.0, 2.0, 2.0, -1.0]])
    assert oc.select_argmax(lg).tolist() == [1]  # first max on ties
    # inverse CDF: the chosen index is the first whose cumsum passes u * total
    for step in range(50):
        c = oc.select_invcdf(lg, 7, np.array([0]), step)[0]
        u = noise.step_uniform(7, np.array([0]), step)[0]
        e = np.exp(lg[0] - 2.0)
        cs = np.cumsum(e)
        assert cs[c] > u * cs[-1] and (c == 0 or cs[c - 1] <= u * cs[-1])
    # Gumbel-max is the argmax of logits + noise
    c = oc.select_gumbel(lg, 3, np.array([9]), 4)
    assert c[0] == np.argmax(lg[0] + noise.gumbel(3, np.array([9]), 4, 4)[0])


def test_gumbel_sampling_frequencies():
    lg = np.log(np.array([[0.1, 0.2, 0.3, 0.4]]))
    picks = np.array([oc.select_gumbel(lg, 1, np.array([0]), s)[0] for s in range(4000)])
    freq = np.bincount(picks, minlength=4) / 4000
    assert np.allclose(freq, [0.1, 0.2, 0.3, 0.4], atol=0.03)


def test_generate_teacher_then_feedback():
    cfg = SMALL[0]
    o = oc.CellOracle(build_cell_model(cfg))
    inputs = np.array([[1, 2], [3, 4]])
    out, lg = oc.generate(o, inputs, 6, 0)
    # steps 0,1 are teacher-forced; step 2 consumes the choice of step 1
    hist = np.concatenate([inputs[:, 0], out[1:5, 0]])
    full = o.forward_full(hist)
    assert np.array_equal(full, lg[:, 0])
    assert np.array_equal(out[:, 0], np.argmax(full, axis=1))


def test_bf16_rounding():
    x = np.array([1.0, 1.0 + 2**-9, 1.0 + 3 * 2**-9, -2.5e-3, 3.0e38], dtype=np.float32)
    r = round_to_bf16(x)
    assert r[0] == 1.0 and r[1] == 1.0 and r[2] == 1.0 + 2**-7 * 1  # ties to even
    assert (r.view(np.uint32) & 0xFFFF).max() == 0


def test_baseline_configs_shape_facts():
    c1, c3, c4, c5 = configs.cfg1(), configs.cfg3(), configs.cfg4(), configs.cfg5()
    assert c1.cell.receptive_field() == 1024
    assert c3.cell.receptive_field() == 5116
    assert c4.cell.receptive_field() == 4093
    assert c5.cell.receptive_field() == 32761
    # queue bytes (fp32): cfg4 8.58 GB, cfg5 8.59 GB
    assert abs(c4.cell.queue_slots() * c4.batch * 128 * 4 / 1e9 - 8.58) < 0.01
    assert abs(c5.cell.queue_slots() * c5.batch * 64 * 4 / 1e9 - 8.59) < 0.01
    m4 = c4.cell.macs_per_sample()
    assert m4 == 40 * (4 * 128 * 128 + 512 * 128) + 39 * 128 * 128 + 512 * 512 + 512 * 256
