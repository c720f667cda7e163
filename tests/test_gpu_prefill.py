"""GPU full-sequence forward (fw_cell_prefill) against teacher-forced
stepping and the CPU oracle's forward_full (the reference's full-sequence ground truth,
oracle.py:84-123, restated for the cell).

The prefill must leave the handle exactly where T teacher-forced steps leave it: same step
counter, the same ring contents (every layer's last d_l inputs), and the same logits for
every step -- so generation continues identically. Tolerances: fp32 configs (SIMT handles,
fp32 GEMMs without TF32) 1e-4 max-abs on logits; bf16 configs (tcgen05 handles, fp16
operands) the north star's 2e-2.
"""

import os

import numpy as np
import pytest
import torch

from oracle import cell as oc
from paper_1611_09482_b200 import CellGenerator, Sampler, build_cell_model
from paper_1611_09482_b200.cell import CellConfig

pytestmark = pytest.mark.gpu

SIMT_CFG = CellConfig(1, 10, 32, 32, 128, init="normal:0.1", bias="fan_in", init_seed=3)
TC_CFG = CellConfig(2, 4, 128, 128, 256, weight_dtype="bf16", bias="fan_in", init_seed=5)
CASES = {"simt": (SIMT_CFG, 3, 1e-4), "tcgen05": (TC_CFG, 128, 2e-2)}


@pytest.fixture(scope="module")
def models():
    return {k: build_cell_model(c) for k, (c, _, _) in CASES.items()}


def teacher(T, B, seed, A=256):
    return np.random.default_rng(seed).integers(0, A, (T, B)).astype(np.int32)


def queue_values(gen):
    """The handle's ring contents as floats (fp32 SIMT slots, fp16 tcgen05 slots)."""
    nbytes = gen.queue_bytes
    buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    from paper_1611_09482_b200 import _lib
    import ctypes as C

    _lib.check(gen._lib.fw_debug_copy(gen._h, 0, C.c_void_p(buf.data_ptr()), nbytes, None))
    torch.cuda.synchronize()
    dt = torch.float16 if gen.kernel == "tcgen05" else torch.float32
    return buf.view(dt).float().cpu().numpy()


def stepped(model, kernel, B, x):
    gen = CellGenerator(model, B, kernel=kernel)
    _, lg = gen.generate(torch.as_tensor(x, device="cuda"), x.shape[0], Sampler(0),
                         n_logit_steps=x.shape[0])
    torch.cuda.synchronize()
    return gen, lg.cpu().numpy()


@pytest.mark.parametrize("kernel", ["simt", "tcgen05"])
@pytest.mark.parametrize("T", [1, 37, 300])
def test_prefill_matches_teacher_forced_steps(cuda, models, kernel, T):
    cfg, B, tol = CASES[kernel]
    x = teacher(T, B, 11 + T)
    ref_gen, ref = stepped(models[kernel], kernel, B, x)
    gen = CellGenerator(models[kernel], B, kernel=kernel)
    lg = gen.prefill(torch.as_tensor(x, device="cuda"), want_logits=True)
    torch.cuda.synchronize()
    assert gen.step_index == T == ref_gen.step_index
    dev = np.max(np.abs(lg.cpu().numpy() - ref))
    assert dev <= tol, dev
    qd = np.max(np.abs(queue_values(gen) - queue_values(ref_gen)))
    assert qd <= (1e-4 if kernel == "simt" else 2e-2), qd


@pytest.mark.parametrize("kernel", ["simt", "tcgen05"])
def test_prefill_against_oracle_forward_full(cuda, models, kernel):
    cfg, B, tol = CASES[kernel]
    T = 200
    x = teacher(T, B, 99)
    gen = CellGenerator(models[kernel], B, kernel=kernel)
    lg = gen.prefill(torch.as_tensor(x, device="cuda"), want_logits=True).cpu().numpy()
    o = oc.CellOracle(models[kernel])
    for b in sorted({0, B - 1}):
        ref = o.forward_full(x[:, b])
        dev = np.max(np.abs(lg[:, b] - ref))
        assert dev <= tol, (b, dev)


@pytest.mark.parametrize("kernel", ["simt", "tcgen05"])
def test_prefill_then_generation_continues(cuda, models, kernel):
    """Queues only (no logits), from a non-zero step, in two calls, then teacher-forced
    steps: the continuation's logits match an all-stepped run."""
    cfg, B, tol = CASES[kernel]
    x = teacher(150, B, 7)
    head, p1, p2, tail = x[:9], x[9:80], x[80:120], x[120:]
    ref_gen, ref = stepped(models[kernel], kernel, B, x)
    gen = CellGenerator(models[kernel], B, kernel=kernel)
    gen.generate(torch.as_tensor(head, device="cuda"), len(head), Sampler(0))
    assert gen.prefill(torch.as_tensor(p1, device="cuda")) is None
    gen.prefill(torch.as_tensor(p2, device="cuda"))
    assert gen.step_index == 120
    _, lg = gen.generate(torch.as_tensor(tail, device="cuda"), len(tail), Sampler(0),
                         n_logit_steps=len(tail))
    torch.cuda.synchronize()
    dev = np.max(np.abs(lg.cpu().numpy() - ref[120:]))
    assert dev <= tol, dev


@pytest.mark.parametrize("kernel", ["simt", "tcgen05"])
def test_prefill_chunking_invariance(cuda, models, kernel, monkeypatch):
    cfg, B, tol = CASES[kernel]
    x = teacher(90, B, 5)
    outs = []
    for chunk in (1, 7, 90):
        monkeypatch.setenv("FW_PREFILL_CHUNK", str(chunk))
        gen = CellGenerator(models[kernel], B, kernel=kernel)
        outs.append((gen.prefill(torch.as_tensor(x, device="cuda"), want_logits=True).cpu().numpy(),
                     queue_values(gen)))
    for lg, q in outs[1:]:
        assert np.max(np.abs(lg - outs[0][0])) <= tol / 10
        assert np.max(np.abs(q - outs[0][1])) <= (1e-5 if kernel == "simt" else 2e-3)


def test_prefill_argument_errors(cuda, models):
    gen = CellGenerator(models["simt"], 3, kernel="simt")
    with pytest.raises(ValueError):
        gen.prefill(torch.zeros((4, 2), dtype=torch.int32, device="cuda"))
    assert gen.prefill(torch.zeros((0, 3), dtype=torch.int32, device="cuda")) is None
    assert gen.step_index == 0


def test_prefill_modes_agree(cuda, models, monkeypatch):
    """The two implementations behind fw_cell_prefill (time-parallel GEMMs, teacher-forced
    steps of the fused kernel) leave the same state and logits."""
    cfg, B, tol = CASES["tcgen05"]
    x = teacher(64, B, 21)
    res = {}
    for mode in ("gemm", "steps"):
        monkeypatch.setenv("FW_PREFILL_MODE", mode)
        gen = CellGenerator(models["tcgen05"], B, kernel="tcgen05")
        lg = gen.prefill(torch.as_tensor(x, device="cuda"), want_logits=True).cpu().numpy()
        res[mode] = (lg, queue_values(gen), gen.step_index)
    assert res["gemm"][2] == res["steps"][2] == 64
    assert np.max(np.abs(res["gemm"][0] - res["steps"][0])) <= tol
    assert np.max(np.abs(res["gemm"][1] - res["steps"][1])) <= 2e-2


def test_fast_generate_long_primer_uses_prefill(cuda, models):
    """cell_fast_generate with a long primer (time-parallel primer phase) against the
    stepped primer phase: the generated continuation's teacher-forced logits on the GPU's
    own samples agree within tolerance, and the samples agree except near-ties."""
    from paper_1611_09482_b200 import cell_fast_generate

    cfg, B, tol = CASES["simt"]
    primer = teacher(200, 1, 8)[:, 0]
    a = cell_fast_generate(models["simt"], primer, 50, kernel="simt")
    b = cell_fast_generate(models["simt"], primer, 50, kernel="simt", prefill_primer=False)
    assert a.shape == b.shape == (1, 50)
    assert np.mean(a == b) >= 0.9
    # the first sample follows the primer alone: identical unless a tie within 1e-4
    o = oc.CellOracle(models["simt"])
    lg = o.forward_full(primer)[-1]
    top = np.sort(lg)[-2:]
    if top[1] - top[0] > 1e-3:
        assert a[0, 0] == b[0, 0] == int(np.argmax(lg))


# ---- naive (cache-free) generation on the GPU -----------------------

def test_naive_logits_match_oracle_demand_plan(cuda, models):
    """Each naive step's logits against the oracle's demand-driven naive_logits (the
    reference's naive.py plan), inside and beyond the receptive field."""
    from paper_1611_09482_b200 import NaiveCellGenerator

    model = models["simt"]
    rf = model.config.receptive_field()
    hist = teacher(rf + 40, 1, 31)
    g = NaiveCellGenerator(model, 1, kernel="simt")
    o = oc.CellOracle(model)
    h = torch.as_tensor(hist, device="cuda")
    for n in (1, 2, 17, rf - 1, rf, rf + 1, rf + 40):
        lg = g.logits(h[:n]).cpu().numpy()[0]
        ref = o.naive_logits(hist[:n, 0])
        assert np.max(np.abs(lg - ref)) <= 1e-4, n


def test_naive_generation_equals_fast(cuda, models):
    """Greedy generation: naive (recompute per step) and fast (queues) agree."""
    from paper_1611_09482_b200 import cell_fast_generate, cell_naive_generate

    model = models["simt"]
    primer = [5, 17, 128]
    a = cell_naive_generate(model, primer, 60, kernel="simt")
    b = cell_fast_generate(model, primer, 60, kernel="simt")
    assert a.shape == b.shape == (1, 60)
    assert np.array_equal(a, b)


def test_prefill_then_staged_kernel_continues(cuda, models):
    """21 streams run on the weight-staged SIMT kernel: queues filled by the prefill (same fp32
    slot layout) and continued by the kernel give the logits of an all-stepped run and the
    oracle's teacher-forced forward."""
    B = 21
    x = teacher(140, B, 9)
    _, ref = stepped(models["simt"], "simt", B, x)
    gen = CellGenerator(models["simt"], B, kernel="simt")
    gen.prefill(torch.as_tensor(x[:100], device="cuda"))
    _, lg = gen.generate(torch.as_tensor(x[100:], device="cuda"), 40, Sampler(0), n_logit_steps=40)
    torch.cuda.synchronize()
    assert np.max(np.abs(lg.cpu().numpy() - ref[100:])) <= 1e-4
    o = oc.CellOracle(models["simt"])
    for b in (0, 20):
        assert np.max(np.abs(ref[:, b] - o.forward_full(x[:, b]))) <= 1e-4


@pytest.mark.parametrize("cfg", [CellConfig(1, 4, 4, 3, 5, classes=7, bias="fan_in", init_seed=3),
                                 CellConfig(1, 5, 10, 6, 12, classes=11, dilation_base=3,
                                            bias="fan_in", init_seed=9),
                                 CellConfig(2, 2, 20, 20, 40, classes=300, bias="fan_in",
                                            init_seed=1)])
def test_prefill_odd_shapes(cuda, cfg):
    """Channel counts that are not multiples of 8 (or 4) and classes != 256: the prefill
    kernels move one channel per thread and the GEMM predicates its edges, so the result
    matches stepping and the oracle exactly as for aligned shapes."""
    m = build_cell_model(cfg)
    B, T = 5, 70
    x = np.random.default_rng(2).integers(0, cfg.classes, (T, B)).astype(np.int32)
    ref_gen, ref = stepped(m, "simt", B, x)
    gen = CellGenerator(m, B, kernel="simt")
    lg = gen.prefill(torch.as_tensor(x, device="cuda"), want_logits=True).cpu().numpy()
    assert np.max(np.abs(lg - ref)) <= 1e-4
    assert np.max(np.abs(queue_values(gen) - queue_values(ref_gen))) <= 1e-4
    o = oc.CellOracle(m)
    for b in (0, B - 1):
        assert np.max(np.abs(lg[:, b] - o.forward_full(x[:, b]))) <= 1e-4


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_select_matches_oracle_rules(cuda, models, mode):
    """fw_cell_select (the selection stage alone) against oracle/cell.py's rules on random
    logits: identical classes except near-ties (margin below 1e-5)."""
    gen = CellGenerator(models["simt"], 3, kernel="simt")
    lg = np.random.default_rng(mode).normal(0, 3, (20, 3, 256)).astype(np.float32)
    got = gen.select(torch.as_tensor(lg, device="cuda"), 40, Sampler(mode, 17, 5)).cpu().numpy()
    for i in range(20):
        want = oc.select(mode, lg[i].astype(np.float64), 17, np.arange(3) + 5, 40 + i)
        for b in range(3):
            if want[b] != got[i, b]:
                m = oc.selection_margin(mode, lg[i, b:b + 1].astype(np.float64), 17,
                                        np.array([b + 5]), 40 + i, want[b:b + 1], got[i, b:b + 1])
                assert m[0] <= 1e-5, (i, b, got[i, b], want[b])


def test_out_of_range_classes_are_rejected(cuda, models):
    gen = CellGenerator(models["simt"], 3, kernel="simt")
    bad = torch.tensor([[1, 256, 3]], dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError):
        gen.generate(bad, 2)
    with pytest.raises(ValueError):
        gen.step(torch.tensor([0, -1, 2], dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):
        gen.prefill(bad)
    with pytest.raises(ValueError):
        gen.generate_host(np.array([[0, 1, 999]], dtype=np.int32), 2)
    assert gen.step_index == 0
    # the C ABI's host entry point checks the host buffer itself
    import ctypes as C
    from paper_1611_09482_b200 import _lib

    h_in = np.array([[0, 1, 300]], dtype=np.int32)
    h_out = np.empty((2, 3), dtype=np.int32)
    s = Sampler(0).c()
    rc = gen._lib.fw_cell_generate_host(gen._h, C.c_void_p(h_in.ctypes.data), 1, 2,
                                        C.c_void_p(h_out.ctypes.data), C.byref(s), None)
    assert rc == _lib.FW_ERR_INVALID
