"""GPU gated-cell parity against the CPU oracle on all five BASELINE configs.

Tolerances are the north-star's (BASELINE.json): teacher-forced logits within
1e-4 max-abs for fp32 configs and 2e-2 for the bf16 config; selected indices
identical except logged near-ties (margin below the tolerance), checked by
re-running the oracle teacher-forced on the GPU's own history. Large configs
run at full batch on the GPU; the oracle checks a subset of streams (they are
independent) over a shortened horizon, and size-independent properties
(determinism, sharding invariance, step == generate) cover the rest.
"""

import numpy as np
import pytest
import torch

from oracle import cell as oc
from paper_1611_09482_b200 import CellGenerator, Sampler, build_cell_model, cell_fast_generate
from paper_1611_09482_b200 import configs
from paper_1611_09482_b200.cell import CellConfig

from cellcheck import check_streams

pytestmark = pytest.mark.gpu

TOL = {"f32": (1e-4, 2e-4), "bf16": (2e-2, 4e-2)}


def run(gen, inputs, n_steps, sampler, n_logit):
    out, lg = gen.generate(torch.as_tensor(inputs, dtype=torch.int32, device="cuda"), n_steps,
                           sampler, n_logit_steps=n_logit)
    torch.cuda.synchronize()
    return out.cpu().numpy(), (lg.cpu().numpy() if lg is not None else None)


def kernels_for(cfg, batch):
    ks = ["simt"]
    if cfg.weight_dtype == "bf16" and batch >= 128:
        ks.append("tcgen05")
    return ks


@pytest.fixture(scope="module")
def cfg1_model():
    return build_cell_model(configs.cfg1().cell)


def test_cfg1_teacher_forced_logits(cuda, cfg1_model):
    spec = configs.cfg1()
    cls = np.random.default_rng(configs.TEACHER_SEED).integers(0, 256, spec.steps)
    gen = CellGenerator(cfg1_model, 1, kernel="simt")
    out, lg = run(gen, cls.reshape(-1, 1), spec.steps, Sampler(0), spec.steps)
    ref = oc.CellOracle(cfg1_model).forward_full(cls)
    dev = np.max(np.abs(lg[:, 0] - ref))
    assert dev <= 1e-4, dev
    assert np.array_equal(out[:, 0], np.argmax(lg[:, 0], axis=1))


def test_cfg1_greedy_free_run(cuda, cfg1_model):
    spec = configs.cfg1()
    gen = CellGenerator(cfg1_model, 1, kernel="simt")
    out, lg = run(gen, np.array([[spec.primer_class]]), spec.steps, Sampler(0), spec.steps)
    report = []
    ties = check_streams(oc.CellOracle(cfg1_model), np.array([[128]]), out, lg, [0], 0, 0,
                         1e-4, 2e-4, report=report)
    assert ties <= 2, report


def test_cfg1_drop_in_fast_generate_matches_device_loop(cuda, cfg1_model):
    seq = cell_fast_generate(cfg1_model, [128], 300)
    gen = CellGenerator(cfg1_model, 1)
    out, _ = run(gen, np.array([[128]]), 300, Sampler(0), 0)
    assert np.array_equal(seq[0], out[:, 0])
    primer = [5, 17, 128]
    seq2 = cell_fast_generate(cfg1_model, primer, 50)
    gen2 = CellGenerator(cfg1_model, 1)
    out2, _ = run(gen2, np.array(primer).reshape(-1, 1), len(primer) - 1 + 50, Sampler(0), 0)
    assert np.array_equal(seq2[0], out2[len(primer) - 1:, 0])


@pytest.mark.parametrize("L", configs.CFG2_LAYERS)
def test_cfg2_depth_sweep_invcdf(cuda, L):
    spec = configs.cfg2(L)
    m = build_cell_model(spec.cell)
    n = 200
    gen = CellGenerator(m, 1)
    s = Sampler(configs.SAMPLE_INVCDF, configs.NOISE_SEED)
    out, lg = run(gen, np.array([[128]]), n, s, n)
    ties = check_streams(oc.CellOracle(m, exact=False), np.array([[128]]), out, lg, [0],
                         configs.SAMPLE_INVCDF, configs.NOISE_SEED, 1e-4, 1e-5)
    assert ties <= 2


def test_cfg3_wavenet_gumbel(cuda):
    spec = configs.cfg3()
    m = build_cell_model(spec.cell)
    n = 96
    gen = CellGenerator(m, spec.batch)
    s = Sampler(configs.SAMPLE_GUMBEL, configs.NOISE_SEED)
    primer = np.full((1, spec.batch), 128)
    out, lg = run(gen, primer, n, s, n)
    ties = check_streams(oc.CellOracle(m, exact=False), primer, out, lg, [0, 17, 63],
                         configs.SAMPLE_GUMBEL, configs.NOISE_SEED, 1e-4, 2e-4)
    assert ties <= 2


@pytest.mark.parametrize("kernel", ["simt", "tcgen05"])
def test_cfg4_large_batch_bf16(cuda, kernel):
    spec = configs.cfg4()
    m = build_cell_model(spec.cell)
    if kernel == "tcgen05":
        try:
            gen = CellGenerator(m, spec.batch, kernel="tcgen05")
        except ValueError as e:
            pytest.skip(f"tcgen05 path unavailable: {e}")
    else:
        gen = CellGenerator(m, spec.batch, kernel="simt")
    n = 24
    s = Sampler(configs.SAMPLE_GUMBEL, configs.NOISE_SEED)
    primer = np.full((1, spec.batch), 128)
    out, lg = run(gen, primer, n, s, n)
    ties = check_streams(oc.CellOracle(m, exact=False), primer, out, lg, [0, 1, 1000, 4095],
                         configs.SAMPLE_GUMBEL, configs.NOISE_SEED, 2e-2, 4e-2)
    assert ties <= 4


@pytest.mark.parametrize("sampler", [0, 1, 2])
def test_tcgen05_biases_shapes_and_samplers(cuda, sampler):
    """Non-zero biases, S != H, 3 layers, every selection rule through the tcgen05 path."""
    cfg = CellConfig(1, 3, 128, 128, 256, head_channels=384, weight_dtype="bf16",
                     bias="fan_in", init_seed=7)
    m = build_cell_model(cfg)
    B, n = 256, 40
    gen = CellGenerator(m, B, kernel="tcgen05")
    assert gen.kernel == "tcgen05"
    primer = np.random.default_rng(3).integers(0, 256, (3, B))
    out, lg = run(gen, primer, n, Sampler(sampler, 9), n)
    ties = check_streams(oc.CellOracle(m, exact=False), primer, out, lg, [0, 77, 255], sampler, 9,
                         2e-2, 4e-2 if sampler != 1 else 2e-2)
    assert ties <= 3
    # the SIMT kernel on the same model agrees with the oracle as well (fp32 math)
    gen2 = CellGenerator(m, B, kernel="simt")
    out2, lg2 = run(gen2, primer, n, Sampler(sampler, 9), n)
    check_streams(oc.CellOracle(m, exact=False), primer, out2, lg2, [0, 255], sampler, 9,
                  1e-4, 2e-4 if sampler != 1 else 1e-5)


def test_tcgen05_matches_simt_all_streams_many_steps(cuda):
    """Race detector: every stream of cfg4, 32 teacher-forced steps, tcgen05 vs the fp32 SIMT
    kernel. The chain kernel overlaps TMA, tensor-core and epilogue work with mbarriers; a
    missing ordering edge shows up as a whole tile (or a few rows) drifting after a few
    steps, which the 4-stream oracle checks above can miss."""
    spec = configs.cfg4()
    m = build_cell_model(spec.cell)
    n = 32
    cls = np.random.default_rng(11).integers(0, 256, (n, spec.batch)).astype(np.int32)
    lg = {}
    for k in ("tcgen05", "simt"):
        g = CellGenerator(m, spec.batch, kernel=k)
        _, l = run(g, cls, n, Sampler(0), n)
        lg[k] = l
        g.close()
    dev = np.abs(lg["tcgen05"] - lg["simt"]).max(axis=2)
    assert dev.max() <= 2e-2, (dev.max(), np.argwhere(dev > 2e-2)[:8].tolist())


def test_cfg5_deep_teacher_forced_walk(cuda):
    spec = configs.cfg5()
    m = build_cell_model(spec.cell)
    n = 160  # first steps of the 48k-step run; BASELINE's 2,000-step check (run to 2,100 steps,
    # past the 2,048 ring wrap) is tests/test_gpu_long.py::test_cfg5_baseline_check_2100_steps
    walk = teacher_walk(n, spec.batch)
    gen = CellGenerator(m, spec.batch)
    out, lg = run(gen, walk, n, Sampler(0), n)
    ref_o = oc.CellOracle(m, exact=False)
    for s in (0, 511, 1023):
        ref = ref_o.forward_full(walk[:, s])
        dev = np.max(np.abs(lg[:, s] - ref))
        assert dev <= 1e-4, (s, dev)


def teacher_walk(n, batch, seed=configs.WALK_SEED):
    rng = np.random.default_rng(seed)
    steps = rng.choice(np.array([-1, 1]), size=(n, batch))
    return np.clip(128 + np.cumsum(steps, axis=0), 0, 255)


def test_step_equals_generate_and_reset(cuda):
    cfg = CellConfig(2, 3, 16, 16, 32, classes=32, bias="fan_in", init_seed=5)
    m = build_cell_model(cfg)
    B, n = 7, 40
    s = Sampler(configs.SAMPLE_GUMBEL, 11)
    gen = CellGenerator(m, B)
    out, lg = run(gen, np.full((1, B), 3), n, s, n)
    gen2 = CellGenerator(m, B)
    x = torch.full((B,), 3, dtype=torch.int32, device="cuda")
    for i in range(n):
        y, l2 = gen2.step(x, s, want_logits=True)
        assert np.array_equal(y.cpu().numpy(), out[i])
        assert np.array_equal(l2.cpu().numpy(), lg[i])
        x = y
    assert gen2.step_index == n
    gen2.reset()
    assert gen2.step_index == 0
    out3, _ = run(gen2, np.full((1, B), 3), n, s, 0)
    assert np.array_equal(out3, out)


def test_sharding_invariance(cuda):
    """Streams keyed by global id give identical sequences however the batch is split."""
    cfg = CellConfig(1, 4, 8, 8, 16, classes=16, init_seed=2)
    m = build_cell_model(cfg)
    B, n = 8, 30
    s = Sampler(configs.SAMPLE_GUMBEL, 5)
    primer = np.arange(B).reshape(1, B) % 16
    full, _ = run(CellGenerator(m, B), primer, n, s, 0)
    lo, _ = run(CellGenerator(m, 4), primer[:, :4], n, Sampler(2, 5, 0), 0)
    hi, _ = run(CellGenerator(m, 4), primer[:, 4:], n, Sampler(2, 5, 4), 0)
    assert np.array_equal(full, np.concatenate([lo, hi], axis=1))


def test_small_odd_shapes_with_biases(cuda):
    for cfg in (CellConfig(1, 4, 4, 3, 5, classes=7, bias="fan_in", init_seed=3),
                CellConfig(1, 5, 6, 4, 8, classes=11, dilation_base=3, bias="fan_in", init_seed=9),
                CellConfig(2, 2, 300, 20, 40, classes=300, bias="fan_in", init_seed=1)):
        m = build_cell_model(cfg)
        B, n = 3, 60
        primer = np.random.default_rng(0).integers(0, cfg.classes, (4, B))
        out, lg = run(CellGenerator(m, B), primer, n, Sampler(1, 3), n)
        check_streams(oc.CellOracle(m), primer, out, lg, range(B), 1, 3, 1e-4, 1e-5)


def test_invalid_arguments(cuda, cfg1_model):
    with pytest.raises(ValueError):
        CellGenerator(cfg1_model, 0)
    gen = CellGenerator(cfg1_model, 2)
    with pytest.raises(ValueError):
        gen.generate(torch.zeros((1, 3), dtype=torch.int32, device="cuda"), 4)
    with pytest.raises(ValueError):
        cell_fast_generate(cfg1_model, [300], 4)
    assert cell_fast_generate(cfg1_model, [1], 0).shape == (1, 0)


@pytest.mark.parametrize("cluster", ["0", "2", "4", "8", "16"])
def test_small_batch_cluster_kernel_matches_oracle(cuda, cfg1_model, monkeypatch, cluster):
    """The cluster-per-stream SIMT kernel (FW_SIMT_CLUSTER) and the per-CTA kernel give the
    oracle's teacher-forced logits on the same inputs, for 1 and 3 streams."""
    monkeypatch.setenv("FW_SIMT_CLUSTER", cluster)
    for B in (1, 3):
        cls = np.random.default_rng(40 + B).integers(0, 256, (60, B))
        gen = CellGenerator(cfg1_model, B, kernel="simt")
        out, lg = run(gen, cls, 60, Sampler(0), 60)
        o = oc.CellOracle(cfg1_model)
        for b in range(B):
            ref = o.forward_full(cls[:, b])
            assert np.max(np.abs(lg[:, b] - ref)) <= 1e-4, (cluster, B, b)
            assert np.array_equal(out[:, b], np.argmax(lg[:, b], axis=1))


def test_tcgen05_needs_three_layers_and_short_stacks_fall_back(cuda):
    """bf16 stacks of 1-2 layers are outside the tcgen05 kernel (its pops are staged two
    layers ahead); auto selection serves them with the SIMT kernel, at parity."""
    for L in (1, 2):
        m = build_cell_model(CellConfig(1, L, 128, 128, 256, weight_dtype="bf16", bias="fan_in",
                                        init_seed=5))
        with pytest.raises(ValueError):
            CellGenerator(m, 128, kernel="tcgen05")
        gen = CellGenerator(m, 128)
        assert gen.kernel == "simt"
        cls = np.random.default_rng(L).integers(0, 256, (6, 128))
        _, lg = run(gen, cls, 6, Sampler(0), 6)
        o = oc.CellOracle(m, exact=False)
        for b in (0, 127):
            assert np.max(np.abs(lg[:, b] - o.forward_full(cls[:, b]))) <= 2e-2


TC_GRID = [(L, S, H, B) for L in (3, 5, 12) for (S, H) in ((128, 128), (256, 256), (512, 256),
                                                           (512, 512), (1024, 512))
           for B in (128, 384)]


@pytest.mark.parametrize("L,S,H,B", TC_GRID)
def test_tcgen05_shape_grid_teacher_forced(cuda, monkeypatch, L, S, H, B):
    """The tcgen05 kernel over its shape space (fused pair tail, fused global tail, per-step
    path; one and several tile pairs; several steps per launch and one), teacher-forced
    logits against the oracle within the bf16 tolerance on the first, a middle and the last
    stream."""
    m = build_cell_model(CellConfig(1, L, 128, 128, S, head_channels=H, weight_dtype="bf16",
                                    bias="fan_in", init_seed=L + S + H))
    o = oc.CellOracle(m, exact=False)
    cls = np.random.default_rng(B + L).integers(0, 256, (5, B))
    for per_launch in ("0", "2"):
        monkeypatch.setenv("FW_STEPS_PER_LAUNCH", per_launch)
        gen = CellGenerator(m, B, kernel="tcgen05")
        _, lg = run(gen, cls, 5, Sampler(0), 5)
        for b in (0, B // 2 + 1, B - 1):
            dev = np.max(np.abs(lg[:, b] - o.forward_full(cls[:, b])))
            assert dev <= 2e-2, (per_launch, b, dev)
        gen.close()


@pytest.mark.parametrize("B", [200, 129])
def test_tcgen05_padded_batch(cuda, B):
    """Batches that are not a multiple of 128 run on the tcgen05 kernel padded to the next
    multiple (extra streams fed class 0, discarded): teacher-forced logits at parity, the
    host-buffer entry point and the full-sequence forward agree with the device loop."""
    m = build_cell_model(CellConfig(1, 4, 128, 128, 256, weight_dtype="bf16", bias="fan_in",
                                    init_seed=9))
    gen = CellGenerator(m, B)
    assert gen.kernel == "tcgen05"
    cls = np.random.default_rng(B).integers(0, 256, (6, B))
    out, lg = run(gen, cls, 6, Sampler(2, 5), 6)
    o = oc.CellOracle(m, exact=False)
    for b in (0, B // 2, B - 1):
        assert np.max(np.abs(lg[:, b] - o.forward_full(cls[:, b]))) <= 2e-2
    gen.reset()
    host = gen.generate_host(cls.astype(np.int32), 6, Sampler(2, 5))
    assert np.array_equal(host, out)
    gen.reset()
    pf = gen.prefill(torch.as_tensor(cls, dtype=torch.int32, device="cuda"), want_logits=True)
    assert pf.shape == (6, B, 256)
    assert np.max(np.abs(pf.cpu().numpy() - lg)) <= 2e-2
    assert gen.step_index == 6


@pytest.mark.parametrize("bt", ["1", "2", "4", "7", "8"])
def test_staged_simt_kernel_matches_oracle_and_ldg_kernel(cuda, monkeypatch, bt):
    """The weight-staged fp32 kernel (bulk-copied weight ring, FW_SIMT_BT streams per CTA, the
    last CTA partly filled) gives the oracle's teacher-forced logits, including shapes whose
    GEMVs span several stages (R = 128, S = H = 512) and non-zero biases, and continues a
    free run with the __ldg kernel's classes."""
    monkeypatch.setenv("FW_SIMT_BT", bt)
    monkeypatch.setenv("FW_SIMT_CLUSTER", "0")  # (these batches would take the cluster kernel,
    monkeypatch.setenv("FW_SIMT_HMMA", "0")     # and the R = D = 64 shape the warp-MMA one)
    for cfg, B in ((CellConfig(2, 3, 64, 64, 256, bias="fan_in", init_seed=4), 37),
                   (CellConfig(1, 4, 128, 128, 512, bias="fan_in", init_seed=6), 19)):
        m = build_cell_model(cfg)
        n = 24
        cls = np.random.default_rng(7).integers(0, 256, (n, B))
        monkeypatch.setenv("FW_SIMT_STAGED", "1")
        out, lg = run(CellGenerator(m, B, kernel="simt"), cls, n, Sampler(0), n)
        o = oc.CellOracle(m)
        for b in (0, B // 2, B - 1):
            ref = o.forward_full(cls[:, b])
            assert np.max(np.abs(lg[:, b] - ref)) <= 1e-4, (bt, B, b)
        primer = cls[:3]
        for mode in (configs.SAMPLE_GUMBEL, configs.SAMPLE_INVCDF):
            s = Sampler(mode, 11)
            tie = 2e-4 if mode == configs.SAMPLE_GUMBEL else 1e-5
            monkeypatch.setenv("FW_SIMT_STAGED", "1")
            got, _ = run(CellGenerator(m, B, kernel="simt"), primer, 40, s, 0)
            monkeypatch.setenv("FW_SIMT_STAGED", "0")
            monkeypatch.delenv("FW_SIMT_BT")
            want, _ = run(CellGenerator(m, B, kernel="simt"), primer, 40, s, 0)
            monkeypatch.setenv("FW_SIMT_BT", bt)
            # both free runs: every choice is the oracle's on the kernel's own history, up
            # to near-ties below the tolerance (a flipped near-tie forks the run, so the two
            # kernels' sequences are each checked, not compared with each other)
            for seq in (got, want):
                check_streams(o, primer, seq, None, [0, B // 2, B - 1], mode, 11, 1e-4, tie)


@pytest.mark.parametrize("sampler", [configs.SAMPLE_GUMBEL, configs.SAMPLE_ARGMAX])
def test_tcgen05_pair_tail_scores_folded_into_head2(cuda, sampler):
    """Pair-mode steps without logits output accumulate head2 onto the bias (+ Gumbel noise)
    in TMEM and select from those scores; steps with logits keep them separate. Both give
    the same classes (up to near-ties), and the logits run matches the oracle."""
    cfg = CellConfig(1, 4, 128, 128, 512, weight_dtype="bf16", bias="fan_in", init_seed=8)
    m = build_cell_model(cfg)
    B, n = 256, 24
    primer = np.random.default_rng(3).integers(0, 256, (2, B))
    s = Sampler(sampler, 21)
    folded, _ = run(CellGenerator(m, B, kernel="tcgen05"), primer, n, s, 0)
    plain, lg = run(CellGenerator(m, B, kernel="tcgen05"), primer, n, s, n)
    o = oc.CellOracle(m, exact=False)
    check_streams(o, primer, plain, lg, [0, 200], sampler, 21, *TOL["bf16"])
    # the folded run (no logits): every choice margin-checked on its own history
    check_streams(o, primer, folded, None, [0, 1, 127, 128, 200, 255], sampler, 21,
                  *TOL["bf16"])


@pytest.mark.parametrize("cluster", ["2", "8", "16"])
def test_small_batch_kernel_streamed_weights(cuda, monkeypatch, cluster):
    """The small-batch cluster kernel with weights streamed through its two-slot ring (cfg2's
    128-channel layers do not fit shared memory), non-zero biases (folded into the next
    layer's taps), teacher-forced logits against the oracle past the ring wraps of d <= 32."""
    monkeypatch.setenv("FW_SIMT_CLUSTER", cluster)
    cfg = CellConfig(1, 6, 128, 128, 256, bias="fan_in", init_seed=12)
    m = build_cell_model(cfg)
    B, n = 2, 80
    cls = np.random.default_rng(8).integers(0, 256, (n, B))
    out, lg = run(CellGenerator(m, B, kernel="simt"), cls, n, Sampler(0), n)
    o = oc.CellOracle(m)
    for b in range(B):
        ref = o.forward_full(cls[:, b])
        assert np.max(np.abs(lg[:, b] - ref)) <= 1e-4, (cluster, b)
        assert np.array_equal(out[:, b], np.argmax(lg[:, b], axis=1))


@pytest.mark.parametrize("B,nt", [(37, "1"), (130, "1"), (37, "2")])
def test_warp_mma_kernel_matches_oracle(cuda, monkeypatch, B, nt):
    """The fp32 configs' warp-MMA kernel (cell_hmma.cu: 3-term fp16 split products on
    mma.sync, skip of layer l - 1 interleaved with the dilated GEMM of layer l, the running
    sums in fp32): teacher-forced logits within 1e-4 of the oracle with non-zero biases, a
    partly filled last CTA (8 or 16 streams per CTA), and free runs (Gumbel, inverse CDF)
    choice by choice on the kernel's own history."""
    monkeypatch.setenv("FW_SIMT_CLUSTER", "0")
    monkeypatch.setenv("FW_HMMA_NT", nt)
    cfg = CellConfig(2, 4, 64, 64, 256, bias="fan_in", init_seed=9)
    m = build_cell_model(cfg)
    n = 40
    cls = np.random.default_rng(B).integers(0, 256, (n, B))
    out, lg = run(CellGenerator(m, B, kernel="simt"), cls, n, Sampler(0), n)
    o = oc.CellOracle(m)
    for b in (0, 7, 8, B // 2, B - 1):
        ref = o.forward_full(cls[:, b])
        assert np.max(np.abs(lg[:, b] - ref)) <= 1e-4, (B, b, np.max(np.abs(lg[:, b] - ref)))
    primer = cls[:3]
    for mode in (configs.SAMPLE_GUMBEL, configs.SAMPLE_INVCDF):
        tie = 2e-4 if mode == configs.SAMPLE_GUMBEL else 1e-5
        got, _ = run(CellGenerator(m, B, kernel="simt"), primer, 60, Sampler(mode, 13), 0)
        check_streams(o, primer, got, None, [0, 9, B - 1], mode, 13, 1e-4, tie)


def test_warp_mma_kernel_agrees_with_staged_kernel(cuda, monkeypatch):
    """cfg5's shape on 300 streams: the warp-MMA kernel and the weight-staged SIMT kernel
    (exact fp32 FMAs) give the same teacher-forced logits to 1e-4 over 100 steps."""
    spec = configs.cfg5()
    m = build_cell_model(spec.cell)
    B, n = 300, 100
    cls = np.random.default_rng(5).integers(0, 256, (n, B))
    _, lg_m = run(CellGenerator(m, B, kernel="simt"), cls, n, Sampler(0), n)
    monkeypatch.setenv("FW_SIMT_HMMA", "0")
    _, lg_s = run(CellGenerator(m, B, kernel="simt"), cls, n, Sampler(0), n)
    assert np.max(np.abs(lg_m - lg_s)) <= 1e-4

