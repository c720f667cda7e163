"""Long-horizon GPU parity: every BASELINE config run past the wrap of its largest ring.

A ring of dilation d is read back as its initial zeros for the first d steps; only after
that do the pops return values the kernel pushed. These tests run each benched kernel for
more steps than its largest dilation, so a wrong per-layer ring offset, slot stride or wrap
in any layer changes the logits (the reference exercises the same thing with a marker
cycling through a dilation-sized queue, pkg/tests/test_fast.py:53, and 10,000-step queue
invariants, pkg/tests/test_acceptance.py:139-155).

* cfg4 on the tcgen05 kernel (d_max 512): all 4,096 streams, 600 teacher-forced steps;
  logits of 8 streams spread over tile pairs checked against the fp64 oracle; every
  stream's logits checked against the fp32 SIMT kernel (which shares no code with it).
* cfg4's benched configuration: free-running Gumbel sampling with no logits output (the
  folded pair tail, head2 accumulating onto bias + noise), every choice of 8 streams
  margin-checked against the oracle on the GPU's own history.
* cfg5 (d_max 2,048): BASELINE's own check -- 1,024 streams teacher-forced on the seeded
  random walk, logits compared on 2,100 steps (past the 2,048 wrap), on the warp-MMA kernel
  and on the weight-staged SIMT kernel.
* cfg3 (d_max 512): 600 Gumbel steps, 64 streams; cfg2: the full 1,000 steps at every L.

Tolerances are the north-star's: logits 1e-4 (fp32 configs) / 2e-2 (bf16 config) max-abs;
choices identical except near-ties below the tolerance (logged).
"""

import numpy as np
import pytest
import torch

from oracle import cell as oc
from paper_1611_09482_b200 import CellGenerator, Sampler, build_cell_model, configs

from cellcheck import check_streams

pytestmark = pytest.mark.gpu

CFG4_STREAMS = [0, 63, 64, 127, 128, 2047, 2113, 4095]  # both tiles of several pairs


def _teacher_walk(n, batch, seed=configs.WALK_SEED):
    rng = np.random.default_rng(seed)
    steps = rng.choice(np.array([-1, 1]), size=(n, batch))
    return np.clip(128 + np.cumsum(steps, axis=0), 0, 255)


def _run(gen, inputs, n_steps, sampler, n_logit, streams):
    """Generate on the GPU; return all choices and the logits of ``streams`` only."""
    out, lg = gen.generate(torch.as_tensor(inputs, dtype=torch.int32, device="cuda"), n_steps,
                           sampler, n_logit_steps=n_logit)
    torch.cuda.synchronize()
    sel = lg[:, streams].cpu().numpy() if lg is not None else None
    return out.cpu().numpy(), sel, lg


@pytest.fixture(scope="module")
def cfg4_model():
    return build_cell_model(configs.cfg4().cell)


def test_cfg4_tcgen05_teacher_forced_past_ring_wrap(cuda, cfg4_model):
    spec = configs.cfg4()
    n = 600  # > d_max = 512: every ring has wrapped
    cls = np.random.default_rng(31).integers(0, 256, (n, spec.batch)).astype(np.int32)
    gen = CellGenerator(cfg4_model, spec.batch, kernel="tcgen05")
    out, lg, lg_all = _run(gen, cls, n, Sampler(0), n, CFG4_STREAMS)
    gen.close()
    report = []
    check_streams(oc.CellOracle(cfg4_model, exact=False), cls[:, CFG4_STREAMS],
                  out[:, CFG4_STREAMS], lg, range(len(CFG4_STREAMS)), 0, 0, 2e-2, 4e-2,
                  report=report, gids=CFG4_STREAMS)
    worst = report[-1][1]
    assert worst <= 2e-2, report
    # every stream, every step: the fp32 SIMT kernel on the same inputs
    sim = CellGenerator(cfg4_model, spec.batch, kernel="simt")
    _, _, lg_simt = _run(sim, cls, n, Sampler(0), n, CFG4_STREAMS)
    sim.close()
    dev = torch.zeros((), device="cuda")
    for t0 in range(0, n, 50):  # chunked: the difference of 2 x 2.5 GB tensors
        dev = torch.maximum(dev, (lg_all[t0:t0 + 50] - lg_simt[t0:t0 + 50]).abs().max())
    assert float(dev) <= 2e-2, float(dev)


def test_cfg4_tcgen05_gumbel_free_run_folded_tail(cuda, cfg4_model):
    """The benched configuration: Gumbel sampling, no logits output -> the pair tail folds
    head2 onto the bias + noise columns and selects from finished scores."""
    spec = configs.cfg4()
    n = 600
    gen = CellGenerator(cfg4_model, spec.batch, kernel="tcgen05")
    primer = np.full((1, spec.batch), spec.primer_class)
    out, _, _ = _run(gen, primer, n, Sampler(configs.SAMPLE_GUMBEL, configs.NOISE_SEED), 0,
                     CFG4_STREAMS)
    gen.close()
    report = []
    ties = check_streams(oc.CellOracle(cfg4_model, exact=False), primer[:, CFG4_STREAMS],
                         out[:, CFG4_STREAMS], None, range(len(CFG4_STREAMS)),
                         configs.SAMPLE_GUMBEL, configs.NOISE_SEED, 2e-2, 4e-2, report=report,
                         gids=CFG4_STREAMS)
    assert ties <= 8, report
    # the run really is a free run (the model is not stuck on one class)
    assert len(np.unique(out[:, CFG4_STREAMS])) > 20


@pytest.mark.parametrize("hmma", ["1", "0"])
def test_cfg5_baseline_check_2100_steps(cuda, monkeypatch, hmma):
    """BASELINE cfg5: 1,024 streams teacher-forced on the random walk, logits compared with
    the CPU path on the first steps -- here 2,100 (> d_max = 2,048); on the warp-MMA kernel
    (the default) and on the weight-staged SIMT kernel."""
    monkeypatch.setenv("FW_SIMT_HMMA", hmma)
    spec = configs.cfg5()
    m = build_cell_model(spec.cell)
    n = 2100
    walk = _teacher_walk(n, spec.batch)
    streams = [0, 6, 7, 511, 1023]  # CTA boundaries of the staged kernel (7 streams per CTA)
    gen = CellGenerator(m, spec.batch)
    out, lg, _ = _run(gen, walk, n, Sampler(0), n, streams)
    gen.close()
    report = []
    check_streams(oc.CellOracle(m, exact=False), walk[:, streams], out[:, streams], lg,
                  range(len(streams)), 0, 0, 1e-4, 2e-4, report=report, gids=streams)
    assert report[-1][1] <= 1e-4, report


def test_cfg3_gumbel_600_steps(cuda):
    spec = configs.cfg3()
    m = build_cell_model(spec.cell)
    n = 600
    gen = CellGenerator(m, spec.batch)
    primer = np.full((1, spec.batch), spec.primer_class)
    streams = [0, 17, 31, 63]
    out, lg, _ = _run(gen, primer, n, Sampler(configs.SAMPLE_GUMBEL, configs.NOISE_SEED), n,
                      streams)
    gen.close()
    report = []
    ties = check_streams(oc.CellOracle(m, exact=False), primer[:, streams], out[:, streams], lg,
                         range(len(streams)), configs.SAMPLE_GUMBEL, configs.NOISE_SEED, 1e-4,
                         2e-4, report=report, gids=streams)
    assert ties <= 2, report


@pytest.mark.parametrize("L", configs.CFG2_LAYERS)
def test_cfg2_full_1000_steps(cuda, L):
    spec = configs.cfg2(L)
    m = build_cell_model(spec.cell)
    gen = CellGenerator(m, 1)
    s = Sampler(configs.SAMPLE_INVCDF, configs.NOISE_SEED)
    out, lg, _ = _run(gen, np.array([[128]]), spec.steps, s, spec.steps, [0])
    gen.close()
    report = []
    ties = check_streams(oc.CellOracle(m, exact=False), np.array([[128]]), out, lg, [0],
                         configs.SAMPLE_INVCDF, configs.NOISE_SEED, 1e-4, 1e-5, report=report)
    assert ties <= 2, report


@pytest.mark.parametrize("B", [512, 1152])
def test_cfg4_split_chain_matches_unsplit_and_oracle(cuda, cfg4_model, monkeypatch, B):
    """Batches whose tiles fit twice on the SMs run each 64-stream tile over a 2-CTA cluster
    (one dilated N-half per CTA, z halves exchanged through DSMEM, the residual accumulated
    in both). 600 teacher-forced steps (past the d = 512 ring wrap): every stream's logits
    against the unsplit kernel, a few against the oracle, and the folded-tail Gumbel free
    run choice by choice."""
    n = 600
    cls = np.random.default_rng(B).integers(0, 256, (n, B)).astype(np.int32)
    gen = CellGenerator(cfg4_model, B, kernel="tcgen05")
    streams = [0, 63, 64, 200, B - 1]
    out, lg, lg_split = _run(gen, cls, n, Sampler(0), n, streams)
    gen.close()
    report = []
    check_streams(oc.CellOracle(cfg4_model, exact=False), cls[:, streams], out[:, streams], lg,
                  range(len(streams)), 0, 0, 2e-2, 4e-2, report=report, gids=streams)
    monkeypatch.setenv("FW_CHAIN_SPLIT", "0")
    ref = CellGenerator(cfg4_model, B, kernel="tcgen05")
    _, _, lg_ref = _run(ref, cls, n, Sampler(0), n, streams)
    ref.close()
    dev = max(float((lg_split[t:t + 100] - lg_ref[t:t + 100]).abs().max()) for t in range(0, n, 100))
    assert dev <= 2e-2, dev
    monkeypatch.delenv("FW_CHAIN_SPLIT")
    gen = CellGenerator(cfg4_model, B, kernel="tcgen05")
    primer = np.full((1, B), 128)
    free, _, _ = _run(gen, primer, 300, Sampler(configs.SAMPLE_GUMBEL, configs.NOISE_SEED), 0, streams)
    gen.close()
    check_streams(oc.CellOracle(cfg4_model, exact=False), primer[:, streams], free[:, streams], None,
                  range(len(streams)), configs.SAMPLE_GUMBEL, configs.NOISE_SEED, 2e-2, 4e-2,
                  gids=streams)


@pytest.mark.parametrize("B,split", [(2048, "1"), (2048, "0"), (4096, "1")])
def test_tcgen05_repeated_runs_are_bit_identical(cuda, cfg4_model, monkeypatch, B, split):
    """Race detector: the persistent step kernel's warps, tiles and tail blocks hand data to
    each other through mbarriers, DSMEM and global counters; a missing ordering edge shows up
    as an occasional step whose logits differ between identical runs (this found the z-stash
    publication and the pair tail's image reuse). Four identical 600-step teacher-forced
    runs must agree bit for bit."""
    monkeypatch.setenv("FW_CHAIN_SPLIT", split)
    n = 600
    cls = torch.as_tensor(np.random.default_rng(B + 7).integers(0, 256, (n, B)), dtype=torch.int32,
                          device="cuda")
    ref = None
    for _ in range(4):
        gen = CellGenerator(cfg4_model, B, kernel="tcgen05")
        _, lg = gen.generate(cls, n, Sampler(0), n_logit_steps=n)
        torch.cuda.synchronize()
        gen.close()
        if ref is None:
            ref = lg
            continue
        bad = torch.nonzero((lg - ref).abs().amax(dim=2) > 0)
        assert bad.shape[0] == 0, bad[:8].tolist()
        del lg


@pytest.mark.parametrize("config,batch,cluster,hmma", [("cfg1", 1, "", "1"), ("cfg2_L8", 2, "16", "1"),
                                                       ("cfg3", 64, "", "1"), ("cfg5", 1024, "", "1"),
                                                       ("cfg5", 1024, "", "0")])
def test_simt_repeated_runs_are_bit_identical(cuda, monkeypatch, config, batch, cluster, hmma):
    """Race detector for the fp32 kernels (the small-batch cluster kernel's st.async
    exchanges and weight ring, the warp-MMA and staged kernels' producer/consumer rings):
    three identical teacher-forced runs, past the largest ring wrap where affordable, agree
    bit for bit."""
    if cluster:
        monkeypatch.setenv("FW_SIMT_CLUSTER", cluster)
    monkeypatch.setenv("FW_SIMT_HMMA", hmma)
    spec = configs.by_name(config)
    m = build_cell_model(spec.cell)
    n = 300 if config == "cfg5" else 600
    cls = torch.as_tensor(np.random.default_rng(3).integers(0, 256, (n, batch)), dtype=torch.int32,
                          device="cuda")
    ref = None
    for _ in range(3):
        gen = CellGenerator(m, batch, kernel="simt")
        _, lg = gen.generate(cls, n, Sampler(0), n_logit_steps=n)
        torch.cuda.synchronize()
        gen.close()
        if ref is None:
            ref = lg
            continue
        bad = torch.nonzero((lg - ref).abs().amax(dim=2) > 0)
        assert bad.shape[0] == 0, bad[:8].tolist()


@pytest.mark.parametrize("variant,env,val", [("2sm", "FW_CHAIN_2SM", "1"), ("fold", "FW_CHAIN_FOLD", "1"),
                                             ("2sm-fold", "FW_CHAIN_2SM", "2")])
def test_opt_in_tcgen05_chains(cuda, cfg4_model, monkeypatch, variant, env, val):
    """The opt-in chain variants on all 4,096 cfg4 streams, 120 teacher-forced steps: the
    2-SM chain (cta_group::2 MMAs, chain_2sm.cuh) does the same arithmetic as the default
    chain, so its logits are bit-identical; the folded chain (chain_fold.cuh) rounds the
    folded weights once more and stays within the bf16 tolerance of the default and the
    oracle, as does the folded 2-SM chain. Each twice, bit for bit (race check)."""
    B, n = configs.cfg4().batch, 120
    cls = np.random.default_rng(11).integers(0, 256, (n, B)).astype(np.int32)
    ref = CellGenerator(cfg4_model, B, kernel="tcgen05")
    _, lg_ref, lg_ref_all = _run(ref, cls, n, Sampler(0), n, CFG4_STREAMS)
    ref.close()
    monkeypatch.setenv(env, val)
    runs = []
    for _ in range(2):
        gen = CellGenerator(cfg4_model, B, kernel="tcgen05")
        out, lg, lg_all = _run(gen, cls, n, Sampler(0), n, CFG4_STREAMS)
        gen.close()
        runs.append(lg_all)
    assert torch.equal(runs[0], runs[1])
    if variant == "2sm":
        assert torch.equal(runs[0], lg_ref_all)
    else:
        dev = max(float((runs[0][t:t + 40] - lg_ref_all[t:t + 40]).abs().max()) for t in range(0, n, 40))
        assert dev <= 2e-2, dev
        report = []
        check_streams(oc.CellOracle(cfg4_model, exact=False), cls[:, CFG4_STREAMS], out[:, CFG4_STREAMS],
                      lg, range(len(CFG4_STREAMS)), 0, 0, 2e-2, 4e-2, report=report, gids=CFG4_STREAMS)

