"""GPU parity: every pt_* call through the C ABI against the CPU oracle on the
same seeded inputs.

Bar (BASELINE.json north_star): selected indices bit-exact whenever the top-two
gap in G exceeds 1e-9; scores within 1e-6 relative.  When the gap is <= 1e-9
(reading c6) any tied set is correct: the test then checks the GPU's set scores
(by the oracle) within 1e-9 of the oracle's best.
"""
import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import Oracle
from paper_2507_15277_b200 import pt, synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
# exh_kernel values a PT_EXH_TIER setting may report (the tc tier falls back to u8
# when its threshold is unusable or its filter leaves more than 2^20 survivors)
TIER_KERNELS = {"tc": (5, 4), "u8": (4,), "fp16": (0,)}

RTOL = 1e-6
GAP = 1e-9


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def check_exh(o, res, k, mask=None, want=None):
    b, gb, ru, gr = want if want is not None else o.exhaustive(k, mask=mask)
    assert res["G"] == pytest.approx(gb, rel=RTOL)
    gap = gb - gr if ru is not None else math.inf
    if gap > GAP:
        assert res["best"] == tuple(b), (res, b, gb, ru, gr)
    else:
        assert o.score(list(res["best"]), mask=mask) >= gb - GAP
    if ru is not None and res["runner"] is not None:
        assert res["G_runner"] == pytest.approx(gr, rel=RTOL)


def check_greedy(o, idx, gt, gp, k, mask=None):
    """Step by step: each GPU pick must be the oracle's pick given the GPU's prefix
    (unless that step's gap <= 1e-9)."""
    oidx, ogt, ogp = o.greedy(k, mask=mask)
    for t in range(k):
        step_idx, step_g, step_gap = o.greedy(1, mask=mask, init=idx[:t])
        if step_gap[0] > GAP:
            assert idx[t] == step_idx[0], (t, idx, oidx)
        assert gt[t] == pytest.approx(step_g[0], rel=RTOL)
        assert gt[t] == pytest.approx(o.score(idx[:t + 1], mask=mask), rel=RTOL)
    if np.all(ogp > GAP):
        assert idx == oidx


# ---------------------------------------------------------------- tiny (config 1)
@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("flags", [0, pt.PT_EXACT_FP64 | pt.PT_GREEDY_STREAM])
def test_tiny(seed, flags):
    T, dev = synth.tiny(seed)
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev, flags=flags)
    for k in (1, 2, 3, 4, 16):
        check_exh(o, pt.pt_exhaustive_best(ctx, k), k)
    idx, gt, gp = pt.pt_greedy_select(ctx, 16)
    check_greedy(o, idx, gt, gp, 16)
    assert gt[-1] == 1.0


def test_pow2_ties():
    for seed in range(1, 6):
        T, m = synth.pow2(seed, n_cfg=70, n_env=13, max_exp=3)
        o = Oracle(T)
        ctx = pt.pt_load_perf(T)
        for k in (1, 2, 3):
            check_exh(o, pt.pt_exhaustive_best(ctx, k), k)
        idx, gt, gp = pt.pt_greedy_select(ctx, 6)
        check_greedy(o, idx, gt, gp, 6)


def test_planted():
    for g in (1, 2, 3):
        for seed in range(1, 6):
            T, dev, cols = synth.planted(seed, n_cfg=200, n_env=40, g=g, gamma=2.0)
            ctx = pt.pt_load_perf(T, dev)
            r = pt.pt_exhaustive_best(ctx, g)
            assert r["best"] == tuple(cols) and r["G"] == 1.0


# ------------------------------------------------------- medium (several tiles)
@pytest.mark.parametrize("tier", ["tc", "u8", "fp16"])
@pytest.mark.parametrize("seed,C,ndev,nin", [(1, 300, 3, 16), (2, 257, 2, 19), (3, 129, 5, 7)])
def test_medium_exhaustive(seed, C, ndev, nin, tier, monkeypatch):
    """Every filter tier of the tiled search (tc default, u8 / fp16 by PT_EXH_TIER; the
    tc tier may fall back to u8 when its filter is too weak for the data)."""
    monkeypatch.setenv("PT_EXH_TIER", tier)
    T, dev = synth.small_matrix(seed, n_cfg=C, n_dev=ndev, n_inputs=nin)
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    for k in (2, 3):
        check_exh(o, pt.pt_exhaustive_best(ctx, k), k)
        st = pt.pt_get_stats(ctx)
        assert st["exh_kernel"] in TIER_KERNELS[tier] and st["exh_sets"] == math.comb(C, k)
    # sharded on one GPU (fake multi-GPU): merged shards == unsharded
    for k in (2, 3):
        want = o.exhaustive(k)
        for shards in (2, 3, 8, 50):   # 50: more shards than tasks (empty shards)
            recs_s, recs_t = [], []
            total = 0
            for r in range(shards):
                res = pt.pt_exhaustive_best(ctx, k, shard_rank=r, shard_count=shards)
                total += pt.pt_get_stats(ctx)["exh_sets"]
                for sv, tup in ((res["s"][0], res["best"]), (res["s"][1], res["runner"])):
                    recs_s.append(sv)
                    recs_t.append(tup if tup is not None else (-1,) * k)
            assert total == math.comb(C, k)
            b, ru, _ = pt.pt_merge_top2(recs_s, recs_t, k)
            assert b == want[0]


def test_medium_masked_and_k4():
    T, dev = synth.small_matrix(4, n_cfg=90, n_dev=3, n_inputs=8)
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    mask = (dev != 1).astype(np.uint8)
    for k in (2, 3):
        check_exh(o, pt.pt_exhaustive_best(ctx, k, env_mask=mask), k, mask=mask)
    check_exh(o, pt.pt_exhaustive_best(ctx, 4), 4)
    idx, gt, gp = pt.pt_greedy_select(ctx, 10, env_mask=mask)
    check_greedy(o, idx, gt, gp, 10, mask=mask)


def test_score_sets_host_and_device():
    T, dev = synth.small_matrix(5, n_cfg=500, n_dev=4, n_inputs=12)
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    rng = np.random.default_rng(0)
    for k in (1, 2, 3, 5, 8):
        sets = rng.integers(0, 500, size=(64, k)).astype(np.int32)
        want = o.score(sets)
        got = pt.pt_score_sets(ctx, sets)
        np.testing.assert_allclose(got, want, rtol=1e-12)
        dsets = torch.from_numpy(sets).cuda()
        dout = torch.empty(64, dtype=torch.float64, device="cuda")
        pt.pt_score_sets(ctx, dsets, out=dout)
        np.testing.assert_allclose(dout.cpu().numpy(), want, rtol=1e-12)
        mask = (dev % 2 == 0).astype(np.uint8)
        np.testing.assert_allclose(pt.pt_score_sets(ctx, sets, env_mask=mask),
                                   o.score(sets, mask=mask), rtol=1e-12)


def test_greedy_stream_vs_resident():
    T, dev = synth.small_matrix(6, n_cfg=700, n_dev=5, n_inputs=20)
    o = Oracle(T, dev)
    for flags in (0, pt.PT_GREEDY_STREAM):
        ctx = pt.pt_load_perf(T, dev, flags=flags)
        idx, gt, gp = pt.pt_greedy_select(ctx, 24)
        check_greedy(o, idx, gt, gp, 24)


def test_missing_cells_and_errors():
    T, dev = synth.small_matrix(7, n_cfg=60, n_dev=2, n_inputs=5)
    T[3, 7] = np.nan
    T[5, 11] = np.inf
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    check_exh(o, pt.pt_exhaustive_best(ctx, 2), 2)
    np.testing.assert_allclose(pt.pt_score_sets(ctx, [[7], [11]]), o.score([[7], [11]]), rtol=1e-12)
    bad = T.copy()
    bad[0, 0] = -1.0
    with pytest.raises(pt.PTError) as ei:
        pt.pt_load_perf(bad, dev)
    assert ei.value.code == pt.PT_EDATA
    with pytest.raises(pt.PTError) as ei:
        pt.pt_exhaustive_best(ctx, 2, env_mask=np.zeros(len(dev), np.uint8))
    assert ei.value.code == pt.PT_EEMPTY
    with pytest.raises(pt.PTError) as ei:
        pt.pt_score_sets(ctx, [[0, 60]])
    assert ei.value.code == pt.PT_EINVAL
    with pytest.raises(pt.PTError) as ei:
        pt.pt_exhaustive_best(ctx, 61)
    assert ei.value.code == pt.PT_EINVAL
    big = np.ones((2, 100000), np.float32)
    ctx2 = pt.pt_load_perf(big)
    with pytest.raises(pt.PTError) as ei:
        pt.pt_exhaustive_best(ctx2, 4)
    assert ei.value.code == pt.PT_ECAP


# ------------------------------------------------ paper shape (configs 2, 3, 4)
@pytest.fixture(scope="module")
def paper1():
    T, dev = synth.paper_matrix(1)
    return T, dev, Oracle(T, dev)


def test_paper_greedy_24(paper1):
    T, dev, o = paper1
    ctx = pt.pt_load_perf(torch.from_numpy(T).cuda(), dev)
    idx, gt, gp = pt.pt_greedy_select(ctx, 24)
    check_greedy(o, idx, gt, gp, 24)


def test_paper_exhaustive_k2(paper1):
    T, dev, o = paper1
    ctx = pt.pt_load_perf(T, dev)
    check_exh(o, pt.pt_exhaustive_best(ctx, 2), 2)


@pytest.mark.parametrize("tier", ["tc", "u8", "fp16"])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_paper_exhaustive_k3_golden(seed, tier, monkeypatch):
    """Full size: 930,485,175 triples vs the oracle's stored result
    (tests/golden/paper_exhaustive.json, written by scripts/make_golden.py), with
    either filter tier."""
    monkeypatch.setenv("PT_EXH_TIER", tier)
    gold = json.load(open(os.path.join(GOLDEN, "paper_exhaustive.json")))[f"seed{seed}_k3"]
    T, dev = synth.paper_matrix(seed)
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    want = (tuple(gold["best"]), gold["G"], tuple(gold["runner"]), gold["G_runner"])
    res = pt.pt_exhaustive_best(ctx, 3)
    check_exh(o, res, 3, want=want)
    assert res["runner"] == want[2]
    st = pt.pt_get_stats(ctx)
    assert st["exh_sets"] == 930_485_175 and st["exh_kernel"] == {"tc": 5, "u8": 4, "fp16": 0}[tier]
    # the oracle re-scores the GPU's pick one by one
    assert o.score(list(res["best"])) == pytest.approx(res["G"], rel=1e-12)
    # 8-way sharded on one device (the multi-GPU partition), merged
    recs_s, recs_t, total = [], [], 0
    for r in range(8):
        x = pt.pt_exhaustive_best(ctx, 3, shard_rank=r, shard_count=8)
        total += pt.pt_get_stats(ctx)["exh_sets"]
        for sv, tup in ((x["s"][0], x["best"]), (x["s"][1], x["runner"])):
            recs_s.append(sv)
            recs_t.append(tup if tup is not None else (-1, -1, -1))
    assert total == 930_485_175
    b, ru, _ = pt.pt_merge_top2(recs_s, recs_t, 3)
    assert b == want[0] and ru == want[2]


def test_paper_holdout(paper1):
    T, dev, o = paper1
    ctx = pt.pt_load_perf(T, dev)
    for d in range(5):
        for k, method in ((5, 0), (2, 1)):
            h = pt.pt_eval_holdout(ctx, d, k, method)
            idx, gtr, gun, gkn, kidx = o.holdout(d, k, method=method)
            assert h["idx"] == idx and h["known_idx"] == kidx
            assert h["G_train"] == pytest.approx(gtr, rel=RTOL)
            assert h["G_unseen"] == pytest.approx(gun, rel=RTOL)
            assert h["G_known"] == pytest.approx(gkn, rel=RTOL)
            assert h["G_known"] >= h["G_unseen"] - 1e-12


# ------------------------------------------------------------ scaled (config 5)
def test_scaled_greedy_32():
    """65,536 configs x 4,096 envs, k=32 (streamed path).  Every step is re-derived
    by the oracle from the GPU's prefix (check_greedy's step rule): the pick must be
    the oracle's whenever that step's top-two gap exceeds 1e-9, and G must match."""
    T, dev = synth.scaled(1)
    ctx = pt.pt_load_perf(torch.from_numpy(T).cuda(), dev)
    idx, gt, gp = pt.pt_greedy_select(ctx, 32)
    assert len(set(idx)) == 32
    del ctx
    o = Oracle(T, dev)
    for t in range(32):
        sidx, sg, sgap = o.greedy(1, init=idx[:t])
        if sgap[0] > GAP:
            assert sidx[0] == idx[t], (t, idx)
        assert gt[t] == pytest.approx(sg[0], rel=RTOL)
        assert gt[t] == pytest.approx(o.score(idx[:t + 1]), rel=RTOL)


def test_greedy_lazy_medium():
    T, dev = synth.small_matrix(6, n_cfg=700, n_dev=5, n_inputs=20)
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev, flags=pt.PT_GREEDY_LAZY)
    idx, gt, gp = pt.pt_greedy_select(ctx, 24)
    oidx, ogt, ogp = o.greedy(24)
    for t in range(24):
        assert gt[t] == pytest.approx(o.score(idx[:t + 1]), rel=RTOL)
    if np.all(ogp > GAP):
        assert idx == oidx
    mask = (dev != 3).astype(np.uint8)
    assert pt.pt_greedy_select(ctx, 10, env_mask=mask)[0] == o.greedy(10, mask=mask)[0]


def test_greedy_lazy_scaled_equals_plain():
    """Lazy greedy on the scaled matrix: same picks as the plain streamed greedy,
    far fewer exact evaluations."""
    T, dev = synth.scaled(1)
    dT = torch.from_numpy(T).cuda()
    ctx = pt.pt_load_perf(dT, dev)
    idx, gt, _ = pt.pt_greedy_select(ctx, 32)
    pt.pt_free(ctx)
    ctx = pt.pt_load_perf(dT, dev, flags=pt.PT_GREEDY_LAZY)
    lidx, lgt, _ = pt.pt_greedy_select(ctx, 32)
    assert lidx == idx
    np.testing.assert_allclose(lgt, gt, rtol=1e-12)
    assert pt.pt_get_stats(ctx)["greedy_candidates"] < 32 * 65536 // 10


def test_holdout_all_batched(paper1):
    T, dev, o = paper1
    ctx = pt.pt_load_perf(T, dev)
    res = pt.pt_eval_holdout_all(ctx, 5, 5)
    for d in range(5):
        h = pt.pt_eval_holdout(ctx, d, 5, 0)
        idx, gtr, gun, gkn, kidx = o.holdout(d, 5, method=0)
        assert res[d]["idx"] == idx == h["idx"] and res[d]["known_idx"] == kidx
        for key, want in (("G_train", gtr), ("G_unseen", gun), ("G_known", gkn)):
            assert res[d][key] == pytest.approx(want, rel=RTOL)
