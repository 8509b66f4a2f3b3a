"""GPU parity of the host-side fast paths added for the bench step: the exhaustive
search seeded from a cached greedy trace, the batched holdout whose host transfers
exceed the pinned staging buffer (pageable fallback), and repeated calls on one
context (the staging buffer is reused).  Same bar as test_gpu_parity.py."""
import math

import numpy as np
import pytest

from oracle import Oracle
from paper_2507_15277_b200 import pt, synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RTOL = 1e-6
GAP = 1e-9


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _check_exh(o, res, k):
    b, gb, ru, gr = o.exhaustive(k)
    assert res["G"] == pytest.approx(gb, rel=RTOL)
    if ru is None or gb - gr > GAP:
        assert res["best"] == tuple(b)
    else:
        assert o.score(list(res["best"])) >= gb - GAP
    if ru is not None:
        assert res["G_runner"] == pytest.approx(gr, rel=RTOL)


@pytest.mark.parametrize("seed", [3, 4])
def test_exhaustive_seed_from_cached_greedy(seed):
    """k=2/3 after a longer greedy run on the same view (seed read from the cached
    trace) equals a fresh context (seed from its own greedy run) and the oracle."""
    T, dev = synth.small_matrix(seed, n_cfg=300, n_dev=3, n_inputs=32)
    o = Oracle(T, dev)
    warm = pt.pt_load_perf(torch.from_numpy(T).cuda(), dev)
    pt.pt_greedy_select(warm, 12)
    cold = pt.pt_load_perf(torch.from_numpy(T).cuda(), dev)
    for k in (2, 3):
        a = pt.pt_exhaustive_best(warm, k)
        b = pt.pt_exhaustive_best(cold, k)
        assert a["best"] == b["best"] and a["s"] == b["s"] and a["runner"] == b["runner"]
        _check_exh(o, a, k)
    # a shorter greedy after the longer one leaves the cache valid (prefix)
    idx, _, _ = pt.pt_greedy_select(warm, 3)
    assert list(idx) == o.greedy(3)[0]
    _check_exh(o, pt.pt_exhaustive_best(warm, 3), 3)
    pt.pt_free(warm)
    pt.pt_free(cold)


def test_holdout_all_many_devices_pageable_fallback():
    """64 devices x 32 inputs: the batched holdout's weight upload (128 problems x
    2,048 envs x 8 B = 2 MiB) exceeds the 1 MiB pinned staging buffer."""
    T, dev = synth.scaled(5, n_cfg=96, n_dev=64, n_inputs=32)
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(torch.from_numpy(T).cuda(), dev)
    res = pt.pt_eval_holdout_all(ctx, 3, 64)
    assert len(res) == 64
    for d in (0, 1, 17, 63):
        idx, gtr, gun, gkn, kidx = o.holdout(d, 3, method=0)
        assert res[d]["idx"] == idx and res[d]["known_idx"] == kidx
        for key, want in (("G_train", gtr), ("G_unseen", gun), ("G_known", gkn)):
            assert res[d][key] == pytest.approx(want, rel=RTOL)
    pt.pt_free(ctx)


def test_repeated_calls_reuse_staging():
    """Many small calls on one context return the same answers every time."""
    T, dev = synth.small_matrix(6, n_cfg=120, n_dev=2, n_inputs=16)
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(torch.from_numpy(T).cuda(), dev)
    ref = None
    for _ in range(5):
        g = pt.pt_greedy_select(ctx, 6)[0]
        e = pt.pt_exhaustive_best(ctx, 2)
        got = (tuple(g), e["best"], e["s"])
        ref = ref or got
        assert got == ref
    assert list(ref[0]) == o.greedy(6)[0]
    _check_exh(o, pt.pt_exhaustive_best(ctx, 2), 2)
    assert not math.isnan(e["G"])
    pt.pt_free(ctx)


def test_weighted_shards():
    """pt_set_shard_weights: shards of a weighted partition merge to the unsharded
    result, cover every set exactly once, and take work in proportion to the weights."""
    T, dev = synth.small_matrix(7, n_cfg=400, n_dev=3, n_inputs=16)
    ctx = pt.pt_load_perf(torch.from_numpy(T).cuda(), dev)
    full = pt.pt_exhaustive_best(ctx, 3)
    w = [0.5, 1.0, 1.5]
    pt.pt_set_shard_weights(ctx, w)
    recs_s, recs_t, sets = [], [], []
    for r in range(3):
        res = pt.pt_exhaustive_best(ctx, 3, shard_rank=r, shard_count=3)
        sets.append(pt.pt_get_stats(ctx)["exh_sets"])
        for sv, tup in ((res["s"][0], res["best"]), (res["s"][1], res["runner"])):
            recs_s.append(sv)
            recs_t.append(tup if tup is not None else (-1,) * 3)
    assert sum(sets) == math.comb(400, 3)
    assert sets[0] < sets[1] < sets[2]
    assert abs(sets[0] / sum(sets) - 0.5 / 3) < 0.05
    b, ru, (s1, s2) = pt.pt_merge_top2(recs_s, recs_t, 3)
    assert b == full["best"] and s1 == full["s"][0] and s2 == full["s"][1]
    with pytest.raises(pt.PTError):
        pt.pt_set_shard_weights(ctx, [1.0, 0.0])
    pt.pt_set_shard_weights(ctx, None)   # equal shares again
    pt.pt_free(ctx)
