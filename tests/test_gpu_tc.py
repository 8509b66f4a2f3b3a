"""The threshold-count tier of the tiled exhaustive search (k_exh_tc):
every set's lower bound u * P(S) (P = a 0/1 dot product of thresholded rows, on the
tensor cores) is compared with tau, an upper bound of the second-best score from a
device-side swap search; survivors are re-scored in fp64.  These tests check the
answers against the oracle and the other tiers, the fall-backs (unusable tau, too
weak a filter, scopes wider than the kernel's K), and that the tier really ran."""
import math

import numpy as np
import pytest

from oracle import Oracle
from paper_2507_15277_b200 import pt, synth
from test_gpu_parity import check_exh

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def run_tier(ctx, k, tier, monkeypatch, **kw):
    monkeypatch.setenv("PT_EXH_TIER", tier)
    r = pt.pt_exhaustive_best(ctx, k, **kw)
    st = pt.pt_get_stats(ctx)
    monkeypatch.delenv("PT_EXH_TIER")
    return r, st


@pytest.mark.parametrize("k", [2, 3])
def test_tc_equals_u8_paper_shape(k, monkeypatch):
    """Paper shape: the tc tier runs (kernel 5) with a small survivor set and returns
    the u8 tier's best, runner-up and bit-identical fp64 scores."""
    T, dev = synth.paper_matrix(1)
    ctx = pt.pt_load_perf(T, dev)
    rt, st = run_tier(ctx, k, "tc", monkeypatch)
    ru, su = run_tier(ctx, k, "u8", monkeypatch)
    assert st["exh_kernel"] == 5 and su["exh_kernel"] == 4
    assert 0 < st["exh_tc_survivors"] < 200_000 and st["exh_tc_nt"] >= 1
    assert rt["best"] == ru["best"] and rt["runner"] == ru["runner"]
    assert rt["s"][0] == ru["s"][0] and rt["s"][1] == ru["s"][1]
    assert st["exh_sets"] == math.comb(1775, k)


@pytest.mark.parametrize("nt", [1, 2, 3])
@pytest.mark.parametrize("seed,C,ndev,nin", [(31, 300, 3, 16), (32, 520, 4, 20), (33, 1100, 5, 9)])
def test_tc_small_vs_oracle(seed, C, ndev, nin, nt, monkeypatch):
    """k = 2, 3, 4 (k=4 only below 500 configs) against the oracle, with 1-3
    thresholds per environment (PT_TC_NT); several row and column tiles, ragged
    column tails (C not a multiple of 256)."""
    monkeypatch.setenv("PT_TC_NT", str(nt))
    T, dev = synth.small_matrix(seed, n_cfg=C, n_dev=ndev, n_inputs=nin)
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    for k in ((2, 3, 4) if C < 500 else (2, 3)):
        r = pt.pt_exhaustive_best(ctx, k)
        st = pt.pt_get_stats(ctx)
        check_exh(o, r, k)
        assert st["exh_kernel"] in (5, 4)
        if st["exh_kernel"] == 5:
            assert st["exh_tc_nt"] == nt


def test_tc_ran_on_medium_data(monkeypatch):
    """Data with a clear optimum: the tc tier is the one that answers (forced for k=2,
    where the default is the u8 tier)."""
    monkeypatch.setenv("PT_EXH_TIER", "tc")
    T, dev = synth.small_matrix(34, n_cfg=700, n_dev=5, n_inputs=64)
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    for k in (2, 3):
        check_exh(o, pt.pt_exhaustive_best(ctx, k), k)
        assert pt.pt_get_stats(ctx)["exh_kernel"] == 5


def test_tc_masked_scopes(monkeypatch):
    """Leave-one-device-out scopes (each its own thresholds, tau and operands)."""
    T, dev = synth.small_matrix(35, n_cfg=400, n_dev=4, n_inputs=30)
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    for d in range(4):
        mask = (dev != d).astype(np.uint8)
        rt, st = run_tier(ctx, 3, "tc", monkeypatch, env_mask=mask)
        check_exh(o, rt, 3, mask=mask)
        ru, _ = run_tier(ctx, 3, "u8", monkeypatch, env_mask=mask)
        assert rt["s"] == ru["s"] and rt["best"] == ru["best"]


def test_tc_missing_cells():
    """NaN cells take the dataset penalty before the thresholds."""
    T, dev = synth.small_matrix(36, n_cfg=350, n_dev=3, n_inputs=21)
    T = T.copy()
    rng = np.random.default_rng(9)
    T[rng.integers(0, T.shape[0], 90), rng.integers(0, T.shape[1], 90)] = np.nan
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    for k in (2, 3):
        check_exh(o, pt.pt_exhaustive_best(ctx, k), k)


def test_tc_after_greedy_host_trace():
    """A greedy run first (host-side trace): the swap search starts from its picks."""
    T, dev = synth.small_matrix(37, n_cfg=450, n_dev=4, n_inputs=16)
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    pt.pt_greedy_select(ctx, 8)
    for k in (2, 3, 4):
        check_exh(o, pt.pt_exhaustive_best(ctx, k), k)


def test_tc_weak_filter_falls_back():
    """Near-ties everywhere (every config within 1e-3 of the best): the lower bound
    separates nothing, the survivor buffer overflows, and the u8 tier answers."""
    rng = np.random.default_rng(3)
    T = (1.0 + 1e-3 * rng.random((40, 600))).astype(np.float32)
    o = Oracle(T)
    ctx = pt.pt_load_perf(T)
    r = pt.pt_exhaustive_best(ctx, 3)
    st = pt.pt_get_stats(ctx)
    check_exh(o, r, 3)
    assert st["exh_kernel"] in (4, 0)


def test_tc_wide_scope_not_eligible():
    """E_pad > 1024: the tc tier's A buffer does not fit (and above 768 environments the
    tiled tiers give way to the generic fp64 kernel)."""
    rng = np.random.default_rng(38)
    T = np.exp(rng.normal(size=(1100, 200))).astype(np.float32)   # E_pad 1152 > 1024
    o = Oracle(T)
    ctx = pt.pt_load_perf(T)
    check_exh(o, pt.pt_exhaustive_best(ctx, 3), 3)
    assert pt.pt_get_stats(ctx)["exh_kernel"] in (4, 1)


def test_tc_sharded_partition():
    """Shards of the tc task list partition the subset space: merged == unsharded."""
    T, dev = synth.small_matrix(39, n_cfg=640, n_dev=5, n_inputs=20)
    ctx = pt.pt_load_perf(T, dev)
    full = pt.pt_exhaustive_best(ctx, 3)
    assert pt.pt_get_stats(ctx)["exh_kernel"] == 5
    recs, sets = [], 0
    for s in range(5):
        r = pt.pt_exhaustive_best(ctx, 3, shard_rank=s, shard_count=5)
        sets += pt.pt_get_stats(ctx)["exh_sets"]
        recs.append(r)
    assert sets == math.comb(640, 3)
    cand = sorted([(r["s"][0], r["best"]) for r in recs if r["best"] is not None] +
                  [(r["s"][1], r["runner"]) for r in recs if r["runner"] is not None])
    assert cand[0][1] == full["best"] and cand[0][0] == full["s"][0]
    assert cand[1][1] == full["runner"] and cand[1][0] == full["s"][1]


def test_tc_overflow_paths(monkeypatch):
    """A tiny survivor buffer (PT_TC_CAP=16): unsharded, the search falls back to the
    u8 tier; sharded, every shard must stay on the tc task list (the tiers partition
    the subset space differently), so it reruns with room for every survivor -- and
    the merged shards still equal the unsharded answer."""
    T, dev = synth.small_matrix(40, n_cfg=500, n_dev=5, n_inputs=20)
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    want = pt.pt_exhaustive_best(ctx, 3)
    assert pt.pt_get_stats(ctx)["exh_kernel"] == 5
    check_exh(o, want, 3)
    monkeypatch.setenv("PT_TC_CAP", "16")
    r = pt.pt_exhaustive_best(ctx, 3)
    st = pt.pt_get_stats(ctx)
    assert st["exh_kernel"] == 4 and st["exh_tc_survivors"] > 16
    assert r["best"] == want["best"] and r["s"] == want["s"]
    recs, sets = [], 0
    for s in range(3):
        rr = pt.pt_exhaustive_best(ctx, 3, shard_rank=s, shard_count=3)
        st = pt.pt_get_stats(ctx)
        assert st["exh_kernel"] == 5
        sets += st["exh_sets"]
        recs.append(rr)
    assert sets == math.comb(500, 3)
    cand = sorted([(x["s"][0], x["best"]) for x in recs if x["best"] is not None] +
                  [(x["s"][1], x["runner"]) for x in recs if x["runner"] is not None])
    assert cand[0] == (want["s"][0], want["best"]) and cand[1] == (want["s"][1], want["runner"])
