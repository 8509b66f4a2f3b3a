"""GPU edge cases: degenerate shapes, all-tied data that overflows the candidate
buffer (the second-pass path), wide scopes (generic kernel), tiny scopes."""
import math

import numpy as np
import pytest

from oracle import Oracle
from paper_2507_15277_b200 import pt, synth
from test_gpu_parity import check_exh, check_greedy

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("C,E", [(3, 1), (4, 2), (5, 33), (9, 31), (65, 7), (70, 64), (129, 65)])
def test_small_shapes(C, E):
    rng = np.random.default_rng(C * 100 + E)
    T = np.exp(rng.normal(size=(E, C))).astype(np.float32)
    o = Oracle(T)
    ctx = pt.pt_load_perf(T)
    for k in range(1, min(C, 4) + 1):
        check_exh(o, pt.pt_exhaustive_best(ctx, k), k)
    kk = min(C, 5)
    idx, gt, gp = pt.pt_greedy_select(ctx, kk)
    check_greedy(o, idx, gt, gp, kk)


def test_all_tied_overflow_second_pass():
    """300 identical configurations: every one of C(300,3) = 4,455,100 triples
    ties, overflowing the 1 M-entry candidate buffer -> the search re-runs with
    the final threshold and a buffer of the reported size; the answer is the
    lexicographically first triple (reading c5)."""
    rng = np.random.default_rng(7)
    col = np.exp(rng.normal(size=(40, 1))).astype(np.float32)
    T = np.repeat(col, 300, axis=1)
    T[:, 0] *= 1.0                                    # keep exact copies
    ctx = pt.pt_load_perf(T)
    r = pt.pt_exhaustive_best(ctx, 3)
    st = pt.pt_get_stats(ctx)
    assert r["best"] == (0, 1, 2) and r["runner"] == (0, 1, 3)
    assert r["G"] == 1.0
    # pass 1: the tc tier finds tau = 0 (every score is 0) and does not run; pass 2:
    # the u8 tier overflows; pass 3: its rerun with room for every survivor
    assert st["exh_tc_survivors"] == -1 and st["exh_kernel"] == 4
    assert st["exh_passes"] == 3 and st["exh_candidates"] == math.comb(300, 3)


def test_near_ties_duplicates():
    """Duplicated good columns: many exact ties near the top."""
    T, dev = synth.small_matrix(9, n_cfg=150, n_dev=2, n_inputs=10)
    T[:, 100:110] = T[:, [3]]                          # ten copies of config 3
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    for k in (2, 3):
        check_exh(o, pt.pt_exhaustive_best(ctx, k), k)
    idx, gt, gp = pt.pt_greedy_select(ctx, 8)
    check_greedy(o, idx, gt, gp, 8)


def test_wide_scope_generic_kernel():
    """E_pad > 768 -> thread-per-subset fp64 kernel."""
    T, dev = synth.small_matrix(4, n_cfg=40, n_dev=13, n_inputs=64)   # 832 envs
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    r = pt.pt_exhaustive_best(ctx, 2)
    assert pt.pt_get_stats(ctx)["exh_kernel"] == 1
    check_exh(o, r, 2)


def test_single_env_scope():
    T, dev = synth.small_matrix(5, n_cfg=50, n_dev=2, n_inputs=3)
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    mask = np.zeros(len(dev), np.uint8)
    mask[4] = 1
    for k in (1, 2, 3):
        check_exh(o, pt.pt_exhaustive_best(ctx, k, env_mask=mask), k, mask=mask)


@pytest.mark.parametrize("tier", ["tc", "u8", "fp16"])
@pytest.mark.parametrize("C", [9, 61, 64, 65, 71, 72, 127, 130])
@pytest.mark.parametrize("k", [2, 3, 4])
def test_every_subset_is_evaluated(C, k, tier, monkeypatch):
    """All-tied data: every k-subset lands in the candidate window, so the count
    of refined candidates must equal C(C, k) -- a direct coverage check of the
    tiling (row tiles, column tiles, the 8-config column alignment, masks) --
    and the shards must partition the subset space."""
    if math.comb(C, k) > 900_000:
        pytest.skip("stays under the 1 M candidate buffer")
    monkeypatch.setenv("PT_EXH_TIER", tier)
    T = np.ones((37, C), np.float32)
    ctx = pt.pt_load_perf(T)
    r = pt.pt_exhaustive_best(ctx, k)
    st = pt.pt_get_stats(ctx)
    # tc: every score is 0, so tau = 0 gives no threshold step -> the u8 tier runs
    assert st["exh_kernel"] == {"tc": 4, "u8": 4, "fp16": 0}[tier]
    assert r["best"] == tuple(range(k))
    assert st["exh_candidates"] == math.comb(C, k) == st["exh_sets"]
    tot = 0
    for s in range(3):
        pt.pt_exhaustive_best(ctx, k, shard_rank=s, shard_count=3)
        st = pt.pt_get_stats(ctx)
        assert st["exh_candidates"] == st["exh_sets"]
        tot += st["exh_candidates"]
    assert tot == math.comb(C, k)


def test_near_tie_below_fp16_resolution():
    """Clones of the best triple's members, each 2e-6 slower everywhere: every
    triple using a clone is worse than the best by ~1e-7..1e-6 in G -- far below
    what the packed-fp16 filter resolves (2^-11 relative), far above the 1e-9
    bar: the window must keep them and the fp64 refine must order them exactly
    (best, runner-up and both G), as the oracle does."""
    T, dev = synth.small_matrix(17, n_cfg=160, n_dev=3, n_inputs=12)
    b = Oracle(T, dev).exhaustive(3)[0]
    T = T.copy()
    T[:, 150:153] = T[:, list(b)] * np.float32(1.0 + 2e-6)
    o = Oracle(T, dev)
    ob, og, orr, ogr = o.exhaustive(3)
    assert ob == b and any(c >= 150 for c in orr)
    assert 1e-9 < og - ogr < 1e-5
    ctx = pt.pt_load_perf(T, dev)
    r = pt.pt_exhaustive_best(ctx, 3)
    assert r["best"] == ob and r["runner"] == orr
    assert r["G"] == pytest.approx(og, rel=1e-12) and r["G_runner"] == pytest.approx(ogr, rel=1e-12)
    assert pt.pt_get_stats(ctx)["exh_candidates"] >= 4   # the near-tied sets all reached the refine
