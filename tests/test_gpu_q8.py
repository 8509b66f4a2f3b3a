"""The u8 filter tier of the tiled exhaustive search (k_exh_q8):
every set is scored exactly on the matrix quantised to bytes, q = rint(l / Delta)
with Delta = (scope max of l) / 255; the per-term error |Delta q - l| <= Delta / 2
gives each set a rigorous window and the survivors are re-scored in fp64.  These
tests stress what is particular to it: a coarse quantum (one huge outlier sets
Delta), missing cells, masked scopes (Delta per scope), identical answers from the
two tiers, and the hand-over to the fp16 tier when the window holds > 2^24 sets."""
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


@pytest.fixture(autouse=True)
def _u8_tier(monkeypatch):
    """These tests are about the u8 tier: select it (the default is the tc tier)."""
    monkeypatch.setenv("PT_EXH_TIER", "u8")


def both_tiers(ctx, k, monkeypatch, **kw):
    out = {}
    for tier in ("u8", "fp16"):
        monkeypatch.setenv("PT_EXH_TIER", tier)
        r = pt.pt_exhaustive_best(ctx, k, **kw)
        out[tier] = (r, pt.pt_get_stats(ctx))
    monkeypatch.setenv("PT_EXH_TIER", "u8")
    return out


@pytest.mark.parametrize("k", [2, 3])
def test_tiers_identical_paper_shape(k, monkeypatch):
    """Same best, runner-up and bit-identical fp64 scores from both tiers at the
    paper shape (the refine is common; only the filter differs)."""
    T, dev = synth.paper_matrix(2)
    ctx = pt.pt_load_perf(T, dev)
    res = both_tiers(ctx, k, monkeypatch)
    (ru, su), (rf, sf) = res["u8"], res["fp16"]
    assert su["exh_kernel"] == 4 and sf["exh_kernel"] == 0
    assert ru["best"] == rf["best"] and ru["runner"] == rf["runner"]
    assert ru["s"][0] == rf["s"][0] and ru["s"][1] == rf["s"][1]
    assert su["exh_sets"] == sf["exh_sets"] == math.comb(1775, k)


@pytest.mark.parametrize("k", [2, 3, 4])
def test_coarse_quantum_outlier(k):
    """One cell 10^6 x slower than its environment's best: Delta grows to
    ln(1e6)/255 ~ 0.054 and the window to ~ E * Delta, so many more sets reach
    the refine -- the answer must not change."""
    T, dev = synth.small_matrix(21, n_cfg=140, n_dev=3, n_inputs=9)
    T = T.copy()
    T[4, 17] = T[4].min() * 1e6
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    check_exh(o, pt.pt_exhaustive_best(ctx, k), k)
    assert pt.pt_get_stats(ctx)["exh_kernel"] == 4


def test_missing_cells():
    """NaN cells take the dataset penalty before quantisation."""
    T, dev = synth.small_matrix(22, n_cfg=200, n_dev=3, n_inputs=11)
    T = T.copy()
    rng = np.random.default_rng(5)
    T[rng.integers(0, T.shape[0], 60), rng.integers(0, T.shape[1], 60)] = np.nan
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    for k in (2, 3):
        check_exh(o, pt.pt_exhaustive_best(ctx, k), k)
        assert pt.pt_get_stats(ctx)["exh_kernel"] == 4


def test_masked_scopes_have_their_own_quantum(monkeypatch):
    """Leave-one-device-out scopes: each scope view is quantised with its own
    Delta; both tiers agree with the oracle on every scope."""
    T, dev = synth.small_matrix(23, n_cfg=260, n_dev=4, n_inputs=13)
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    for d in range(4):
        mask = (dev != d).astype(np.uint8)
        res = both_tiers(ctx, 3, monkeypatch, env_mask=mask)
        for tier, (r, st) in res.items():
            check_exh(o, r, 3, mask=mask)
        assert res["u8"][0]["s"] == res["fp16"][0]["s"]


def test_handover_to_fp16_tier():
    """470 identical configurations: all C(470,3) = 17,202,340 triples tie, which
    is more than the u8 tier keeps (2^24 = 16,777,216): the search hands over to the
    fp16 tier (its own overflow rerun follows) and still returns the
    lexicographically first triples."""
    rng = np.random.default_rng(11)
    col = np.exp(rng.normal(size=(24, 1))).astype(np.float32)
    T = np.repeat(col, 470, axis=1)
    ctx = pt.pt_load_perf(T)
    r = pt.pt_exhaustive_best(ctx, 3)
    st = pt.pt_get_stats(ctx)
    assert r["best"] == (0, 1, 2) and r["runner"] == (0, 1, 3) and r["G"] == 1.0
    assert st["exh_kernel"] == 0 and st["exh_passes"] == 3
    assert st["exh_candidates"] == math.comb(470, 3)
