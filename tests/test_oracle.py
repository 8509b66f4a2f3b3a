"""Pins for the CPU oracle (oracle/oracle.c) against what the paper and the
mathematics fix -- never against the oracle itself.

Pins used:
  * paper worked values: the Quadro rows of "Sample Data From Dataset"
    (P:L406-408), SPEC worked examples S:L109, S:L182;
  * closed forms: power-of-two matrices, G = 2^(-sum min m / E) exactly;
  * brute force over every subset of tiny inputs with exact integer arithmetic;
  * hand enumerations (tests/golden/hand_3x4.txt, greedy_vs_opt.txt);
  * invariants: k = C -> 1.0, monotone in k, per-env scale invariance,
    permutation invariance, greedy submodularity and the (1 - 1/e) bound;
  * planted specialists: unique known optimum.
"""
import itertools
import math

import numpy as np
import pytest

from conftest import read_golden
from oracle import Oracle, OracleError
from paper_2507_15277_b200 import synth


def pow2_matrix(m):
    m = np.asarray(m)
    return np.ldexp(np.ones(m.shape, np.float32), m.astype(np.int32))


def lex_key(sumv, tup):
    return (sumv, tuple(tup))


# --------------------------------------------------------------------------
# paper / SPEC worked values
# --------------------------------------------------------------------------

def test_quadro_sample_rows():
    """times 0.693 and 0.157 ms on one env; S/O printed 4.41 and 1.0."""
    rows = read_golden("quadro_sample.txt")
    t = np.array([[float(r[1]) for r in rows]], np.float32)
    o = Oracle(t)
    assert o.best[0] == pytest.approx(0.157, rel=1e-7)        # the Oracle
    for c, r in enumerate(rows):
        so = 1.0 / o.score([c])                                # S/O = A/O
        assert round(so, 2) == pytest.approx(float(r[2]))
    # best-member reading of Eq. 1 (reading c1): the pair performs as its best
    assert o.score([0, 1]) == 1.0
    # the literal "max runtime" reading would give 0.157/0.693; ours does not
    assert o.score([0, 1]) != pytest.approx(0.157 / 0.693)
    # worst-speedup column is consistent with the same Oracle (sanity on the fixture)
    worst = float(rows[0][1]) * float(rows[0][3])
    assert worst == pytest.approx(float(rows[1][1]) * float(rows[1][3]), rel=2e-3)


def test_spec_examples():
    # one env, runtimes {2.0, 4.0} -> slowdowns [1.0, 2.0]
    o = Oracle(np.array([[2.0, 4.0]], np.float32))
    assert o.score([0]) == 1.0
    assert 1.0 / o.score([1]) == pytest.approx(2.0, rel=1e-15)
    # two envs, best-in-set slowdowns 1 and 4 -> geomean 2 -> G = 0.5
    o = Oracle(np.array([[1.0, 3.0], [4.0, 1.0]], np.float32))
    assert o.score([0]) == pytest.approx(0.5, rel=1e-15)


def test_hand_3x4_fixture():
    g = read_golden("hand_3x4.txt")
    m = np.array([[int(x) for x in r[1:]] for r in g if r[0] == "m"])
    o = Oracle(pow2_matrix(m))
    E = m.shape[0]
    for r in g:
        if r[0] in ("pair", "single", "triple"):
            idx = [int(x) for x in r[1:-1]]
            assert o.score(idx) == pytest.approx(2.0 ** (-int(r[-1]) / E), rel=1e-15)
    for r in g:
        if r[0] == "best":
            k = int(r[1].split("=")[1])
            b = tuple(int(x) for x in r[2].split(","))
            ru = tuple(int(x) for x in r[4].split(","))
            sb, sr = int(r[6]), int(r[7])
            got = o.exhaustive(k, threads=2)
            assert got[0] == b and got[2] == ru
            assert got[1] == pytest.approx(2.0 ** (-sb / E), rel=1e-15)
            assert got[3] == pytest.approx(2.0 ** (-sr / E), rel=1e-15)
        if r[0] == "greedy":
            picks = [int(x) for x in r[1:4]]
            sums = [int(x) for x in r[5:8]]
            nxt = [int(x) for x in r[9:12]]
            idx, gt, gp = o.greedy(3)
            assert idx == picks
            for t in range(3):
                assert gt[t] == pytest.approx(2.0 ** (-sums[t] / E), rel=1e-15)
                assert gp[t] == pytest.approx(2.0 ** (-sums[t] / E) - 2.0 ** (-nxt[t] / E),
                                              rel=1e-12)


def test_greedy_vs_opt_fixture():
    g = read_golden("greedy_vs_opt.txt")
    m = np.array([[int(x) for x in r[1:]] for r in g if r[0] == "m"])
    o = Oracle(pow2_matrix(m))
    E = m.shape[0]
    idx, gt, gp = o.greedy(2)
    assert idx == [0, 1]
    assert gt[1] == pytest.approx(2.0 ** (-2 / E), rel=1e-15)
    assert gp[1] == 0.0                         # exact tie at step 2 -> lowest index
    b, gb, ru, gr = o.exhaustive(2)
    assert b == (1, 2) and gb == 1.0 and ru == (0, 1)
    assert gr == pytest.approx(2.0 ** (-2 / E), rel=1e-15)


# --------------------------------------------------------------------------
# closed forms and brute force with exact integer arithmetic
# --------------------------------------------------------------------------

def brute_force_pow2(m, k, mask=None):
    """Every k-subset, exact integer score sum_e min m (lower is better)."""
    E, C = m.shape
    rows = range(E) if mask is None else [e for e in range(E) if mask[e]]
    allsets = []
    for s in itertools.combinations(range(C), k):
        allsets.append((sum(min(m[e][c] for c in s) for e in rows), s))
    allsets.sort()
    return allsets, len(rows)


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_pow2_closed_form_all_subsets(seed):
    _, m = synth.pow2(seed, n_cfg=9, n_env=7, max_exp=5)
    o = Oracle(pow2_matrix(m))
    E = m.shape[0]
    for k in range(1, 10):
        for s in itertools.combinations(range(9), k):
            want = 2.0 ** (-sum(min(m[e][c] for c in s) for e in range(E)) / E)
            assert o.score(list(s)) == pytest.approx(want, rel=1e-15)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_pow2_exhaustive_matches_brute_force_with_ties(seed):
    """pow2 data is tie-rich: pins the lexicographic tie-break (reading c5)."""
    _, m = synth.pow2(seed, n_cfg=12, n_env=6, max_exp=3)
    o = Oracle(pow2_matrix(m))
    mask = np.array([1, 0, 1, 1, 0, 1], np.uint8)
    for msk in (None, mask):
        for k in (1, 2, 3, 4):
            allsets, E = brute_force_pow2(m, k, msk)
            b, gb, ru, gr = o.exhaustive(k, mask=msk, threads=3)
            assert b == allsets[0][1] and ru == allsets[1][1]
            assert gb == pytest.approx(2.0 ** (-allsets[0][0] / E), rel=1e-15)
            assert gr == pytest.approx(2.0 ** (-allsets[1][0] / E), rel=1e-15)


def test_tiny_all_subsets_brute_force():
    """BASELINE config 1: brute force over all 2^16 subsets (grouped by size)."""
    T, dev = synth.tiny(1)
    o = Oracle(T, dev)
    lg = np.log(T.astype(np.float64))
    # independent route: log T and row minimum via numpy, sum of log slowdowns
    ell = lg - lg.min(axis=1, keepdims=True)
    best = {}
    for mask_bits in range(1, 1 << 16):
        s = [c for c in range(16) if mask_bits >> c & 1]
        v = ell[:, s].min(axis=1).sum()
        k = len(s)
        cur = best.get(k)
        if cur is None or (v, s) < cur:
            best[k] = (v, s)
    for k in (1, 2, 3, 4):
        b, gb, _, _ = o.exhaustive(k)
        v, s = best[k]
        assert b == tuple(s)
        assert gb == pytest.approx(math.exp(-v / 8), rel=1e-12)
    b, gb, _, _ = o.exhaustive(16)
    assert gb == 1.0 and b == tuple(range(16))


# --------------------------------------------------------------------------
# invariants
# --------------------------------------------------------------------------

def test_full_set_and_best_cover_give_one():
    T, _ = synth.small_matrix(5, n_cfg=40, n_dev=2, n_inputs=6)
    o = Oracle(T)
    assert o.score(list(range(40))) == 1.0
    cover = sorted(set(int(c) for c in np.argmin(T, axis=1)))
    assert o.score(cover) == 1.0
    # monotone in k: best G non-decreasing; best k=1 is a column mean argmax
    prev = 0.0
    for k in (1, 2, 3):
        _, gb, _, _ = o.exhaustive(k)
        assert gb >= prev
        prev = gb
    col = np.log(T.astype(np.float64)) - np.log(T.astype(np.float64)).min(1, keepdims=True)
    assert o.exhaustive(1)[0] == (int(np.argmin(col.sum(0))),)


def test_scale_and_permutation_invariance():
    T, _ = synth.small_matrix(7, n_cfg=30, n_dev=3, n_inputs=4)
    o = Oracle(T)
    scale = np.exp(np.random.default_rng(0).uniform(-3, 3, size=(T.shape[0], 1)))
    scale = np.ldexp(1.0, np.round(np.log2(scale)).astype(int))   # exact powers of two
    o2 = Oracle((T * scale).astype(np.float32))
    b, gb, ru, gr = o.exhaustive(3)
    b2, gb2, ru2, gr2 = o2.exhaustive(3)
    assert (b, ru) == (b2, ru2) and gb == gb2 and gr == gr2
    # config permutation: same optimum under the index map (no ties in this data)
    perm = np.random.default_rng(1).permutation(30)
    o3 = Oracle(np.ascontiguousarray(T[:, perm]))
    b3, gb3, _, _ = o3.exhaustive(3)
    assert tuple(sorted(int(perm[c]) for c in b3)) == b
    assert gb3 == pytest.approx(gb, rel=1e-14)
    # env permutation
    ep = np.random.default_rng(2).permutation(T.shape[0])
    o4 = Oracle(np.ascontiguousarray(T[ep]))
    b4, gb4, _, _ = o4.exhaustive(3)
    assert b4 == b and gb4 == pytest.approx(gb, rel=1e-14)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_greedy_properties(seed):
    T, dev = synth.small_matrix(seed, n_cfg=14, n_dev=2, n_inputs=5)
    o = Oracle(T, dev)
    E = T.shape[0]
    idx, gt, gp = o.greedy(6)
    # greedy k=1 = exhaustive k=1
    assert (idx[0],) == o.exhaustive(1)[0]
    # prefix consistency: greedy(k) = first k of greedy(6)
    for k in range(1, 6):
        assert o.greedy(k)[0] == idx[:k]
    # init continuation: greedy from the first t picks continues identically
    for t in range(1, 6):
        assert o.greedy(6 - t, init=idx[:t])[0] == idx[t:]
    # scores along the trace equal the set scores
    for t in range(6):
        assert gt[t] == pytest.approx(o.score(idx[:t + 1]), rel=1e-14)
    # facility location: marginal gains of L = E log G are non-increasing
    # (submodularity), and greedy >= (1 - 1/e) OPT for f(S) = L(S) - L_min
    L = E * np.log(gt)
    gains = np.diff(L)
    assert np.all(gains[1:] <= gains[:-1] + 1e-12)
    lmin = np.log(T.astype(np.float64)).min(1, keepdims=True) - np.log(T.astype(np.float64))
    f0 = lmin.min(axis=1).sum()          # L of the worst possible "set" baseline
    for k in (2, 3):
        opt = E * math.log(o.exhaustive(k)[1])
        assert (L[k - 1] - f0) >= (1 - 1 / math.e) * (opt - f0) - 1e-9


@pytest.mark.parametrize("g", [1, 2, 3])
def test_planted_recovery(g):
    for seed in range(1, 21):
        T, dev, cols = synth.planted(seed, n_cfg=15, n_env=12, g=g, gamma=2.0)
        o = Oracle(T, dev)
        b, gb, ru, gr = o.exhaustive(g)
        assert b == tuple(cols) and gb == 1.0
        assert gr <= 2.0 ** (-1.0 / 12) + 1e-12     # any other set misses a block env by >= gamma


def test_holdout_clone_and_scopes():
    T, dev = synth.small_matrix(3, n_cfg=20, n_dev=2, n_inputs=6)
    # device 1 is a clone of device 0 (identical rows)
    T[6:12] = T[0:6]
    o = Oracle(T, dev)
    for method in (0, 1):
        idx, gtr, gun, gkn, kidx = o.holdout(1, 2, method=method)
        assert gun == gkn and idx == kidx
        assert gtr == gun
    # holdout = select on masked scope + score on the complementary scope
    T, dev = synth.small_matrix(4, n_cfg=20, n_dev=3, n_inputs=4)
    o = Oracle(T, dev)
    idx, gtr, gun, gkn, kidx = o.holdout(2, 2, method=1)
    assert gkn >= gun
    assert list(o.exhaustive(2, mask=(dev != 2))[0]) == idx
    assert o.score(idx, mask=(dev == 2)) == gun


def test_missing_cells_penalty():
    # one missing cell -> global max slowdown (reading c4)
    T = np.array([[1.0, 2.0, 8.0, np.nan],
                  [4.0, 1.0, 2.0, 2.0],
                  [1.0, 1.0, 1.0, 4.0]], np.float32)
    o = Oracle(T)
    assert o.penalty == 8.0
    assert o.score([3]) == pytest.approx((1 / 8 * 1 / 2 * 1 / 4) ** (1 / 3), rel=1e-15)


def test_errors():
    with pytest.raises(OracleError) as ei:
        Oracle(np.array([[1.0, -1.0]], np.float32))
    assert ei.value.code == -7
    with pytest.raises(OracleError) as ei:
        Oracle(np.array([[np.nan, np.inf]], np.float32))
    assert ei.value.code == -7
    o = Oracle(np.array([[1.0, 2.0]], np.float32))
    with pytest.raises(OracleError) as ei:
        o.score([0], mask=np.zeros(1, np.uint8))
    assert ei.value.code == -6
    with pytest.raises(OracleError) as ei:
        o.exhaustive(3)
    assert ei.value.code == -1


def test_counting_pins():
    """1,343 Quadro variants, best 3, 10 inputs -> "over 24 billion"."""
    assert 1343 ** 3 * 10 == 24_223_006_070 > 24e9
    assert math.comb(1343, 3) * 10 == 4_028_153_910
    assert math.comb(1775, 2) == 1_574_425
    assert math.comb(1775, 3) == 930_485_175
    assert sum(1775 - t for t in range(24)) == 42_324


def test_holdout_known_leg_hand():
    """The 'known' baseline of Sec. 5.8 ("combinations ... selected on the
    known device") is selected on the HELD-OUT envs, the unseen set on the
    others.  Hand-worked pow2 fixture, 2 devices x 2 envs, 3 configs (log2 slowdowns):
        device 0 envs: c0 = 0, c1 = 3, c2 = 1      -> train selects c0 (k=1)
        device 1 envs: c0 = 2, c1 = 0, c2 = 1      -> known selects c1, G_known = 1
    G_unseen = G({c0} on device 1) = 2^-2 exactly; G_train = 1 exactly.
    A holdout whose known leg selected on the train scope would report {c0}, 1/4."""
    m = np.array([[0, 3, 1], [0, 3, 1], [2, 0, 1], [2, 0, 1]])
    dev = np.array([0, 0, 1, 1], np.int32)
    o = Oracle(pow2_matrix(m), dev)
    for method in (0, 1):
        idx, gtr, gun, gkn, kidx = o.holdout(1, 1, method=method)
        assert idx == [0] and kidx == [1]
        assert gtr == 1.0 and gkn == 1.0 and gun == pytest.approx(0.25, rel=1e-15)
        # the other fold: train on device 1 -> c1; unseen on device 0 = 2^-3; known c0
        idx, gtr, gun, gkn, kidx = o.holdout(0, 1, method=method)
        assert idx == [1] and kidx == [0]
        assert gtr == 1.0 and gkn == 1.0 and gun == pytest.approx(0.125, rel=1e-15)
    # k=2 on the 3-device variant: known = the held-out device's own best pair
    m3 = np.array([[0, 3, 1, 2], [1, 0, 3, 2], [3, 3, 0, 2], [3, 3, 2, 0]])
    dev3 = np.array([0, 1, 2, 2], np.int32)
    o3 = Oracle(pow2_matrix(m3), dev3)
    idx, gtr, gun, gkn, kidx = o3.holdout(2, 2, method=1)
    assert idx == [0, 1] and gtr == 1.0             # c0, c1 are exact on devices 0, 1
    assert kidx == [2, 3] and gkn == 1.0            # c2, c3 exact on device 2's two envs
    assert gun == pytest.approx(2.0 ** -3, rel=1e-15)   # {c0,c1} on device 2: min(3,3) twice
