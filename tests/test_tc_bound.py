"""CPU pins of the threshold-count filter's mathematics, independent of
the CUDA kernel: with thresholds t_j = j u (j = 1..nt) and Q(x) = u #{j : x >= t_j},

  * Q(min_c l_c) = min_c Q(l_c), and [min_c l_c >= t] = AND_c [l_c >= t];
  * u P(S) <= s(S) for every set S, P(S) = the 0/1 dot product of the thresholded
    row of S's first k-1 members (ANDed) and of its last member;
  * hence every set of the exact top-2 (the oracle's exhaustive search) has
    u P <= s_(2) <= tau for any tau >= s_(2): the filter cannot drop an answer.

Exact scores come from the oracle (s = -E log G); the log-slowdowns from the
oracle's own normalisation (l = -logeff); the bound is computed here with numpy."""
import itertools
import math

import numpy as np
import pytest

from oracle import Oracle
from paper_2507_15277_b200 import synth

pytestmark = pytest.mark.filterwarnings("ignore")


def thresholded(l, u, nt):
    """[l >= j u] for j = 1..nt, concatenated along the environment axis: [C][nt E]."""
    return np.concatenate([(l >= (j + 1) * u) for j in range(nt)], axis=1).astype(np.int64)


@pytest.mark.parametrize("seed,nt,alpha", [(1, 1, 1.5), (2, 2, 1.5), (3, 3, 2.0), (4, 2, 0.7)])
def test_threshold_count_is_a_lower_bound(seed, nt, alpha):
    T, dev = synth.small_matrix(seed, n_cfg=40, n_dev=3, n_inputs=8)
    o = Oracle(T, dev)
    l = -o.logeff.T.copy()                       # [C][E] log-slowdowns >= 0
    C, E = l.shape
    # every 3-set: exact score from the oracle, bound from the thresholded bits
    sets = np.array(list(itertools.combinations(range(C), 3)), dtype=np.int32)
    s = -E * np.log(o.score(sets))
    best, gb, runner, gr = o.exhaustive(3)
    s2 = -E * math.log(gr)
    u = float(np.float32(alpha * s2 / E))        # a float step, as k_tc_const
    bits = thresholded(l, u, nt)
    A = bits[sets[:, 0]] & bits[sets[:, 1]]      # the row's bits = AND of its members
    P = (A * bits[sets[:, 2]]).sum(axis=1)       # 0/1 dot product
    lb = u * P
    assert np.all(lb <= s * (1 + 1e-12) + 1e-12), "threshold-count bound above an exact score"
    # the top-2 survive any tau >= s_(2)
    key = {tuple(x): i for i, x in enumerate(sets.tolist())}
    for t in (best, runner):
        assert lb[key[tuple(t)]] <= s2 * (1 + 1e-12)
    # and the bound is not vacuous: it excludes most sets
    assert (lb <= s2).mean() < 0.5


def test_min_commutes_with_the_floor_quantisation():
    rng = np.random.default_rng(5)
    x = rng.exponential(0.5, size=(6, 1000))
    u, nt = 0.17, 3
    Q = lambda v: u * sum((v >= (j + 1) * u) for j in range(nt))   # noqa: E731
    assert np.array_equal(Q(x.min(axis=0)), np.min(np.stack([Q(r) for r in x]), axis=0))
    for j in range(nt):
        t = (j + 1) * u
        assert np.array_equal(x.min(axis=0) >= t, np.logical_and.reduce(x >= t, axis=0))
    assert np.all(Q(x) <= x)
