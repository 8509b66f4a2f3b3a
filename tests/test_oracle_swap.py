"""Pins for the oracle's swap local search."""
import itertools

import numpy as np
import pytest

from conftest import read_golden
from oracle import Oracle
from paper_2507_15277_b200 import synth
from test_oracle import pow2_matrix


def test_hand_fixture():
    g = read_golden("greedy_vs_opt.txt")
    m = np.array([[int(x) for x in r[1:]] for r in g if r[0] == "m"])
    o = Oracle(pow2_matrix(m))
    row = next(r for r in g if r[0] == "swap")
    s, G, moves = o.swap_search(2)
    assert s == tuple(int(x) for x in row[1].split(",")) and moves == int(row[3]) and G == 1.0


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_local_optimum_and_improvement(seed):
    T, dev = synth.small_matrix(seed, n_cfg=14, n_dev=2, n_inputs=5)
    o = Oracle(T, dev)
    for k in (2, 3, 4):
        s, G, moves = o.swap_search(k)
        gidx, gt, _ = o.greedy(k)
        assert G >= gt[-1] - 1e-15                      # never worse than its greedy seed
        assert G == pytest.approx(o.score(list(s)), rel=1e-14)
        # local optimum: brute force over every single swap
        for a in s:
            for b in range(14):
                if b in s:
                    continue
                t = sorted(set(s) - {a} | {b})
                assert o.score(t) <= G + 1e-15
        # and never better than the exhaustive optimum
        assert G <= o.exhaustive(k)[1] + 1e-15


def test_planted_recovery_and_init():
    for seed in range(1, 11):
        T, dev, cols = synth.planted(seed, n_cfg=20, n_env=12, g=3, gamma=2.0)
        o = Oracle(T, dev)
        s, G, _ = o.swap_search(3)
        assert s == tuple(cols) and G == 1.0
    # starting from an explicit set
    T, dev = synth.small_matrix(5, n_cfg=12, n_dev=2, n_inputs=4)
    o = Oracle(T, dev)
    s, G, moves = o.swap_search(3, init=[0, 1, 2], max_moves=0)
    assert s == (0, 1, 2) and moves == 0


def test_tied_best_move_takes_smallest_tuple():
    """S:L258-266 + reading c5: among equally good swaps the lexicographically
    smallest resulting sorted tuple wins.  Hand fixture (log2 slowdowns, 2 envs):
        c0 = [0, 3], c1 = [3, 0], c2 = [5, 5], c3 = [0, 3]   (c3 duplicates c0)
    From {0, 3} (s = 3) the swaps reach {1,3}: 0, {2,3}: 3, {0,1}: 0, {0,2}: 3, in
    that enumeration order; {1,3} and {0,1} tie at the optimum s = 0, so the move
    is to (0, 1) -- a first-encountered rule would stop at (1, 3).  One move, G = 1."""
    o = Oracle(pow2_matrix(np.array([[0, 3, 5, 0], [3, 0, 5, 3]])))
    s, G, moves = o.swap_search(2, init=[0, 3])
    assert s == (0, 1) and G == 1.0 and moves == 1
    s, G, moves = o.swap_search(2, init=[3, 0])        # init order is irrelevant
    assert s == (0, 1) and moves == 1
