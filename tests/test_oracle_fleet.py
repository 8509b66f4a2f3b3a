"""Pins for the oracle's fleet objective (Eq. 2): hand-worked
fixture, SPEC worked examples, an event-level simulation of the
fleet, brute force over all subsets, invariants."""
import heapq
import itertools
from fractions import Fraction

import numpy as np
import pytest

from conftest import read_golden
from oracle import Oracle
from paper_2507_15277_b200 import synth


def fixture():
    g = read_golden("fleet_hand.txt")
    dev = np.array([int(x) for x in next(r for r in g if r[0] == "dev")[1:]], np.int32)
    qenv = [float(x) for x in next(r for r in g if r[0] == "qenv")[1:]]
    qdev = [float(x) for x in next(r for r in g if r[0] == "qdev")[1:]]
    T = np.array([[float(x) for x in r[1:]] for r in g if r[0] == "t"], np.float32)
    o = Oracle(T, dev)
    o.set_fleet(qdev, qenv)
    return g, o


def test_fleet_hand_fixture():
    g, o = fixture()
    for r in g:
        if r[0] == "rate":
            s = [int(x) for x in r[1].split(",")]
            assert o.fleet_rate(s) == pytest.approx(float(Fraction(r[2])), rel=1e-15)
        if r[0] == "best":
            k = int(r[1].split("=")[1])
            b, rb, ru, rr = o.fleet_exhaustive(k)
            assert b == tuple(int(x) for x in r[2].split(","))
            assert ru == tuple(int(x) for x in r[4].split(","))
        if r[0] == "greedy":
            idx, rt, gp = o.fleet_greedy(2)
            assert idx == [int(r[1]), int(r[2])]
            assert gp[1] == pytest.approx(7 / 120, rel=1e-12)
        if r[0] == "geomean_best_k1":
            assert o.exhaustive(1)[0] == (int(r[1]),)


def test_spec_examples():
    # one device (quantity 1), one input (quantity 1), best runtime 2.0 ms -> 0.5 tasks/ms
    o = Oracle(np.array([[2.0, 5.0]], np.float32), np.array([0], np.int32))
    o.set_fleet([1.0], [1.0])
    assert o.fleet_rate([0, 1]) == 0.5
    # doubling every quantity(d) doubles the rate
    T, dev = synth.small_matrix(2, n_cfg=12, n_dev=3, n_inputs=4)
    o = Oracle(T, dev)
    rng = np.random.default_rng(1)
    qd, qe = rng.uniform(1, 5, 3), rng.uniform(1, 3, len(dev))
    o.set_fleet(qd, qe)
    r1 = o.fleet_rate([1, 4, 7])
    o.set_fleet(2 * qd, qe)
    assert o.fleet_rate([1, 4, 7]) == pytest.approx(2 * r1, rel=1e-15)


def simulate(T_sel, dev, qdev, qenv, horizon):
    """Event-level fleet simulation: quantity(d) identical devices of
    each type; each device runs its task = every input i of its device,
    quantity(i) times, back to back; count tasks completed by `horizon`."""
    events = []
    for d in range(len(qdev)):
        envs = [e for e in range(len(dev)) if dev[e] == d]
        runs = [T_sel[e] for e in envs for _ in range(int(qenv[e]))]
        for unit in range(int(qdev[d])):
            heapq.heappush(events, (0.0, d, unit, 0, runs))
    done = 0
    while events:
        t, d, unit, pos, runs = heapq.heappop(events)
        t += runs[pos]
        if t > horizon:
            continue
        pos += 1
        if pos == len(runs):
            done += 1
            pos = 0
        heapq.heappush(events, (t, d, unit, pos, runs))
    return done / horizon


def test_event_simulation():
    T, dev = synth.small_matrix(3, n_cfg=10, n_dev=2, n_inputs=3)
    qdev = np.array([3.0, 2.0])
    qenv = np.array([1.0, 2.0, 3.0] * 2)
    o = Oracle(T, dev)
    o.set_fleet(qdev, qenv)
    S = [2, 5]
    y = T[:, S].astype(np.float64).min(axis=1)
    tau = [sum(y[e] * qenv[e] for e in range(len(dev)) if dev[e] == d) for d in range(2)]
    horizon = 2000.0 * max(tau)
    sim = simulate(y, dev, qdev, qenv, horizon)
    R = o.fleet_rate(S)
    assert abs(sim - R) <= qdev.sum() / horizon * 1.0001


def test_brute_force_and_invariants():
    T, dev = synth.small_matrix(4, n_cfg=9, n_dev=3, n_inputs=3)
    T[2, 4] = np.nan                                       # a missing cell (reading c4)
    o = Oracle(T, dev)
    rng = np.random.default_rng(2)
    qd, qe = rng.uniform(1, 4, 3), rng.integers(1, 4, len(dev)).astype(float)
    o.set_fleet(qd, qe)
    Tp = T.astype(np.float64).copy()
    miss = ~np.isfinite(Tp)
    Tp[miss] = (o.penalty * o.best[:, None] * np.ones_like(Tp))[miss]
    for k in (1, 2, 3):
        scores = []
        for s in itertools.combinations(range(9), k):
            y = Tp[:, list(s)].min(axis=1)
            den = np.bincount(dev, weights=y * qe, minlength=3)
            scores.append((-(qd / den).sum(), s))
        scores.sort()
        b, rb, ru, rr = o.fleet_exhaustive(k)
        assert b == scores[0][1] and ru == scores[1][1]
        assert rb == pytest.approx(-scores[0][0], rel=1e-13)
    # monotone under set inclusion; the full set reaches the row-minimum rate
    assert o.fleet_rate([0, 1, 2]) >= o.fleet_rate([0, 1]) >= o.fleet_rate([0])
    full = o.fleet_rate(list(range(9)))
    den = np.bincount(dev, weights=Tp.min(axis=1) * qe, minlength=3)
    assert full == pytest.approx((qd / den).sum(), rel=1e-14)
    # greedy k=1 = exhaustive k=1; greedy value >= (1-1/e) ... not submodular: only check k=1
    assert o.fleet_greedy(1)[0] == [o.fleet_exhaustive(1)[0][0]]


def test_missing_cell_costs_penalty_times_best():
    """Reading c4 carried to Eq. 2: a missing cell costs
    penalty x best[e], penalty = the dataset-max slowdown.  Hand fixture:
        env 0 (device 0): T = [1, NaN]   best 1
        env 1 (device 1): T = [2, 1]     best 1      -> penalty = 2/1 = 2
    q = 1 everywhere.  R({c1}) = 1/(2*1) + 1/1 = 3/2 (the missing cell costs 2 ms);
    R({c0}) = 1/1 + 1/2 = 3/2; R({c0, c1}) = 1/1 + 1/1 = 2."""
    T = np.array([[1.0, np.nan], [2.0, 1.0]], np.float32)
    o = Oracle(T, np.array([0, 1], np.int32))
    o.set_fleet([1.0, 1.0], [1.0, 1.0])
    assert o.penalty == 2.0
    assert o.fleet_rate([1]) == 1.5
    assert o.fleet_rate([0]) == 1.5
    assert o.fleet_rate([0, 1]) == 2.0
    # a larger penalty (env 1's worst cell 8x its best) moves only the missing cell's cost
    T2 = np.array([[1.0, np.nan], [8.0, 1.0]], np.float32)
    o2 = Oracle(T2, np.array([0, 1], np.int32))
    o2.set_fleet([1.0, 1.0], [1.0, 1.0])
    assert o2.fleet_rate([1]) == pytest.approx(1 / 8 + 1, rel=1e-15)
    b, rb, ru, rr = o2.fleet_exhaustive(1)
    assert b == (0,) and rb == pytest.approx(1 + 1 / 8, rel=1e-15)   # ties by R; lex-first c0


def test_parallel_exhaustive_equals_sequential():
    """or_fleet_exhaustive_par (first index dealt to threads, used for the full-size
    golden) returns exactly the sequential search's best, runner-up and rates."""
    for seed in (13, 14):
        T, dev = synth.small_matrix(seed, n_cfg=36, n_dev=3, n_inputs=6)
        o = Oracle(T, dev)
        o.set_fleet([1.0, 2.0, 3.0], np.linspace(1.0, 2.0, T.shape[0]))
        for k in (1, 2, 3):
            for th in (1, 3, 8):
                assert o.fleet_exhaustive_par(k, threads=th) == o.fleet_exhaustive(k)
