"""GPU parity for the fleet objective (Eq. 2) through the
C ABI against the CPU oracle's fleet functions (tests/test_oracle_fleet.py pins)."""
from fractions import Fraction

import numpy as np
import pytest

from conftest import read_golden
from oracle import Oracle
from paper_2507_15277_b200 import pt, synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
RTOL = 1e-9
GAP = 1e-9


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def both(T, dev, qd, qe):
    o = Oracle(T, dev)
    o.set_fleet(qd, qe)
    ctx = pt.pt_load_perf(T, dev)
    pt.pt_set_fleet(ctx, qd, qe)
    return o, ctx


def check_exh(o, ctx, k, mask=None, shards=1):
    b, rb, ru, rr = o.fleet_exhaustive(k, mask=mask)
    if shards == 1:
        r = pt.pt_exhaustive_best(ctx, k, env_mask=mask, objective=pt.PT_OBJ_FLEET)
        got_b, got_R = r["best"], r["G"]
    else:
        ss, tt = [], []
        for s in range(shards):
            r = pt.pt_exhaustive_best(ctx, k, env_mask=mask, shard_rank=s, shard_count=shards,
                                      objective=pt.PT_OBJ_FLEET)
            for sv, tup in zip(r["s"], (r["best"], r["runner"])):
                ss.append(sv)
                tt.append(tup if tup is not None else (-1,) * k)
        got_b, _, (c1, _) = pt.pt_merge_top2(ss, tt, k)
        got_R = 1.0 / c1
    assert got_R == pytest.approx(rb, rel=RTOL)
    if ru is None or rb - rr > GAP * rb:
        assert got_b == b
    else:
        assert o.fleet_rate(list(got_b), mask=mask) >= rb * (1 - GAP)


def test_hand_fixture():
    g = read_golden("fleet_hand.txt")
    dev = np.array([int(x) for x in next(r for r in g if r[0] == "dev")[1:]], np.int32)
    qe = [float(x) for x in next(r for r in g if r[0] == "qenv")[1:]]
    qd = [float(x) for x in next(r for r in g if r[0] == "qdev")[1:]]
    T = np.array([[float(x) for x in r[1:]] for r in g if r[0] == "t"], np.float32)
    o, ctx = both(T, dev, qd, qe)
    for r in g:
        if r[0] == "rate":
            s = np.array([[int(x) for x in r[1].split(",")]], np.int32)
            got = pt.pt_score_sets(ctx, s, objective=pt.PT_OBJ_FLEET)[0]
            assert got == pytest.approx(float(Fraction(r[2])), rel=1e-15)
        if r[0] == "best":
            k = int(r[1].split("=")[1])
            res = pt.pt_exhaustive_best(ctx, k, objective=pt.PT_OBJ_FLEET)
            assert res["best"] == tuple(int(x) for x in r[2].split(","))
            assert res["runner"] == tuple(int(x) for x in r[4].split(","))
        if r[0] == "greedy":
            idx, rt, gp = pt.pt_greedy_select(ctx, 2, objective=pt.PT_OBJ_FLEET)
            assert idx == [int(r[1]), int(r[2])]
            assert gp[1] == pytest.approx(7 / 120, rel=1e-12)


@pytest.mark.parametrize("seed", [1, 2])
def test_small_random(seed):
    T, dev = synth.small_matrix(seed, n_cfg=120, n_dev=4, n_inputs=9)
    T[5, 17] = np.nan
    rng = np.random.default_rng(seed)
    qd, qe = rng.uniform(1, 5, 4), rng.integers(1, 4, len(dev)).astype(float)
    o, ctx = both(T, dev, qd, qe)
    sets = rng.integers(0, 120, size=(40, 3)).astype(np.int32)
    np.testing.assert_allclose(pt.pt_score_sets(ctx, sets, objective=pt.PT_OBJ_FLEET),
                               o.fleet_rate(sets), rtol=1e-12)
    mask = (dev != 2).astype(np.uint8)
    np.testing.assert_allclose(pt.pt_score_sets(ctx, sets, env_mask=mask, objective=pt.PT_OBJ_FLEET),
                               o.fleet_rate(sets, mask=mask), rtol=1e-12)
    for k in (1, 2, 3):
        check_exh(o, ctx, k)
    check_exh(o, ctx, 2, mask=mask)
    check_exh(o, ctx, 3, shards=3)
    idx, rt, gp = pt.pt_greedy_select(ctx, 8, objective=pt.PT_OBJ_FLEET)
    oidx, ort, ogp = o.fleet_greedy(8)
    for t in range(8):
        assert rt[t] == pytest.approx(o.fleet_rate(idx[:t + 1]), rel=1e-12)
    if np.all(ogp > GAP * ort):
        assert idx == oidx
    idx_m, rt_m, _ = pt.pt_greedy_select(ctx, 4, env_mask=mask, objective=pt.PT_OBJ_FLEET)
    assert idx_m == o.fleet_greedy(4, mask=mask)[0]


def test_paper_shape():
    T, dev = synth.paper_matrix(1)
    qd = np.array([5.0, 2.0, 1.0, 3.0, 4.0])                   # fleet mix (invented)
    qe = np.ones(len(dev))                                    # one of each input per task
    o, ctx = both(T, dev, qd, qe)
    idx, rt, gp = pt.pt_greedy_select(ctx, 5, objective=pt.PT_OBJ_FLEET)
    assert idx == o.fleet_greedy(5)[0]
    check_exh(o, ctx, 2)
    # fleet and geomean pick different sets (the rate is dominated by fast devices)
    assert pt.pt_exhaustive_best(ctx, 1, objective=pt.PT_OBJ_FLEET)["best"] != \
        pt.pt_exhaustive_best(ctx, 1)["best"]


def test_errors():
    T, dev = synth.tiny(1)
    ctx = pt.pt_load_perf(T, dev)
    with pytest.raises(pt.PTError) as ei:
        pt.pt_greedy_select(ctx, 2, objective=pt.PT_OBJ_FLEET)
    assert ei.value.code == pt.PT_EINVAL
    with pytest.raises(pt.PTError):
        pt.pt_set_fleet(ctx, [1.0], np.ones(len(dev)))        # device id 4 out of range
    with pytest.raises(pt.PTError):
        pt.pt_set_fleet(ctx, np.ones(5), -np.ones(len(dev)))


def test_tiled_fleet_path():
    """The full-scope fleet search runs the (min,+) tiled kernel with the per-device
    fold (exh_kernel 3); a masked scope the thread-per-subset fp64 search (2).
    Uneven device segments (9 envs each, padded to 64-env stages) and a missing cell."""
    T, dev = synth.small_matrix(4, n_cfg=300, n_dev=4, n_inputs=9)
    T[7, 33] = np.nan
    rng = np.random.default_rng(4)
    qd, qe = rng.uniform(1, 5, 4), rng.integers(1, 4, len(dev)).astype(float)
    o, ctx = both(T, dev, qd, qe)
    for k in (2, 3):
        check_exh(o, ctx, k)
        assert pt.pt_get_stats(ctx)["exh_kernel"] == 3
        check_exh(o, ctx, k, shards=5)
    check_exh(o, ctx, 2, mask=(dev != 1).astype(np.uint8))
    assert pt.pt_get_stats(ctx)["exh_kernel"] == 2


def test_paper_fleet_k3_golden():
    """Config 3b with the fleet objective (Eq. 2): k=2 and k=3 over 1,775 x 320 against
    the oracle's full search (tests/golden/paper_exhaustive.json, written by
    scripts/make_golden.py --fleet, which calls only oracle/)."""
    import json
    import os
    from conftest import GOLDEN
    gold = json.load(open(os.path.join(GOLDEN, "paper_exhaustive.json")))
    if "seed1_fleet_k3" not in gold:
        pytest.skip("fleet golden not generated")
    T, dev = synth.paper_matrix(1)
    qd = np.array(gold["seed1_fleet_k3"]["q_dev"])
    ctx = pt.pt_load_perf(T, dev)
    pt.pt_set_fleet(ctx, qd, np.ones(len(dev)))
    for k in (2, 3):
        g = gold[f"seed1_fleet_k{k}"]
        r = pt.pt_exhaustive_best(ctx, k, objective=pt.PT_OBJ_FLEET)
        st = pt.pt_get_stats(ctx)
        assert st["exh_kernel"] == 3
        assert r["G"] == pytest.approx(g["R"], rel=RTOL) and r["G_runner"] == pytest.approx(g["R_runner"], rel=RTOL)
        if g["R"] - g["R_runner"] > GAP * g["R"]:
            assert r["best"] == tuple(g["best"])
        assert r["runner"] == tuple(g["runner"]) or abs(r["G_runner"] - g["R_runner"]) <= GAP * g["R"]
    # 8 shards through the library's own exchange + merge (thread-emulated ranks)
    r8 = []
    for rank in range(8):
        r8.append(pt.pt_exhaustive_best(ctx, 3, shard_rank=rank, shard_count=8, objective=pt.PT_OBJ_FLEET))
    ss = [x for r in r8 for x in r["s"]]
    tt = [t if t is not None else (-1, -1, -1) for r in r8 for t in (r["best"], r["runner"])]
    b, ru, (c1, c2) = pt.pt_merge_top2(ss, tt, 3)
    assert b == tuple(gold["seed1_fleet_k3"]["best"]) and 1.0 / c1 == pytest.approx(gold["seed1_fleet_k3"]["R"], rel=RTOL)


def test_fleet_many_small_devices_falls_back():
    """12 devices of 5 environments: each segment padded to a 64-env stage gives 768+ rows,
    beyond the tiled kernel's shared-memory A tile -> the fp64 thread-per-subset search,
    still equal to the oracle."""
    T, _ = synth.small_matrix(17, n_cfg=80, n_dev=13, n_inputs=5)
    dev = np.repeat(np.arange(13, dtype=np.int32), 5)        # 13 device ids, 5 envs each
    rng = np.random.default_rng(17)
    qd, qe = rng.uniform(1, 3, 13), np.ones(len(dev))
    o, ctx = both(T, dev, qd, qe)
    check_exh(o, ctx, 2)
    assert pt.pt_get_stats(ctx)["exh_kernel"] == 2
