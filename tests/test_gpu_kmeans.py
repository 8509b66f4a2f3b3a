"""GPU parity for the k-means selector: the whole Lloyd
trajectory is computed in the same order without FMA contraction, so the
selection AND the iteration count must equal the oracle's exactly."""
import numpy as np
import pytest

from conftest import read_golden
from oracle import Oracle
from paper_2507_15277_b200 import pt, synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_hand_fixture():
    g = read_golden("kmeans_hand.txt")
    T = np.array([[float(x) for x in r[1:]] for r in g if r[0] == "t"], np.float32)
    ctx = pt.pt_load_perf(T)
    sel, G, it = pt.pt_kmeans_select(ctx, 2)
    row = next(r for r in g if r[0] == "select")
    assert sel == tuple(int(x) for x in row[1].split(",")) and it == int(row[3])


@pytest.mark.parametrize("seed,C,nd,ni", [(1, 60, 3, 6), (2, 300, 4, 12), (3, 130, 2, 40)])
def test_random(seed, C, nd, ni):
    T, dev = synth.small_matrix(seed, n_cfg=C, n_dev=nd, n_inputs=ni)
    T[1, 3] = np.nan
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    for k in (1, 2, 5, 9):
        sel, G, it = pt.pt_kmeans_select(ctx, k)
        osel, oit, _ = o.kmeans(k)
        assert sel == osel and it == oit
        assert G == pytest.approx(o.score(list(sel)), rel=1e-12)
    mask = (dev != 0).astype(np.uint8)
    assert pt.pt_kmeans_select(ctx, 4, env_mask=mask)[0] == o.kmeans(4, mask=mask)[0]


def test_paper_shape():
    T, dev = synth.paper_matrix(1)
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    for k in (3, 10, 24):
        sel, G, it = pt.pt_kmeans_select(ctx, k)
        osel, oit, _ = o.kmeans(k)
        assert sel == osel and it == oit


def test_many_points_per_pass_init():
    """1,280 environments: above the pairwise-init limit (1,024 points), so the
    maximin initialisation takes one distance pass per centroid."""
    T, dev = synth.scaled(4, n_cfg=48, n_dev=20, n_inputs=64)
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    for k in (3, 7):
        sel, G, it = pt.pt_kmeans_select(ctx, k)
        osel, oit, _ = o.kmeans(k)
        assert sel == osel and it == oit


def test_k32_many_tiles_and_chunks():
    """k = 32 (8 warps of 4 centroids), 2,048 points (64 point tiles), 2,050 configs
    (33 staged chunks, the last one config wide: the bulk-copy padding double): the device
    Lloyd loop stays bit-identical to the oracle (selection and iteration count)."""
    T, dev = synth.scaled(5, n_cfg=2049, n_dev=32, n_inputs=64)
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    for k in (32, 5):
        sel, G, it = pt.pt_kmeans_select(ctx, k)
        osel, oit, _ = o.kmeans(k)
        assert sel == osel and it == oit
    sel, G, it = pt.pt_kmeans_select(ctx, 32, max_iter=3)    # stopped by max_iter, not convergence
    osel, oit, _ = o.kmeans(32, max_iter=3)
    assert sel == osel and it == oit == 3


def test_given_start_reseed():
    """pt_kmeans_select_from against or_kmeans_from: the hand fixture whose start empties
    a cluster (the re-seed rule, tests/test_oracle_kmeans.py), and random scopes started
    with one centroid far from every point (a re-seed on the first pass)."""
    T = np.array([[1, 5], [1, 6], [4, 1]], np.float32)
    init = np.array([[1.0, 5.5], [100.0, 100.0]])
    ctx = pt.pt_load_perf(T)
    sel, G, it = pt.pt_kmeans_select_from(ctx, init)
    assert (sel, it) == ((0, 1), 3)
    for seed, C, nd, ni in ((1, 60, 3, 6), (2, 300, 4, 12)):
        T, dev = synth.small_matrix(seed, n_cfg=C, n_dev=nd, n_inputs=ni)
        o = Oracle(T, dev)
        ctx = pt.pt_load_perf(T, dev)
        X = T.astype(np.float64) / T.astype(np.float64).min(axis=1, keepdims=True)
        for k in (3, 6):
            init = X[:k].copy()
            init[-1] = 1e6                     # far from every point: empty on pass 1
            sel, G, it = pt.pt_kmeans_select_from(ctx, init)
            osel, oit, _ = o.kmeans_from(init)
            assert sel == osel and it == oit
