"""GPU parity for the swap local search vs the oracle."""
import numpy as np
import pytest

from conftest import read_golden
from oracle import Oracle
from paper_2507_15277_b200 import pt, synth
from test_oracle import pow2_matrix

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_hand_fixture():
    g = read_golden("greedy_vs_opt.txt")
    m = np.array([[int(x) for x in r[1:]] for r in g if r[0] == "m"])
    ctx = pt.pt_load_perf(pow2_matrix(m))
    s, G, moves = pt.pt_swap_search(ctx, 2)
    assert s == (1, 2) and G == 1.0 and moves == 1


@pytest.mark.parametrize("seed,C,nd,ni,k", [(1, 60, 2, 8, 3), (2, 200, 3, 12, 6), (3, 300, 5, 10, 10)])
def test_random(seed, C, nd, ni, k):
    T, dev = synth.small_matrix(seed, n_cfg=C, n_dev=nd, n_inputs=ni)
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    s, G, moves = pt.pt_swap_search(ctx, k)
    os_, oG, omoves = o.swap_search(k)
    assert s == os_ and moves == omoves
    assert G == pytest.approx(oG, rel=1e-12)
    mask = (dev != 0).astype(np.uint8)
    s, G, moves = pt.pt_swap_search(ctx, k, env_mask=mask)
    os_, oG, omoves = o.swap_search(k, mask=mask)
    assert s == os_ and G == pytest.approx(oG, rel=1e-12)
    init = list(range(k))
    assert pt.pt_swap_search(ctx, k, init=init, max_moves=2)[0] == o.swap_search(k, init=init, max_moves=2)[0]


def test_paper_shape_k10():
    T, dev = synth.paper_matrix(1)
    o = Oracle(T, dev)
    ctx = pt.pt_load_perf(T, dev)
    s, G, moves = pt.pt_swap_search(ctx, 5)
    os_, oG, omoves = o.swap_search(5)
    assert s == os_ and moves == omoves and G == pytest.approx(oG, rel=1e-12)
    gidx, gt, _ = pt.pt_greedy_select(ctx, 5)
    assert G >= gt[-1]
