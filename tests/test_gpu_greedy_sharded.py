"""Column-sharded greedy (pt_greedy_sharded) on one GPU.

W ranks are emulated by W threads, each with its own context (own stream, own
replica of the matrix), exchanging their per-step top-2 records through a
barrier-based all-gather -- the same protocol greedy_select_distributed runs
over NCCL.  Every rank must return the unsharded streamed greedy's picks and
G trace (the exact fp64 re-score of a candidate is the same arithmetic on any
shard, so they are bit-identical), and those must match the oracle.
"""
import threading

import numpy as np
import pytest

from oracle import Oracle
from paper_2507_15277_b200 import pt, synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


class _Exchange:
    def __init__(self, world):
        self.buf = [None] * world
        self.bar = threading.Barrier(world, timeout=120)

    def rank_fn(self, r):
        def allgather(mine):
            self.buf[r] = np.array(mine, np.float64)
            self.bar.wait()
            out = np.concatenate(self.buf)
            self.bar.wait()
            return out
        return allgather


    def dev_rank_fn(self, r):
        """stream-ordered flavour: device views in, host-staged exchange"""
        def allgather(mine, out, stream):
            stream.synchronize()
            self.buf[r] = mine.cpu().numpy().copy()
            self.bar.wait()
            cat = torch.from_numpy(np.concatenate(self.buf))
            self.bar.wait()
            with torch.cuda.stream(stream):
                out.copy_(cat)
        return allgather


def run_sharded(T, dev, k, world, mask=None, on_device=False):
    ctxs = [pt.pt_load_perf(T, dev) for _ in range(world)]
    ex = _Exchange(world)
    res, errs = [None] * world, []

    def body(r):
        try:
            if on_device:
                res[r] = pt.pt_greedy_sharded_dev(ctxs[r], k, ex.dev_rank_fn(r), r, world, env_mask=mask)
            else:
                res[r] = pt.pt_greedy_sharded(ctxs[r], k, ex.rank_fn(r), r, world, env_mask=mask)
        except BaseException as e:   # surface in the main thread
            errs.append(e)
            ex.bar.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return res


def plain(T, dev, k, mask=None):
    ctx = pt.pt_load_perf(T, dev, flags=pt.PT_GREEDY_STREAM)
    return pt.pt_greedy_select(ctx, k, env_mask=mask)


@pytest.mark.parametrize("on_device", [False, True])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_sharded_equals_streamed(world, on_device):
    T, dev = synth.small_matrix(11, n_cfg=700, n_dev=5, n_inputs=20)
    idx, gt, gp = plain(T, dev, 24)
    for ridx, rgt, rgp in run_sharded(T, dev, 24, world, on_device=on_device):
        assert ridx == idx
        np.testing.assert_array_equal(rgt, gt)
        np.testing.assert_array_equal(rgp, gp)
    o = Oracle(T, dev)
    oidx, ogt, ogp = o.greedy(24)
    np.testing.assert_allclose(gt, ogt, rtol=1e-9)
    if np.all(ogp > 1e-9):
        assert idx == oidx


def test_sharded_empty_shards_and_k_equals_C():
    """C=100 over 8 ranks: 64-config shard boundaries leave 6 ranks empty; k=C
    takes every configuration (last step: one candidate, no runner-up)."""
    T, dev = synth.small_matrix(12, n_cfg=100, n_dev=3, n_inputs=10)
    idx, gt, gp = plain(T, dev, 100)
    assert sorted(idx) == list(range(100))
    for on_device in (False, True):
        for ridx, rgt, rgp in run_sharded(T, dev, 100, 8, on_device=on_device):
            assert ridx == idx
            np.testing.assert_array_equal(rgt, gt)
            assert np.isinf(rgp[-1])
    assert np.isinf(gp[-1])


def test_sharded_masked():
    T, dev = synth.small_matrix(13, n_cfg=500, n_dev=4, n_inputs=16)
    mask = (dev != 2).astype(np.uint8)
    o = Oracle(T, dev)
    oidx, ogt, ogp = o.greedy(12, mask=mask)
    for ridx, rgt, _ in run_sharded(T, dev, 12, 4, mask=mask):
        np.testing.assert_allclose(rgt, ogt, rtol=1e-9)
        if np.all(ogp > 1e-9):
            assert ridx == oidx


def test_sharded_scaled_8():
    """Config 5 (65,536 configs x 4,096 envs), 8 shards of 8,192 configs: every
    step's pick and G re-derived by the oracle from the sharded run's own prefix."""
    T, dev = synth.scaled(1)
    dT = torch.from_numpy(T).cuda()
    runs = [r for on_device in (False, True) for r in run_sharded(dT, dev, 32, 8, on_device=on_device)]
    del dT
    o = Oracle(T, dev)
    ridx, rgt, _ = runs[0]
    for t in range(32):
        sidx, sg, sgap = o.greedy(1, init=ridx[:t])
        if sgap[0] > 1e-9:
            assert sidx[0] == ridx[t], (t, ridx)
        assert rgt[t] == pytest.approx(sg[0], rel=1e-6)
    for idx, gt, _ in runs[1:]:          # every rank, both exchange flavours: identical
        assert idx == ridx
        np.testing.assert_array_equal(gt, rgt)


def test_callback_failure_reported():
    T, dev = synth.small_matrix(14, n_cfg=200, n_dev=3, n_inputs=8)
    ctx = pt.pt_load_perf(T, dev)

    def bad(mine):
        raise RuntimeError("peer lost")

    with pytest.raises(RuntimeError, match="peer lost"):
        pt.pt_greedy_sharded(ctx, 4, bad, 0, 2)
    with pytest.raises(pt.PTError):
        pt.pt_greedy_sharded(ctx, 4, lambda m: m, 2, 2)   # shard_rank >= shard_count

    def bad_dev(mine, out, stream):
        raise RuntimeError("nccl down")

    with pytest.raises(RuntimeError, match="nccl down"):
        pt.pt_greedy_sharded_dev(ctx, 4, bad_dev, 0, 2)
