"""The multi-GPU exhaustive path on a real GPU, all through the C ABI:
shard search on the device, the record exchange (NCCL over a communicator the
library builds, or a caller's stream-ordered all-gather), the device merge and the
objective transform in libpt.  A world-size-1 NCCL group (all this box has), two
gloo processes sharing the GPU, and 8 thread-emulated ranks must each equal the
unsharded search and the oracle.  The 2-rank protocol on CPU: tests/test_dist.py."""
import threading
import os
import socket

import numpy as np
import pytest

from oracle import Oracle
from paper_2507_15277_b200 import pt, synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_nccl_world1_distributed_search():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        T, dev = synth.small_matrix(8, n_cfg=400, n_dev=3, n_inputs=16)
        o = Oracle(T, dev)
        ctx = pt.pt_load_perf(torch.from_numpy(T).cuda(), dev)
        for k in (2, 3):
            r = pt.exhaustive_best_distributed(ctx, k)
            b, gb, ru, gr = o.exhaustive(k)
            assert r["best"] == b and r["runner"] == ru
            assert r["G"] == pytest.approx(gb, rel=1e-12)
        # column-sharded greedy with the record exchange (world 1): host and
        # stream-ordered (device) flavours
        oidx, ogt, ogp = o.greedy(12)
        for on_device in (False, True):
            idx, gt, _ = pt.greedy_select_distributed(ctx, 12, on_device=on_device)
            np.testing.assert_allclose(gt, ogt, rtol=1e-9)
            if np.all(ogp > 1e-9):
                assert idx == oidx
        # the all-gather itself on the nccl group
        t = torch.tensor([[1.0, 2.0]], device="cuda")
        out = [torch.empty_like(t)]
        dist.all_gather(out, t)
        assert torch.equal(out[0], t)
        assert dist.get_backend() == "nccl"
    finally:
        dist.destroy_process_group()


def _gpu_worker(rank, world, port, q):
    """One rank of a 2-process gloo group sharing cuda:0 (all this box has):
    the real shard kernels + the collective exchange, end to end."""
    try:
        import torch as th
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        th.cuda.set_device(0)
        T, dev = synth.small_matrix(31, n_cfg=500, n_dev=4, n_inputs=16)
        ctx = pt.pt_load_perf(th.from_numpy(T).cuda(), dev)
        r3 = pt.exhaustive_best_distributed(ctx, 3)
        idx, gt, _ = pt.greedy_select_distributed(ctx, 16)
        didx, dgt, _ = pt.greedy_select_distributed(ctx, 16, on_device=True)   # host-staged over gloo
        assert didx == idx and list(dgt) == list(gt)
        q.put((rank, r3["best"], r3["runner"], r3["G"], idx, [float(x) for x in gt]))
        dist.destroy_process_group()
    except BaseException as e:   # report instead of hanging the parent
        q.put((rank, "error", repr(e)))


def test_two_process_gloo_on_one_gpu():
    """2 processes, one GPU, gloo: exhaustive_best_distributed and
    greedy_select_distributed (sharded scan + per-step record all-gather) must
    equal the unsharded searches and the oracle."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    T, dev = synth.small_matrix(31, n_cfg=500, n_dev=4, n_inputs=16)
    o = Oracle(T, dev)
    ctx0 = pt.pt_load_perf(T, dev, flags=pt.PT_GREEDY_STREAM)
    want3 = pt.pt_exhaustive_best(ctx0, 3)
    widx, wgt, _ = pt.pt_greedy_select(ctx0, 16)
    b, gb, ru, gr = o.exhaustive(3)
    assert want3["best"] == b
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    port = _port()
    procs = [mpc.Process(target=_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for g in got:
        assert g[1] != "error", g
        _, best, runner, G, idx, gt = g
        assert best == want3["best"] and runner == want3["runner"]
        assert G == pytest.approx(want3["G"], rel=1e-12)
        assert idx == widx
        np.testing.assert_array_equal(np.array(gt), wgt)


class _Gather:
    """An in-process all-gather for thread-emulated ranks (one GPU): each rank's
    device record is copied into every rank's output at its slot."""

    def __init__(self, world):
        self.world, self.bar, self.parts = world, threading.Barrier(world), [None] * world

    def fn(self, r):
        def gather(mine, out, stream):
            stream.synchronize()
            self.parts[r] = mine.clone()
            self.bar.wait()
            with torch.cuda.stream(stream):
                out.copy_(torch.cat(self.parts))
            self.bar.wait()
        return gather


def _emulate(T, dev, k, world, weights=None, objective=pt.PT_OBJ_GEOMEAN, fleet=None):
    ctxs = [pt.pt_load_perf(T, dev) for _ in range(world)]
    for r, c in enumerate(ctxs):
        if weights is not None:
            pt.pt_set_shard_weights(c, weights[r])
        if fleet is not None:
            pt.pt_set_fleet(c, *fleet)
    g = _Gather(world)
    res, errs = [None] * world, []

    def body(r):
        try:
            res[r] = pt.pt_exhaustive_best_sharded(ctxs[r], k, r, world, allgather=g.fn(r), objective=objective)
        except BaseException as e:
            errs.append(e)
            g.bar.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return res, errs


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_library_exchange_emulated_ranks(world):
    """pt_exhaustive_best_sharded with `world` thread-emulated ranks: the device merge
    and G = exp(-s/E) in the library equal the oracle on every rank."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    T, dev = synth.small_matrix(12, n_cfg=300, n_dev=3, n_inputs=16)
    o = Oracle(T, dev)
    for k in (2, 3):
        b, gb, ru, gr = o.exhaustive(k)
        res, errs = _emulate(T, dev, k, world)
        assert not errs, errs
        for r in res:
            assert r["best"] == b and r["runner"] == ru
            assert r["G"] == pytest.approx(gb, rel=1e-12) and r["G_runner"] == pytest.approx(gr, rel=1e-12)


def test_library_exchange_fleet_objective():
    """The sharded Eq. 2 search: records carry the cost 1/R, the library returns R."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    T, dev = synth.small_matrix(13, n_cfg=90, n_dev=3, n_inputs=8)
    qd, qe = np.array([1.0, 2.0, 3.0]), np.linspace(1.0, 2.0, T.shape[0])
    o = Oracle(T, dev)
    o.set_fleet(qd, qe)
    b, rb, ru, rr = o.fleet_exhaustive(2)
    res, errs = _emulate(T, dev, 2, 4, objective=pt.PT_OBJ_FLEET, fleet=(qd, qe))
    assert not errs, errs
    for r in res:
        assert r["best"] == b and r["G"] == pytest.approx(rb, rel=1e-12)


def test_mismatched_shard_plans_are_an_error():
    """ranks that deal the task list with different weights would skip or
    repeat subsets; the plan fingerprint in the records turns that into PT_EINVAL."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    T, dev = synth.small_matrix(14, n_cfg=200, n_dev=2, n_inputs=16)
    res, errs = _emulate(T, dev, 3, 2, weights=[[1.0, 1.0], [1.0, 3.0]])
    assert len(errs) == 2 and all(isinstance(e, pt.PTError) and e.code == pt.PT_EINVAL for e in errs)
    res, errs = _emulate(T, dev, 3, 2, weights=[[1.0, 3.0], [1.0, 3.0]])   # same weights: fine
    assert not errs and res[0]["best"] == res[1]["best"] == Oracle(T, dev).exhaustive(3)[0]


def test_library_nccl_comm_world1():
    """pt_comm_unique_id + pt_comm_init without torch.distributed: the library's own
    NCCL communicator (world 1) carries the record exchange."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    T, dev = synth.small_matrix(15, n_cfg=260, n_dev=2, n_inputs=16)
    o = Oracle(T, dev)
    comm = pt.pt_comm_init(pt.pt_comm_unique_id(), 0, 1, 0)
    ctx = pt.pt_load_perf(torch.from_numpy(T).cuda(), dev)
    for k in (2, 3):
        r = pt.pt_exhaustive_best_sharded(ctx, k, 0, 1, comm=comm)
        b, gb, ru, gr = o.exhaustive(k)
        assert r["best"] == b and r["runner"] == ru and r["G"] == pytest.approx(gb, rel=1e-12)
    with pytest.raises(pt.PTError) as ei:                 # rank/world must match the comm
        pt.pt_exhaustive_best_sharded(ctx, 2, 0, 2, comm=comm)
    assert ei.value.code == pt.PT_EINVAL
    comm.close()


def test_library_exchange_callback_failure():
    """A failing exchange is reported as PT_ENCCL (pt.h) -- the caller's exception is
    re-raised by the binding after the C call returns."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    T, dev = synth.small_matrix(16, n_cfg=120, n_dev=2, n_inputs=8)
    ctx = pt.pt_load_perf(T, dev)

    def broken(mine, out, stream):
        raise RuntimeError("link down")
    with pytest.raises(RuntimeError, match="link down"):
        pt.pt_exhaustive_best_sharded(ctx, 2, 0, 1, allgather=broken)
    # the context stays usable afterwards
    assert pt.pt_exhaustive_best_sharded(ctx, 2, 0, 1, allgather=lambda m, o, s: o.copy_(m))["best"] == \
        pt.pt_exhaustive_best(ctx, 2)["best"]
    with pytest.raises(pt.PTError) as ei:               # neither comm nor callback
        lib = pt.lib()
        import ctypes as ct
        b = (ct.c_int32 * 2)()
        g = (ct.c_double * 2)()
        rc = lib.pt_exhaustive_best_sharded(ctx.handle, 2, None, 0, 0, 1, None, ct.cast(None, pt.DEV_ALLGATHER_FN),
                                            None, b, ct.byref(g, 0), None, None, None)
        pt._chk(rc, "pt_exhaustive_best_sharded")
    assert ei.value.code == pt.PT_EINVAL
