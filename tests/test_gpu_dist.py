"""The multi-GPU exhaustive path on a real GPU: a world-size-1 NCCL process
group (all this box has) drives exhaustive_best_distributed end to end --
shard search on the device, NCCL all-gather of the (s, tuple) records, merge
with pt_merge_top2 -- and must equal the unsharded search.  The 2-rank protocol
is covered by tests/test_dist.py (gloo, CPU)."""
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
