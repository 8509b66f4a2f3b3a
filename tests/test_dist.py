"""World-size-2 gloo test of the multi-GPU exhaustive protocol on CPU: each
rank searches its shard, the (s, tuple) top-2 records are all-gathered and
merged with pt_merge_top2.  The shard search itself is the GPU kernel on a B200;
here a stand-in shard search (the oracle over a split of the subset space)
drives the same collective + merge code path."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import Oracle
from paper_2507_15277_b200 import pt, synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, k, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    T, dev = synth.small_matrix(21, n_cfg=40, n_dev=2, n_inputs=6)
    o = Oracle(T, dev)
    E = T.shape[0]

    def local(r, w):
        lo, hi = r * o.C // w, (r + 1) * o.C // w    # split by first index
        b, gb, ru, gr = o.exhaustive(k, lo=lo, hi=hi, threads=1)
        recs = [(-E * np.log(gb), b)]
        if ru is not None:
            recs.append((-E * np.log(gr), ru))
        return recs

    res = pt.exhaustive_best_distributed(None, k, local_search=local, n_env=E)
    q.put((rank, res["best"], res["runner"], res["G"]))
    dist.destroy_process_group()


def test_two_rank_gloo_merge_equals_unsharded():
    T, dev = synth.small_matrix(21, n_cfg=40, n_dev=2, n_inputs=6)
    o = Oracle(T, dev)
    for k in (2, 3):
        want = o.exhaustive(k, threads=1)
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, 2, port, k, q)) for r in range(2)]
        for p in procs:
            p.start()
        got = [q.get(timeout=120) for _ in procs]
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
        for rank, best, runner, G in got:
            assert best == want[0] and runner == want[2]
            assert abs(G - want[1]) <= 1e-12
