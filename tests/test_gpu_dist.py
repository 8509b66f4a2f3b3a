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
        # column-sharded greedy with the NCCL record exchange (world 1)
        idx, gt, _ = pt.greedy_select_distributed(ctx, 12)
        oidx, ogt, ogp = o.greedy(12)
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
