"""Thin ctypes binding of libpt.so (include/pt.h) -- argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C ABI; this
module only converts numpy arrays / torch tensors to pointers, picks the
current CUDA stream, and hands the library a process group's ncclUniqueId (or, for
gloo test groups, a host-staged all-gather callback); the record exchange, merge and
objective transform of the multi-GPU search run inside the library.  There is no CPU
fallback: if libpt.so is missing or cannot initialise a GPU, calls raise.

Names follow the C ABI: pt_load_perf, pt_score_sets, pt_greedy_select,
pt_exhaustive_best, pt_merge_top2, pt_eval_holdout, pt_get_stats, pt_free.
"""
from __future__ import annotations

import ctypes as ct
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PT_LIB") or os.path.join(_HERE, "libpt.so")   # PT_LIB: a variant build (tests)

PT_OK, PT_EINVAL, PT_ENOMEM, PT_ECUDA, PT_ENCCL, PT_ECAP, PT_EEMPTY, PT_EDATA = 0, -1, -2, -3, -4, -5, -6, -7
PT_OBJ_GEOMEAN, PT_OBJ_FLEET = 0, 1
PT_MISSING_PENALTY_MAX, PT_EXACT_FP64, PT_GREEDY_STREAM, PT_GREEDY_LAZY = 0x1, 0x2, 0x4, 0x8

EXPORTS = ("pt_load_perf", "pt_score_sets", "pt_greedy_select", "pt_exhaustive_best",
           "pt_merge_top2", "pt_eval_holdout", "pt_eval_holdout_all", "pt_swap_search",
           "pt_kmeans_select", "pt_set_fleet", "pt_get_stats", "pt_greedy_sharded",
           "pt_greedy_sharded_dev", "pt_set_shard_weights", "pt_comm_unique_id", "pt_comm_init",
           "pt_comm_free", "pt_exhaustive_best_sharded", "pt_record_len", "pt_merge_records",
           "pt_kmeans_select_from",
           "pt_free", "pt_last_error")
PT_COMM_ID_BYTES = 128


# int (*)(void *user, const double *mine, int32_t n, double *all)
ALLGATHER_FN = ct.CFUNCTYPE(ct.c_int, ct.c_void_p, ct.POINTER(ct.c_double), ct.c_int32,
                            ct.POINTER(ct.c_double))


# int (*)(void *user, const double *mine, int32_t n, double *all, void *stream)  (device pointers)
DEV_ALLGATHER_FN = ct.CFUNCTYPE(ct.c_int, ct.c_void_p, ct.c_void_p, ct.c_int32, ct.c_void_p, ct.c_void_p)


class _DevView:
    """Zero-copy view of n float64 at a device pointer (for torch.as_tensor)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 2, "strides": None}


class pt_stats(ct.Structure):
    _fields_ = [("launches", ct.c_int64), ("exh_main_ms", ct.c_double), ("exh_sets", ct.c_int64),
                ("exh_slots", ct.c_int64), ("exh_env_pad", ct.c_int64),
                ("exh_candidates", ct.c_int64), ("exh_passes", ct.c_int32),
                ("exh_kernel", ct.c_int32), ("greedy_ms", ct.c_double),
                ("greedy_candidates", ct.c_int64), ("exh_tc_nt", ct.c_int32), ("exh_tc_pad", ct.c_int32),
                ("exh_tc_survivors", ct.c_int64)]


class PTError(RuntimeError):
    def __init__(self, code, where, msg):
        super().__init__(f"{where}: status {code}: {msg}")
        self.code = code


_lib = None


def lib():
    """Load libpt.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (or make)")
        L = ct.CDLL(LIB_PATH)
        P, i64, i32, u32, dbl = ct.c_void_p, ct.c_int64, ct.c_int32, ct.c_uint32, ct.c_double
        L.pt_load_perf.argtypes = [ct.POINTER(P), P, i64, i64, i64, P, u32, ct.c_int, P]
        L.pt_score_sets.argtypes = [P, P, i64, i32, P, i32, P]
        L.pt_greedy_select.argtypes = [P, i32, P, i32, P, P, P]
        L.pt_exhaustive_best.argtypes = [P, i32, P, i32, i32, i32, P, P, P, P, P]
        L.pt_merge_top2.argtypes = [P, P, i32, i32, P, P, P]
        L.pt_set_shard_weights.argtypes = [P, P, i32]
        L.pt_eval_holdout.argtypes = [P, i32, i32, i32, P, P, P, P, P]
        L.pt_get_stats.argtypes = [P, ct.POINTER(pt_stats)]
        L.pt_set_fleet.argtypes = [P, P, i32, P]
        L.pt_swap_search.argtypes = [P, i32, P, i32, i32, P, P, P, P]
        L.pt_eval_holdout_all.argtypes = [P, i32, i32, P, P, P, P, P, P]
        L.pt_kmeans_select.argtypes = [P, i32, P, i32, P, P, P, P]
        L.pt_kmeans_select_from.argtypes = [P, i32, P, i32, P, P, P, P, P]
        L.pt_greedy_sharded.argtypes = [P, i32, P, i32, i32, ALLGATHER_FN, P, P, P, P]
        L.pt_greedy_sharded_dev.argtypes = [P, i32, P, i32, i32, DEV_ALLGATHER_FN, P, P, P, P]
        L.pt_comm_unique_id.argtypes = [P]
        L.pt_comm_init.argtypes = [ct.POINTER(P), P, i32, i32, ct.c_int]
        L.pt_comm_free.argtypes = [P]
        L.pt_comm_free.restype = None
        L.pt_exhaustive_best_sharded.argtypes = [P, i32, P, i32, i32, i32, P, DEV_ALLGATHER_FN, P,
                                                 P, P, P, P, P]
        L.pt_record_len.argtypes = [i32]
        L.pt_record_len.restype = i32
        L.pt_merge_records.argtypes = [P, i32, i32, i64, i32, P, P, P, P, P]
        L.pt_free.argtypes = [P]
        L.pt_free.restype = None
        L.pt_last_error.argtypes = []
        L.pt_last_error.restype = ct.c_char_p
        for f in ("pt_load_perf", "pt_score_sets", "pt_greedy_select", "pt_exhaustive_best",
                  "pt_merge_top2", "pt_eval_holdout", "pt_get_stats", "pt_set_fleet",
                  "pt_swap_search", "pt_eval_holdout_all", "pt_kmeans_select", "pt_comm_unique_id",
                  "pt_comm_init", "pt_exhaustive_best_sharded", "pt_merge_records", "pt_kmeans_select_from"):
            getattr(L, f).restype = ct.c_int
        _lib = L
    return _lib


def _chk(rc, where):
    if rc != PT_OK:
        raise PTError(rc, where, lib().pt_last_error().decode())


def _ptr(a):
    """Pointer of a numpy array or torch tensor (host or device); None -> NULL."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return ct.c_void_p(a.data_ptr())
    return a.ctypes.data_as(ct.c_void_p)


def _np(a, dtype):
    return np.ascontiguousarray(np.asarray(a), dtype=dtype)


def _mask(m):
    return None if m is None else _np(m, np.uint8)


def _stream(stream, device=None):
    if stream is not None:
        return stream if isinstance(stream, ct.c_void_p) else ct.c_void_p(int(stream))
    try:
        import torch
        if torch.cuda.is_available():
            return ct.c_void_p(torch.cuda.current_stream(device).cuda_stream)
    except ImportError:
        pass
    return None


class PtContext:
    """Owner of a pt_ctx handle (freed on close / garbage collection)."""

    def __init__(self, handle, n_env, n_cfg):
        self.handle = handle
        self.E, self.C = n_env, n_cfg

    def close(self):
        if self.handle:
            lib().pt_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pt_load_perf(times_ms, env_device=None, flags=0, device=None, stream=None) -> PtContext:
    """times_ms: [E][C] float32 numpy array (host) or torch tensor (host or cuda).
    device: CUDA ordinal (default: a cuda tensor's own device, else torch's current
    device); stream: a cudaStream_t handle (default: torch's current stream OF THAT
    device)."""
    if device is None:
        if hasattr(times_ms, "is_cuda") and times_ms.is_cuda:
            device = times_ms.device.index
        else:
            try:
                import torch
                device = torch.cuda.current_device() if torch.cuda.is_available() else 0
            except ImportError:
                device = 0
    if stream is None:
        stream = _stream(None, device)
    if hasattr(times_ms, "data_ptr"):
        assert times_ms.dtype.__str__() == "torch.float32" and times_ms.is_contiguous()
        E, C = times_ms.shape
        keep = times_ms
    else:
        keep = _np(times_ms, np.float32)
        E, C = keep.shape
    dev = None if env_device is None else _np(env_device, np.int32)
    h = ct.c_void_p()
    _chk(lib().pt_load_perf(ct.byref(h), _ptr(keep), E, C, C, _ptr(dev), flags, device,
                            _stream(stream)), "pt_load_perf")
    return PtContext(h, E, C)


def pt_set_fleet(ctx, q_device, q_env):
    """Quantities for the fleet objective (Eq. 2): quantity(d) per device id, quantity(i) per env."""
    qd = _np(q_device, np.float64)
    qe = _np(q_env, np.float64)
    _chk(lib().pt_set_fleet(ctx.handle, _ptr(qd), len(qd), _ptr(qe)), "pt_set_fleet")


def pt_score_sets(ctx, sets, env_mask=None, out=None, objective=PT_OBJ_GEOMEAN):
    """G (or fleet rate R) of each set.  sets: [n][k] int32 (numpy or torch); returns numpy
    (or fills `out`)."""
    if hasattr(sets, "data_ptr"):
        n, k = sets.shape
        s = sets
    else:
        s = np.atleast_2d(_np(sets, np.int32))
        n, k = s.shape
    res = out if out is not None else np.empty(n, np.float64)
    _chk(lib().pt_score_sets(ctx.handle, _ptr(s), n, k, _ptr(_mask(env_mask)), objective,
                             _ptr(res)), "pt_score_sets")
    return res


def pt_greedy_select(ctx, k, env_mask=None, objective=PT_OBJ_GEOMEAN):
    """Greedy forward selection: (indices, G_trace (or R_trace), gap_trace)."""
    idx = (ct.c_int32 * k)()          # ctypes buffers: ~1 us of marshalling instead of ~15 with numpy
    gt = (ct.c_double * k)()
    gp = (ct.c_double * k)()
    _chk(lib().pt_greedy_select(ctx.handle, k, _ptr(_mask(env_mask)), objective, idx, gt, gp),
         "pt_greedy_select")
    return list(idx), np.frombuffer(gt, np.float64).copy(), np.frombuffer(gp, np.float64).copy()


def pt_greedy_sharded(ctx, k, allgather, shard_rank=0, shard_count=1, env_mask=None):
    """Column-sharded greedy: this rank scans configurations shard `shard_rank` of
    `shard_count`; `allgather(mine)` takes this rank's 4 float64 record values
    and returns the (shard_count * 4) values of every rank in rank order.
    Returns (indices, G_trace, gap_trace), the same on every rank."""
    err = []

    def _cb(_user, mine, n, all_out):
        try:
            got = np.ascontiguousarray(allgather(np.ctypeslib.as_array(mine, (n,)).copy()),
                                       dtype=np.float64).reshape(-1)
            if got.size != n * shard_count:
                raise ValueError(f"allgather returned {got.size} values, want {n * shard_count}")
            ct.memmove(all_out, got.ctypes.data, got.nbytes)
            return 0
        except BaseException as ex:   # reported after the C call returns
            err.append(ex)
            return 1

    cb = ALLGATHER_FN(_cb)
    idx = np.zeros(k, np.int32)
    gt = np.zeros(k, np.float64)
    gp = np.zeros(k, np.float64)
    rc = lib().pt_greedy_sharded(ctx.handle, k, _ptr(_mask(env_mask)), shard_rank, shard_count, cb,
                                 None, _ptr(idx), _ptr(gt), _ptr(gp))
    if err:
        raise err[0]
    _chk(rc, "pt_greedy_sharded")
    return [int(x) for x in idx], gt, gp


def pt_greedy_sharded_dev(ctx, k, allgather, shard_rank=0, shard_count=1, env_mask=None):
    """Column-sharded greedy with a stream-ordered exchange (no host sync inside
    the k-step loop).  `allgather(mine, out, stream)` gets torch CUDA views of
    this rank's 4 record values and of the (shard_count * 4) output, and the
    context's stream (torch.cuda stream object); it must enqueue the gather so
    `out` is complete in that stream's order.  Returns (indices, G_trace, gap_trace)."""
    import torch
    err = []

    views = {}   # the pointers and stream are fixed for the whole call: build the views once

    def _cb(_user, mine, n, all_out, stream):
        try:
            key = (mine, all_out, stream)
            if key not in views:
                views[key] = (torch.as_tensor(_DevView(mine, n), device="cuda"),
                              torch.as_tensor(_DevView(all_out, n * shard_count), device="cuda"),
                              torch.cuda.ExternalStream(stream) if stream else torch.cuda.default_stream())
            mt, at, st = views[key]
            allgather(mt, at, st)
            return 0
        except BaseException as ex:   # reported after the C call returns
            err.append(ex)
            return 1

    cb = DEV_ALLGATHER_FN(_cb)
    idx = np.zeros(k, np.int32)
    gt = np.zeros(k, np.float64)
    gp = np.zeros(k, np.float64)
    rc = lib().pt_greedy_sharded_dev(ctx.handle, k, _ptr(_mask(env_mask)), shard_rank, shard_count, cb,
                                     None, _ptr(idx), _ptr(gt), _ptr(gp))
    if err:
        raise err[0]
    _chk(rc, "pt_greedy_sharded_dev")
    return [int(x) for x in idx], gt, gp


def greedy_select_distributed(ctx, k, env_mask=None, group=None, on_device=None):
    """Column-sharded greedy over a torch.distributed group: rank r of world W
    scans configuration shard r of W and the 2 exact records per rank are
    all-gathered every step.  on_device (default: True for an NCCL group) uses
    pt_greedy_sharded_dev with an NCCL all_gather_into_tensor enqueued on the
    library's stream (over NVLink; no host round trip per step); otherwise the
    records go through the host (pt_greedy_sharded; gloo)."""
    import torch
    import torch.distributed as dist
    init = dist.is_available() and dist.is_initialized()
    rank = dist.get_rank(group) if init else 0
    world = dist.get_world_size(group) if init else 1
    nccl = init and dist.get_backend(group) == "nccl"
    if on_device is None:
        on_device = nccl

    if on_device:
        def dev_allgather(mine, out, stream):
            if nccl:   # enqueued on the library's stream: no host round trip
                with torch.cuda.stream(stream):
                    dist.all_gather_into_tensor(out, mine, group=group)
            elif world == 1:
                with torch.cuda.stream(stream):
                    out.copy_(mine)
            else:   # host-staged (gloo)
                stream.synchronize()
                parts = [torch.empty(mine.numel(), dtype=torch.float64) for _ in range(world)]
                dist.all_gather(parts, mine.cpu(), group=group)
                with torch.cuda.stream(stream):
                    out.copy_(torch.cat(parts))
        return pt_greedy_sharded_dev(ctx, k, dev_allgather, rank, world, env_mask)

    def allgather(mine):
        if world == 1 and not nccl:
            return mine
        t = torch.from_numpy(mine)
        if nccl:
            t = t.cuda()
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t, group=group)
        return torch.cat([o.cpu() for o in out]).numpy()

    return pt_greedy_sharded(ctx, k, allgather, rank, world, env_mask)


def pt_exhaustive_best(ctx, k, env_mask=None, shard_rank=0, shard_count=1,
                       objective=PT_OBJ_GEOMEAN):
    """Exhaustive k-subset search (one shard): dict(best, G, runner, G_runner, s).
    For PT_OBJ_FLEET, G/G_runner hold the fleet rates and s the costs 1/R."""
    b = (ct.c_int32 * k)()
    r = (ct.c_int32 * k)()
    g = (ct.c_double * 2)()
    s = (ct.c_double * 2)()
    _chk(lib().pt_exhaustive_best(ctx.handle, k, _ptr(_mask(env_mask)), objective, shard_rank, shard_count,
                                  b, ct.byref(g, 0), r, ct.byref(g, 8), s), "pt_exhaustive_best")
    return _result(b, g, r, s)


def pt_swap_search(ctx, k, env_mask=None, init=None, max_moves=1000):
    """Swap local search from greedy (or init): (sorted set, G, moves)."""
    out = np.zeros(k, np.int32)
    g = np.zeros(1)
    mv = np.zeros(1, np.int32)
    ini = None if init is None else _np(init, np.int32)
    _chk(lib().pt_swap_search(ctx.handle, k, _ptr(_mask(env_mask)), PT_OBJ_GEOMEAN, max_moves,
                              _ptr(ini), _ptr(out), _ptr(g), _ptr(mv)), "pt_swap_search")
    return tuple(int(x) for x in out), float(g[0]), int(mv[0])


def pt_kmeans_select(ctx, k, env_mask=None, max_iter=100):
    """k-means selector (Sec. 4.3.2): (sorted unique selection, G, iterations)."""
    out = np.zeros(k, np.int32)
    n = np.zeros(1, np.int32)
    g = np.zeros(1)
    it = np.zeros(1, np.int32)
    _chk(lib().pt_kmeans_select(ctx.handle, k, _ptr(_mask(env_mask)), max_iter, _ptr(out), _ptr(n),
                                _ptr(g), _ptr(it)), "pt_kmeans_select")
    return tuple(int(x) for x in out[:n[0]]), float(g[0]), int(it[0])


def pt_kmeans_select_from(ctx, init, env_mask=None, max_iter=100):
    """k-means from given initial centroids (init: [k][C] slowdowns): (selection, G, iterations)."""
    ini = _np(init, np.float64)
    k = ini.shape[0]
    out = np.zeros(k, np.int32)
    n = np.zeros(1, np.int32)
    g = np.zeros(1)
    it = np.zeros(1, np.int32)
    _chk(lib().pt_kmeans_select_from(ctx.handle, k, _ptr(_mask(env_mask)), max_iter, _ptr(ini), _ptr(out),
                                     _ptr(n), _ptr(g), _ptr(it)), "pt_kmeans_select_from")
    return tuple(int(x) for x in out[:n[0]]), float(g[0]), int(it[0])


def pt_set_shard_weights(ctx, weights=None):
    """Relative work shares of the shards of later sharded exhaustive searches with
    shard_count == len(weights); None restores equal shares."""
    if weights is None:
        _chk(lib().pt_set_shard_weights(ctx.handle, None, 0), "pt_set_shard_weights")
        return
    w = _np(weights, np.float64)
    _chk(lib().pt_set_shard_weights(ctx.handle, _ptr(w), len(w)), "pt_set_shard_weights")


def pt_merge_top2(s, tuples, k):
    """Merge (s, tuple) records -> (best, runner, (s1, s2)); host-only."""
    s = _np(s, np.float64)
    t = _np(tuples, np.int32).reshape(len(s), k)
    b = np.zeros(k, np.int32)
    r = np.zeros(k, np.int32)
    o = np.zeros(2, np.float64)
    _chk(lib().pt_merge_top2(_ptr(s), _ptr(t), len(s), k, _ptr(b), _ptr(r), _ptr(o)),
         "pt_merge_top2")
    runner = tuple(int(x) for x in r) if np.isfinite(o[1]) else None
    return tuple(int(x) for x in b), runner, (float(o[0]), float(o[1]))


def pt_eval_holdout(ctx, heldout_device, k, method=0):
    """Leave-one-device-out: dict(idx, G_train, G_unseen, G_known, known_idx)."""
    idx = np.zeros(k, np.int32)
    kidx = np.zeros(k, np.int32)
    g = np.zeros(3, np.float64)
    _chk(lib().pt_eval_holdout(ctx.handle, heldout_device, k, method, _ptr(idx), _ptr(g[0:1]),
                               _ptr(g[1:2]), _ptr(g[2:3]), _ptr(kidx)), "pt_eval_holdout")
    return {"idx": [int(x) for x in idx], "G_train": float(g[0]), "G_unseen": float(g[1]),
            "G_known": float(g[2]), "known_idx": [int(x) for x in kidx]}


def pt_eval_holdout_all(ctx, k, n_device):
    """All leave-one-device-out folds (greedy) in one batched call: list of dicts like
    pt_eval_holdout, one per device id 0..n_device-1."""
    D = n_device
    idx = np.zeros((D, k), np.int32)
    kidx = np.zeros((D, k), np.int32)
    gtr, gun, gkn = np.zeros(D), np.zeros(D), np.zeros(D)
    nd = np.zeros(1, np.int32)
    _chk(lib().pt_eval_holdout_all(ctx.handle, k, D, _ptr(idx), _ptr(gtr), _ptr(gun), _ptr(gkn),
                                   _ptr(kidx), _ptr(nd)), "pt_eval_holdout_all")
    D = int(nd[0])   # the library writes D <= n_device rows
    return [{"idx": [int(x) for x in idx[d]], "G_train": float(gtr[d]), "G_unseen": float(gun[d]),
             "G_known": float(gkn[d]), "known_idx": [int(x) for x in kidx[d]]} for d in range(D)]


def pt_get_stats(ctx):
    st = pt_stats()   # ctypes structure: no numpy marshalling
    _chk(lib().pt_get_stats(ctx.handle, ct.byref(st)), "pt_get_stats")
    return {f: getattr(st, f) for f, _ in pt_stats._fields_}


def pt_free(ctx):
    ctx.close()


class PtComm:
    """Owner of a library-built NCCL communicator (pt_comm_init)."""

    def __init__(self, handle, rank, world, device):
        self.handle, self.rank, self.world, self.device = handle, rank, world, device

    def close(self):
        if self.handle:
            lib().pt_comm_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pt_comm_unique_id():
    """A fresh ncclUniqueId (bytes) for pt_comm_init; create on one rank, broadcast."""
    buf = (ct.c_uint8 * PT_COMM_ID_BYTES)()
    _chk(lib().pt_comm_unique_id(ct.cast(buf, ct.c_void_p)), "pt_comm_unique_id")
    return bytes(buf)


def pt_comm_init(uid, rank, world, device=None):
    """Collective: every rank passes the same id bytes and its rank -> PtComm."""
    if device is None:
        import torch
        device = torch.cuda.current_device()
    buf = (ct.c_uint8 * PT_COMM_ID_BYTES).from_buffer_copy(uid)
    h = ct.c_void_p()
    _chk(lib().pt_comm_init(ct.byref(h), ct.cast(buf, ct.c_void_p), rank, world, device), "pt_comm_init")
    return PtComm(h, rank, world, device)


def pt_record_len(k):
    return int(lib().pt_record_len(k))


def _result(b, g, r, s):
    has1, has2 = math.isfinite(s[0]), math.isfinite(s[1])
    return {"best": tuple(int(x) for x in b) if has1 else None, "G": float(g[0]),
            "runner": tuple(int(x) for x in r) if has2 else None, "G_runner": float(g[1]),
            "s": (float(s[0]), float(s[1]))}


def pt_exhaustive_best_sharded(ctx, k, shard_rank, shard_count, comm=None, allgather=None,
                               env_mask=None, objective=PT_OBJ_GEOMEAN):
    """The sharded search end to end in the library: shard search, record exchange over
    `comm` (PtComm, NCCL) or `allgather(mine, out, stream)` (torch CUDA views of this
    rank's record and of the gathered records, the library's stream; must enqueue the
    gather in that stream's order), device merge, G.  Returns the pt_exhaustive_best dict."""
    import torch
    err = []
    cb = None
    if allgather is not None:
        def _cb(_user, mine, n, all_out, stream):
            try:
                mt = torch.as_tensor(_DevView(mine, n), device="cuda")
                at = torch.as_tensor(_DevView(all_out, n * shard_count), device="cuda")
                st = torch.cuda.ExternalStream(stream) if stream else torch.cuda.default_stream()
                allgather(mt, at, st)
                return 0
            except BaseException as ex:   # reported after the C call returns
                err.append(ex)
                return 1
        cb = DEV_ALLGATHER_FN(_cb)
    else:
        cb = ct.cast(None, DEV_ALLGATHER_FN)
    b = (ct.c_int32 * k)()
    r = (ct.c_int32 * k)()
    g = (ct.c_double * 2)()
    s = (ct.c_double * 2)()
    rc = lib().pt_exhaustive_best_sharded(ctx.handle, k, _ptr(_mask(env_mask)), objective, shard_rank,
                                          shard_count, comm.handle if comm is not None else None, cb, None,
                                          b, ct.byref(g, 0), r, ct.byref(g, 8), s)
    if err:
        raise err[0]
    _chk(rc, "pt_exhaustive_best_sharded")
    return _result(b, g, r, s)


def pt_merge_records(records, k, n_env, objective=PT_OBJ_GEOMEAN):
    """Host merge of gathered rank records ([n_rank][pt_record_len(k)] float64)."""
    rec = _np(records, np.float64).reshape(-1)
    L = pt_record_len(k)
    b = np.zeros(k, np.int32)
    r = np.zeros(k, np.int32)
    g = np.zeros(2, np.float64)
    s = np.zeros(2, np.float64)
    _chk(lib().pt_merge_records(_ptr(rec), rec.size // L, k, n_env, objective, _ptr(b), _ptr(g[0:1]), _ptr(r),
                                _ptr(g[1:2]), _ptr(s)), "pt_merge_records")
    return _result(b, g, r, s)


_COMMS = {}


def _library_comm(group, rank, world):
    """One library-built NCCL communicator per (process group, device), created on
    first use: rank 0 makes the ncclUniqueId, the group broadcasts it."""
    import torch
    import torch.distributed as dist
    key = (id(group), world, torch.cuda.current_device())
    if key not in _COMMS:
        # rank 0 makes the id (or reports why it cannot); every rank sees the same outcome,
        # so either all ranks build the communicator or all take the fallback
        obj = [None]
        if rank == 0:
            try:
                obj = [pt_comm_unique_id()]
            except PTError as ex:
                obj = [f"error: {ex}"]
        dist.broadcast_object_list(obj, src=0 if group is None else dist.get_global_rank(group, 0),
                                   group=group)
        if isinstance(obj[0], str):
            _COMMS[key] = None
        else:
            _COMMS[key] = pt_comm_init(obj[0], rank, world)
    if _COMMS[key] is None:
        raise PTError(PT_ENCCL, "pt_comm_unique_id", "NCCL unavailable on rank 0")
    return _COMMS[key]


def exhaustive_best_distributed(ctx, k, env_mask=None, group=None, objective=PT_OBJ_GEOMEAN,
                                local_search=None, n_env=None):
    """Sharded exhaustive search over a torch.distributed group: rank r of W searches
    shard r, and the library exchanges and merges the (s, tuple) records --
    over its own NCCL communicator for an nccl group (built once per group from a
    broadcast ncclUniqueId), or through a host-staged gloo all-gather (tests).
    `local_search(shard_rank, shard_count) -> [(s, tuple), ...]` replaces the GPU shard
    search (CPU protocol tests); its records are merged by pt_merge_records."""
    import torch
    import torch.distributed as dist
    init = dist.is_available() and dist.is_initialized()
    rank = dist.get_rank(group) if init else 0
    world = dist.get_world_size(group) if init else 1
    if local_search is not None:        # CPU: marshal the records, gather, merge in C
        L = pt_record_len(k)
        rec = np.full(L, np.inf)
        rec[0] = 0.0
        for q, (sv, tup) in enumerate(local_search(rank, world)[:2]):
            rec[1 + q] = sv
            rec[3 + q * k:3 + (q + 1) * k] = tup
        allr = [torch.empty(L, dtype=torch.float64) for _ in range(world)]
        if world > 1:
            dist.all_gather(allr, torch.from_numpy(rec), group=group)
        else:
            allr = [torch.from_numpy(rec)]
        E = n_env if env_mask is None else int(np.count_nonzero(env_mask))
        return pt_merge_records(torch.cat(allr).numpy(), k, E, objective)
    if init and dist.get_backend(group) == "nccl":
        comm = None
        try:
            comm = _library_comm(group, rank, world)
        except PTError as ex:   # e.g. no libnccl.so.2 visible to dlopen: same exchange via torch's NCCL
            import warnings
            warnings.warn(f"library NCCL communicator unavailable ({ex}); exchanging records through "
                          "torch.distributed on the library's stream")
        if comm is not None:
            return pt_exhaustive_best_sharded(ctx, k, rank, world, comm=comm, env_mask=env_mask,
                                              objective=objective)

        def nccl_allgather(mine, out, stream):
            with torch.cuda.stream(stream):
                dist.all_gather_into_tensor(out, mine, group=group)
        return pt_exhaustive_best_sharded(ctx, k, rank, world, allgather=nccl_allgather, env_mask=env_mask,
                                          objective=objective)

    def host_allgather(mine, out, stream):      # gloo (or no group): host-staged
        if world == 1:
            with torch.cuda.stream(stream):
                out.copy_(mine)
            return
        stream.synchronize()
        parts = [torch.empty(mine.numel(), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, mine.cpu(), group=group)
        with torch.cuda.stream(stream):
            out.copy_(torch.cat(parts))
    return pt_exhaustive_best_sharded(ctx, k, rank, world, allgather=host_allgather, env_mask=env_mask,
                                      objective=objective)
