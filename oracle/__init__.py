"""CPU oracle for portability tuning (arXiv 2507.15277) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2507_15277_b200``) never imports it; the two share no code.

This module is a thin ctypes wrapper around ``oracle.c`` (plain C, fp64,
definitions written out; see that file for the paper citations).  It compiles
``oracle.c`` with gcc on first use if the shared object is missing or stale.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (plain -O2; no vectorisation flags)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-D_POSIX_C_SOURCE=200809L", "-fPIC",
                               "-shared", "-o", _LIB, _SRC, "-lm", "-lpthread"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ct.CDLL(_LIB)
        P = ct.c_void_p
        i64, i32, dbl = ct.c_int64, ct.c_int32, ct.c_double
        lib.or_normalize.argtypes = [P, i64, i64, i64, P, P, P]
        lib.or_score.argtypes = [P, i64, i64, P, P, ct.c_int, P, P]
        lib.or_exhaustive.argtypes = [P, i64, i64, P, ct.c_int, i64, i64, ct.c_int,
                                      P, P, P, P, P]
        lib.or_greedy.argtypes = [P, i64, i64, P, ct.c_int, P, ct.c_int, P, P, P]
        lib.or_holdout.argtypes = [P, i64, i64, P, i32, ct.c_int, ct.c_int, ct.c_int,
                                   P, P, P, P, P]
        lib.or_fleet_rate.argtypes = [P, i64, i64, P, dbl, P, i32, P, P, P, P, ct.c_int, P]
        lib.or_fleet_exhaustive.argtypes = [P, i64, i64, P, dbl, P, i32, P, P, P, ct.c_int,
                                            P, P, P, P, P]
        lib.or_fleet_greedy.argtypes = [P, i64, i64, P, dbl, P, i32, P, P, P, ct.c_int, P, P, P]
        lib.or_fleet_exhaustive_par.argtypes = [P, i64, i64, P, dbl, P, i32, P, P, P, ct.c_int, ct.c_int,
                                                P, P, P, P, P]
        lib.or_swap_search.argtypes = [P, i64, i64, P, ct.c_int, P, ct.c_int, P, P, P]
        lib.or_kmeans.argtypes = [P, i64, i64, P, dbl, P, ct.c_int, ct.c_int, P, P, P, P]
        lib.or_kmeans_from.argtypes = [P, i64, i64, P, dbl, P, ct.c_int, ct.c_int, P, P, P, P, P]
        for f in (lib.or_normalize, lib.or_score, lib.or_exhaustive, lib.or_greedy,
                  lib.or_holdout, lib.or_fleet_rate, lib.or_fleet_exhaustive, lib.or_fleet_greedy,
                  lib.or_swap_search, lib.or_kmeans, lib.or_fleet_exhaustive_par, lib.or_kmeans_from):
            f.restype = ct.c_int
        _lib = lib
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where} failed with status {code}")
        self.code = code


def _chk(rc: int, where: str):
    if rc != 0:
        raise OracleError(rc, where)


def _p(a):
    return None if a is None else a.ctypes.data_as(ct.c_void_p)


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


class Oracle:
    """Normalised performance data + the oracle's search functions."""

    def __init__(self, T, env_device=None):
        T = np.ascontiguousarray(T, dtype=np.float32)
        self.T = T
        assert T.ndim == 2
        self.E, self.C = T.shape
        self.best = np.empty(self.E, np.float64)
        self.logeff = np.empty((self.E, self.C), np.float64)
        pen = np.zeros(1, np.float64)
        _chk(_load().or_normalize(_p(T), self.E, self.C, self.C, _p(self.best),
                                  _p(self.logeff), _p(pen)), "or_normalize")
        self.penalty = float(pen[0])
        self.env_device = (None if env_device is None
                           else np.ascontiguousarray(env_device, dtype=np.int32))

    @staticmethod
    def _mask(mask):
        return None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)

    def score(self, sets, mask=None):
        """G for one set (1-D) or a batch of sets (2-D)."""
        sets = np.asarray(sets, dtype=np.int32)
        one = sets.ndim == 1
        sets = np.atleast_2d(sets)
        m = self._mask(mask)
        out = np.empty(len(sets), np.float64)
        g = np.zeros(1, np.float64)
        lib = _load()
        for r, s in enumerate(sets):
            s = np.ascontiguousarray(s)
            _chk(lib.or_score(_p(self.logeff), self.E, self.C, _p(m), _p(s), len(s),
                              _p(g), None), "or_score")
            out[r] = g[0]
        return float(out[0]) if one else out

    def exhaustive(self, k, mask=None, lo=0, hi=None, threads=None):
        """Best and runner-up k-subsets: (best_tuple, G_best, runner_tuple, G_runner)."""
        hi = self.C if hi is None else hi
        threads = default_threads() if threads is None else threads
        m = self._mask(mask)
        b = np.zeros(k, np.int32)
        r = np.zeros(k, np.int32)
        gb = np.zeros(1, np.float64)
        gr = np.full(1, np.nan)
        nf = np.zeros(1, np.int32)
        _chk(_load().or_exhaustive(_p(self.logeff), self.E, self.C, _p(m), k, lo, hi, threads,
                                   _p(b), _p(gb), _p(r), _p(gr), _p(nf)), "or_exhaustive")
        runner = tuple(int(x) for x in r) if nf[0] >= 2 else None
        return tuple(int(x) for x in b), float(gb[0]), runner, float(gr[0])

    def greedy(self, k, mask=None, init=()):
        """Greedy forward selection: (indices, G_trace, gap_trace)."""
        m = self._mask(mask)
        init = np.ascontiguousarray(np.asarray(init, dtype=np.int32))
        idx = np.zeros(k, np.int32)
        gt = np.zeros(k, np.float64)
        gp = np.zeros(k, np.float64)
        _chk(_load().or_greedy(_p(self.logeff), self.E, self.C, _p(m), k,
                               _p(init) if len(init) else None, len(init),
                               _p(idx), _p(gt), _p(gp)), "or_greedy")
        return [int(x) for x in idx], gt, gp

    def holdout(self, device, k, method=0, threads=None):
        """Leave-one-device-out: (idx, G_train, G_unseen, G_known, known_idx)."""
        assert self.env_device is not None
        threads = default_threads() if threads is None else threads
        idx = np.zeros(k, np.int32)
        kidx = np.zeros(k, np.int32)
        g = np.zeros(3, np.float64)
        lib = _load()
        _chk(lib.or_holdout(_p(self.logeff), self.E, self.C, _p(self.env_device), device, k,
                            method, threads, _p(idx), _p(g[0:1]), _p(g[1:2]), _p(g[2:3]),
                            _p(kidx)), "or_holdout")
        return ([int(x) for x in idx], float(g[0]), float(g[1]), float(g[2]),
                [int(x) for x in kidx])

    def swap_search(self, k, mask=None, init=None, max_moves=1000):
        """Best-improvement swap local search from greedy (or init): (set, G, moves)."""
        m = self._mask(mask)
        ini = None if init is None else np.ascontiguousarray(np.asarray(init, dtype=np.int32))
        out = np.zeros(k, np.int32)
        g = np.zeros(1)
        mv = np.zeros(1, np.int32)
        _chk(_load().or_swap_search(_p(self.logeff), self.E, self.C, _p(m), k, _p(ini), max_moves,
                                    _p(out), _p(g), _p(mv)), "or_swap_search")
        return tuple(int(x) for x in out), float(g[0]), int(mv[0])

    def kmeans(self, k, mask=None, max_iter=100):
        """k-means selector: (sorted unique selection, iterations, wcss trace)."""
        m = self._mask(mask)
        sel = np.zeros(k, np.int32)
        n = np.zeros(1, np.int32)
        it = np.zeros(1, np.int32)
        w = np.zeros(max_iter)
        _chk(_load().or_kmeans(_p(self.T), self.E, self.C, _p(self.best), self.penalty, _p(m), k,
                               max_iter, _p(sel), _p(n), _p(it), _p(w)), "or_kmeans")
        return tuple(int(x) for x in sel[:n[0]]), int(it[0]), w[:it[0]]

    def kmeans_from(self, init, mask=None, max_iter=100):
        """k-means from given initial centroids (init: [k][C] slowdowns): (selection, iterations, wcss)."""
        m = self._mask(mask)
        init = np.ascontiguousarray(init, dtype=np.float64)
        k = init.shape[0]
        sel = np.zeros(k, np.int32)
        n = np.zeros(1, np.int32)
        it = np.zeros(1, np.int32)
        w = np.zeros(max_iter)
        _chk(_load().or_kmeans_from(_p(self.T), self.E, self.C, _p(self.best), self.penalty, _p(m), k, max_iter,
                                    _p(init), _p(sel), _p(n), _p(it), _p(w)), "or_kmeans_from")
        return tuple(int(x) for x in sel[:n[0]]), int(it[0]), w[:it[0]]

    # ---- fleet objective (Eq. 2) --------------------------------------------
    def set_fleet(self, q_dev, q_env):
        """quantity(d) per device id and quantity(i) per environment."""
        assert self.env_device is not None
        self.q_dev = np.ascontiguousarray(q_dev, dtype=np.float64)
        self.q_env = np.ascontiguousarray(q_env, dtype=np.float64)

    def _fleet_args(self):
        return (_p(self.T), self.E, self.C, _p(self.best), self.penalty, _p(self.env_device),
                len(self.q_dev), _p(self.q_dev), _p(self.q_env))

    def fleet_rate(self, sets, mask=None):
        sets = np.asarray(sets, dtype=np.int32)
        one = sets.ndim == 1
        sets = np.atleast_2d(sets)
        m = self._mask(mask)
        out = np.empty(len(sets))
        r = np.zeros(1)
        for q, s in enumerate(sets):
            s = np.ascontiguousarray(s)
            _chk(_load().or_fleet_rate(*self._fleet_args(), _p(m), _p(s), len(s), _p(r)), "or_fleet_rate")
            out[q] = r[0]
        return float(out[0]) if one else out

    def fleet_exhaustive(self, k, mask=None):
        m = self._mask(mask)
        b = np.zeros(k, np.int32)
        ru = np.zeros(k, np.int32)
        rb = np.zeros(1)
        rr = np.full(1, np.nan)
        nf = np.zeros(1, np.int32)
        _chk(_load().or_fleet_exhaustive(*self._fleet_args(), _p(m), k, _p(b), _p(rb), _p(ru), _p(rr),
                                         _p(nf)), "or_fleet_exhaustive")
        return (tuple(int(x) for x in b), float(rb[0]),
                tuple(int(x) for x in ru) if nf[0] >= 2 else None, float(rr[0]))

    def fleet_exhaustive_par(self, k, mask=None, threads=None):
        """fleet_exhaustive with the first index dealt to `threads` threads (same result)."""
        threads = default_threads() if threads is None else threads
        m = self._mask(mask)
        b = np.zeros(k, np.int32)
        ru = np.zeros(k, np.int32)
        rb = np.zeros(1)
        rr = np.full(1, np.nan)
        nf = np.zeros(1, np.int32)
        _chk(_load().or_fleet_exhaustive_par(*self._fleet_args(), _p(m), k, threads, _p(b), _p(rb), _p(ru),
                                             _p(rr), _p(nf)), "or_fleet_exhaustive_par")
        return (tuple(int(x) for x in b), float(rb[0]),
                tuple(int(x) for x in ru) if nf[0] >= 2 else None, float(rr[0]))

    def fleet_greedy(self, k, mask=None):
        m = self._mask(mask)
        idx = np.zeros(k, np.int32)
        rt = np.zeros(k)
        gp = np.zeros(k)
        _chk(_load().or_fleet_greedy(*self._fleet_args(), _p(m), k, _p(idx), _p(rt), _p(gp)),
             "or_fleet_greedy")
        return [int(x) for x in idx], rt, gp

