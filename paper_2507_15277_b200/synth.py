"""Seeded synthetic runtime matrices shaped like the paper's workloads.

This module is the ONE piece shared by the CUDA path's tests/bench and the CPU
oracle's tests: it only draws runtimes.  It holds none of the method's
arithmetic (no Oracle/best, no slowdowns, no scores).

Every generator returns ``(T, env_device)``:
  * ``T``           float32 [E][C], runtimes in ms, env-major (row = environment
                    = device x GEMM input (M,N,K); column = parameter
                    configuration);
  * ``env_device``  int32 [E], the device id of every environment.

Recipe: environments are device-major, then inputs
(M,N,K) in lexicographic order over {256,512,1024,4096}^3.  Per device d,
input i and configuration c:

  log T = log m_d + alpha*log(W_i/W_med) + s_d * exp(kappa * <z_c, a_{d,b(i)}>)
          + beta * h(t_c, b(i)) + tau * eps_{d,i,c}

  m_d      median runtimes of the "GEMM: Runtime vs Compilation" table
           (P:L180-184): Mali 95.00, Iris 19.45, HD500 39.49, Vega 1.92,
           Quadro 0.89 ms;
  W_i      2*M*N*K (work of the GEMM);
  z_c      config latent in R^4, N(0, I);
  a_{d,b}  unit-norm affinity of device d and input-size bucket b(i)
           (bucket = large/small per dimension, 8 buckets);
  t_c      tile class 0..7; h penalises large tiles on small inputs, which makes
           input-dependent specialists;
  s_d      per-device spread, kappa = 0.6 the skew of the log-slowdown
           distribution; both chosen so that the middle 50 % of variants have
           the slowdown IQRs quoted at P:L313 (Quadro 1.8-4.3x, Mali 2.6-13.2x);
           Iris/HD500/Vega are interpolated -- invented, flagged in DESIGN.md;
  tau      0.05 iid noise.
"""
from __future__ import annotations

import itertools

import numpy as np

SIZES = (256, 512, 1024, 4096)
#: GEMM inputs in lexicographic (M, N, K) order, 64 of them.
INPUTS = list(itertools.product(SIZES, SIZES, SIZES))

#: (name, median runtime ms [P:L180-184], spread s_d).
#: s_d fitted offline to the IQRs at P:L313 (Quadro, Mali); Iris, HD500, Vega
#: are interpolated (invented).
DEVICES = [
    ("Mali", 95.00, 1.81),
    ("Iris", 19.45, 1.50),
    ("HD500", 39.49, 1.60),
    ("Vega", 1.92, 1.30),
    ("Quadro", 0.89, 1.11),
]
KAPPA = 0.6
#: the latent is capped so the worst variant is a few hundred x slower than the
#: best, the range of the "Sample Data" rows (Quadro worst/best ~ 475x).
LAT_CAP = 2.2

ALPHA = 0.9
BETA = 0.8
TAU = 0.05
LATENT = 4


def _bucket(inp):
    m, n, k = inp
    return (m >= 1024) * 4 + (n >= 1024) * 2 + (k >= 1024)


def _nlarge(inp):
    return sum(x >= 1024 for x in inp)


def _config_draws(rng, C):
    z = rng.standard_normal((C, LATENT))
    tile = rng.integers(0, 8, size=C)
    return z, tile


def _device_affinity(rng, n_dev):
    w = rng.standard_normal((n_dev, LATENT))
    v = rng.standard_normal((8, LATENT))
    return w, v


def _rows(rng, med, sigma, w_d, v, z, tile, inputs):
    """Runtimes of one device on the given inputs: float32 [len(inputs)][C]."""
    W = np.array([2.0 * m * n * k for (m, n, k) in inputs])
    Wmed = 2.0 * 1024 ** 3
    out = np.empty((len(inputs), z.shape[0]), np.float32)
    for r, inp in enumerate(inputs):
        a = w_d + 0.7 * v[_bucket(inp)]
        a = a / np.linalg.norm(a)
        lat = z @ a                                   # N(0,1) per config
        small = 1.0 - _nlarge(inp) / 3.0              # 1 = all dims small
        h = np.maximum(0.0, tile / 7.0 - (1.0 - small)) * small
        eps = rng.standard_normal(z.shape[0])
        logt = (np.log(med) + ALPHA * np.log(W[r] / Wmed) + sigma * np.exp(KAPPA * np.minimum(lat, LAT_CAP))
                + BETA * h + TAU * eps)
        out[r] = np.exp(logt).astype(np.float32)
    return out


def paper_matrix(seed: int = 1, n_cfg: int = 1775, n_inputs: int = 64, devices=None):
    """Paper-shaped dense matrix: 1,775 configs x 64 inputs x 5 devices.

    ``devices`` selects a subset of DEVICES by index (default all five, in the
    "GPUs Studied" order); ``n_inputs`` takes the first inputs of
    the lexicographic grid.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    devs = list(range(len(DEVICES))) if devices is None else list(devices)
    z, tile = _config_draws(rng, n_cfg)
    w, v = _device_affinity(rng, len(DEVICES))
    inputs = INPUTS[:n_inputs]
    blocks, dev = [], []
    for d in devs:
        _, med, sig = DEVICES[d]
        blocks.append(_rows(rng, med, sig, w[d], v, z, tile, inputs))
        dev += [d] * len(inputs)
    return np.ascontiguousarray(np.vstack(blocks)), np.array(dev, np.int32)


def small_matrix(seed: int, n_cfg: int, n_dev: int, n_inputs: int):
    """Same model at arbitrary small shape (parity-test sizes)."""
    return paper_matrix(seed, n_cfg=n_cfg, n_inputs=n_inputs,
                        devices=[d % len(DEVICES) for d in range(n_dev)])


TINY_INPUTS = [(256, 1024, 256), (256, 1024, 4096), (4096, 1024, 256), (4096, 1024, 4096)]


def tiny(seed: int = 1):
    """BASELINE config 1: 16 configs x (4 inputs x 2 devices {Quadro, Mali}) = 8 envs."""
    rng = np.random.Generator(np.random.PCG64(seed))
    z, tile = _config_draws(rng, 16)
    w, v = _device_affinity(rng, len(DEVICES))
    blocks, dev = [], []
    for d in (4, 0):                                  # Quadro, Mali
        _, med, sig = DEVICES[d]
        blocks.append(_rows(rng, med, sig, w[d], v, z, tile, TINY_INPUTS))
        dev += [d] * 4
    return np.ascontiguousarray(np.vstack(blocks)), np.array(dev, np.int32)


def scaled(seed: int = 1, n_cfg: int = 65536, n_dev: int = 64, n_inputs: int = 64):
    """BASELINE config 5: 65,536 configs x (64 devices x 64 inputs) = 4,096 envs.

    Devices interpolate between the five archetypes (median, spread and
    affinity are convex blends of two neighbouring archetypes).
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    z, tile = _config_draws(rng, n_cfg)
    w, v = _device_affinity(rng, len(DEVICES))
    inputs = INPUTS[:n_inputs]
    T = np.empty((n_dev * len(inputs), n_cfg), np.float32)
    dev = np.repeat(np.arange(n_dev, dtype=np.int32), len(inputs))
    for d in range(n_dev):
        pos = d * (len(DEVICES) - 1) / max(1, n_dev - 1)
        a0 = int(np.floor(pos))
        a1 = min(a0 + 1, len(DEVICES) - 1)
        f = pos - a0
        med = np.exp((1 - f) * np.log(DEVICES[a0][1]) + f * np.log(DEVICES[a1][1]))
        sig = (1 - f) * DEVICES[a0][2] + f * DEVICES[a1][2]
        wd = (1 - f) * w[a0] + f * w[a1] + 0.3 * rng.standard_normal(LATENT)
        T[d * len(inputs):(d + 1) * len(inputs)] = _rows(rng, med, sig, wd, v, z, tile, inputs)
    return T, dev


def planted(seed: int, n_cfg: int, n_env: int, g: int, gamma: float = 2.0, n_dev: int = 1):
    """Planted g-specialist family.

    The environments are split into g contiguous blocks; specialist s (at a
    seeded random column) runs at the base runtime b_e on block s and at
    >= gamma * b_e elsewhere; every other configuration runs at
    >= gamma * b_e everywhere.  Returns (T, env_device, planted_columns sorted).
    """
    if gamma <= 1.0 or n_cfg < g or n_env < g:
        raise ValueError("need gamma > 1, n_cfg >= g, n_env >= g")
    rng = np.random.Generator(np.random.PCG64(seed))
    base = np.exp(rng.uniform(np.log(0.5), np.log(100.0), size=n_env))
    T = (base[:, None] * gamma * np.exp(rng.uniform(0.0, 1.5, size=(n_env, n_cfg))))
    cols = np.sort(rng.choice(n_cfg, size=g, replace=False))
    blocks = np.array_split(np.arange(n_env), g)
    for s, c in enumerate(cols):
        T[:, c] = base * gamma * np.exp(rng.uniform(0.0, 1.5, size=n_env))
        T[blocks[s], c] = base[blocks[s]]
    dev = (np.arange(n_env) * n_dev // n_env).astype(np.int32)
    return T.astype(np.float32), dev, [int(c) for c in cols]


def pow2(seed: int, n_cfg: int, n_env: int, max_exp: int = 6):
    """Power-of-two fixture: T = 2^m with integer m >= 0 and a 1.0 in every row,
    so every efficiency is an exact power of two (closed-form scores).
    Returns (T, m) with m int [E][C]."""
    rng = np.random.Generator(np.random.PCG64(seed))
    m = rng.integers(0, max_exp + 1, size=(n_env, n_cfg))
    zero_at = rng.integers(0, n_cfg, size=n_env)
    m[np.arange(n_env), zero_at] = 0
    return np.ldexp(np.ones_like(m, dtype=np.float32), m.astype(np.int32)), m
