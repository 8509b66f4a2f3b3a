// greedy.cu -- greedy forward selection (north_star): k dependent steps; each
// step scores S u {c} for every unselected configuration c in parallel and
// takes the argmax (ties -> lowest c).  Score of a set S (Eq. 1 under the
// best-member reading, P:L222 / P:L305-310), in log-slowdown form:
//     s(S u {c}) = sum_e min(cur[e], l[c][e]),  cur[e] = min_{c' in S} l[c'][e]
// (G = exp(-s/E) is monotone, so argmax G = argmin s).
//
// Two kernels families:
//  * RESIDENT (paper shape, matrix in L2): one cooperative persistent kernel for
//    all k steps.  cur[] lives in shared memory of every CTA, candidates are
//    scored in fp64 by one warp each (lanes over envs, xor-shuffle tree), the
//    per-CTA top-2 goes through global memory and a grid barrier, every CTA
//    merges the same list (deterministic) and updates its own cur[].
//    Latency-bound: k grid barriers.
//  * STREAM (scaled shape, 1 GiB fp32 matrix in HBM): per step one HBM-bound
//    scan kernel computes an fp32 key per config (direct sum at step 1, the
//    facility-location gain sum_e max(0, cur - l) afterwards), then one
//    single-CTA kernel derives a rigorous error window,
//    re-scores every config inside it in fp64 and commits the exact argmin.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include <map>
#include <mutex>
#include "pt_internal.cuh"

namespace cg = cooperative_groups;

#define PT_BIGI 0x7fffffff
#ifndef GR_PAIR
#define GR_PAIR 1   // resident greedy scores two candidates per warp pass (loads together; 0: one)
#endif
#ifndef GR_BPS
#define GR_BPS 1    // resident greedy: blocks per SM (with GR_PAIR, 1 and 2 measure the same)
#endif

__device__ __forceinline__ void top2_ins(double &s1, int &c1, double &s2, int &c2, double s,
                                         int c)
{
    if (s < s1 || (s == s1 && c < c1)) {
        s2 = s1;
        c2 = c1;
        s1 = s;
        c1 = c;
    } else if (c != c1 && (s < s2 || (s == s2 && c < c2))) {
        s2 = s;
        c2 = c;
    }
}

__device__ __forceinline__ void warp_top2(double &s1, int &c1, double &s2, int &c2)
{
    for (int o = 16; o; o >>= 1) {
        double a1 = __shfl_xor_sync(0xffffffffu, s1, o);
        double a2 = __shfl_xor_sync(0xffffffffu, s2, o);
        int b1 = __shfl_xor_sync(0xffffffffu, c1, o);
        int b2 = __shfl_xor_sync(0xffffffffu, c2, o);
        top2_ins(s1, c1, s2, c2, a1, b1);
        top2_ins(s1, c1, s2, c2, a2, b2);
    }
}

// s = sum_e min(cur[e], col[e]) over this lane's envs (e = lane, lane+32, ...,
// ascending: the fixed order of the reduction).  The column's loads are issued
// before the sums so one candidate costs one L2 round trip, not E_pad/32.
__device__ __forceinline__ double lane_sum_min(const double *cur, const double *__restrict__ col,
                                               int64_t E_pad, int lane)
{
    double acc = 0.0;
    for (int64_t e0 = lane; e0 < E_pad; e0 += 32 * 16) {
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; u++) v[u] = e0 + 32 * u < E_pad ? __ldg(col + e0 + 32 * u) : 0.0;
#pragma unroll
        for (int u = 0; u < 16; u++)
            if (e0 + 32 * u < E_pad) acc += fmin(cur[e0 + 32 * u], v[u]);
    }
    return acc;
}

// ---------------------------------------------------------------------------
// RESIDENT fp64 cooperative kernel
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_greedy_resident(const double *__restrict__ l64,
                                                          int64_t C, int64_t E_pad, int k,
                                                          double4 *__restrict__ blk,
                                                          int32_t *__restrict__ out_idx,
                                                          double *__restrict__ s1_tr,
                                                          double *__restrict__ s2_tr)
{
    extern __shared__ double sm[];
    double *cur = sm;
    uint32_t *taken = (uint32_t *)(cur + E_pad);
    __shared__ double ws1[8], ws2[8];
    __shared__ int wc1[8], wc2[8];
    __shared__ int cstar;
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t nwords = (C + 31) / 32;
    for (int64_t e = threadIdx.x; e < E_pad; e += blockDim.x) cur[e] = INFINITY;
    for (int64_t w = threadIdx.x; w < nwords; w += blockDim.x) taken[w] = 0u;
    __syncthreads();
    const int64_t gw = (int64_t)blockIdx.x * 8 + warp, nw = (int64_t)gridDim.x * 8;
    for (int t = 0; t < k; t++) {
        double s1 = INFINITY, s2 = INFINITY;
        int c1 = PT_BIGI, c2 = PT_BIGI;
#if GR_PAIR
        // two candidates per pass, both columns' loads in flight together
        for (int64_t c = gw; c < C; c += 2 * nw) {
            const int64_t c2n = c + nw;
            const bool ok1 = !(taken[c >> 5] >> (c & 31) & 1u);
            const bool ok2 = c2n < C && !(taken[c2n >> 5] >> (c2n & 31) & 1u);
            double a1 = 0.0, a2 = 0.0;
            for (int64_t e0 = lane; e0 < E_pad; e0 += 32 * 16) {   // lane's envs ascending
                double v1[16], v2[16];
#pragma unroll
                for (int u = 0; u < 16; u++) {
                    const int64_t e = e0 + 32 * u;
                    v1[u] = ok1 && e < E_pad ? __ldg(l64 + c * E_pad + e) : 0.0;
                    v2[u] = ok2 && e < E_pad ? __ldg(l64 + c2n * E_pad + e) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 16; u++) {
                    const int64_t e = e0 + 32 * u;
                    if (e < E_pad) {
                        const double cu = cur[e];
                        a1 += fmin(cu, v1[u]);
                        a2 += fmin(cu, v2[u]);
                    }
                }
            }
            for (int o = 16; o; o >>= 1) {
                a1 += __shfl_xor_sync(0xffffffffu, a1, o);
                a2 += __shfl_xor_sync(0xffffffffu, a2, o);
            }
            if (ok1) top2_ins(s1, c1, s2, c2, a1, (int)c);
            if (ok2) top2_ins(s1, c1, s2, c2, a2, (int)c2n);
        }
        if (false)
#endif
        for (int64_t c = gw; c < C; c += nw) {
            if (taken[c >> 5] >> (c & 31) & 1u) continue;
            const double *col = l64 + c * E_pad;
            double acc = lane_sum_min(cur, col, E_pad, lane);
            for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            top2_ins(s1, c1, s2, c2, acc, (int)c);
        }
        if (lane == 0) {
            ws1[warp] = s1;
            ws2[warp] = s2;
            wc1[warp] = c1;
            wc2[warp] = c2;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < 8; w++) {
                top2_ins(s1, c1, s2, c2, ws1[w], wc1[w]);
                top2_ins(s1, c1, s2, c2, ws2[w], wc2[w]);
            }
            blk[(t & 1) * gridDim.x + blockIdx.x] = make_double4(s1, s2, (double)c1, (double)c2);
        }
        grid.sync();
        if (warp == 0) {
            s1 = s2 = INFINITY;
            c1 = c2 = PT_BIGI;
            for (int b0 = lane; b0 < (int)gridDim.x; b0 += 32 * 10) {   // 10 records in flight per lane
                double4 r[10];
#pragma unroll
                for (int u = 0; u < 10; u++)
                    if (b0 + 32 * u < (int)gridDim.x) r[u] = blk[(t & 1) * gridDim.x + b0 + 32 * u];
#pragma unroll
                for (int u = 0; u < 10; u++)
                    if (b0 + 32 * u < (int)gridDim.x) {
                        top2_ins(s1, c1, s2, c2, r[u].x, (int)r[u].z);
                        top2_ins(s1, c1, s2, c2, r[u].y, (int)r[u].w);
                    }
            }
            warp_top2(s1, c1, s2, c2);
            if (lane == 0) {
                cstar = c1;
                if (blockIdx.x == 0) {
                    out_idx[t] = c1;
                    s1_tr[t] = s1;
                    s2_tr[t] = s2;
                }
            }
        }
        __syncthreads();
        const int cs = cstar;
        if (threadIdx.x == 0) taken[cs >> 5] |= 1u << (cs & 31);
        const double *col = l64 + (int64_t)cs * E_pad;
        for (int64_t e = threadIdx.x; e < E_pad; e += blockDim.x) cur[e] = fmin(cur[e], col[e]);
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// STREAM: fp32 scan + single-CTA fp64 window refine
// ---------------------------------------------------------------------------
// key[c] (minimised): step 0 -> sum_e l32[c][e];  later -> -sum_e max(0, cur-l).
// Each block also writes the two smallest keys it produced (blk2[blockIdx]).
// Odd steps scan the configurations in reverse so the L2-resident tail of the
// previous step's stream is read first.
__global__ void __launch_bounds__(256) k_greedy_scan(const float *__restrict__ l32, int64_t C,
                                                      int64_t E_pad,
                                                      const float *__restrict__ cur32,
                                                      const uint32_t *__restrict__ taken,
                                                      int gain_mode, int reverse,
                                                      int64_t cached_from, int64_t c_lo,
                                                      int64_t c_hi, float *__restrict__ key,
                                                      float2 *__restrict__ blk2)
{
    extern __shared__ float cur_s[];
    __shared__ float w1[8], w2[8];
    for (int64_t e = threadIdx.x; e < E_pad; e += blockDim.x) cur_s[e] = cur32[e];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nq = E_pad >> 2;
    const float4 *cur4 = reinterpret_cast<const float4 *>(cur_s);
    float k1 = INFINITY, k2 = INFINITY;
    const int64_t ns = c_hi - c_lo;   // this shard's configs [c_lo, c_hi)
    for (int64_t cc = gw; cc < ns; cc += nw) {
        const int64_t c = c_lo + (reverse ? ns - 1 - cc : cc);
        const float4 *col = reinterpret_cast<const float4 *>(l32 + c * E_pad);
        // the tail of this step's stream stays in L2 (normal loads) for the next,
        // reversed, step; the rest streams with evict-first loads
        const bool keep = cc >= cached_from;
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
        if (gain_mode) {
#pragma unroll 8
            for (int64_t q = lane; q < nq; q += 32) {
                float4 v = keep ? __ldg(col + q) : __ldcs(col + q);
                float4 m = cur4[q];
                a0 += fmaxf(m.x - v.x, 0.f);
                a1 += fmaxf(m.y - v.y, 0.f);
                a2 += fmaxf(m.z - v.z, 0.f);
                a3 += fmaxf(m.w - v.w, 0.f);
            }
        } else {
#pragma unroll 8
            for (int64_t q = lane; q < nq; q += 32) {
                float4 v = keep ? __ldg(col + q) : __ldcs(col + q);
                a0 += v.x;
                a1 += v.y;
                a2 += v.z;
                a3 += v.w;
            }
        }
        float acc = (a0 + a1) + (a2 + a3);
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        const bool tk = taken[c >> 5] >> (c & 31) & 1u;
        const float kv = tk ? INFINITY : (gain_mode ? -acc : acc);
        if (lane == 0) key[c] = kv;
        if (kv < k1) {
            k2 = k1;
            k1 = kv;
        } else if (kv < k2) {
            k2 = kv;
        }
    }
    // block: two smallest key values (each warp holds them for distinct configs)
    if (lane == 0) {
        w1[warp] = k1;
        w2[warp] = k2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float b1 = INFINITY, b2 = INFINITY;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
            const float xs[2] = {w1[w], w2[w]};
            for (int u = 0; u < 2; u++) {
                if (xs[u] < b1) {
                    b2 = b1;
                    b1 = xs[u];
                } else if (xs[u] < b2) {
                    b2 = xs[u];
                }
            }
        }
        blk2[blockIdx.x] = make_float2(b1, b2);
    }
}

struct pick_state {
    double S;       // sum_e cur64[e] over real envs (finite from step 1 on)
    double delta;   // gain-mode error bound of the last scan (see k_greedy_pick)
};

// one CTA of 1024 threads
__global__ void __launch_bounds__(1024) k_greedy_pick(
    const float *__restrict__ key, const float2 *__restrict__ blk2, int nblk, int64_t C,
    const double *__restrict__ l64, int64_t E_pad,
    int64_t E, float *__restrict__ cur32, double *__restrict__ cur64,
    uint32_t *__restrict__ taken, pick_state *__restrict__ st, int t, int gain_mode,
    double gamma, int32_t *__restrict__ cand, int32_t *__restrict__ out_idx,
    double *__restrict__ s1_tr, double *__restrict__ s2_tr, int32_t *__restrict__ ncand_tr,
    int64_t c_lo, int64_t c_hi, double4 *__restrict__ local_rec)
{
    __shared__ double rs1[32], rs2[32];
    __shared__ int ncand;
    __shared__ double thr;
    __shared__ int cstar;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double s1, s2;
    int c1, c2;
    // 1. two smallest key values over all configurations (from the per-block pairs)
    float f1 = INFINITY, f2 = INFINITY;
    for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
        const float2 r = blk2[b];
        const float xs[2] = {r.x, r.y};
        for (int u = 0; u < 2; u++) {
            if (xs[u] < f1) {
                f2 = f1;
                f1 = xs[u];
            } else if (xs[u] < f2) {
                f2 = xs[u];
            }
        }
    }
    for (int o = 16; o; o >>= 1) {
        const float a1 = __shfl_xor_sync(0xffffffffu, f1, o);
        const float a2 = __shfl_xor_sync(0xffffffffu, f2, o);
        // merge two sorted pairs (values of distinct configurations)
        const float n1 = fminf(f1, a1);
        const float n2 = fminf(fmaxf(f1, a1), fminf(f2, a2));
        f1 = n1;
        f2 = n2;
    }
    if (lane == 0) {
        rs1[warp] = f1;
        rs2[warp] = f2;
    }
    if (threadIdx.x == 0) ncand = 0;
    __syncthreads();
    if (warp == 0) {
        f1 = rs1[lane];
        f2 = rs2[lane];
        for (int o = 16; o; o >>= 1) {
            const float a1 = __shfl_xor_sync(0xffffffffu, f1, o);
            const float a2 = __shfl_xor_sync(0xffffffffu, f2, o);
            const float n1 = fminf(f1, a1);
            const float n2 = fminf(fmaxf(f1, a1), fminf(f2, a2));
            f1 = n1;
            f2 = n2;
        }
        if (lane == 0) {
            const double s1k = f1, s2k = f2;
            // window: keep every c that could be one of the
            // two exact best configurations
            const double u = 5.9604644775390625e-08;   // 2^-24
            if (!gain_mode) {
                // key = s_hat >= 0, |s_hat - s| <= gamma*s
                thr = (s2k == INFINITY) ? INFINITY : s2k * (1.0 + gamma) / (1.0 - gamma) * (1.0 + 1e-12);
            } else {
                // key = -g_hat; |g_hat - g| <= delta = 2u*S + gamma*g_max
                const double gmax = -s1k;
                const double delta = (2.0 * u * st->S + gamma * gmax) * 1.01 + 1e-300;
                st->delta = delta;
                thr = (s2k == INFINITY) ? INFINITY : s2k + 2.0 * delta;
            }
        }
    }
    __syncthreads();
    // 2. collect candidates (float4 sweep of the keys)
    const double th = thr;
    // (shard [c_lo, c_hi): c_lo is a multiple of 4 -- see pt_greedy_sharded)
    const int64_t C4 = c_lo / 4 + ((c_hi - c_lo) >> 2);
    const float4 *key4 = reinterpret_cast<const float4 *>(key);
    for (int64_t q0 = c_lo / 4; q0 < C4; q0 += 8 * (int64_t)blockDim.x) {
        float4 kv[8];   // 8 independent loads in flight per thread
#pragma unroll
        for (int r = 0; r < 8; r++) {
            const int64_t q = q0 + r * (int64_t)blockDim.x + threadIdx.x;
            kv[r] = q < C4 ? key4[q] : make_float4(INFINITY, INFINITY, INFINITY, INFINITY);
        }
#pragma unroll
        for (int r = 0; r < 8; r++) {
            const int64_t q = q0 + r * (int64_t)blockDim.x + threadIdx.x;
            const float xs[4] = {kv[r].x, kv[r].y, kv[r].z, kv[r].w};
#pragma unroll
            for (int u = 0; u < 4; u++)
                if (xs[u] != INFINITY && (double)xs[u] <= th) cand[atomicAdd(&ncand, 1)] = (int32_t)(4 * q + u);
        }
    }
    for (int64_t c = 4 * C4 + threadIdx.x; c < c_hi; c += blockDim.x) {
        const float kv = key[c];
        if (kv != INFINITY && (double)kv <= th) cand[atomicAdd(&ncand, 1)] = (int32_t)c;
    }
    __syncthreads();
    // 3. exact fp64 re-score of each candidate by the whole block (envs strided
    //    over 1024 threads, fixed-order block reduction: deterministic)
    const int n = ncand;
    s1 = s2 = INFINITY;
    c1 = c2 = PT_BIGI;
    for (int q = 0; q < n; q++) {
        const int c = cand[q];
        const double *col = l64 + (int64_t)c * E_pad;
        double part = 0.0;
        for (int64_t e = threadIdx.x; e < E_pad; e += blockDim.x) part += fmin(cur64[e], col[e]);
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) rs2[warp] = part;
        __syncthreads();
        if (threadIdx.x == 0) {
            double acc = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); w++) acc += rs2[w];
            top2_ins(s1, c1, s2, c2, acc, c);
        }
        __syncthreads();
    }
    if (local_rec) {   // sharded: report this shard's exact top-2, commit later
        if (threadIdx.x == 0) {
            *local_rec = make_double4(s1, s2, (double)c1, (double)c2);
            ncand_tr[t] = n;
        }
        return;
    }
    if (threadIdx.x == 0) {
        cstar = c1;
        out_idx[t] = c1;
        s1_tr[t] = s1;
        s2_tr[t] = s2;
        ncand_tr[t] = n;
        taken[c1 >> 5] |= 1u << (c1 & 31);
    }
    __syncthreads();
    // 4. commit: cur <- min(cur, l[c*]); S = sum over real envs (block reduce)
    const double *col = l64 + (int64_t)cstar * E_pad;
    double part = 0.0;
    for (int64_t e = threadIdx.x; e < E_pad; e += blockDim.x) {
        double v = fmin(cur64[e], col[e]);
        cur64[e] = v;
        cur32[e] = (float)v;
        if (e < E) part += v;
    }
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) rs1[warp] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
        double S = 0.0;
        for (int w = 0; w < 32; w++) S += rs1[w];
        st->S = S;
    }
}

// sharded greedy: merge the n_rank x 2 all-gathered records (s1, s2, c1, c2 per
// rank) into the global top-2 (s asc, config asc; identical on every rank) and
// commit the winner
__global__ void __launch_bounds__(1024) k_greedy_commit(const double *__restrict__ all, int n_rank,
                                                         int *__restrict__ fail,
                                                         const double *__restrict__ l64,
                                                         int64_t E_pad, int64_t E,
                                                         float *__restrict__ cur32,
                                                         double *__restrict__ cur64,
                                                         uint32_t *__restrict__ taken,
                                                         pick_state *__restrict__ st, int t,
                                                         int32_t *__restrict__ out_idx,
                                                         double *__restrict__ s1_tr,
                                                         double *__restrict__ s2_tr)
{
    __shared__ double rs[32];
    __shared__ double4 gsh;
    if (threadIdx.x == 0) {
        double s1 = INFINITY, s2 = INFINITY, c1 = (double)PT_BIGI, c2 = (double)PT_BIGI;
        for (int r = 0; r < n_rank; r++)
            for (int q = 0; q < 2; q++) {
                const double sv = all[4 * r + q], cv = all[4 * r + 2 + q];
                if (!(sv < INFINITY)) continue;
                if (sv < s1 || (sv == s1 && cv < c1)) {
                    s2 = s1;
                    c2 = c1;
                    s1 = sv;
                    c1 = cv;
                } else if (cv != c1 && (sv < s2 || (sv == s2 && cv < c2))) {
                    s2 = sv;
                    c2 = cv;
                }
            }
        if (!(s1 < INFINITY)) {
            *fail = 1;
            c1 = 0.0;   // stay in bounds; the host reports the failure
        }
        gsh = make_double4(s1, s2, c1, c2);
    }
    __syncthreads();
    const double4 g = gsh;
    const int cs = (int)g.z;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        out_idx[t] = cs;
        s1_tr[t] = g.x;
        s2_tr[t] = g.y;
        taken[cs >> 5] |= 1u << (cs & 31);
    }
    const double *col = l64 + (int64_t)cs * E_pad;
    double part = 0.0;
    for (int64_t e = threadIdx.x; e < E_pad; e += blockDim.x) {
        double v = fmin(cur64[e], col[e]);
        cur64[e] = v;
        cur32[e] = (float)v;
        if (e < E) part += v;
    }
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) rs[warp] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
        double S = 0.0;
        for (int w = 0; w < 32; w++) S += rs[w];
        st->S = S;
    }
}

// ---------------------------------------------------------------------------
// LAZY greedy (Minoux), opt-in PT_GREEDY_LAZY, streamed path.
// The facility-location gain g_c(S) = sum_e max(0, cur_e - l[c][e]) is
// submodular, so a gain measured at an earlier step is an upper bound later.
// After the second full scan ub[c] = g_hat_c + delta (rigorous: the scan's
// fp32 error bound); every later step re-scores exactly only the configs whose
// bound can still reach the best exact gain, and tightens their bounds.
// ---------------------------------------------------------------------------
__global__ void k_lazy_init(const float *__restrict__ key, int64_t C, const uint32_t *__restrict__ taken,
                            const pick_state *__restrict__ st, double *__restrict__ ub)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    const bool tk = taken[c >> 5] >> (c & 31) & 1u;
    ub[c] = tk ? -INFINITY : -(double)key[c] + st->delta;
}

// one CTA (1024 threads) per lazy step
__global__ void __launch_bounds__(1024) k_lazy_step(
    int64_t C, const double *__restrict__ l64, int64_t E_pad, int64_t E, float *__restrict__ cur32,
    double *__restrict__ cur64, uint32_t *__restrict__ taken, pick_state *__restrict__ st,
    double *__restrict__ ub, int32_t *__restrict__ cand, double *__restrict__ cs, int t,
    int32_t *__restrict__ out_idx, double *__restrict__ s1_tr, double *__restrict__ s2_tr,
    int32_t *__restrict__ ncand_tr)
{
    __shared__ double rs1[32], rs2[32];
    __shared__ int rc1[32], rc2[32];
    __shared__ int ncand, c0s, cstar;
    __shared__ double thr_s;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double S = st->S;
    const double slack = 1e-12 * S + 1e-300;
    // a. argmax of the upper bounds (ties -> lowest index)
    double bu = -INFINITY;
    int bc = PT_BIGI;
    for (int64_t c = threadIdx.x; c < C; c += blockDim.x) {
        const double v = ub[c];
        if (v > bu) { bu = v; bc = (int)c; }
    }
    for (int o = 16; o; o >>= 1) {
        const double v = __shfl_xor_sync(0xffffffffu, bu, o);
        const int c = __shfl_xor_sync(0xffffffffu, bc, o);
        if (v > bu || (v == bu && c < bc)) { bu = v; bc = c; }
    }
    if (lane == 0) { rs1[warp] = bu; rc1[warp] = bc; }
    if (threadIdx.x == 0) ncand = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 32; w++)
            if (rs1[w] > bu || (rs1[w] == bu && rc1[w] < bc)) { bu = rs1[w]; bc = rc1[w]; }
        c0s = bc;
    }
    __syncthreads();
    // b. exact score of c0 (block reduction) -> the gain every candidate must reach
    {
        const double *col = l64 + (int64_t)c0s * E_pad;
        double part = 0.0;
        for (int64_t e = threadIdx.x; e < E_pad; e += blockDim.x) part += fmin(cur64[e], col[e]);
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) rs2[warp] = part;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s0 = 0.0;
            for (int w = 0; w < 32; w++) s0 += rs2[w];
            thr_s = (S - s0) - slack;   // gain of c0, lowered by the rounding slack
        }
        __syncthreads();
    }
    // c. every config whose bound reaches that gain is a candidate
    const double thr = thr_s;
    for (int64_t c = threadIdx.x; c < C; c += blockDim.x)
        if (ub[c] >= thr) cand[atomicAdd(&ncand, 1)] = (int32_t)c;
    __syncthreads();
    // d. exact scores of the candidates (warp each), then the argmin (ties -> lowest c)
    const int n = ncand;
    double s1 = INFINITY, s2 = INFINITY;
    int c1 = PT_BIGI, c2 = PT_BIGI;
    for (int q = warp; q < n; q += 32) {
        const int c = cand[q];
        const double *col = l64 + (int64_t)c * E_pad;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int64_t e = lane;
        for (; e + 96 < E_pad; e += 128) {
            a0 += fmin(cur64[e], col[e]);
            a1 += fmin(cur64[e + 32], col[e + 32]);
            a2 += fmin(cur64[e + 64], col[e + 64]);
            a3 += fmin(cur64[e + 96], col[e + 96]);
        }
        for (; e < E_pad; e += 32) a0 += fmin(cur64[e], col[e]);
        double acc = (a0 + a1) + (a2 + a3);
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
            cs[q] = acc;
            ub[c] = (S - acc) + slack;          // e. tightened bound for later steps
        }
        top2_ins(s1, c1, s2, c2, acc, c);
    }
    if (lane == 0) { rs1[warp] = s1; rs2[warp] = s2; rc1[warp] = c1; rc2[warp] = c2; }
    __syncthreads();
    if (warp == 0) {
        s1 = rs1[lane]; s2 = rs2[lane]; c1 = rc1[lane]; c2 = rc2[lane];
        warp_top2(s1, c1, s2, c2);
        if (lane == 0) {
            cstar = c1;
            out_idx[t] = c1;
            s1_tr[t] = s1;
            s2_tr[t] = s2;        // second best among the candidates (gap: lower bound)
            ncand_tr[t] = n;
            taken[c1 >> 5] |= 1u << (c1 & 31);
            ub[c1] = -INFINITY;
        }
    }
    __syncthreads();
    // f. commit
    const double *col = l64 + (int64_t)cstar * E_pad;
    double part = 0.0;
    for (int64_t e = threadIdx.x; e < E_pad; e += blockDim.x) {
        double v = fmin(cur64[e], col[e]);
        cur64[e] = v;
        cur32[e] = (float)v;
        if (e < E) part += v;
    }
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) rs1[warp] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
        double Sn = 0.0;
        for (int w = 0; w < 32; w++) Sn += rs1[w];
        st->S = Sn;
    }
}

__global__ void k_fill_f64(double *p, int64_t n, double v)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}
__global__ void k_fill_f32(float *p, int64_t n, float v)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

// ---------------------------------------------------------------------------
static bool use_stream(const pt_ctx *ctx, const pt_view *v)
{
    if (ctx->flags & (PT_GREEDY_STREAM | PT_GREEDY_LAZY)) return true;
    const double bytes = (double)v->C * (double)v->E_pad * 8.0;
    return bytes > 64.0 * (1 << 20) || v->E_pad * 8 > 160 * 1024;
}

pt_status pt_greedy_seed_enqueue(pt_ctx *ctx, const pt_view *v, int32_t k)
{
    if (k < 1 || k > v->C || use_stream(ctx, v)) return PT_EINVAL;   // caller takes the host path
    const int64_t C = v->C, E_pad = v->E_pad;
    const int64_t nwords = (C + 31) / 32;
    cudaStream_t s = ctx->stream;
    const size_t smem = sizeof(double) * E_pad + sizeof(uint32_t) * nwords;
    static std::mutex mu;
    static std::map<std::pair<int, size_t>, int> occ_cache;   // (device, dynamic smem) -> blocks per SM
    int occ = 0;
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = occ_cache.find(std::make_pair(ctx->dev, smem));
        if (it == occ_cache.end()) {
            PT_TRY(pt_smem_optin(ctx, (const void *)k_greedy_resident));
            PT_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_greedy_resident, 256, smem));
            occ_cache[std::make_pair(ctx->dev, smem)] = occ;
        } else {
            occ = it->second;
        }
    }
    if (occ < 1) return PT_EINVAL;
    const int nblk = ctx->num_sms * std::min(occ, GR_BPS);
    pt_view *mv = const_cast<pt_view *>(v);
    if (mv->d_seed_s2) pt_dfree(ctx, mv->d_seed_s2);
    if (mv->d_seed_idx) pt_dfree(ctx, mv->d_seed_idx);
    mv->d_seed_s2 = nullptr;
    mv->d_seed_idx = nullptr;
    mv->d_seed_k = 0;
    PT_TRY(pt_dalloc(ctx, (void **)&mv->d_seed_s2, sizeof(double) * k));
    PT_TRY(pt_dalloc(ctx, (void **)&mv->d_seed_idx, sizeof(int32_t) * k));
    char *tmp = nullptr;
    const size_t o_s1 = pt_round_up(sizeof(double4) * 2 * nblk, 256) + 256;
    PT_TRY(pt_dalloc(ctx, (void **)&tmp, o_s1 + pt_round_up(sizeof(double) * k, 256)));
    double4 *blk = (double4 *)tmp;
    int32_t *d_idx = mv->d_seed_idx;
    double *d_s1 = (double *)(tmp + o_s1), *d_s2 = mv->d_seed_s2;
    const double *l64 = v->l64;
    int kk = k;
    int64_t CC = C, EE = E_pad;
    void *args[] = {(void *)&l64, (void *)&CC, (void *)&EE, (void *)&kk, (void *)&blk,
                    (void *)&d_idx, (void *)&d_s1, (void *)&d_s2};
    PT_CK(cudaLaunchCooperativeKernel((void *)k_greedy_resident, dim3(nblk), dim3(256), args, smem, s));
    ctx->stats.launches++;
    pt_dfree(ctx, tmp);   // stream-ordered: released after the kernel
    mv->d_seed_k = k;
    return PT_OK;
}

pt_status pt_greedy_view(pt_ctx *ctx, const pt_view *v, int32_t k, int32_t *out_idx,
                         double *s1_trace, double *s2_trace)
{
    if (k < 1 || k > v->C) return pt_fail(PT_EINVAL, "k=%d outside [1, %lld]", k, (long long)v->C);
    const int64_t C = v->C, E_pad = v->E_pad;
    const int64_t nwords = (C + 31) / 32;
    cudaStream_t s = ctx->stream;
    pt_hostio io(ctx);
    std::vector<int32_t> nc;   // stream path: fp64 re-scores per step
    PT_CK(cudaEventRecord(ctx->ev0, s));
    if (!use_stream(ctx, v)) {
        size_t smem = sizeof(double) * E_pad + sizeof(uint32_t) * nwords;
        if (smem > 48 * 1024)
            PT_CK(cudaFuncSetAttribute(k_greedy_resident, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
        int occ = 0;
        PT_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_greedy_resident, 256, smem));
        if (occ < 1) return pt_fail(PT_ECUDA, "resident greedy kernel cannot be co-resident");
        // 2 blocks per SM when they fit: at most one candidate per warp per step at the paper shape
        const int nblk = ctx->num_sms * std::min(occ, GR_BPS);
        size_t bytes = pt_round_up(sizeof(double4) * 2 * nblk, 256) + 256 +
                       pt_round_up(sizeof(int32_t) * k, 256) + 2 * pt_round_up(sizeof(double) * k, 256);
        void *scr = nullptr;
        PT_TRY(pt_scratch(ctx, bytes, &scr));
        char *p = (char *)scr;
        double4 *blk = (double4 *)p;
        p += pt_round_up(sizeof(double4) * 2 * nblk, 256) + 256;
        int32_t *d_idx = (int32_t *)p;
        p += pt_round_up(sizeof(int32_t) * k, 256);
        double *d_s1 = (double *)p;
        p += pt_round_up(sizeof(double) * k, 256);
        double *d_s2 = (double *)p;
        const double *l64 = v->l64;
        int kk = k;
        void *args[] = {(void *)&l64, (void *)&C, (void *)&E_pad, (void *)&kk, (void *)&blk,
                        (void *)&d_idx, (void *)&d_s1, (void *)&d_s2};
        PT_CK(cudaLaunchCooperativeKernel((void *)k_greedy_resident, dim3(nblk), dim3(256), args,
                                          smem, s));
        ctx->stats.launches++;
        PT_TRY(io.d2h(out_idx, d_idx, sizeof(int32_t) * k));
        PT_TRY(io.d2h(s1_trace, d_s1, sizeof(double) * k));
        PT_TRY(io.d2h(s2_trace, d_s2, sizeof(double) * k));
    } else {
        // buffers: key[C] f32, cand[C] i32, taken[nwords], cur32[E_pad], cur64[E_pad],
        // st, traces
        size_t off = 0;
        auto take = [&](size_t b) { size_t o = off; off += pt_round_up(b, 256); return o; };
        size_t o_key = take(sizeof(float) * C), o_cand = take(sizeof(int32_t) * C),
               o_taken = take(sizeof(uint32_t) * nwords), o_c32 = take(sizeof(float) * E_pad),
               o_c64 = take(sizeof(double) * E_pad), o_st = take(sizeof(pick_state)),
               o_idx = take(sizeof(int32_t) * k), o_s1 = take(sizeof(double) * k),
               o_s2 = take(sizeof(double) * k), o_nc = take(sizeof(int32_t) * k),
               o_blk = take(sizeof(float2) * (size_t)ctx->num_sms * 32);
        void *scr = nullptr;
        PT_TRY(pt_scratch(ctx, off, &scr));
        char *b = (char *)scr;
        float *key = (float *)(b + o_key);
        int32_t *cand = (int32_t *)(b + o_cand);
        uint32_t *taken = (uint32_t *)(b + o_taken);
        float *cur32 = (float *)(b + o_c32);
        double *cur64 = (double *)(b + o_c64);
        pick_state *st = (pick_state *)(b + o_st);
        int32_t *d_idx = (int32_t *)(b + o_idx), *d_nc = (int32_t *)(b + o_nc);
        double *d_s1 = (double *)(b + o_s1), *d_s2 = (double *)(b + o_s2);
        float2 *blk2 = (float2 *)(b + o_blk);
        PT_CK(cudaMemsetAsync(taken, 0, sizeof(uint32_t) * nwords, s));
        PT_CK(cudaMemsetAsync(st, 0, sizeof(pick_state), s));
        k_fill_f64<<<(unsigned)((E_pad + 255) / 256), 256, 0, s>>>(cur64, E_pad, INFINITY);
        k_fill_f32<<<(unsigned)((E_pad + 255) / 256), 256, 0, s>>>(cur32, E_pad, INFINITY);
        ctx->stats.launches += 2;
        const size_t smem = sizeof(float) * E_pad;
        if (smem > 48 * 1024)
            PT_CK(cudaFuncSetAttribute(k_greedy_scan, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
        // k_greedy_scan's fp32 sum: each lane keeps 4 accumulators over E_pad/128
        // float4 slots, then (a0+a1)+(a2+a3) and a 5-level xor tree: every term
        // passes through at most E_pad/128 + 7 roundings (plus 1 for the term
        // itself in gain mode) -> Higham gamma_n with n = E_pad/128 + 8.
        const double u = 5.9604644775390625e-08;
        const double n = (double)((E_pad + 127) / 128) + 8.0;
        const double gamma = n * u / (1.0 - n * u) * 1.01;
        int occ = 0;
        PT_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_greedy_scan, 256, smem));
        const int64_t want_blocks = (C * 32 + 255) / 256;
        const int grid = (int)std::min<int64_t>(want_blocks, (int64_t)ctx->num_sms * std::max(occ, 1));
        // keep the last ~80 MB of each step's stream L2-resident (L2 is ~126 MB)
        const int64_t keep_cfgs = (int64_t)(80.0 * (1 << 20) / (4.0 * (double)E_pad));
        const int64_t cached_from = std::max<int64_t>(0, C - keep_cfgs);
        const bool lazy = (ctx->flags & PT_GREEDY_LAZY) != 0;
        double *ub = nullptr, *cs = nullptr;
        if (lazy && k > 2) {
            PT_TRY(pt_dalloc(ctx, (void **)&ub, sizeof(double) * C));
            PT_TRY(pt_dalloc(ctx, (void **)&cs, sizeof(double) * C));
        }
        // lazy mode: a step re-scores only configs whose upper bound can still win;
        // when the previous lazy step needed more than `lazy_max` re-scores the
        // bounds have gone stale and the step does a full scan instead (which
        // also refreshes every bound)
        const int32_t lazy_max = (int32_t)std::max<int64_t>(64, C / 256);
        bool ub_fresh = false, full_next = true;
        for (int t = 0; t < k; t++) {
            if (lazy && t >= 2 && !full_next) {
                if (!ub_fresh) {
                    k_lazy_init<<<(unsigned)((C + 255) / 256), 256, 0, s>>>(key, C, taken, st, ub);
                    ctx->stats.launches++;
                    ub_fresh = true;
                }
                k_lazy_step<<<1, 1024, 0, s>>>(C, v->l64, E_pad, v->E, cur32, cur64, taken, st, ub, cand,
                                               cs, t, d_idx, d_s1, d_s2, d_nc);
                ctx->stats.launches++;
                int32_t nc_t = 0;
                PT_CK(cudaMemcpyAsync(&nc_t, d_nc + t, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
                PT_CK(cudaStreamSynchronize(s));
                full_next = nc_t > lazy_max;
                continue;
            }
            if (lazy && t >= 1) {
                ub_fresh = false;     // this full scan's keys become the new bounds
                full_next = false;
            }
            k_greedy_scan<<<grid, 256, smem, s>>>(v->l32, C, E_pad, cur32, taken, t > 0, t & 1,
                                                  cached_from, 0, C, key, blk2);
            k_greedy_pick<<<1, 1024, 0, s>>>(key, blk2, grid, C, v->l64, E_pad, v->E, cur32, cur64, taken, st,
                                             t, t > 0, gamma, cand, d_idx, d_s1, d_s2, d_nc, 0, C, nullptr);
            ctx->stats.launches += 2;
        }
        PT_CK(cudaGetLastError());
        PT_TRY(io.d2h(out_idx, d_idx, sizeof(int32_t) * k));
        PT_TRY(io.d2h(s1_trace, d_s1, sizeof(double) * k));
        PT_TRY(io.d2h(s2_trace, d_s2, sizeof(double) * k));
        pt_dfree(ctx, ub);
        pt_dfree(ctx, cs);
        nc.resize(k);
        PT_TRY(io.d2h(nc.data(), d_nc, sizeof(int32_t) * k));
    }
    PT_CK(cudaEventRecord(ctx->ev1, s));
    PT_TRY(io.finish());
    if ((size_t)k > v->greedy_s2.size()) {
        v->greedy_s2.assign(s2_trace, s2_trace + k);
        v->greedy_idx.assign(out_idx, out_idx + k);
    }
    if (!nc.empty()) {
        int64_t tot = 0;
        for (int t = 0; t < k; t++) tot += nc[t];
        ctx->stats.greedy_candidates = tot;
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    ctx->stats.greedy_ms = ms;
    return PT_OK;
}

extern "C" pt_status pt_greedy_select(pt_ctx *ctx, int32_t k, const uint8_t *env_mask,
                                      int32_t objective, int32_t *out_idx, double *out_G_trace,
                                      double *out_gap_trace)
{
    PT_NVTX();
    if (!ctx || !out_idx) return pt_fail(PT_EINVAL, "NULL argument");
    if (objective != PT_OBJ_GEOMEAN && objective != PT_OBJ_FLEET)
        return pt_fail(PT_EINVAL, "unknown objective %d", objective);
    PT_CK(cudaSetDevice(ctx->dev));
    if (objective == PT_OBJ_FLEET) return pt_fleet_greedy(ctx, k, env_mask, out_idx, out_G_trace, out_gap_trace);
    const pt_view *v = nullptr;
    PT_TRY(pt_get_view(ctx, env_mask, &v));
    std::vector<double> s1(k > 0 ? k : 1), s2(k > 0 ? k : 1);
    PT_TRY(pt_greedy_view(ctx, v, k, out_idx, s1.data(), s2.data()));
    const double invE = 1.0 / (double)v->E;
    for (int t = 0; t < k; t++) {
        double g1 = exp(-s1[t] * invE);
        if (out_G_trace) out_G_trace[t] = g1;
        if (out_gap_trace) out_gap_trace[t] = std::isinf(s2[t]) ? INFINITY : g1 - exp(-s2[t] * invE);
    }
    return PT_OK;
}

// ---------------------------------------------------------------------------
// pt_greedy_sharded (SURVEY §8(e) "greedy, scaled", NEXT #3): the configurations
// are cut into shard_count contiguous ranges; this rank streams only its range
// (1/N of the matrix per step -- L2-sized at N = 8 for the scaled matrix), picks
// its exact local top-2 (fp32 window + fp64 refine, as the streamed path), and
// the ranks all-gather those 2 records (4 doubles) through the caller's
// callback; every rank merges them identically and commits the winner from its
// own replica of the matrix (no column broadcast needed).
// ---------------------------------------------------------------------------
static pt_status greedy_sharded_impl(pt_ctx *ctx, int32_t k, const uint8_t *env_mask, int32_t shard_rank,
                                     int32_t shard_count, pt_allgather_fn allgather,
                                     pt_dev_allgather_fn dev_allgather, void *user, int32_t *out_idx,
                                     double *out_G_trace, double *out_gap_trace)
{
    if (!ctx || !out_idx || (!allgather && !dev_allgather)) return pt_fail(PT_EINVAL, "NULL argument");
    if (shard_count < 1 || shard_rank < 0 || shard_rank >= shard_count)
        return pt_fail(PT_EINVAL, "bad shard %d of %d", shard_rank, shard_count);
    PT_CK(cudaSetDevice(ctx->dev));
    const pt_view *v = nullptr;
    PT_TRY(pt_get_view(ctx, env_mask, &v));
    const int64_t C = v->C, E_pad = v->E_pad;
    if (k < 1 || k > C) return pt_fail(PT_EINVAL, "k=%d outside [1, %lld]", k, (long long)C);
    // shard boundaries on multiples of 64 configs
    auto bound = [&](int64_t r) { return std::min(C, (C * r / shard_count + 63) / 64 * 64); };
    const int64_t c_lo = bound(shard_rank), c_hi = bound(shard_rank + 1);
    cudaStream_t s = ctx->stream;
    const int64_t nwords = (C + 31) / 32;
    size_t off = 0;
    auto take = [&](size_t b) { size_t o = off; off += pt_round_up(b, 256); return o; };
    const size_t o_key = take(sizeof(float) * C), o_cand = take(sizeof(int32_t) * C),
                 o_taken = take(sizeof(uint32_t) * nwords), o_c32 = take(sizeof(float) * E_pad),
                 o_c64 = take(sizeof(double) * E_pad), o_st = take(sizeof(pick_state)),
                 o_idx = take(sizeof(int32_t) * k), o_s1 = take(sizeof(double) * k),
                 o_s2 = take(sizeof(double) * k), o_nc = take(sizeof(int32_t) * k),
                 o_blk = take(sizeof(float2) * (size_t)ctx->num_sms * 32), o_rec = take(sizeof(double4) * 2),
                 o_all = take(sizeof(double) * 4 * (size_t)shard_count), o_fail = take(sizeof(int));
    void *scr = nullptr;
    PT_TRY(pt_scratch(ctx, off, &scr));
    char *b = (char *)scr;
    float *key = (float *)(b + o_key);
    int32_t *cand = (int32_t *)(b + o_cand), *d_idx = (int32_t *)(b + o_idx), *d_nc = (int32_t *)(b + o_nc);
    uint32_t *taken = (uint32_t *)(b + o_taken);
    float *cur32 = (float *)(b + o_c32);
    double *cur64 = (double *)(b + o_c64), *d_s1 = (double *)(b + o_s1), *d_s2 = (double *)(b + o_s2);
    pick_state *st = (pick_state *)(b + o_st);
    float2 *blk2 = (float2 *)(b + o_blk);
    double4 *rec = (double4 *)(b + o_rec);   // [0] this rank's local top-2
    double *d_all = (double *)(b + o_all);
    int *d_fail = (int *)(b + o_fail);
    PT_CK(cudaMemsetAsync(d_fail, 0, sizeof(int), s));
    // a rank with an empty shard reports no candidate
    const double4 none = make_double4(INFINITY, INFINITY, (double)PT_BIGI, (double)PT_BIGI);
    if (!(c_hi > c_lo)) PT_CK(cudaMemcpyAsync(rec, &none, sizeof(double4), cudaMemcpyHostToDevice, s));
    PT_CK(cudaMemsetAsync(taken, 0, sizeof(uint32_t) * nwords, s));
    PT_CK(cudaMemsetAsync(st, 0, sizeof(pick_state), s));
    PT_CK(cudaMemsetAsync(key, 0x7f, sizeof(float) * C, s));   // large finite: never a candidate
    k_fill_f64<<<(unsigned)((E_pad + 255) / 256), 256, 0, s>>>(cur64, E_pad, INFINITY);
    k_fill_f32<<<(unsigned)((E_pad + 255) / 256), 256, 0, s>>>(cur32, E_pad, INFINITY);
    ctx->stats.launches += 2;
    const size_t smem = sizeof(float) * E_pad;
    if (smem > 48 * 1024)
        PT_CK(cudaFuncSetAttribute(k_greedy_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const double u = 5.9604644775390625e-08;
    const double n = (double)((E_pad + 127) / 128) + 8.0;
    const double gamma = n * u / (1.0 - n * u) * 1.01;
    int occ = 0;
    PT_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_greedy_scan, 256, smem));
    const int64_t ns = std::max<int64_t>(c_hi - c_lo, 1);
    const int grid = (int)std::min<int64_t>((ns * 32 + 255) / 256, (int64_t)ctx->num_sms * std::max(occ, 1));
    const int64_t keep_cfgs = (int64_t)(80.0 * (1 << 20) / (4.0 * (double)E_pad));
    const int64_t cached_from = std::max<int64_t>(0, ns - keep_cfgs);
    std::vector<double> mine(4), all(4 * (size_t)shard_count);
    int64_t n_cand = 0;
    PT_CK(cudaEventRecord(ctx->ev0, s));
    for (int t = 0; t < k; t++) {
        if (dev_allgather) {
            // stream-ordered exchange: no host synchronisation inside the loop
            if (c_hi > c_lo) {
                k_greedy_scan<<<grid, 256, smem, s>>>(v->l32, C, E_pad, cur32, taken, t > 0, t & 1,
                                                      cached_from, c_lo, c_hi, key, blk2);
                k_greedy_pick<<<1, 1024, 0, s>>>(key, blk2, grid, C, v->l64, E_pad, v->E, cur32, cur64, taken,
                                                 st, t, t > 0, gamma, cand, d_idx, d_s1, d_s2, d_nc, c_lo,
                                                 c_hi, rec);
                ctx->stats.launches += 2;
            }
            PT_CK(cudaGetLastError());
            if (dev_allgather(user, (const double *)rec, 4, d_all, (void *)s) != 0)
                return pt_fail(PT_ENCCL, "device all-gather callback failed at step %d", t);
            k_greedy_commit<<<1, 1024, 0, s>>>(d_all, shard_count, d_fail, v->l64, E_pad, v->E, cur32, cur64,
                                               taken, st, t, d_idx, d_s1, d_s2);
            ctx->stats.launches += 1;
            continue;
        }
        double4 hl = none;
        if (c_hi > c_lo) {
            k_greedy_scan<<<grid, 256, smem, s>>>(v->l32, C, E_pad, cur32, taken, t > 0, t & 1, cached_from,
                                                  c_lo, c_hi, key, blk2);
            k_greedy_pick<<<1, 1024, 0, s>>>(key, blk2, grid, C, v->l64, E_pad, v->E, cur32, cur64, taken,
                                             st, t, t > 0, gamma, cand, d_idx, d_s1, d_s2, d_nc, c_lo, c_hi,
                                             rec);
            ctx->stats.launches += 2;
            PT_CK(cudaMemcpyAsync(&hl, rec, sizeof(double4), cudaMemcpyDeviceToHost, s));
            int32_t nc = 0;
            PT_CK(cudaMemcpyAsync(&nc, d_nc + t, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
            PT_CK(cudaStreamSynchronize(s));
            n_cand += nc;
        }
        mine[0] = hl.x;
        mine[1] = hl.y;
        mine[2] = hl.z;
        mine[3] = hl.w;
        if (allgather(user, mine.data(), 4, all.data()) != 0)
            return pt_fail(PT_ENCCL, "all-gather callback failed at step %d", t);
        // the merge runs in the commit kernel (same code as the device-exchange path);
        // the host only checks that some rank still had a candidate
        bool any = false;
        for (int r = 0; r < shard_count; r++) any = any || all[4 * r] < INFINITY;
        if (!any) return pt_fail(PT_EINVAL, "no candidate left at step %d", t);
        PT_CK(cudaMemcpyAsync(d_all, all.data(), sizeof(double) * 4 * shard_count, cudaMemcpyHostToDevice, s));
        k_greedy_commit<<<1, 1024, 0, s>>>(d_all, shard_count, d_fail, v->l64, E_pad, v->E, cur32, cur64, taken,
                                           st, t, d_idx, d_s1, d_s2);
        ctx->stats.launches++;
    }
    PT_CK(cudaEventRecord(ctx->ev1, s));
    PT_CK(cudaGetLastError());
    if (dev_allgather) {
        int fail = 0;
        std::vector<int32_t> nc(k, 0);
        PT_CK(cudaMemcpyAsync(&fail, d_fail, sizeof(int), cudaMemcpyDeviceToHost, s));
        if (c_hi > c_lo) PT_CK(cudaMemcpyAsync(nc.data(), d_nc, sizeof(int32_t) * k, cudaMemcpyDeviceToHost, s));
        PT_CK(cudaStreamSynchronize(s));
        if (fail) return pt_fail(PT_EINVAL, "no candidate left (all-gathered records empty)");
        for (int t = 0; t < k; t++) n_cand += nc[t];
    }
    std::vector<double> h1(k), h2(k);
    PT_CK(cudaMemcpyAsync(out_idx, d_idx, sizeof(int32_t) * k, cudaMemcpyDeviceToHost, s));
    PT_CK(cudaMemcpyAsync(h1.data(), d_s1, sizeof(double) * k, cudaMemcpyDeviceToHost, s));
    PT_CK(cudaMemcpyAsync(h2.data(), d_s2, sizeof(double) * k, cudaMemcpyDeviceToHost, s));
    PT_CK(cudaStreamSynchronize(s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    ctx->stats.greedy_ms = ms;
    ctx->stats.greedy_candidates = n_cand;
    const double invE = 1.0 / (double)v->E;
    for (int t = 0; t < k; t++) {
        const double g1 = exp(-h1[t] * invE);
        if (out_G_trace) out_G_trace[t] = g1;
        if (out_gap_trace) out_gap_trace[t] = std::isinf(h2[t]) ? INFINITY : g1 - exp(-h2[t] * invE);
    }
    return PT_OK;
}

extern "C" pt_status pt_greedy_sharded(pt_ctx *ctx, int32_t k, const uint8_t *env_mask, int32_t shard_rank,
                                       int32_t shard_count, pt_allgather_fn allgather, void *user,
                                       int32_t *out_idx, double *out_G_trace, double *out_gap_trace)
{
    PT_NVTX();
    if (!allgather) return pt_fail(PT_EINVAL, "NULL argument");
    return greedy_sharded_impl(ctx, k, env_mask, shard_rank, shard_count, allgather, nullptr, user, out_idx,
                               out_G_trace, out_gap_trace);
}

extern "C" pt_status pt_greedy_sharded_dev(pt_ctx *ctx, int32_t k, const uint8_t *env_mask, int32_t shard_rank,
                                           int32_t shard_count, pt_dev_allgather_fn allgather, void *user,
                                           int32_t *out_idx, double *out_G_trace, double *out_gap_trace)
{
    PT_NVTX();
    if (!allgather) return pt_fail(PT_EINVAL, "NULL argument");
    return greedy_sharded_impl(ctx, k, env_mask, shard_rank, shard_count, nullptr, allgather, user, out_idx,
                               out_G_trace, out_gap_trace);
}
