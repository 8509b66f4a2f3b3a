// holdout.cu -- pt_eval_holdout: leave-one-device-out generalization, the
// analogue of the paper's unseen-device experiment (Sec. 5.8):
// select on the environments of the other devices (train scope), evaluate the
// chosen set on the held-out device's environments, each normalised by its own
// Oracle best[e], and compare with a selection made directly on the
// held-out environments (the "known" baseline).
#include <algorithm>
#include <cmath>
#include <vector>

#include "pt_internal.cuh"

static pt_status select_on(pt_ctx *ctx, const uint8_t *mask, int32_t k, int32_t method,
                           int32_t *idx, double *G)
{
    if (method == 0) {
        std::vector<double> gt(k), gp(k);
        PT_TRY(pt_greedy_select(ctx, k, mask, PT_OBJ_GEOMEAN, idx, gt.data(), gp.data()));
        *G = gt[k - 1];
    } else {
        PT_TRY(pt_exhaustive_best(ctx, k, mask, PT_OBJ_GEOMEAN, 0, 1, idx, G, nullptr, nullptr,
                                  nullptr));
    }
    return PT_OK;
}

extern "C" pt_status pt_eval_holdout(pt_ctx *ctx, int32_t heldout_device, int32_t k, int32_t method,
                                     int32_t *out_idx, double *out_G_train, double *out_G_unseen,
                                     double *out_G_known, int32_t *out_known_idx)
{
    PT_NVTX();
    if (!ctx || !out_idx || !out_G_train || !out_G_unseen || !out_G_known)
        return pt_fail(PT_EINVAL, "NULL argument");
    if (!ctx->have_device) return pt_fail(PT_EINVAL, "pt_load_perf was given no env_device");
    if (method != 0 && method != 1) return pt_fail(PT_EINVAL, "method must be 0 or 1");
    if (k < 1) return pt_fail(PT_EINVAL, "k < 1");
    std::vector<uint8_t> train(ctx->E), test(ctx->E);
    int64_t ntr = 0, nte = 0;
    for (int64_t e = 0; e < ctx->E; e++) {
        train[e] = ctx->env_device[e] != heldout_device;
        test[e] = !train[e];
        ntr += train[e];
        nte += test[e];
    }
    if (ntr == 0 || nte == 0)
        return pt_fail(PT_EEMPTY, "device %d leaves an empty train or test scope", heldout_device);
    PT_TRY(select_on(ctx, train.data(), k, method, out_idx, out_G_train));
    PT_TRY(pt_score_sets(ctx, out_idx, 1, k, test.data(), PT_OBJ_GEOMEAN, out_G_unseen));
    std::vector<int32_t> kidx(k);
    PT_TRY(select_on(ctx, test.data(), k, method, kidx.data(), out_G_known));
    if (out_known_idx)
        for (int u = 0; u < k; u++) out_known_idx[u] = kidx[u];
    return PT_OK;
}

// ---------------------------------------------------------------------------
// pt_eval_holdout_all: every fold at once (greedy method).  2*D greedy problems
// (train scope and held-out scope of each device d) run in lockstep in ONE
// cooperative launch on the full matrix, each with its own 0/1 env weights (no
// scope compaction, no per-fold host round trips); a second small kernel scores
// each train selection on its held-out envs.  Same definitions as
// pt_eval_holdout (reading c13); fp64, deterministic.
// ---------------------------------------------------------------------------
#include <cooperative_groups.h>
namespace cgh = cooperative_groups;

#define HB_BIGI 0x7fffffff
#ifndef XH_BPS
#define XH_BPS 4   // batched holdout: co-resident blocks per SM
#endif

__device__ __forceinline__ void hb_top2(double &s1, int &c1, double &s2, int &c2, double s, int c)
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

// blocks are dealt to problems round-robin; per step each block scores its share
// of the configs for its problem, the per-block top-2 goes through global memory
// and one grid barrier, every block merges its problem's records (fixed order)
__global__ void __launch_bounds__(256) k_greedy_multi(const double *__restrict__ l64, int64_t C,
                                                       int64_t E_pad, int k, int P,
                                                       const double *__restrict__ w,     // [P][E_pad]
                                                       double4 *__restrict__ blk,        // [2][nblk]
                                                       int32_t *__restrict__ out_idx,    // [P][k]
                                                       double *__restrict__ out_s)       // [P] final s
{
    extern __shared__ double smh[];
    double *cur = smh;                              // [E_pad] this block's problem
    uint32_t *taken = (uint32_t *)(cur + E_pad);
    __shared__ double ws1[8], ws2[8];
    __shared__ int wc1[8], wc2[8];
    __shared__ int cstar;
    cgh::grid_group grid = cgh::this_grid();
    const int p = blockIdx.x % P;
    const int bpp = (int)((gridDim.x - p + P - 1) / P);   // blocks of this problem
    const int bi = blockIdx.x / P;                        // index among them
    const double *wp = w + (int64_t)p * E_pad;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t nwords = (C + 31) / 32;
    for (int64_t e = threadIdx.x; e < E_pad; e += blockDim.x) cur[e] = INFINITY;
    for (int64_t q = threadIdx.x; q < nwords; q += blockDim.x) taken[q] = 0u;
    __syncthreads();
    const int64_t gw = (int64_t)bi * 8 + warp, nw = (int64_t)bpp * 8;
    double last_s = 0.0;
    for (int t = 0; t < k; t++) {
        double s1 = INFINITY, s2 = INFINITY;
        int c1 = HB_BIGI, c2 = HB_BIGI;
        for (int64_t c = gw; c < C; c += nw) {
            if (taken[c >> 5] >> (c & 31) & 1u) continue;
            const double *col = l64 + c * E_pad;
            // loads issued together (one L2 round trip per candidate); e ascending per lane
            double acc = 0.0;
            for (int64_t e0 = lane; e0 < E_pad; e0 += 32 * 16) {
                double v[16];
#pragma unroll
                for (int u = 0; u < 16; u++) v[u] = e0 + 32 * u < E_pad ? __ldg(col + e0 + 32 * u) : 0.0;
#pragma unroll
                for (int u = 0; u < 16; u++)
                    if (e0 + 32 * u < E_pad) acc += wp[e0 + 32 * u] * fmin(cur[e0 + 32 * u], v[u]);
            }
            for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            hb_top2(s1, c1, s2, c2, acc, (int)c);
        }
        if (lane == 0) {
            ws1[warp] = s1;
            ws2[warp] = s2;
            wc1[warp] = c1;
            wc2[warp] = c2;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int q = 1; q < 8; q++) {
                hb_top2(s1, c1, s2, c2, ws1[q], wc1[q]);
                hb_top2(s1, c1, s2, c2, ws2[q], wc2[q]);
            }
            blk[(t & 1) * gridDim.x + blockIdx.x] = make_double4(s1, s2, (double)c1, (double)c2);
        }
        grid.sync();
        if (warp == 0) {
            // this problem's block records, read in parallel by the lanes; the top-2 of a
            // strict (s, c) order does not depend on the merge order
            s1 = s2 = INFINITY;
            c1 = c2 = HB_BIGI;
            for (int b0 = p + P * lane; b0 < (int)gridDim.x; b0 += P * 32 * 2) {
                double4 r[2];
#pragma unroll
                for (int u = 0; u < 2; u++)
                    if (b0 + P * 32 * u < (int)gridDim.x) r[u] = blk[(t & 1) * gridDim.x + b0 + P * 32 * u];
#pragma unroll
                for (int u = 0; u < 2; u++)
                    if (b0 + P * 32 * u < (int)gridDim.x) {
                        hb_top2(s1, c1, s2, c2, r[u].x, (int)r[u].z);
                        hb_top2(s1, c1, s2, c2, r[u].y, (int)r[u].w);
                    }
            }
            for (int o = 16; o; o >>= 1) {
                const double a1 = __shfl_xor_sync(0xffffffffu, s1, o), a2 = __shfl_xor_sync(0xffffffffu, s2, o);
                const int b1 = __shfl_xor_sync(0xffffffffu, c1, o), b2 = __shfl_xor_sync(0xffffffffu, c2, o);
                hb_top2(s1, c1, s2, c2, a1, b1);
                hb_top2(s1, c1, s2, c2, a2, b2);
            }
            if (lane == 0) {
                cstar = c1;
                last_s = s1;
                if (bi == 0) out_idx[(int64_t)p * k + t] = c1;
            }
        }
        __syncthreads();
        const int cs = cstar;
        if (threadIdx.x == 0) taken[cs >> 5] |= 1u << (cs & 31);
        const double *col = l64 + (int64_t)cs * E_pad;
        for (int64_t e = threadIdx.x; e < E_pad; e += blockDim.x) cur[e] = fmin(cur[e], col[e]);
        __syncthreads();
    }
    if (threadIdx.x == 0 && bi == 0) out_s[p] = last_s;
}

// warp per fold: s of the fold's train selection on its held-out envs
__global__ void k_holdout_unseen(const double *__restrict__ l64, int64_t E_pad, int k, int D,
                                 const int32_t *__restrict__ idx, const double *__restrict__ w,
                                 double *__restrict__ out_s)
{
    const int f = ((int)(blockIdx.x * blockDim.x + threadIdx.x)) >> 5;
    const int lane = threadIdx.x & 31;
    if (f >= D) return;
    const int32_t *set = idx + (int64_t)(2 * f) * k;          // problem 2f = train of fold f
    const double *wt = w + (int64_t)(2 * f + 1) * E_pad;      // problem 2f+1 = test envs of fold f
    double acc = 0.0;
    for (int64_t e = lane; e < E_pad; e += 32) {
        double m = l64[(int64_t)set[0] * E_pad + e];
        for (int u = 1; u < k; u++) m = fmin(m, l64[(int64_t)set[u] * E_pad + e]);
        acc += wt[e] * m;
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out_s[f] = acc;
}

extern "C" pt_status pt_eval_holdout_all(pt_ctx *ctx, int32_t k, int32_t n_device_cap, int32_t *out_idx,
                                         double *out_G_train, double *out_G_unseen, double *out_G_known,
                                         int32_t *out_known_idx, int32_t *out_n_device)
{
    PT_NVTX();
    if (!ctx || !out_idx || !out_G_train || !out_G_unseen || !out_G_known)
        return pt_fail(PT_EINVAL, "NULL argument");
    if (!ctx->have_device) return pt_fail(PT_EINVAL, "pt_load_perf was given no env_device");
    const pt_view &v = ctx->full;
    const int64_t C = v.C, E_pad = v.E_pad;
    if (k < 1 || k > C) return pt_fail(PT_EINVAL, "k=%d outside [1, %lld]", k, (long long)C);
    int32_t D = 0;
    for (int32_t d : ctx->env_device) D = std::max(D, d + 1);
    if (out_n_device) *out_n_device = D;
    if (D > n_device_cap)
        return pt_fail(PT_EINVAL, "%d devices but output room for %d (n_device_cap)", D, n_device_cap);
    std::vector<int64_t> cnt(D, 0);
    for (int32_t d : ctx->env_device) cnt[d]++;
    for (int32_t d = 0; d < D; d++)
        if (cnt[d] == 0 || cnt[d] == ctx->E)
            return pt_fail(PT_EEMPTY, "device %d leaves an empty train or test scope", d);
    if (out_n_device) *out_n_device = D;
    PT_CK(cudaSetDevice(ctx->dev));
    cudaStream_t s = ctx->stream;
    const int P = 2 * D;
    std::vector<double> hw((size_t)P * E_pad, 0.0);
    for (int32_t d = 0; d < D; d++)
        for (int64_t e = 0; e < ctx->E; e++) {
            hw[(size_t)(2 * d) * E_pad + e] = ctx->env_device[e] != d;
            hw[(size_t)(2 * d + 1) * E_pad + e] = ctx->env_device[e] == d;
        }
    const int64_t nwords = (C + 31) / 32;
    const size_t smem = sizeof(double) * E_pad + sizeof(uint32_t) * nwords;
    if (smem > 48 * 1024)
        PT_CK(cudaFuncSetAttribute(k_greedy_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    PT_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_greedy_multi, 256, smem));
    // up to XH_BPS co-resident blocks per SM: more warps per problem, fewer candidates per warp
    // (each candidate costs one L2 round trip per step)
    const int nblk = std::max(P, ctx->num_sms * std::min(occ, XH_BPS));
    if (occ * ctx->num_sms < nblk) return pt_fail(PT_ECUDA, "batched greedy cannot be co-resident");
    double *w = nullptr, *d_s = nullptr, *d_u = nullptr;
    double4 *blk = nullptr;
    int32_t *d_idx = nullptr;
    PT_TRY(pt_dalloc(ctx, (void **)&w, sizeof(double) * hw.size()));
    PT_TRY(pt_dalloc(ctx, (void **)&blk, sizeof(double4) * 2 * nblk));
    PT_TRY(pt_dalloc(ctx, (void **)&d_idx, sizeof(int32_t) * P * k));
    PT_TRY(pt_dalloc(ctx, (void **)&d_s, sizeof(double) * P));
    PT_TRY(pt_dalloc(ctx, (void **)&d_u, sizeof(double) * D));
    pt_hostio io(ctx);
    PT_TRY(io.h2d(w, hw.data(), sizeof(double) * hw.size()));
    const double *l64 = v.l64;
    int kk = k, PP = P;
    void *args[] = {(void *)&l64, (void *)&C, (void *)&E_pad, (void *)&kk, (void *)&PP, (void *)&w,
                    (void *)&blk, (void *)&d_idx, (void *)&d_s};
    PT_CK(cudaLaunchCooperativeKernel((void *)k_greedy_multi, dim3(nblk), dim3(256), args, smem, s));
    k_holdout_unseen<<<(unsigned)((D * 32 + 127) / 128), 128, 0, s>>>(v.l64, E_pad, k, D, d_idx, w, d_u);
    ctx->stats.launches += 2;
    PT_CK(cudaGetLastError());
    std::vector<int32_t> hidx((size_t)P * k);
    std::vector<double> hs(P), hu(D);
    PT_TRY(io.d2h(hidx.data(), d_idx, sizeof(int32_t) * P * k));
    PT_TRY(io.d2h(hs.data(), d_s, sizeof(double) * P));
    PT_TRY(io.d2h(hu.data(), d_u, sizeof(double) * D));
    for (void *p : {(void *)w, (void *)blk, (void *)d_idx, (void *)d_s, (void *)d_u}) pt_dfree(ctx, p);
    PT_TRY(io.finish());
    for (int32_t d = 0; d < D; d++) {
        const double etr = (double)(ctx->E - cnt[d]), ete = (double)cnt[d];
        for (int u = 0; u < k; u++) {
            out_idx[(size_t)d * k + u] = hidx[(size_t)(2 * d) * k + u];
            if (out_known_idx) out_known_idx[(size_t)d * k + u] = hidx[(size_t)(2 * d + 1) * k + u];
        }
        out_G_train[d] = std::exp(-hs[2 * d] / etr);
        out_G_known[d] = std::exp(-hs[2 * d + 1] / ete);
        out_G_unseen[d] = std::exp(-hu[d] / ete);
    }
    return PT_OK;
}
