// load.cu -- pt_load_perf (ingest + normalise), scopes, context lifetime.
//
// The post-processing pass of the paper (Sec. 5.3: performance
// "relative to the best ... kernels for that device and input") and the
// Oracle best[e] run here once per matrix:
//   k_rowstats : best[e] = min_c T[e][c] over measured cells, the row's max
//                slowdown (for the missing-cell penalty, reading c4), data checks
//   k_ell      : l[c][e] = log(T'/best[e]) in fp64 (T' = T, or penalty*best
//                for a missing cell), written config-major fp64 + fp32 and
//                env-major fp32 (smem-tiled transpose, coalesced both ways)
// HBM-bound elementwise work: one read of T, 16 B written per cell.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <cmath>
#include <set>
#include <vector>

#include <cuda_fp16.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <climits>
#include "pt_internal.cuh"

static thread_local std::string g_err;

pt_status pt_fail(pt_status st, const char *fmt, ...)
{
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

extern "C" const char *pt_last_error(void) { return g_err.c_str(); }

bool pt_is_device_ptr(const void *p)
{
    PT_NVTX();
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Device memory comes from the device's default stream-ordered pool with the
// release threshold lifted, so repeated loads / scopes / scratch reuse memory
// without cudaMalloc/cudaFree (and their implicit device synchronisation).
static void keep_pool(int dev)
{
    static std::mutex mu;
    static std::vector<int> done;
    std::lock_guard<std::mutex> g(mu);
    if (std::find(done.begin(), done.end(), dev) != done.end()) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    done.push_back(dev);
}

pt_status pt_dalloc(pt_ctx *ctx, void **p, size_t bytes)
{
    *p = nullptr;
    if (cudaMallocAsync(p, std::max<size_t>(bytes, 16), ctx->stream) != cudaSuccess) {
        cudaGetLastError();
        *p = nullptr;
        return pt_fail(PT_ENOMEM, "device allocation of %zu bytes failed", bytes);
    }
    return PT_OK;
}

void pt_dfree(pt_ctx *ctx, void *p)
{
    if (p) cudaFreeAsync(p, ctx->stream);
}

static constexpr size_t kPinnedBytes = 1 << 20;
static char *pinned_buffer()
{
    static thread_local char *buf = nullptr;   // lives for the thread (never freed)
    if (!buf && cudaMallocHost((void **)&buf, kPinnedBytes) != cudaSuccess) {
        cudaGetLastError();
        buf = nullptr;
    }
    return buf;
}

pt_status pt_hostio::h2d(void *dev_dst, const void *host_src, size_t n)
{
    char *pin = pinned_buffer();
    const size_t a = pt_round_up(off, 16);
    if (pin && a + n <= kPinnedBytes) {
        memcpy(pin + a, host_src, n);
        off = a + n;
        PT_CK(cudaMemcpyAsync(dev_dst, pin + a, n, cudaMemcpyHostToDevice, ctx->stream));
    } else {
        PT_CK(cudaMemcpyAsync(dev_dst, host_src, n, cudaMemcpyHostToDevice, ctx->stream));
    }
    return PT_OK;
}

pt_status pt_hostio::d2h(void *host_dst, const void *dev_src, size_t n)
{
    char *pin = pinned_buffer();
    const size_t a = pt_round_up(off, 16);
    if (pin && a + n <= kPinnedBytes) {
        off = a + n;
        PT_CK(cudaMemcpyAsync(pin + a, dev_src, n, cudaMemcpyDeviceToHost, ctx->stream));
        items.push_back({host_dst, a, n});
    } else {
        PT_CK(cudaMemcpyAsync(host_dst, dev_src, n, cudaMemcpyDeviceToHost, ctx->stream));
    }
    return PT_OK;
}

pt_status pt_hostio::finish()
{
    PT_CK(cudaStreamSynchronize(ctx->stream));
    char *pin = pinned_buffer();
    for (const item &it : items) memcpy(it.dst, pin + it.off, it.n);
    items.clear();
    off = 0;
    return PT_OK;
}

pt_status pt_scratch(pt_ctx *ctx, size_t bytes, void **p)
{
    if (bytes > ctx->scratch_bytes) {
        pt_dfree(ctx, ctx->scratch);
        ctx->scratch = nullptr;
        ctx->scratch_bytes = 0;
        size_t nb = std::max(bytes, (size_t)1 << 20);
        PT_TRY(pt_dalloc(ctx, &ctx->scratch, nb));
        ctx->scratch_bytes = nb;
    }
    *p = ctx->scratch;
    return PT_OK;
}

void pt_view_free(pt_ctx *ctx, pt_view &v)
{
    if (v.owned) {
        pt_dfree(ctx, v.l32);
        pt_dfree(ctx, v.l64);
        pt_dfree(ctx, v.hT);
        pt_dfree(ctx, v.hTile);
        pt_dfree(ctx, v.qC);
        pt_dfree(ctx, v.qTile);
        pt_dfree(ctx, v.qSum);
        pt_dfree(ctx, v.qConst);
        pt_dfree(ctx, v.hC);
        pt_dfree(ctx, v.hPair);
    }
    // allocated per view object (owned or not)
    pt_dfree(ctx, v.d_seed_s2);
    pt_dfree(ctx, v.d_seed_idx);
    pt_dfree(ctx, v.tcA);
    pt_dfree(ctx, v.tcB);
    pt_dfree(ctx, v.tcConst);
    v = pt_view();
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------

// one block per environment row: best (min over finite cells), max slowdown,
// status bits (1 = a finite runtime <= 0, 2 = no measured cell)
__global__ void k_rowstats(const float *__restrict__ T, int64_t C, double *__restrict__ best,
                           double *__restrict__ rowmax, int *__restrict__ status)
{
    const int64_t e = blockIdx.x;
    const float *row = T + e * C;
    __shared__ float red[32];
    __shared__ int bad;
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    float mn = INFINITY;
    int nonpos = 0;
    for (int64_t c = threadIdx.x; c < C; c += blockDim.x) {
        float t = row[c];
        if (isfinite(t)) {
            if (t <= 0.0f) nonpos = 1;
            mn = fminf(mn, t);
        }
    }
    if (nonpos) atomicOr(&bad, 1);
    for (int o = 16; o; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mn;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : INFINITY;
        for (int o = 16; o; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    const double b = (double)red[0];
    __syncthreads();
    double mx = 1.0;
    for (int64_t c = threadIdx.x; c < C; c += blockDim.x) {
        float t = row[c];
        if (isfinite(t) && t > 0.0f) mx = fmax(mx, (double)t / b);
    }
    __shared__ double redd[32];
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) redd[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double v = 1.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) v = fmax(v, redd[w]);
        rowmax[e] = v;
        best[e] = b;
        status[e] = bad | (isfinite(red[0]) ? 0 : 2);
    }
}

// 32x32 tiles: read T[e][c] coalesced along c, write l64/l32[c][e] through a
// shared transpose (coalesced along e).
// dataset penalty (the largest measured slowdown, >= 1) and the first
// environment whose status is bad (bit 1: a runtime <= 0, bit 2: no measured cell),
// computed on the device so the load needs one host round trip, at its end
__global__ void k_penalty(const double *__restrict__ rowmax, const int *__restrict__ status, int64_t E,
                          double *__restrict__ pen, long long *__restrict__ bad)
{
    __shared__ double smax[256];
    __shared__ long long sbad;
    if (threadIdx.x == 0) sbad = LLONG_MAX;
    __syncthreads();
    double m = 1.0;
    for (int64_t e = threadIdx.x; e < E; e += blockDim.x) {
        m = fmax(m, rowmax[e]);
        if (status[e]) atomicMin(&sbad, (long long)e);
    }
    smax[threadIdx.x] = m;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *pen = smax[0];
        bad[0] = sbad;
        bad[1] = sbad == LLONG_MAX ? 0 : status[sbad];
    }
}

__global__ void k_ell(const float *__restrict__ T, int64_t E, int64_t C,
                      const double *__restrict__ best, const double *__restrict__ pen, int64_t E_pad,
                      float *__restrict__ l32, double *__restrict__ l64)
{
    __shared__ double tile[32][33];
    const double penalty = *pen;
    const int64_t c0 = (int64_t)blockIdx.x * 32, e0 = (int64_t)blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
    for (int r = ty; r < 32; r += 8) {
        int64_t e = e0 + r, c = c0 + tx;
        double v = 0.0;
        if (e < E && c < C) {
            float t = T[e * C + c];
            double b = best[e];
            double tt = isfinite(t) ? (double)t : penalty * b;
            v = log(tt / b);
        }
        tile[r][tx] = v;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        int64_t c = c0 + r, e = e0 + tx;
        if (c < C && e < E_pad) {
            double v = tile[tx][r];
            l64[c * E_pad + e] = v;
            l32[c * E_pad + e] = (float)v;
        }
    }
}

// gather the environments of a scope (list idx[E_s]) out of the full view
__global__ void k_gather_cfg_major(const float *__restrict__ s32, const double *__restrict__ s64,
                                   int64_t E_pad_src, const int32_t *__restrict__ idx,
                                   int64_t E_s, int64_t E_pad_dst, int64_t C,
                                   float *__restrict__ d32, double *__restrict__ d64)
{
    const int64_t c = blockIdx.x;
    for (int64_t q = threadIdx.x; q < E_pad_dst; q += blockDim.x) {
        float v32 = 0.0f;
        double v64 = 0.0;
        if (q < E_s) {
            int64_t e = idx[q];
            v32 = s32[c * E_pad_src + e];
            v64 = s64[c * E_pad_src + e];
        }
        d32[c * E_pad_dst + q] = v32;
        d64[c * E_pad_dst + q] = v64;
    }
}

// hT[e][c] = fp16(l64[c][e]) (round to nearest), 32x32 smem transpose
__global__ void k_half(const double *__restrict__ l64, int64_t E, int64_t C, int64_t E_pad,
                       int64_t C_pad, uint16_t *__restrict__ hT)
{
    __shared__ uint16_t tile[32][34];
    const int64_t c0 = (int64_t)blockIdx.x * 32, e0 = (int64_t)blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
    for (int r = ty; r < 32; r += 8) {
        int64_t c = c0 + r, e = e0 + tx;
        uint16_t h = 0;
        if (c < C && e < E) h = __half_as_ushort(__double2half(l64[c * E_pad + e]));
        tile[r][tx] = h;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        int64_t e = e0 + r, c = c0 + tx;
        if (e < E_pad && c < C_pad) hT[e * C_pad + c] = tile[tx][r];
    }
}

// ---------------------------------------------------------------------------
static pt_status alloc_view(pt_ctx *ctx, pt_view &v, int64_t E, int64_t C)
{
    v.E = E;
    v.C = C;
    v.E_pad = pt_round_up(std::max<int64_t>(E, 1), 64);   // a whole number of 64-env stages
    v.C_pad = pt_round_up(C + 64, 64);   // >= C + 64: a 64-column bulk row copy never leaves the row
    v.owned = true;
    if (pt_dalloc(ctx, (void **)&v.l32, sizeof(float) * v.C * v.E_pad) != PT_OK ||
        pt_dalloc(ctx, (void **)&v.l64, sizeof(double) * v.C * v.E_pad) != PT_OK) {
        pt_view_free(ctx, v);
        return pt_fail(PT_ENOMEM, "device allocation for a %lld x %lld view failed",
                       (long long)E, (long long)C);
    }
    return PT_OK;
}

pt_status pt_smem_optin(pt_ctx *ctx, const void *kfn)
{
    static std::mutex mu;
    static std::set<std::pair<int, const void *>> done;
    std::lock_guard<std::mutex> g(mu);
    if (done.count(std::make_pair(ctx->dev, kfn))) return PT_OK;
    int optin = 0;
    PT_CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->dev));
    cudaFuncAttributes fa;
    PT_CK(cudaFuncGetAttributes(&fa, kfn));
    // static + dynamic shared memory of a block must fit the opt-in maximum
    PT_CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes));
    done.insert(std::make_pair(ctx->dev, kfn));
    return PT_OK;
}

// fp16 tier of a view (env-major copy of l64 rounded to nearest fp16), built on
// the first exhaustive search that needs it
pt_status pt_view_fp16(pt_ctx *ctx, const pt_view *cv)
{
    pt_view &v = *const_cast<pt_view *>(cv);
    if (v.hT) return PT_OK;
    PT_TRY(pt_dalloc(ctx, (void **)&v.hT, sizeof(uint16_t) * v.E_pad * v.C_pad));
    PT_CK(cudaMemsetAsync(v.hT, 0, sizeof(uint16_t) * v.E_pad * v.C_pad, ctx->stream));
    dim3 grid((unsigned)((v.C + 31) / 32), (unsigned)((v.E_pad + 31) / 32));
    k_half<<<grid, dim3(32, 8), 0, ctx->stream>>>(v.l64, v.E, v.C, v.E_pad, v.C_pad, v.hT);
    ctx->stats.launches += 1;
    PT_CK(cudaGetLastError());
    return PT_OK;
}

pt_status pt_get_view(pt_ctx *ctx, const uint8_t *env_mask, const pt_view **out)
{
    if (!env_mask) {
        *out = &ctx->full;
        return PT_OK;
    }
    bool all = true;
    for (int64_t e = 0; e < ctx->E; e++) all = all && env_mask[e];
    if (all) {
        *out = &ctx->full;
        return PT_OK;
    }
    ctx->tick++;
    for (auto &sc : ctx->scopes)
        if (sc.mask.size() == (size_t)ctx->E && memcmp(sc.mask.data(), env_mask, (size_t)ctx->E) == 0) {
            sc.last_use = ctx->tick;
            *out = &sc.view;
            return PT_OK;
        }
    std::vector<int32_t> idx;
    for (int64_t e = 0; e < ctx->E; e++)
        if (env_mask[e]) idx.push_back((int32_t)e);
    if (idx.empty()) return pt_fail(PT_EEMPTY, "env_mask selects no environment");
    // reuse the least recently used slot once the cache is full
    const size_t kMaxScopes = 8;
    pt_scope *slot = nullptr;
    if (ctx->scopes.size() < kMaxScopes) {
        ctx->scopes.emplace_back();
        slot = &ctx->scopes.back();
    } else {
        slot = &ctx->scopes[0];
        for (auto &sc : ctx->scopes)
            if (sc.last_use < slot->last_use) slot = &sc;
        pt_view_free(ctx, slot->view);
        slot->mask.clear();
    }
    pt_view &s = slot->view;
    PT_TRY(alloc_view(ctx, s, (int64_t)idx.size(), ctx->C));
    int32_t *d_idx = nullptr;
    PT_TRY(pt_dalloc(ctx, (void **)&d_idx, sizeof(int32_t) * idx.size()));
    PT_CK(cudaMemcpyAsync(d_idx, idx.data(), sizeof(int32_t) * idx.size(),
                          cudaMemcpyHostToDevice, ctx->stream));
    k_gather_cfg_major<<<(unsigned)s.C, 128, 0, ctx->stream>>>(
        ctx->full.l32, ctx->full.l64, ctx->full.E_pad, d_idx, s.E, s.E_pad, s.C, s.l32, s.l64);
    ctx->stats.launches += 1;
    PT_CK(cudaGetLastError());
    pt_dfree(ctx, d_idx);
    slot->mask.assign(env_mask, env_mask + ctx->E);
    slot->last_use = ctx->tick;
    *out = &s;
    return PT_OK;
}

extern "C" pt_status pt_load_perf(pt_ctx **out, const float *times_ms, int64_t n_env,
                                  int64_t n_cfg, int64_t ld, const int32_t *env_device,
                                  uint32_t flags, int cuda_device, void *cuda_stream)
{
    PT_NVTX();
    static const bool trace = getenv("PT_TRACE") != nullptr;
    const auto t_entry = std::chrono::steady_clock::now();
    auto mark = [&](const char *what) {
        if (trace)
            fprintf(stderr, "[pt load] %-12s %8.1f us\n", what,
                    std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_entry).count());
    };
    if (!out) return pt_fail(PT_EINVAL, "out is NULL");
    *out = nullptr;
    if (!times_ms || n_env < 1 || n_cfg < 1 || ld < n_cfg)
        return pt_fail(PT_EINVAL, "bad matrix arguments (n_env=%lld n_cfg=%lld ld=%lld)",
                       (long long)n_env, (long long)n_cfg, (long long)ld);
    if (n_cfg >= (1 << 21))
        return pt_fail(PT_EINVAL, "n_cfg must be < 2^21 (subset keys pack 21-bit indices)");
    if (env_device)
        for (int64_t e = 0; e < n_env; e++)
            if (env_device[e] < 0)
                return pt_fail(PT_EINVAL, "env_device[%lld] = %d is negative", (long long)e, env_device[e]);
    PT_CK(cudaSetDevice(cuda_device));
    pt_ctx *ctx = new pt_ctx();
    ctx->dev = cuda_device;
    ctx->stream = (cudaStream_t)cuda_stream;
    ctx->flags = flags;
    ctx->E = n_env;
    ctx->C = n_cfg;
    if (env_device) {
        ctx->env_device.assign(env_device, env_device + n_env);
        ctx->have_device = true;
    } else {
        ctx->env_device.assign((size_t)n_env, 0);
    }
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, cuda_device);
    auto bail = [&](pt_status st) {
        pt_free(ctx);
        return st;
    };
    if (cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess)
        return bail(pt_fail(PT_ECUDA, "cudaEventCreate failed"));

    mark("ctx");
    const int64_t E = n_env, C = n_cfg;
    keep_pool(cuda_device);
    float *dT = nullptr;
    double *rowmax = nullptr;
    int *status = nullptr;
    if (pt_dalloc(ctx, (void **)&dT, sizeof(float) * E * C) != PT_OK ||
        pt_dalloc(ctx, (void **)&ctx->best, sizeof(double) * E) != PT_OK ||
        pt_dalloc(ctx, (void **)&rowmax, sizeof(double) * E) != PT_OK ||
        pt_dalloc(ctx, (void **)&status, sizeof(int) * E) != PT_OK) {
        pt_dfree(ctx, dT);
        pt_dfree(ctx, rowmax);
        pt_dfree(ctx, status);
        return bail(pt_fail(PT_ENOMEM, "device allocation for %lld x %lld failed",
                            (long long)E, (long long)C));
    }
    auto cleanup = [&]() {
        pt_dfree(ctx, dT);
        pt_dfree(ctx, rowmax);
        pt_dfree(ctx, status);
    };
    const cudaMemcpyKind kind =
        pt_is_device_ptr(times_ms) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (cudaMemcpy2DAsync(dT, sizeof(float) * C, times_ms, sizeof(float) * ld,
                          sizeof(float) * C, E, kind, ctx->stream) != cudaSuccess) {
        cleanup();
        return bail(pt_fail(PT_ECUDA, "copy of the runtime matrix failed: %s",
                            cudaGetErrorString(cudaGetLastError())));
    }
    mark("copied");
    k_rowstats<<<(unsigned)E, 256, 0, ctx->stream>>>(dT, C, ctx->best, rowmax, status);
    double *d_pen = nullptr;
    long long *d_bad = nullptr;
    if (pt_dalloc(ctx, (void **)&d_pen, 256 + 2 * sizeof(long long)) != PT_OK) {
        cleanup();
        return bail(pt_fail(PT_ENOMEM, "device allocation failed"));
    }
    d_bad = (long long *)((char *)d_pen + 256);
    k_penalty<<<1, 256, 0, ctx->stream>>>(rowmax, status, E, d_pen, d_bad);
    ctx->stats.launches += 2;
    pt_status st = alloc_view(ctx, ctx->full, E, C);
    if (st != PT_OK) {
        cleanup();
        pt_dfree(ctx, d_pen);
        return bail(st);
    }
    pt_view &v = ctx->full;
    dim3 grid((unsigned)((C + 31) / 32), (unsigned)((v.E_pad + 31) / 32));
    k_ell<<<grid, dim3(32, 8), 0, ctx->stream>>>(dT, E, C, ctx->best, d_pen, v.E_pad, v.l32, v.l64);
    ctx->stats.launches++;
    // keep the runtimes (env-major fp32) for objectives on raw times (Eq. 2)
    ctx->T32 = dT;
    pt_dfree(ctx, rowmax);
    pt_dfree(ctx, status);
    mark("launched");
    double pen = 1.0;
    long long bad[2] = {0, 0};
    pt_hostio io(ctx);
    if (io.d2h(&pen, d_pen, sizeof(double)) != PT_OK || io.d2h(bad, d_bad, sizeof bad) != PT_OK ||
        io.finish() != PT_OK || cudaGetLastError() != cudaSuccess)
        return bail(pt_fail(PT_ECUDA, "load: %s", cudaGetErrorString(cudaGetLastError())));
    mark("synced");
    pt_dfree(ctx, d_pen);
    if (bad[1] & 1) return bail(pt_fail(PT_EDATA, "environment %lld has a runtime <= 0", bad[0]));
    if (bad[1] & 2) return bail(pt_fail(PT_EDATA, "environment %lld has no measured cell", bad[0]));
    ctx->penalty = pen;
    *out = ctx;
    return PT_OK;
}

extern "C" pt_status pt_get_stats(const pt_ctx *ctx, pt_stats *out)
{
    PT_NVTX();
    if (!ctx || !out) return pt_fail(PT_EINVAL, "NULL argument");
    *out = ctx->stats;
    return PT_OK;
}

extern "C" void pt_free(pt_ctx *ctx)
{
    PT_NVTX();
    if (!ctx) return;
    cudaSetDevice(ctx->dev);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    pt_view_free(ctx, ctx->full);
    for (auto &sc : ctx->scopes) pt_view_free(ctx, sc.view);
    pt_dfree(ctx, ctx->best);
    pt_dfree(ctx, ctx->scratch);
    pt_dfree(ctx, ctx->T32);
    pt_dfree(ctx, ctx->fl.tcm);
    pt_dfree(ctx, ctx->fl.tem);
    pt_dfree(ctx, ctx->fl.w);
    pt_dfree(ctx, ctx->fl.qdev);
    pt_dfree(ctx, ctx->fl.seg);
    pt_fleet_tiled_free(ctx);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    delete ctx;
}
