// kmeans.cu -- the paper's k-means selector (Sec. 4.3.2; SURVEY
// §8(f) NEXT #4).  Environments are points of their slowdowns T/best over the
// configurations (reading k1); k = |kappa| centroids; per centroid the config
// with the smallest centroid slowdown is selected, duplicates
// collapse.  Deterministic maximin init and Lloyd iterations (reading k2).
//
// Every sum runs in the same order as the oracle's and products/sums use
// explicit round-to-nearest intrinsics (no FMA contraction), so the whole
// trajectory -- init, every assignment, every centroid -- is bit-identical to
// the CPU oracle's.  The whole loop runs on the device: points are stored in
// 32-point tiles Xt[tile][c][32] (one tile's configurations are contiguous), a
// distance pass is one CTA per tile (warp = centroid, lane = point) fed by bulk
// copies (TMA engine) of 128-config chunks, so the 2 GiB scaled matrix streams
// once per pass; the assignment, the convergence test, the centroid update and
// the empty-cluster re-seed are kernels too, and the host only reads a stop flag
// every few passes (no round trip per pass).
#include <algorithm>
#include <cmath>
#include <mutex>
#include <vector>

#include "pt_internal.cuh"

#define KM_MAXK 32
#define KM_CB 64    // configs per staged chunk: the tile's 64 x 32 points + the centroids' 64-config rows
#define KM_NS 3     // chunk ring depth

namespace {
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t n)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity)
{
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok)
                     : "r"(su32(b)), "r"(parity), "r"(1000000u)
                     : "memory");
}
// control block of the device-side Lloyd loop
struct KmCtl {
    int it;         // assignment passes done
    int stop;       // 1: converged or max_iter reached -- every later kernel returns at once
    int changed;    // some assignment changed in the current pass
    int max_iter;
};
}  // namespace

// Xt[t][c][p] = T/best of point q = 32 t + p (missing -> penalty), 0 for padding points
__global__ void k_km_build(const float *__restrict__ T, int64_t C, const double *__restrict__ best,
                           double penalty, const int32_t *__restrict__ envs, int64_t ne,
                           double *__restrict__ Xt)
{
    const int64_t c = blockIdx.x, t = blockIdx.y;
    const int p = threadIdx.x;   // 32 threads
    const int64_t q = 32 * t + p;
    double v = 0.0;
    if (q < ne) {
        const int64_t e = envs[q];
        const float x = T[e * C + c];
        const double tt = isfinite(x) ? (double)x : penalty * best[e];
        v = tt / best[e];
    }
    Xt[(t * C + c) * 32 + p] = v;
}

// mean over points (q ascending), thread per config
__global__ void k_km_mean(const double *__restrict__ Xt, int64_t ne, int64_t C, double *__restrict__ mean)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    double s = 0.0;
    for (int64_t q = 0; q < ne; q++) s = __dadd_rn(s, Xt[((q >> 5) * C + c) * 32 + (q & 31)]);
    mean[c] = s / (double)ne;
}

// D[q][j] = sum_c (x_q[c] - Mt[c][j])^2, c ascending, j < nc: one CTA per 32-point tile,
// lane = point, warp w = centroids 4w .. 4w+3 (x is read once per c for four chains);
// each chunk of KM_CB configs -- the tile's 32 points and the centroids' values, stored
// config-major Mt[c][nc] so a chunk is contiguous -- arrives by bulk copies (TMA engine)
// in a KM_NS-deep ring, so no load latency sits in the sequential sums.  `ctl` (may be
// NULL): skip the pass when the loop has stopped.
#define KM_JW 4   // centroids per warp (JW = 1 for the single-centroid passes of the init)
template <int JW>
__global__ void __launch_bounds__(32 * KM_MAXK / KM_JW) k_km_dist(const double *__restrict__ Xt, int64_t ne,
                                                                  int64_t C, const double *__restrict__ Mt, int nc,
                                                                  double *__restrict__ D,
                                                                  const KmCtl *__restrict__ ctl)
{
    if (ctl && ctl->stop) return;
    extern __shared__ __align__(128) unsigned char smem[];
    double *Xs = reinterpret_cast<double *>(smem);                        // [NS][CB][32]
    double *Ms = Xs + KM_NS * KM_CB * 32;                                  // [NS][CB][nc]
    uint64_t *full = reinterpret_cast<uint64_t *>(Ms + KM_NS * KM_CB * nc);
    const int64_t t = blockIdx.x;
    const int lane = threadIdx.x & 31, j0 = JW * (threadIdx.x >> 5);
    const int nch = (int)((C + KM_CB - 1) / KM_CB);
    const double *src = Xt + t * C * 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < KM_NS; s++) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int ch) {
        const int64_t c0 = (int64_t)ch * KM_CB;
        const int64_t n = min((int64_t)KM_CB, C - c0);
        const int sl = ch % KM_NS;
        // (bulk copies move multiples of 16 bytes: an odd n * nc reads one padding double,
        // which the centroid buffers carry and the sums never use)
        const uint32_t xb = (uint32_t)(n * 32 * sizeof(double)), mb = (uint32_t)((n * nc * sizeof(double) + 15) & ~15);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[sl])), "r"(xb + mb)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(Xs + sl * KM_CB * 32)),
                     "l"(src + c0 * 32), "r"(xb), "r"(su32(&full[sl]))
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(Ms + sl * KM_CB * nc)),
                     "l"(Mt + c0 * nc), "r"(mb), "r"(su32(&full[sl]))
                     : "memory");
    };
    if (threadIdx.x == 0)
        for (int ch = 0; ch < KM_NS && ch < nch; ch++) issue(ch);
    double acc[JW];
#pragma unroll
    for (int u = 0; u < JW; u++) acc[u] = 0.0;
    const int nj = min(JW, nc - j0);
    for (int ch = 0; ch < nch; ch++) {
        mbar_wait(&full[ch % KM_NS], (uint32_t)(ch / KM_NS) & 1u);
        const int64_t c0 = (int64_t)ch * KM_CB;
        const int n = (int)min((int64_t)KM_CB, C - c0);
        const double *xs = Xs + (ch % KM_NS) * KM_CB * 32;
        const double *ms = Ms + (ch % KM_NS) * KM_CB * nc + j0;
        int cc = 0;
        for (; cc + 8 <= n; cc += 8) {   // operands of 8 configs in registers, then the sums in c order
            double x[8], y[8][JW];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                x[u] = xs[(cc + u) * 32 + lane];
#pragma unroll
                for (int v = 0; v < JW; v++) y[u][v] = v < nj ? ms[(cc + u) * nc + v] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; u++)
#pragma unroll
                for (int v = 0; v < JW; v++) {
                    const double d = __dsub_rn(x[u], y[u][v]);
                    acc[v] = __dadd_rn(acc[v], __dmul_rn(d, d));
                }
        }
        for (; cc < n; cc++) {
            const double x = xs[cc * 32 + lane];
#pragma unroll
            for (int v = 0; v < JW; v++) {
                const double d = __dsub_rn(x, v < nj ? ms[cc * nc + v] : 0.0);
                acc[v] = __dadd_rn(acc[v], __dmul_rn(d, d));
            }
        }
        __syncthreads();   // every warp is done with this chunk: refill it
        if (threadIdx.x == 0 && ch + KM_NS < nch) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(ch + KM_NS);
        }
    }
    const int64_t q = 32 * t + lane;
    if (q < ne)
#pragma unroll
        for (int v = 0; v < JW; v++)
            if (v < nj) D[q * KM_MAXK + j0 + v] = acc[v];
}

// init helper: index of the smallest (pick_max = 0, ties -> lowest q) or the largest
// (pick_max = 1, first strictly larger than -1 -- the oracle's "farthest" loop) of
// v[q * stride] over q < ne; copies that point into centroid j of Mt (j >= 0) and cent1
__global__ void __launch_bounds__(1024) k_km_pick(const double *__restrict__ v, int64_t stride, int64_t ne,
                                                  int pick_max, const double *__restrict__ Xt, int64_t C, int j,
                                                  int k, double *__restrict__ Mt, double *__restrict__ cent1,
                                                  int64_t *__restrict__ out_q)
{
    __shared__ double bv[1024];
    __shared__ int64_t bq[1024];
    double b = pick_max ? -1.0 : INFINITY;
    int64_t bi = -1;
    for (int64_t q = threadIdx.x; q < ne; q += blockDim.x) {
        const double x = v[q * stride];
        if (pick_max ? x > b : x < b) {
            b = x;
            bi = q;
        }
    }
    bv[threadIdx.x] = b;
    bq[threadIdx.x] = bi;
    __syncthreads();
    for (int h = blockDim.x / 2; h > 0; h >>= 1) {
        if ((int)threadIdx.x < h) {
            const double o = bv[threadIdx.x + h];
            const int64_t oq = bq[threadIdx.x + h];
            const double me = bv[threadIdx.x];
            const int64_t mq = bq[threadIdx.x];
            const bool better = oq >= 0 && (mq < 0 || (pick_max ? o > me : o < me) || (o == me && oq < mq));
            if (better) {
                bv[threadIdx.x] = o;
                bq[threadIdx.x] = oq;
            }
        }
        __syncthreads();
    }
    const int64_t qs = bq[0] < 0 ? 0 : bq[0];
    if (threadIdx.x == 0 && out_q) *out_q = qs;
    if (j >= 0)
        for (int64_t c = threadIdx.x; c < C; c += blockDim.x) {
            const double x = Xt[((qs >> 5) * C + c) * 32 + (qs & 31)];
            Mt[c * k + j] = x;    // centroid j (config-major)
            cent1[c] = x;         // and alone, for the next single-centroid distance pass
        }
}

// small scopes (ne <= KM_PAIR_MAX): every point's distance to every point and to the mean
// (column ne) in one pass -- P[q][r] is exactly what k_km_dist returns for point q and a
// centroid that is a copy of point r (same c-ascending sum) -- so the maximin init needs
// no further distance pass
#define KM_PAIR_MAX 1024
__global__ void __launch_bounds__(128) k_km_pair(const double *__restrict__ Xt, int64_t ne, int64_t C,
                                                const double *__restrict__ mean, double *__restrict__ P)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ne * (ne + 1)) return;
    const int64_t q = i % ne, r = i / ne;
    const double *xq = Xt + (q >> 5) * C * 32 + (q & 31);
    const double *xr = r < ne ? Xt + (r >> 5) * C * 32 + (r & 31) : nullptr;
    double acc = 0.0;
    int64_t c = 0;
    for (; c + 8 <= C; c += 8) {   // 8 operand pairs in flight, then the sums in c order
        double x[8], y[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            x[u] = xq[(c + u) * 32];
            y[u] = xr ? xr[(c + u) * 32] : mean[c + u];
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const double d = __dsub_rn(x[u], y[u]);
            acc = __dadd_rn(acc, __dmul_rn(d, d));
        }
    }
    for (; c < C; c++) {
        const double d = __dsub_rn(xq[c * 32], xr ? xr[c * 32] : mean[c]);
        acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
    P[q * (ne + 1) + r] = acc;
}

// init helper (pairwise path): dmin[q] = P[q][*col] (first) or min(dmin[q], P[q][*col])
__global__ void k_km_dmin_col(const double *__restrict__ P, int64_t ne, const int64_t *__restrict__ col, int first,
                              double *__restrict__ dmin)
{
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= ne) return;
    const double d = P[q * (ne + 1) + *col];
    dmin[q] = first ? d : fmin(dmin[q], d);
}

// init helper: dmin[q] = D[q][0] (first) or min(dmin[q], D[q][0])
__global__ void k_km_dmin(const double *__restrict__ D, int64_t ne, int first, double *__restrict__ dmin)
{
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= ne) return;
    const double d = D[q * KM_MAXK];
    dmin[q] = first ? d : fmin(dmin[q], d);
}

// Lloyd assignment: nearest centroid (ties -> lowest j), dmin, counts, changed flag
__global__ void k_km_assign(const double *__restrict__ D, int64_t ne, int k, int32_t *__restrict__ asg,
                            double *__restrict__ dmin, int32_t *__restrict__ cnt, KmCtl *__restrict__ ctl)
{
    if (ctl->stop) return;
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= ne) return;
    int bj = 0;
    double bd = INFINITY;
    for (int j = 0; j < k; j++) {
        const double d = D[q * KM_MAXK + j];
        if (d < bd) {
            bd = d;
            bj = j;
        }
    }
    if (asg[q] != bj) ctl->changed = 1;   // benign race: every writer stores 1
    asg[q] = bj;
    dmin[q] = bd;
    atomicAdd(&cnt[bj], 1);
}

// after an assignment pass: count it; converged (no change, not the first pass) -> stop
__global__ void k_km_ctl_assigned(KmCtl *ctl)
{
    if (ctl->stop) return;
    ctl->it++;
    if (!ctl->changed && ctl->it > 1) ctl->stop = 1;
    ctl->changed = 0;
}

// centroid update: Mt[c][j] = (sum of the cluster's points, q ascending) / count,
// thread per config (empty clusters keep their row for the re-seed)
__global__ void k_km_update(const double *__restrict__ Xt, int64_t ne, int64_t C, const int32_t *__restrict__ asg,
                            int k, const int32_t *__restrict__ cnt, double *__restrict__ Mt,
                            const KmCtl *__restrict__ ctl)
{
    if (ctl->stop) return;
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    double acc[KM_MAXK];
#pragma unroll
    for (int j = 0; j < KM_MAXK; j++) acc[j] = 0.0;
    for (int64_t q = 0; q < ne; q++) {
        const int a = __ldg(asg + q);
        const double x = Xt[((q >> 5) * C + c) * 32 + (q & 31)];
#pragma unroll
        for (int j = 0; j < KM_MAXK; j++)
            if (j == a) acc[j] = __dadd_rn(acc[j], x);
    }
    for (int j = 0; j < k; j++)
        if (cnt[j] > 0) Mt[c * k + j] = acc[j] / (double)cnt[j];
}

// empty clusters, j ascending: re-seed with the point farthest from its own centroid
// (first strictly larger than -1), then dmin[far] = 0; one CTA.  Clears the
// counts for the next pass and stops the loop at max_iter.
__global__ void __launch_bounds__(1024) k_km_reseed(const double *__restrict__ Xt, int64_t ne, int64_t C, int k,
                                                    double *__restrict__ dmin, int32_t *__restrict__ cnt,
                                                    double *__restrict__ Mt, KmCtl *__restrict__ ctl)
{
    if (ctl->stop) return;
    __shared__ double bv[1024];
    __shared__ int64_t bq[1024];
    for (int j = 0; j < k; j++) {
        if (cnt[j] != 0) continue;   // uniform across the block
        double b = -1.0;
        int64_t bi = -1;
        for (int64_t q = threadIdx.x; q < ne; q += blockDim.x)
            if (dmin[q] > b) {
                b = dmin[q];
                bi = q;
            }
        bv[threadIdx.x] = b;
        bq[threadIdx.x] = bi;
        __syncthreads();
        for (int h = blockDim.x / 2; h > 0; h >>= 1) {
            if ((int)threadIdx.x < h) {
                const double o = bv[threadIdx.x + h], me = bv[threadIdx.x];
                const int64_t oq = bq[threadIdx.x + h], mq = bq[threadIdx.x];
                if (oq >= 0 && (mq < 0 || o > me || (o == me && oq < mq))) {
                    bv[threadIdx.x] = o;
                    bq[threadIdx.x] = oq;
                }
            }
            __syncthreads();
        }
        const int64_t far = bq[0] < 0 ? 0 : bq[0];
        for (int64_t c = threadIdx.x; c < C; c += blockDim.x)
            Mt[c * k + j] = Xt[((far >> 5) * C + c) * 32 + (far & 31)];
        __syncthreads();
        if (threadIdx.x == 0) dmin[far] = 0.0;
        __syncthreads();
    }
    __syncthreads();
    for (int j = threadIdx.x; j < k; j += blockDim.x) cnt[j] = 0;
    if (threadIdx.x == 0 && ctl->it >= ctl->max_iter) ctl->stop = 1;
}

// per centroid: the config with the smallest slowdown (ties -> lowest index)
__global__ void k_km_select(const double *__restrict__ Mt, int64_t C, int k, int32_t *__restrict__ sel)
{
    __shared__ double bv[256];
    __shared__ int bc[256];
    const int j = blockIdx.x;
    double v = INFINITY;
    int ci = 0x7fffffff;
    for (int64_t c = threadIdx.x; c < C; c += blockDim.x) {
        const double m = Mt[c * k + j];
        if (m < v) {
            v = m;
            ci = (int)c;
        }
    }
    bv[threadIdx.x] = v;
    bc[threadIdx.x] = ci;
    __syncthreads();
    for (int h = blockDim.x / 2; h > 0; h >>= 1) {
        if ((int)threadIdx.x < h) {
            const double o = bv[threadIdx.x + h];
            const int oc = bc[threadIdx.x + h];
            if (o < bv[threadIdx.x] || (o == bv[threadIdx.x] && oc < bc[threadIdx.x])) {
                bv[threadIdx.x] = o;
                bc[threadIdx.x] = oc;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) sel[j] = bc[0];
}

// init: NULL = the deterministic maximin start; else host [k][C] initial centroids
static pt_status kmeans_run(pt_ctx *ctx, int32_t k, const uint8_t *env_mask, int32_t max_iter, const double *init,
                            int32_t *out_idx, int32_t *out_n, double *out_G, int32_t *out_iters)
{
    if (!ctx || !out_idx || !out_n) return pt_fail(PT_EINVAL, "NULL argument");
    if (k < 1 || k > KM_MAXK) return pt_fail(PT_EINVAL, "k=%d outside [1, %d]", k, KM_MAXK);
    if (max_iter < 1) return pt_fail(PT_EINVAL, "max_iter must be >= 1");
    PT_CK(cudaSetDevice(ctx->dev));
    std::vector<int32_t> envs;
    for (int64_t e = 0; e < ctx->E; e++)
        if (!env_mask || env_mask[e]) envs.push_back((int32_t)e);
    const int64_t ne = (int64_t)envs.size(), C = ctx->C;
    if (ne == 0) return pt_fail(PT_EEMPTY, "env_mask selects no environment");
    if (k > ne) return pt_fail(PT_EINVAL, "k=%d exceeds the %lld points", k, (long long)ne);
    cudaStream_t s = ctx->stream;
    const int64_t nt = (ne + 31) / 32;
    int32_t *d_envs = nullptr, *d_asg = nullptr, *d_cnt = nullptr, *d_sel = nullptr;
    double *X = nullptr, *M = nullptr, *D = nullptr, *mean = nullptr, *dmin = nullptr, *cent1 = nullptr;
    KmCtl *ctl = nullptr;
    PT_TRY(pt_dalloc(ctx, (void **)&d_envs, sizeof(int32_t) * ne));
    PT_TRY(pt_dalloc(ctx, (void **)&X, sizeof(double) * nt * 32 * C));
    PT_TRY(pt_dalloc(ctx, (void **)&M, sizeof(double) * (k * C + 2)));    // +2: bulk-copy padding
    PT_TRY(pt_dalloc(ctx, (void **)&mean, sizeof(double) * (C + 2)));
    PT_TRY(pt_dalloc(ctx, (void **)&cent1, sizeof(double) * (C + 2)));
    PT_TRY(pt_dalloc(ctx, (void **)&D, sizeof(double) * ne * KM_MAXK));
    PT_TRY(pt_dalloc(ctx, (void **)&dmin, sizeof(double) * ne));
    PT_TRY(pt_dalloc(ctx, (void **)&d_asg, sizeof(int32_t) * ne));
    PT_TRY(pt_dalloc(ctx, (void **)&d_cnt, sizeof(int32_t) * k));
    PT_TRY(pt_dalloc(ctx, (void **)&d_sel, sizeof(int32_t) * k));
    PT_TRY(pt_dalloc(ctx, (void **)&ctl, sizeof(KmCtl)));
    PT_CK(cudaMemcpyAsync(d_envs, envs.data(), sizeof(int32_t) * ne, cudaMemcpyHostToDevice, s));
    PT_CK(cudaMemsetAsync(d_asg, 0xFF, sizeof(int32_t) * ne, s));   // -1: unassigned
    PT_CK(cudaMemsetAsync(d_cnt, 0, sizeof(int32_t) * k, s));
    const KmCtl h_ctl{0, 0, 0, max_iter};
    PT_CK(cudaMemcpyAsync(ctl, &h_ctl, sizeof h_ctl, cudaMemcpyHostToDevice, s));
    k_km_build<<<dim3((unsigned)C, (unsigned)nt), 32, 0, s>>>(ctx->T32, C, ctx->best, ctx->penalty, d_envs, ne, X);
    // M is config-major, Mt[c][k]: a chunk of all centroids is one contiguous block
    auto smem_of = [](int nc) { return sizeof(double) * KM_NS * KM_CB * (32 + nc) + sizeof(uint64_t) * KM_NS; };
    static std::mutex attr_mu;
    static uint64_t attr_done = 0;   // bit d: attributes set on device d
    std::lock_guard<std::mutex> attr_g(attr_mu);
    if (!(attr_done >> (ctx->dev & 63) & 1ull)) {
        PT_CK(cudaFuncSetAttribute(k_km_dist<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_of(1)));
        PT_CK(cudaFuncSetAttribute(k_km_dist<KM_JW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem_of(KM_MAXK)));
        attr_done |= 1ull << (ctx->dev & 63);
    }
    auto dist = [&](const double *cent, int nc, const KmCtl *c) {
        if (nc == 1)
            k_km_dist<1><<<(unsigned)nt, 32, smem_of(1), s>>>(X, ne, C, cent, 1, D, c);
        else
            k_km_dist<KM_JW><<<(unsigned)nt, 32 * ((nc + KM_JW - 1) / KM_JW), smem_of(nc), s>>>(X, ne, C, cent, nc, D, c);
    };
    const unsigned gc = (unsigned)((C + 127) / 128), gq = (unsigned)((ne + 255) / 256);
    // init: the point nearest the mean, then successive farthest points (maximin).  Every
    // init centroid is a copy of a point, so small scopes read one pairwise pass; larger
    // ones run one single-centroid distance pass per centroid.  A given start is copied
    // in (config-major).
    if (init) {
        std::vector<double> mt((size_t)k * C);
        for (int j = 0; j < k; j++)
            for (int64_t c = 0; c < C; c++) mt[(size_t)c * k + j] = init[(size_t)j * C + c];
        PT_CK(cudaMemcpyAsync(M, mt.data(), sizeof(double) * k * C, cudaMemcpyHostToDevice, s));
        PT_CK(cudaStreamSynchronize(s));   // mt is a host temporary
    } else {
    k_km_mean<<<gc, 128, 0, s>>>(X, ne, C, mean);
    ctx->stats.launches++;
    if (ne <= KM_PAIR_MAX) {
        double *P = nullptr;
        int64_t *pq = nullptr;
        PT_TRY(pt_dalloc(ctx, (void **)&P, sizeof(double) * ne * (ne + 1)));
        PT_TRY(pt_dalloc(ctx, (void **)&pq, sizeof(int64_t)));
        k_km_pair<<<(unsigned)((ne * (ne + 1) + 127) / 128), 128, 0, s>>>(X, ne, C, mean, P);
        k_km_pick<<<1, 1024, 0, s>>>(P + ne, ne + 1, ne, 0, X, C, 0, k, M, cent1, pq);
        k_km_dmin_col<<<gq, 256, 0, s>>>(P, ne, pq, 1, dmin);
        ctx->stats.launches += 3;
        for (int j = 1; j < k; j++) {
            k_km_pick<<<1, 1024, 0, s>>>(dmin, 1, ne, 1, X, C, j, k, M, cent1, pq);
            k_km_dmin_col<<<gq, 256, 0, s>>>(P, ne, pq, 0, dmin);
            ctx->stats.launches += 2;
        }
        pt_dfree(ctx, P);
        pt_dfree(ctx, pq);
    } else {
        dist(mean, 1, nullptr);
        k_km_pick<<<1, 1024, 0, s>>>(D, KM_MAXK, ne, 0, X, C, 0, k, M, cent1, nullptr);
        dist(cent1, 1, nullptr);
        k_km_dmin<<<gq, 256, 0, s>>>(D, ne, 1, dmin);
        ctx->stats.launches += 5;
        for (int j = 1; j < k; j++) {
            k_km_pick<<<1, 1024, 0, s>>>(dmin, 1, ne, 1, X, C, j, k, M, cent1, nullptr);
            dist(cent1, 1, nullptr);
            k_km_dmin<<<gq, 256, 0, s>>>(D, ne, 0, dmin);
            ctx->stats.launches += 3;
        }
    }
    }
    PT_CK(cudaGetLastError());
    // Lloyd, enqueued in batches of passes; a pass after the stop flag returns at once
    const int batch = 4;
    KmCtl h{};
    int enq = 0;
    while (enq < max_iter) {
        for (int b = 0; b < batch && enq < max_iter; b++, enq++) {
            dist(M, k, ctl);
            k_km_assign<<<gq, 256, 0, s>>>(D, ne, k, d_asg, dmin, d_cnt, ctl);
            k_km_ctl_assigned<<<1, 1, 0, s>>>(ctl);
            k_km_update<<<gc, 128, 0, s>>>(X, ne, C, d_asg, k, d_cnt, M, ctl);
            k_km_reseed<<<1, 1024, 0, s>>>(X, ne, C, k, dmin, d_cnt, M, ctl);
            ctx->stats.launches += 5;
        }
        PT_CK(cudaGetLastError());
        PT_CK(cudaMemcpyAsync(&h, ctl, sizeof h, cudaMemcpyDeviceToHost, s));
        PT_CK(cudaStreamSynchronize(s));
        if (h.stop) break;
    }
    k_km_select<<<k, 256, 0, s>>>(M, C, k, d_sel);
    ctx->stats.launches++;
    std::vector<int32_t> sel(k);
    PT_CK(cudaMemcpyAsync(sel.data(), d_sel, sizeof(int32_t) * k, cudaMemcpyDeviceToHost, s));
    PT_CK(cudaMemcpyAsync(&h, ctl, sizeof h, cudaMemcpyDeviceToHost, s));
    for (void *p : {(void *)d_envs, (void *)X, (void *)M, (void *)mean, (void *)cent1, (void *)D, (void *)dmin,
                    (void *)d_asg,
                    (void *)d_cnt, (void *)d_sel, (void *)ctl})
        pt_dfree(ctx, p);
    PT_CK(cudaStreamSynchronize(s));
    std::sort(sel.begin(), sel.end());
    sel.erase(std::unique(sel.begin(), sel.end()), sel.end());
    for (size_t u = 0; u < sel.size(); u++) out_idx[u] = sel[u];
    *out_n = (int32_t)sel.size();
    if (out_iters) *out_iters = h.it;
    if (out_G) PT_TRY(pt_score_sets(ctx, sel.data(), 1, (int32_t)sel.size(), env_mask, PT_OBJ_GEOMEAN, out_G));
    return PT_OK;
}

extern "C" pt_status pt_kmeans_select(pt_ctx *ctx, int32_t k, const uint8_t *env_mask, int32_t max_iter,
                                      int32_t *out_idx, int32_t *out_n, double *out_G, int32_t *out_iters)
{
    PT_NVTX();
    return kmeans_run(ctx, k, env_mask, max_iter, nullptr, out_idx, out_n, out_G, out_iters);
}

extern "C" pt_status pt_kmeans_select_from(pt_ctx *ctx, int32_t k, const uint8_t *env_mask, int32_t max_iter,
                                           const double *init, int32_t *out_idx, int32_t *out_n, double *out_G,
                                           int32_t *out_iters)
{
    PT_NVTX();
    if (!init) return pt_fail(PT_EINVAL, "init is NULL");
    return kmeans_run(ctx, k, env_mask, max_iter, init, out_idx, out_n, out_G, out_iters);
}
