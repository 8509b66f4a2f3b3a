// kmeans.cu -- the paper's k-means selector (Sec. 4.3.2; SURVEY
// §8(f) NEXT #4).  Environments are points of their slowdowns T/best over the
// configurations (reading k1); k = |kappa| centroids; per centroid the config
// with the smallest centroid slowdown is selected, duplicates
// collapse.  Deterministic maximin init and Lloyd iterations (reading k2).
//
// Every sum runs in the same order as the oracle's and products/sums use
// explicit round-to-nearest intrinsics (no FMA contraction), so the whole
// trajectory -- init, every assignment, every centroid -- is bit-identical to
// the CPU oracle's.  Work per Lloyd iteration: E x k x C squared differences
// (thread per point, k running sums in registers, centroid chunks staged in
// shared memory) + E x C adds for the update (thread per config).
#include <algorithm>
#include <cmath>
#include <vector>

#include "pt_internal.cuh"

#define KM_MAXK 32
#define KM_CB 64   // configs per staged centroid chunk

// X[c][q] = runtime / best (missing -> penalty), q over the scope's envs
__global__ void k_km_build(const float *__restrict__ T, int64_t C, const double *__restrict__ best,
                           double penalty, const int32_t *__restrict__ envs, int64_t ne,
                           double *__restrict__ X)
{
    const int64_t c = blockIdx.x;
    for (int64_t q = threadIdx.x; q < ne; q += blockDim.x) {
        const int64_t e = envs[q];
        const float t = T[e * C + c];
        const double tt = isfinite(t) ? (double)t : penalty * best[e];
        X[c * ne + q] = tt / best[e];
    }
}

// mean over points (q ascending), thread per config
__global__ void k_km_mean(const double *__restrict__ X, int64_t ne, int64_t C, double *__restrict__ mean)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    double s = 0.0;
    for (int64_t q = 0; q < ne; q++) s = __dadd_rn(s, X[c * ne + q]);
    mean[c] = s / (double)ne;
}

// squared distance of every point to nc centroids M[j][c] (j < nc), c ascending;
// thread per point; out D[q][j]
__global__ void __launch_bounds__(128) k_km_dist(const double *__restrict__ X, int64_t ne, int64_t C,
                                                const double *__restrict__ M, int nc,
                                                double *__restrict__ D)
{
    __shared__ double Ms[KM_MAXK][KM_CB];
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double acc[KM_MAXK];
#pragma unroll
    for (int j = 0; j < KM_MAXK; j++) acc[j] = 0.0;
    for (int64_t c0 = 0; c0 < C; c0 += KM_CB) {
        const int cb = (int)min((int64_t)KM_CB, C - c0);
        __syncthreads();
        for (int i = threadIdx.x; i < nc * KM_CB; i += blockDim.x) {
            const int j = i / KM_CB, cc = i % KM_CB;
            Ms[j][cc] = cc < cb ? M[(int64_t)j * C + c0 + cc] : 0.0;
        }
        __syncthreads();
        if (q < ne) {
            for (int cc = 0; cc < cb; cc++) {
                const double x = X[(c0 + cc) * ne + q];
#pragma unroll
                for (int j = 0; j < KM_MAXK; j++)
                    if (j < nc) {
                        const double t = __dsub_rn(x, Ms[j][cc]);
                        acc[j] = __dadd_rn(acc[j], __dmul_rn(t, t));
                    }
            }
        }
    }
    if (q < ne)
#pragma unroll
        for (int j = 0; j < KM_MAXK; j++)
            if (j < nc) D[q * KM_MAXK + j] = acc[j];
}

// the same distances with one thread per (point, centroid): ne * nc threads instead of
// ne (the per-thread loop over c ascending -- and so every result -- is unchanged)
__global__ void __launch_bounds__(128) k_km_dist1(const double *__restrict__ X, int64_t ne, int64_t C,
                                                 const double *__restrict__ M, int nc,
                                                 double *__restrict__ D)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ne * nc) return;
    const int64_t q = i % ne;
    const int j = (int)(i / ne);
    const double *m = M + (int64_t)j * C;
    double acc = 0.0;
    int64_t c = 0;
    for (; c + 16 <= C; c += 16) {   // 16 loads in flight, then the sums in c order
        double x[16], y[16];
#pragma unroll
        for (int u = 0; u < 16; u++) {
            x[u] = X[(c + u) * ne + q];
            y[u] = __ldg(m + c + u);
        }
#pragma unroll
        for (int u = 0; u < 16; u++) {
            const double t = __dsub_rn(x[u], y[u]);
            acc = __dadd_rn(acc, __dmul_rn(t, t));
        }
    }
    for (; c < C; c++) {
        const double t = __dsub_rn(X[c * ne + q], __ldg(m + c));
        acc = __dadd_rn(acc, __dmul_rn(t, t));
    }
    D[q * KM_MAXK + j] = acc;
}

// every point's distance to every point and to the mean (column ne), for the
// maximin initialisation: P[q][r] is what k_km_dist1 returns for point q and a
// centroid that is a copy of point r (or the mean) -- the same c-ascending sum
__global__ void __launch_bounds__(128) k_km_pair(const double *__restrict__ X, int64_t ne, int64_t C,
                                                const double *__restrict__ mean, double *__restrict__ P)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ne * (ne + 1)) return;
    const int64_t q = i % ne, r = i / ne;
    double acc = 0.0;
    int64_t c = 0;
    for (; c + 16 <= C; c += 16) {
        double x[16], y[16];
#pragma unroll
        for (int u = 0; u < 16; u++) {
            x[u] = X[(c + u) * ne + q];
            y[u] = r < ne ? X[(c + u) * ne + r] : mean[c + u];
        }
#pragma unroll
        for (int u = 0; u < 16; u++) {
            const double t = __dsub_rn(x[u], y[u]);
            acc = __dadd_rn(acc, __dmul_rn(t, t));
        }
    }
    for (; c < C; c++) {
        const double t = __dsub_rn(X[c * ne + q], r < ne ? X[c * ne + r] : mean[c]);
        acc = __dadd_rn(acc, __dmul_rn(t, t));
    }
    P[q * (ne + 1) + r] = acc;
}

// centroid update: M[j][c] = sum over points of cluster j (q ascending); counts on host
__global__ void k_km_update(const double *__restrict__ X, int64_t ne, int64_t C,
                            const int32_t *__restrict__ asg, int k, const int32_t *__restrict__ cnt,
                            double *__restrict__ M)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    double acc[KM_MAXK];
#pragma unroll
    for (int j = 0; j < KM_MAXK; j++) acc[j] = 0.0;
    for (int64_t q = 0; q < ne; q++) {
        const int a = asg[q];
        const double x = X[c * ne + q];
#pragma unroll
        for (int j = 0; j < KM_MAXK; j++)
            if (j == a) acc[j] = __dadd_rn(acc[j], x);
    }
    for (int j = 0; j < k; j++)
        if (cnt[j] > 0) M[(int64_t)j * C + c] = acc[j] / (double)cnt[j];
}

// copy point q into centroid row j
__global__ void k_km_seed(const double *__restrict__ X, int64_t ne, int64_t C, int64_t q, int j,
                          double *__restrict__ M)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c < C) M[(int64_t)j * C + c] = X[c * ne + q];
}

// per centroid: the config with the smallest slowdown (ties -> lowest index)
__global__ void k_km_select(const double *__restrict__ M, int64_t C, int32_t *__restrict__ sel)
{
    __shared__ double bv[256];
    __shared__ int bc[256];
    const int j = blockIdx.x;
    double v = INFINITY;
    int ci = 0x7fffffff;
    for (int64_t c = threadIdx.x; c < C; c += blockDim.x) {
        const double m = M[(int64_t)j * C + c];
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

extern "C" pt_status pt_kmeans_select(pt_ctx *ctx, int32_t k, const uint8_t *env_mask, int32_t max_iter,
                                      int32_t *out_idx, int32_t *out_n, double *out_G, int32_t *out_iters)
{
    PT_NVTX();
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
    int32_t *d_envs = nullptr, *d_asg = nullptr, *d_cnt = nullptr, *d_sel = nullptr;
    double *X = nullptr, *M = nullptr, *D = nullptr, *mean = nullptr;
    PT_TRY(pt_dalloc(ctx, (void **)&d_envs, sizeof(int32_t) * ne));
    PT_TRY(pt_dalloc(ctx, (void **)&X, sizeof(double) * C * ne));
    PT_TRY(pt_dalloc(ctx, (void **)&M, sizeof(double) * k * C));
    PT_TRY(pt_dalloc(ctx, (void **)&mean, sizeof(double) * C));
    PT_TRY(pt_dalloc(ctx, (void **)&D, sizeof(double) * ne * KM_MAXK));
    PT_TRY(pt_dalloc(ctx, (void **)&d_asg, sizeof(int32_t) * ne));
    PT_TRY(pt_dalloc(ctx, (void **)&d_cnt, sizeof(int32_t) * k));
    PT_TRY(pt_dalloc(ctx, (void **)&d_sel, sizeof(int32_t) * k));
    PT_CK(cudaMemcpyAsync(d_envs, envs.data(), sizeof(int32_t) * ne, cudaMemcpyHostToDevice, s));
    // the whole D block is copied back each time, only nc columns are written
    PT_CK(cudaMemsetAsync(D, 0, sizeof(double) * ne * KM_MAXK, s));
    k_km_build<<<(unsigned)C, 128, 0, s>>>(ctx->T32, C, ctx->best, ctx->penalty, d_envs, ne, X);
    const unsigned gc = (unsigned)((C + 127) / 128), gq = (unsigned)((ne + 127) / 128);
    std::vector<double> hD(ne * KM_MAXK), dmin(ne);
    (void)gq;
    auto dist = [&](const double *cent, int nc) -> pt_status {
        k_km_dist1<<<(unsigned)((ne * nc + 127) / 128), 128, 0, s>>>(X, ne, C, cent, nc, D);
        ctx->stats.launches++;
        PT_CK(cudaGetLastError());
        pt_hostio io(ctx);
        PT_TRY(io.d2h(hD.data(), D, sizeof(double) * ne * KM_MAXK));
        return io.finish();
    };
    // init: the point nearest the mean, then successive farthest points (maximin).
    // Every centroid of the init is a copy of a point, so up to 1,024 points one
    // pairwise pass (+ the mean) answers all k distance passes; beyond that, one
    // distance pass per centroid.
    k_km_mean<<<gc, 128, 0, s>>>(X, ne, C, mean);
    ctx->stats.launches += 2;
    const bool pairwise = ne <= 1024;
    std::vector<double> hP;
    if (pairwise) {
        double *P = nullptr;
        PT_TRY(pt_dalloc(ctx, (void **)&P, sizeof(double) * ne * (ne + 1)));
        k_km_pair<<<(unsigned)((ne * (ne + 1) + 127) / 128), 128, 0, s>>>(X, ne, C, mean, P);
        ctx->stats.launches++;
        PT_CK(cudaGetLastError());
        hP.resize((size_t)ne * (ne + 1));
        pt_hostio io(ctx);
        PT_TRY(io.d2h(hP.data(), P, sizeof(double) * ne * (ne + 1)));
        pt_dfree(ctx, P);
        PT_TRY(io.finish());
    }
    // (pairwise) distance of every point to the mean (r = ne) or to a copy of point r
    auto point_dist = [&](int64_t r, std::vector<double> &out) -> pt_status {
        for (int64_t q = 0; q < ne; q++) out[q] = hP[q * (ne + 1) + r];
        return PT_OK;
    };
    std::vector<double> dq(ne);
    int64_t first = 0;
    {
        if (pairwise) {
            PT_TRY(point_dist(ne, dq));
        } else {
            PT_TRY(dist(mean, 1));
            for (int64_t q = 0; q < ne; q++) dq[q] = hD[q * KM_MAXK];
        }
        double bd = INFINITY;
        for (int64_t q = 0; q < ne; q++)
            if (dq[q] < bd) {
                bd = dq[q];
                first = q;
            }
    }
    k_km_seed<<<gc, 128, 0, s>>>(X, ne, C, first, 0, M);
    ctx->stats.launches++;
    if (pairwise) {
        PT_TRY(point_dist(first, dmin));
    } else {
        PT_TRY(dist(M, 1));
        for (int64_t q = 0; q < ne; q++) dmin[q] = hD[q * KM_MAXK];
    }
    for (int j = 1; j < k; j++) {
        int64_t far = 0;
        double fd = -1.0;
        for (int64_t q = 0; q < ne; q++)
            if (dmin[q] > fd) {
                fd = dmin[q];
                far = q;
            }
        k_km_seed<<<gc, 128, 0, s>>>(X, ne, C, far, j, M);
        ctx->stats.launches++;
        if (pairwise) {
            PT_TRY(point_dist(far, dq));
        } else {
            PT_TRY(dist(M + (int64_t)j * C, 1));
            for (int64_t q = 0; q < ne; q++) dq[q] = hD[q * KM_MAXK];
        }
        for (int64_t q = 0; q < ne; q++) dmin[q] = std::min(dmin[q], dq[q]);
    }
    // Lloyd
    std::vector<int32_t> asg(ne, -1), cnt(k);
    int it = 0;
    while (it < max_iter) {
        PT_TRY(dist(M, k));
        bool changed = false;
        for (int64_t q = 0; q < ne; q++) {
            int bj = 0;
            double bdist = INFINITY;
            for (int j = 0; j < k; j++)
                if (hD[q * KM_MAXK + j] < bdist) {
                    bdist = hD[q * KM_MAXK + j];
                    bj = j;
                }
            changed = changed || asg[q] != bj;
            asg[q] = bj;
            dmin[q] = bdist;
        }
        it++;
        if (!changed && it > 1) break;
        std::fill(cnt.begin(), cnt.end(), 0);
        for (int64_t q = 0; q < ne; q++) cnt[asg[q]]++;
        PT_CK(cudaMemcpyAsync(d_asg, asg.data(), sizeof(int32_t) * ne, cudaMemcpyHostToDevice, s));
        PT_CK(cudaMemcpyAsync(d_cnt, cnt.data(), sizeof(int32_t) * k, cudaMemcpyHostToDevice, s));
        k_km_update<<<gc, 128, 0, s>>>(X, ne, C, d_asg, k, d_cnt, M);
        ctx->stats.launches++;
        for (int j = 0; j < k; j++)
            if (cnt[j] == 0) {   // re-seed with the point farthest from its centroid
                int64_t far = 0;
                double fd = -1.0;
                for (int64_t q = 0; q < ne; q++)
                    if (dmin[q] > fd) {
                        fd = dmin[q];
                        far = q;
                    }
                k_km_seed<<<gc, 128, 0, s>>>(X, ne, C, far, j, M);
                ctx->stats.launches++;
                dmin[far] = 0.0;
            }
    }
    k_km_select<<<k, 256, 0, s>>>(M, C, d_sel);
    ctx->stats.launches++;
    std::vector<int32_t> sel(k);
    PT_CK(cudaMemcpyAsync(sel.data(), d_sel, sizeof(int32_t) * k, cudaMemcpyDeviceToHost, s));
    for (void *p : {(void *)d_envs, (void *)X, (void *)M, (void *)mean, (void *)D, (void *)d_asg,
                    (void *)d_cnt, (void *)d_sel})
        pt_dfree(ctx, p);
    PT_CK(cudaStreamSynchronize(s));
    std::sort(sel.begin(), sel.end());
    sel.erase(std::unique(sel.begin(), sel.end()), sel.end());
    for (size_t u = 0; u < sel.size(); u++) out_idx[u] = sel[u];
    *out_n = (int32_t)sel.size();
    if (out_iters) *out_iters = it;
    if (out_G) PT_TRY(pt_score_sets(ctx, sel.data(), 1, (int32_t)sel.size(), env_mask, PT_OBJ_GEOMEAN, out_G));
    return PT_OK;
}
