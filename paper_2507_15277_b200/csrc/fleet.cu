// fleet.cu -- the fleet objective, Eq. 2 (Sec. 4.4.2), on the same
// search drivers as Eq. 1:
//
//     R(S) = sum_d quantity(d) / sum_{i in d} y'_{d,i}(S) * quantity(i),
//     y'_{d,i}(S) = min_{c in S} T[(d,i)][c]          (best member per env)
//
// Only the reduction changes w.r.t. Eq. 1: the per-env min is over raw runtimes,
// then a per-device weighted segmented sum, a reciprocal and a quantity(d)-
// weighted sum.  Environments are permuted so each device is one contiguous
// segment of a config-major fp64 copy of the runtimes (tcm).  Everything is
// fp64 in a fixed order (exact scorer; this objective is not the throughput
// path).  Sets are ranked by R descending, i.e. cost 1/R ascending (the tuner
// minimises the reciprocal), ties to the lexicographically smallest
// tuple / lowest index.
#include <algorithm>
#include <cmath>
#include <vector>

#include <cooperative_groups.h>
#include <cuda_fp16.h>

#include "pt_internal.cuh"

#define FL_MAXDEV 64
#define FL_BIGI 0x7fffffff

// tcm[c][q] = runtime of config c in permuted env q (missing -> penalty*best)
__global__ void k_fleet_build(const float *__restrict__ T, int64_t E, int64_t C,
                              const double *__restrict__ best, double penalty,
                              const int32_t *__restrict__ perm, int64_t E_pad,
                              double *__restrict__ tcm, double *__restrict__ tem)
{
    const int64_t c = blockIdx.x;
    for (int64_t q = threadIdx.x; q < E_pad; q += blockDim.x) {
        double v = 0.0;
        if (q < E) {
            const int64_t e = perm[q];
            const float t = T[e * C + c];
            v = isfinite(t) ? (double)t : penalty * best[e];
        }
        tcm[c * E_pad + q] = v;
        tem[q * C + c] = v;
    }
}

// R of one set given per-env "current" minima cur (may be +inf = empty) and an
// extra member column x (may be NULL): warp-wide, result on every lane
__device__ __forceinline__ double fleet_rate_warp(const double *__restrict__ cur,
                                                  const double *__restrict__ x,
                                                  const double *__restrict__ w,
                                                  const int32_t *__restrict__ seg, int n_dev,
                                                  const double *__restrict__ qdev, int lane)
{
    double R = 0.0;
    for (int d = 0; d < n_dev; d++) {
        double den = 0.0, wsum = 0.0;
        for (int q = seg[d] + lane; q < seg[d + 1]; q += 32) {
            double y = cur[q];
            if (x) y = fmin(y, x[q]);
            den += w[q] * y;
            wsum += w[q];
        }
        for (int o = 16; o; o >>= 1) {
            den += __shfl_xor_sync(0xffffffffu, den, o);
            wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
        }
        if (wsum > 0.0) R += qdev[d] / den;   // device present in scope
    }
    return R;
}

// one warp per set: R(set)
__global__ void k_fleet_score(const double *__restrict__ tcm, int64_t E_pad, int64_t C,
                              const int32_t *__restrict__ sets, int64_t n_sets, int k,
                              const double *__restrict__ w, const int32_t *__restrict__ seg,
                              int n_dev, const double *__restrict__ qdev, double *__restrict__ out,
                              int *__restrict__ bad)
{
    const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= n_sets) return;
    const int32_t *set = sets + s * k;
    for (int u = 0; u < k; u++)
        if (set[u] < 0 || set[u] >= C) {
            if (lane == 0) {
                atomicExch(bad, 1);
                out[s] = NAN;
            }
            return;
        }
    double R = 0.0;
    for (int d = 0; d < n_dev; d++) {
        double den = 0.0, wsum = 0.0;
        for (int q = seg[d] + lane; q < seg[d + 1]; q += 32) {
            double y = tcm[(int64_t)set[0] * E_pad + q];
            for (int u = 1; u < k; u++) y = fmin(y, tcm[(int64_t)set[u] * E_pad + q]);
            den += w[q] * y;
            wsum += w[q];
        }
        for (int o = 16; o; o >>= 1) {
            den += __shfl_xor_sync(0xffffffffu, den, o);
            wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
        }
        if (wsum > 0.0) R += qdev[d] / den;
    }
    if (lane == 0) out[s] = R;
}

// greedy step: warp per unselected candidate -> R(S u {c}) (taken: -inf)
__global__ void k_fleet_greedy_scan(const double *__restrict__ tcm, int64_t E_pad, int64_t C,
                                    const double *__restrict__ cur,
                                    const uint32_t *__restrict__ taken,
                                    const double *__restrict__ w, const int32_t *__restrict__ seg,
                                    int n_dev, const double *__restrict__ qdev,
                                    double *__restrict__ R)
{
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = gw; c < C; c += nw) {
        if (taken[c >> 5] >> (c & 31) & 1u) {
            if (lane == 0) R[c] = -INFINITY;
            continue;
        }
        const double r = fleet_rate_warp(cur, tcm + c * E_pad, w, seg, n_dev, qdev, lane);
        if (lane == 0) R[c] = r;
    }
}

__device__ __forceinline__ void top2_max(double &r1, int &c1, double &r2, int &c2, double r, int c)
{
    if (r > r1 || (r == r1 && c < c1)) {
        r2 = r1;
        c2 = c1;
        r1 = r;
        c1 = c;
    } else if (c != c1 && (r > r2 || (r == r2 && c < c2))) {
        r2 = r;
        c2 = c;
    }
}

// greedy step: one CTA picks the argmax (ties -> lowest c), updates cur/taken
__global__ void __launch_bounds__(1024) k_fleet_greedy_pick(const double *__restrict__ R, int64_t C,
                                                             const double *__restrict__ tcm,
                                                             int64_t E_pad, double *__restrict__ cur,
                                                             uint32_t *__restrict__ taken, int t,
                                                             int32_t *__restrict__ out_idx,
                                                             double *__restrict__ r1_tr,
                                                             double *__restrict__ r2_tr)
{
    __shared__ double sr1[32], sr2[32];
    __shared__ int sc1[32], sc2[32];
    __shared__ int cstar;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double r1 = -INFINITY, r2 = -INFINITY;
    int c1 = FL_BIGI, c2 = FL_BIGI;
    for (int64_t c = threadIdx.x; c < C; c += blockDim.x) top2_max(r1, c1, r2, c2, R[c], (int)c);
    for (int o = 16; o; o >>= 1) {
        const double a1 = __shfl_xor_sync(0xffffffffu, r1, o), a2 = __shfl_xor_sync(0xffffffffu, r2, o);
        const int b1 = __shfl_xor_sync(0xffffffffu, c1, o), b2 = __shfl_xor_sync(0xffffffffu, c2, o);
        top2_max(r1, c1, r2, c2, a1, b1);
        top2_max(r1, c1, r2, c2, a2, b2);
    }
    if (lane == 0) {
        sr1[warp] = r1;
        sr2[warp] = r2;
        sc1[warp] = c1;
        sc2[warp] = c2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); w++) {
            top2_max(r1, c1, r2, c2, sr1[w], sc1[w]);
            top2_max(r1, c1, r2, c2, sr2[w], sc2[w]);
        }
        cstar = c1;
        out_idx[t] = c1;
        r1_tr[t] = r1;
        r2_tr[t] = r2;
        taken[c1 >> 5] |= 1u << (c1 & 31);
    }
    __syncthreads();
    const double *col = tcm + (int64_t)cstar * E_pad;
    for (int64_t q = threadIdx.x; q < E_pad; q += blockDim.x) cur[q] = fmin(cur[q], col[q]);
}

// the whole fleet greedy in one cooperative launch (as k_greedy_resident for Eq. 1): the
// current per-env minima live in every CTA's shared memory; per step every warp scores
// its candidates (fleet_rate_warp, fp64, the scan kernel's order), each CTA keeps its
// (R desc, c asc) top-2, one grid barrier, every CTA merges the same block records and
// commits the same winner.  One launch for k steps instead of 2 k.
namespace cgf = cooperative_groups;
__global__ void __launch_bounds__(256) k_fleet_greedy_resident(
    const double *__restrict__ tcm, int64_t E_pad, int64_t C, int k, const double *__restrict__ w,
    const int32_t *__restrict__ seg, int n_dev, const double *__restrict__ qdev, double4 *__restrict__ blk,
    int32_t *__restrict__ out_idx, double *__restrict__ r1_tr, double *__restrict__ r2_tr)
{
    extern __shared__ double fsm[];
    double *cur = fsm;
    uint32_t *taken = reinterpret_cast<uint32_t *>(cur + E_pad);
    __shared__ double wr1[8], wr2[8];
    __shared__ int wc1[8], wc2[8];
    __shared__ int cstar;
    cgf::grid_group grid = cgf::this_grid();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t nwords = (C + 31) / 32;
    for (int64_t e = threadIdx.x; e < E_pad; e += blockDim.x) cur[e] = INFINITY;
    for (int64_t q = threadIdx.x; q < nwords; q += blockDim.x) taken[q] = 0u;
    __syncthreads();
    const int64_t gw = (int64_t)blockIdx.x * 8 + warp, nw = (int64_t)gridDim.x * 8;
    for (int t = 0; t < k; t++) {
        double r1 = -INFINITY, r2 = -INFINITY;
        int c1 = FL_BIGI, c2 = FL_BIGI;
        for (int64_t c = gw; c < C; c += nw) {
            if (taken[c >> 5] >> (c & 31) & 1u) continue;
            const double r = fleet_rate_warp(cur, tcm + c * E_pad, w, seg, n_dev, qdev, lane);
            top2_max(r1, c1, r2, c2, r, (int)c);
        }
        if (lane == 0) {
            wr1[warp] = r1;
            wr2[warp] = r2;
            wc1[warp] = c1;
            wc2[warp] = c2;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int q = 1; q < 8; q++) {
                top2_max(r1, c1, r2, c2, wr1[q], wc1[q]);
                top2_max(r1, c1, r2, c2, wr2[q], wc2[q]);
            }
            blk[(t & 1) * gridDim.x + blockIdx.x] = make_double4(r1, r2, (double)c1, (double)c2);
        }
        grid.sync();
        if (warp == 0) {
            r1 = r2 = -INFINITY;
            c1 = c2 = FL_BIGI;
            for (int b = lane; b < (int)gridDim.x; b += 32) {
                const double4 rec = blk[(t & 1) * gridDim.x + b];
                top2_max(r1, c1, r2, c2, rec.x, (int)rec.z);
                top2_max(r1, c1, r2, c2, rec.y, (int)rec.w);
            }
            for (int o = 16; o; o >>= 1) {
                const double a1 = __shfl_xor_sync(0xffffffffu, r1, o), a2 = __shfl_xor_sync(0xffffffffu, r2, o);
                const int b1 = __shfl_xor_sync(0xffffffffu, c1, o), b2 = __shfl_xor_sync(0xffffffffu, c2, o);
                top2_max(r1, c1, r2, c2, a1, b1);
                top2_max(r1, c1, r2, c2, a2, b2);
            }
            if (lane == 0) {
                cstar = c1;
                if (blockIdx.x == 0) {
                    out_idx[t] = c1;
                    r1_tr[t] = r1;
                    r2_tr[t] = r2;
                }
            }
        }
        __syncthreads();
        const int cs = cstar;
        if (threadIdx.x == 0) taken[cs >> 5] |= 1u << (cs & 31);
        const double *col = tcm + (int64_t)cs * E_pad;
        for (int64_t e = threadIdx.x; e < E_pad; e += blockDim.x) cur[e] = fmin(cur[e], col[e]);
        __syncthreads();
    }
}

// exhaustive: thread per subset (colex rank), per-device accumulators in
// registers/local memory; per-block (cost = 1/R, tuple) top-2
struct FRec2 {
    double s1, s2;
    int32_t t1[PT_MAXK], t2[PT_MAXK];
};

__device__ __forceinline__ void frec_offer(FRec2 &r, double s, const int32_t *t, int k)
{
    if (!(s < INFINITY)) return;
    if (pt_key_less(s, t, r.s1, r.t1, k)) {
        r.s2 = r.s1;
        for (int u = 0; u < k; u++) r.t2[u] = r.t1[u];
        r.s1 = s;
        for (int u = 0; u < k; u++) r.t1[u] = t[u];
    } else if (pt_key_less(s, t, r.s2, r.t2, k)) {
        bool same = s == r.s1;
        for (int u = 0; u < k && same; u++) same = t[u] == r.t1[u];
        if (!same) {
            r.s2 = s;
            for (int u = 0; u < k; u++) r.t2[u] = t[u];
        }
    }
}

__global__ void __launch_bounds__(128) k_fleet_exh(const double *__restrict__ tem, int64_t E_pad,
                                                  int64_t C, int k, int64_t r0, int64_t r1,
                                                  const double *__restrict__ w,
                                                  const int32_t *__restrict__ seg, int n_dev,
                                                  const double *__restrict__ qdev,
                                                  double *__restrict__ blk_s,
                                                  int32_t *__restrict__ blk_t)
{
    __shared__ FRec2 sh[128];
    FRec2 r;
    r.s1 = r.s2 = INFINITY;
    for (int u = 0; u < PT_MAXK; u++) r.t1[u] = r.t2[u] = FL_BIGI;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t R = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; R < r1; R += stride) {
        int32_t tup[PT_MAXK];
        pt_unrank_colex(R, k, C, tup);
        double rate = 0.0;
        for (int d = 0; d < n_dev; d++) {
            double den = 0.0, wsum = 0.0;
            for (int q = seg[d]; q < seg[d + 1]; q++) {
                // env-major: consecutive subsets share their larger members and step
                // the smallest, so a warp's loads of one env are (mostly) contiguous
                double y = tem[(int64_t)q * C + tup[0]];
                for (int u = 1; u < k; u++) y = fmin(y, tem[(int64_t)q * C + tup[u]]);
                den += w[q] * y;
                wsum += w[q];
            }
            if (wsum > 0.0) rate += qdev[d] / den;
        }
        frec_offer(r, 1.0 / rate, tup, k);
    }
    sh[threadIdx.x] = r;
    __syncthreads();
    for (int h = blockDim.x / 2; h > 0; h >>= 1) {
        if ((int)threadIdx.x < h) {
            FRec2 o = sh[threadIdx.x + h], me = sh[threadIdx.x];
            frec_offer(me, o.s1, o.t1, k);
            frec_offer(me, o.s2, o.t2, k);
            sh[threadIdx.x] = me;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        blk_s[2 * blockIdx.x] = sh[0].s1;
        blk_s[2 * blockIdx.x + 1] = sh[0].s2;
        for (int u = 0; u < k; u++) {
            blk_t[(2 * blockIdx.x) * k + u] = sh[0].t1[u];
            blk_t[(2 * blockIdx.x + 1) * k + u] = sh[0].t2[u];
        }
    }
}

// per device segment: max and min over (env, config < C) of w[q] * tcm[c][q]
__global__ void k_fleet_seg_minmax(const double *__restrict__ tcm, int64_t E_pad, int64_t C,
                                   const double *__restrict__ w, const int32_t *__restrict__ seg,
                                   double *__restrict__ out /* [n_dev][2] */)
{
    const int d = blockIdx.x;
    const int64_t q0 = seg[d], q1 = seg[d + 1];
    double mx = 0.0, mn = INFINITY;
    for (int64_t i = threadIdx.x; i < (q1 - q0) * C; i += blockDim.x) {
        const int64_t q = q0 + i / C, c = i % C;
        const double v = w[q] * tcm[c * E_pad + q];
        mx = fmax(mx, v);
        mn = fmin(mn, v);
    }
    __shared__ double smx[256], smn[256];
    smx[threadIdx.x] = mx;
    smn[threadIdx.x] = mn;
    __syncthreads();
    for (int h = 128; h > 0; h >>= 1) {
        if ((int)threadIdx.x < h) {
            smx[threadIdx.x] = fmax(smx[threadIdx.x], smx[threadIdx.x + h]);
            smn[threadIdx.x] = fmin(smn[threadIdx.x], smn[threadIdx.x + h]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[2 * d] = smx[0];
        out[2 * d + 1] = smn[0];
    }
}

// hWT[r][c] = RN16(w[q] * tcm[c][q] * scale[r]) for the segment row r -> permuted env q
// (rowq[r] = -1: a padding row), 0 past C
__global__ void k_fleet_half(const double *__restrict__ tcm, int64_t E_pad, int64_t C, int64_t C_pad,
                             const double *__restrict__ w, const int32_t *__restrict__ rowq,
                             const double *__restrict__ rscale, int64_t E_fp, uint16_t *__restrict__ hWT)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= E_fp * C_pad) return;
    const int64_t r = i / C_pad, c = i % C_pad;
    const int32_t q = rowq[r];
    double v = 0.0;
    if (q >= 0 && c < C) v = w[q] * tcm[c * E_pad + q] * rscale[r];
    hWT[i] = __half_as_ushort(__double2half(v));
}

void pt_fleet_tiled_free(pt_ctx *ctx)
{
    pt_fleet_tiled &t = ctx->fl.tiled;
    pt_dfree(ctx, t.hWT);
    pt_dfree(ctx, t.hWTile);
    t = pt_fleet_tiled();
}

pt_status pt_fleet_tiled_operands(pt_ctx *ctx, const pt_fleet_tiled **out)
{
    pt_fleet &f = ctx->fl;
    pt_fleet_tiled &t = f.tiled;
    *out = &t;
    if (t.built) return PT_OK;
    t.built = true;
    const int64_t C = ctx->C, E_pad = ctx->full.E_pad, C_pad = ctx->full.C_pad;
    cudaStream_t s = ctx->stream;
    double *mm = nullptr;
    PT_TRY(pt_dalloc(ctx, (void **)&mm, sizeof(double) * 2 * f.n_dev));
    k_fleet_seg_minmax<<<f.n_dev, 256, 0, s>>>(f.tcm, E_pad, C, f.w, f.seg, mm);
    ctx->stats.launches++;
    std::vector<double> h(2 * f.n_dev);
    PT_CK(cudaMemcpyAsync(h.data(), mm, sizeof(double) * 2 * f.n_dev, cudaMemcpyDeviceToHost, s));
    PT_CK(cudaStreamSynchronize(s));
    pt_dfree(ctx, mm);
    // segments -> padded rows; per device sigma_d = 2^(10 - ceil(log2 max))
    std::vector<int32_t> rowq;
    std::vector<double> rscale;
    int nst = 0;
    bool ok = true;
    for (int32_t d = 0; d < f.n_dev; d++) {
        const int64_t n = f.h_seg[d + 1] - f.h_seg[d];
        if (n == 0) continue;                             // a device without environments
        const double sigma = std::ldexp(1.0, 10 - (int)std::ceil(std::log2(h[2 * d])));
        if (!(h[2 * d + 1] * sigma >= std::ldexp(1.0, -14)) || !(h[2 * d] * sigma <= 1024.0)) ok = false;
        const int64_t rows = (n + 63) / 64 * 64;
        for (int64_t r = 0; r < rows; r++) {
            rowq.push_back(r < n ? (int32_t)(f.h_seg[d] + r) : -1);
            rscale.push_back(sigma);
        }
        nst += (int)(rows / 64);
        if (nst > 32) {
            ok = false;
            break;
        }
        t.stage_end_mask |= 1u << (nst - 1);
        t.stage_Q[nst - 1] = (float)(f.h_qdev[d] * sigma);
    }
    // the tiled kernel keeps the row tile's A operand for all E_fp rows in shared memory
    if ((int64_t)rowq.size() > 768) ok = false;
    if (!ok) return PT_OK;    // not eligible: the thread-per-subset search runs instead
    t.E_fp = (int64_t)rowq.size();
    int32_t *d_rowq = nullptr;
    double *d_rs = nullptr;
    PT_TRY(pt_dalloc(ctx, (void **)&d_rowq, sizeof(int32_t) * t.E_fp));
    PT_TRY(pt_dalloc(ctx, (void **)&d_rs, sizeof(double) * t.E_fp));
    PT_TRY(pt_dalloc(ctx, (void **)&t.hWT, sizeof(uint16_t) * t.E_fp * C_pad));
    PT_CK(cudaMemcpyAsync(d_rowq, rowq.data(), sizeof(int32_t) * t.E_fp, cudaMemcpyHostToDevice, s));
    PT_CK(cudaMemcpyAsync(d_rs, rscale.data(), sizeof(double) * t.E_fp, cudaMemcpyHostToDevice, s));
    k_fleet_half<<<(unsigned)((t.E_fp * C_pad + 255) / 256), 256, 0, s>>>(f.tcm, E_pad, C, C_pad, f.w, d_rowq, d_rs,
                                                                          t.E_fp, t.hWT);
    ctx->stats.launches++;
    PT_CK(cudaGetLastError());
    PT_CK(cudaStreamSynchronize(s));   // rowq / rscale are host temporaries
    pt_dfree(ctx, d_rowq);
    pt_dfree(ctx, d_rs);
    t.eligible = true;
    return PT_OK;
}

// ---------------------------------------------------------------------------
// host
// ---------------------------------------------------------------------------
extern "C" pt_status pt_set_fleet(pt_ctx *ctx, const double *q_device, int32_t n_device,
                                  const double *q_env)
{
    PT_NVTX();
    if (!ctx || !q_device || !q_env || n_device < 1) return pt_fail(PT_EINVAL, "bad argument");
    if (n_device > FL_MAXDEV) return pt_fail(PT_EINVAL, "at most %d devices", FL_MAXDEV);
    for (int32_t d = 0; d < n_device; d++)
        if (!(q_device[d] > 0.0)) return pt_fail(PT_EINVAL, "quantity(d=%d) must be > 0", d);
    for (int64_t e = 0; e < ctx->E; e++) {
        if (ctx->env_device[e] < 0 || ctx->env_device[e] >= n_device)
            return pt_fail(PT_EINVAL, "environment %lld has device id %d outside [0,%d)",
                           (long long)e, ctx->env_device[e], n_device);
        if (!(q_env[e] > 0.0)) return pt_fail(PT_EINVAL, "quantity of env %lld must be > 0", (long long)e);
    }
    PT_CK(cudaSetDevice(ctx->dev));
    pt_fleet_tiled_free(ctx);     // new quantities: the fp16 operands are rebuilt on use
    pt_fleet &f = ctx->fl;
    const int64_t E = ctx->E, C = ctx->C, E_pad = ctx->full.E_pad;
    f.perm.clear();
    f.h_seg.assign(1, 0);
    for (int32_t d = 0; d < n_device; d++) {
        for (int64_t e = 0; e < E; e++)
            if (ctx->env_device[e] == d) f.perm.push_back((int32_t)e);
        f.h_seg.push_back((int32_t)f.perm.size());
    }
    f.h_w.assign(E_pad, 0.0);
    for (int64_t q = 0; q < E; q++) f.h_w[q] = q_env[f.perm[q]];
    f.h_qdev.assign(q_device, q_device + n_device);
    f.n_dev = n_device;
    pt_dfree(ctx, f.w);
    pt_dfree(ctx, f.qdev);
    pt_dfree(ctx, f.seg);
    f.w = nullptr;
    f.qdev = nullptr;
    f.seg = nullptr;
    PT_TRY(pt_dalloc(ctx, (void **)&f.w, sizeof(double) * E_pad));
    PT_TRY(pt_dalloc(ctx, (void **)&f.qdev, sizeof(double) * n_device));
    PT_TRY(pt_dalloc(ctx, (void **)&f.seg, sizeof(int32_t) * (n_device + 1)));
    PT_CK(cudaMemcpyAsync(f.w, f.h_w.data(), sizeof(double) * E_pad, cudaMemcpyHostToDevice, ctx->stream));
    PT_CK(cudaMemcpyAsync(f.qdev, f.h_qdev.data(), sizeof(double) * n_device, cudaMemcpyHostToDevice,
                          ctx->stream));
    PT_CK(cudaMemcpyAsync(f.seg, f.h_seg.data(), sizeof(int32_t) * (n_device + 1), cudaMemcpyHostToDevice,
                          ctx->stream));
    if (!f.tcm) {
        PT_TRY(pt_dalloc(ctx, (void **)&f.tcm, sizeof(double) * C * E_pad));
        PT_TRY(pt_dalloc(ctx, (void **)&f.tem, sizeof(double) * C * E_pad));
    }
    int32_t *d_perm = nullptr;
    PT_TRY(pt_dalloc(ctx, (void **)&d_perm, sizeof(int32_t) * E));
    PT_CK(cudaMemcpyAsync(d_perm, f.perm.data(), sizeof(int32_t) * E, cudaMemcpyHostToDevice, ctx->stream));
    k_fleet_build<<<(unsigned)C, 128, 0, ctx->stream>>>(ctx->T32, E, C, ctx->best, ctx->penalty, d_perm,
                                                       E_pad, f.tcm, f.tem);
    ctx->stats.launches++;
    PT_CK(cudaGetLastError());
    pt_dfree(ctx, d_perm);
    PT_CK(cudaStreamSynchronize(ctx->stream));
    f.set = true;
    return PT_OK;
}

// weights for a scope: quantity(i) for in-scope envs, 0 elsewhere (device-major order)
static pt_status fleet_weights(pt_ctx *ctx, const uint8_t *env_mask, const double **d_w)
{
    pt_fleet &f = ctx->fl;
    if (!f.set) return pt_fail(PT_EINVAL, "PT_OBJ_FLEET needs pt_set_fleet first");
    if (!env_mask) {
        *d_w = f.w;
        return PT_OK;
    }
    std::vector<double> w(f.h_w);
    bool any = false;
    for (int64_t q = 0; q < ctx->E; q++) {
        if (!env_mask[f.perm[q]]) w[q] = 0.0;
        any = any || w[q] > 0.0;
    }
    if (!any) return pt_fail(PT_EEMPTY, "env_mask selects no environment");
    double *dw = nullptr;
    PT_TRY(pt_dalloc(ctx, (void **)&dw, sizeof(double) * w.size()));
    PT_CK(cudaMemcpyAsync(dw, w.data(), sizeof(double) * w.size(), cudaMemcpyHostToDevice, ctx->stream));
    *d_w = dw;
    return PT_OK;
}

static void fleet_weights_release(pt_ctx *ctx, const double *d_w)
{
    if (d_w != ctx->fl.w) pt_dfree(ctx, (void *)d_w);
}

pt_status pt_fleet_score(pt_ctx *ctx, const int32_t *d_sets, int64_t n_sets, int32_t k,
                         const uint8_t *env_mask, double *d_R)
{
    const double *w = nullptr;
    PT_TRY(fleet_weights(ctx, env_mask, &w));
    int *d_bad = nullptr;
    PT_TRY(pt_dalloc(ctx, (void **)&d_bad, sizeof(int)));
    PT_CK(cudaMemsetAsync(d_bad, 0, sizeof(int), ctx->stream));
    const int64_t threads = n_sets * 32;
    k_fleet_score<<<(unsigned)((threads + 255) / 256), 256, 0, ctx->stream>>>(
        ctx->fl.tcm, ctx->full.E_pad, ctx->C, d_sets, n_sets, k, w, ctx->fl.seg, ctx->fl.n_dev,
        ctx->fl.qdev, d_R, d_bad);
    ctx->stats.launches++;
    int bad = 0;
    PT_CK(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    pt_dfree(ctx, d_bad);
    fleet_weights_release(ctx, w);
    PT_CK(cudaStreamSynchronize(ctx->stream));
    if (bad) return pt_fail(PT_EINVAL, "a set holds a configuration index outside [0, %lld)", (long long)ctx->C);
    return PT_OK;
}

__global__ void k_fill_inf(double *p, int64_t n)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = INFINITY;
}

pt_status pt_fleet_greedy(pt_ctx *ctx, int32_t k, const uint8_t *env_mask, int32_t *out_idx,
                          double *R_trace, double *gap_trace)
{
    const int64_t C = ctx->C, E_pad = ctx->full.E_pad;
    if (k < 1 || k > C) return pt_fail(PT_EINVAL, "k=%d outside [1, %lld]", k, (long long)C);
    const double *w = nullptr;
    PT_TRY(fleet_weights(ctx, env_mask, &w));
    cudaStream_t s = ctx->stream;
    const int64_t nwords = (C + 31) / 32;
    double *R = nullptr, *cur = nullptr, *r1 = nullptr, *r2 = nullptr;
    uint32_t *taken = nullptr;
    int32_t *d_idx = nullptr;
    PT_TRY(pt_dalloc(ctx, (void **)&R, sizeof(double) * C));
    PT_TRY(pt_dalloc(ctx, (void **)&cur, sizeof(double) * E_pad));
    PT_TRY(pt_dalloc(ctx, (void **)&r1, sizeof(double) * k));
    PT_TRY(pt_dalloc(ctx, (void **)&r2, sizeof(double) * k));
    PT_TRY(pt_dalloc(ctx, (void **)&taken, sizeof(uint32_t) * nwords));
    PT_TRY(pt_dalloc(ctx, (void **)&d_idx, sizeof(int32_t) * k));
    PT_CK(cudaMemsetAsync(taken, 0, sizeof(uint32_t) * nwords, s));
    k_fill_inf<<<(unsigned)((E_pad + 255) / 256), 256, 0, s>>>(cur, E_pad);
    ctx->stats.launches++;
    const int grid = (int)std::min<int64_t>((C * 32 + 255) / 256, (int64_t)ctx->num_sms * 8);
    // one cooperative launch for all k steps when the current minima fit in shared memory
    const size_t rsmem = sizeof(double) * E_pad + sizeof(uint32_t) * nwords;
    int occ = 0;
    if (rsmem <= 200 * 1024) {
        if (rsmem > 48 * 1024)
            PT_CK(cudaFuncSetAttribute(k_fleet_greedy_resident, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)rsmem));
        PT_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fleet_greedy_resident, 256, rsmem));
    }
    PT_CK(cudaEventRecord(ctx->ev0, s));
    if (occ >= 1) {
        const int nblk = ctx->num_sms * std::min(occ, 2);
        double4 *blk = nullptr;
        PT_TRY(pt_dalloc(ctx, (void **)&blk, sizeof(double4) * 2 * nblk));
        const double *tcm = ctx->fl.tcm, *qd = ctx->fl.qdev;
        const int32_t *sg = ctx->fl.seg;
        int nd = ctx->fl.n_dev, kk = k;
        int64_t EE = E_pad, CC = C;
        void *args[] = {(void *)&tcm, (void *)&EE, (void *)&CC, (void *)&kk, (void *)&w, (void *)&sg,
                        (void *)&nd, (void *)&qd, (void *)&blk, (void *)&d_idx, (void *)&r1, (void *)&r2};
        PT_CK(cudaLaunchCooperativeKernel((void *)k_fleet_greedy_resident, dim3(nblk), dim3(256), args, rsmem, s));
        ctx->stats.launches++;
        pt_dfree(ctx, blk);
    } else {
        for (int t = 0; t < k; t++) {
            k_fleet_greedy_scan<<<grid, 256, 0, s>>>(ctx->fl.tcm, E_pad, C, cur, taken, w, ctx->fl.seg,
                                                     ctx->fl.n_dev, ctx->fl.qdev, R);
            k_fleet_greedy_pick<<<1, 1024, 0, s>>>(R, C, ctx->fl.tcm, E_pad, cur, taken, t, d_idx, r1, r2);
            ctx->stats.launches += 2;
        }
    }
    PT_CK(cudaEventRecord(ctx->ev1, s));
    PT_CK(cudaGetLastError());
    std::vector<double> h1(k), h2(k);
    PT_CK(cudaMemcpyAsync(out_idx, d_idx, sizeof(int32_t) * k, cudaMemcpyDeviceToHost, s));
    PT_CK(cudaMemcpyAsync(h1.data(), r1, sizeof(double) * k, cudaMemcpyDeviceToHost, s));
    PT_CK(cudaMemcpyAsync(h2.data(), r2, sizeof(double) * k, cudaMemcpyDeviceToHost, s));
    for (void *p : {(void *)R, (void *)cur, (void *)r1, (void *)r2, (void *)taken, (void *)d_idx})
        pt_dfree(ctx, p);
    fleet_weights_release(ctx, w);
    PT_CK(cudaStreamSynchronize(s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    ctx->stats.greedy_ms = ms;
    for (int t = 0; t < k; t++) {
        if (R_trace) R_trace[t] = h1[t];
        if (gap_trace) gap_trace[t] = std::isinf(h2[t]) ? INFINITY : h1[t] - h2[t];
    }
    return PT_OK;
}

// defined in exhaustive.cu (one-CTA (s, tuple) top-2 over records)
pt_status pt_top2_records(pt_ctx *ctx, const double *d_s, const int32_t *d_t, int64_t n, int k,
                          double *s_out, int32_t *t_out);

pt_status pt_fleet_exhaustive(pt_ctx *ctx, int32_t k, const uint8_t *env_mask, int32_t shard_rank,
                              int32_t shard_count, int32_t *best, int32_t *runner, double *R_out,
                              double *cost_out, int *n_found)
{
    const int64_t C = ctx->C, E_pad = ctx->full.E_pad;
    if (k < 1 || k > C) return pt_fail(PT_EINVAL, "k=%d outside [1, %lld]", k, (long long)C);
    if (k > PT_MAXK) return pt_fail(PT_EINVAL, "k=%d above the supported maximum %d", k, PT_MAXK);
    if (shard_count < 1 || shard_rank < 0 || shard_rank >= shard_count)
        return pt_fail(PT_EINVAL, "bad shard %d of %d", shard_rank, shard_count);
    const double nsets = std::exp(std::lgamma((double)C + 1) - std::lgamma((double)k + 1) -
                                  std::lgamma((double)(C - k) + 1));
    if (nsets > 1e13) return pt_fail(PT_ECAP, "C(%lld,%d) = %.3g exceeds the cap 1e13", (long long)C, k, nsets);
    if (!ctx->fl.set) return pt_fail(PT_EINVAL, "PT_OBJ_FLEET needs pt_set_fleet first");
    // the (min,+) tiled search with a per-device fold (exhaustive.cu) for the full scope
    if (!env_mask && k >= 2 && k <= 4 && k < C && !(ctx->flags & PT_EXACT_FP64) && E_pad <= 768) {
        const pt_fleet_tiled *ft = nullptr;
        PT_TRY(pt_fleet_tiled_operands(ctx, &ft));
        if (ft->eligible)
            return pt_fleet_exhaustive_tiled(ctx, k, shard_rank, shard_count, ft, best, runner, R_out, cost_out,
                                             n_found);
    }
    const double *w = nullptr;
    PT_TRY(fleet_weights(ctx, env_mask, &w));
    const int64_t n = pt_binom(C, k);
    const int64_t r0 = n * shard_rank / shard_count, r1 = n * (shard_rank + 1) / shard_count;
    double sv[2] = {INFINITY, INFINITY};
    std::vector<int32_t> t(2 * k, 0);
    if (r1 > r0) {
        cudaStream_t s = ctx->stream;
        const int nblk = (int)std::max<int64_t>(1, std::min<int64_t>((r1 - r0 + 127) / 128, (int64_t)ctx->num_sms * 16));
        double *bs = nullptr;
        int32_t *bt = nullptr;
        PT_TRY(pt_dalloc(ctx, (void **)&bs, sizeof(double) * 2 * nblk));
        PT_TRY(pt_dalloc(ctx, (void **)&bt, sizeof(int32_t) * 2 * nblk * k));
        PT_CK(cudaEventRecord(ctx->ev0, s));
        k_fleet_exh<<<nblk, 128, 0, s>>>(ctx->fl.tem, E_pad, C, k, r0, r1, w, ctx->fl.seg, ctx->fl.n_dev,
                                        ctx->fl.qdev, bs, bt);
        PT_CK(cudaEventRecord(ctx->ev1, s));
        ctx->stats.launches++;
        PT_CK(cudaGetLastError());
        PT_TRY(pt_top2_records(ctx, bs, bt, 2 * nblk, k, sv, t.data()));
        pt_dfree(ctx, bs);
        pt_dfree(ctx, bt);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        ctx->stats.exh_main_ms = ms;
        ctx->stats.exh_kernel = 2;
        ctx->stats.exh_sets = r1 - r0;
        ctx->stats.exh_slots = r1 - r0;
        ctx->stats.exh_candidates = 0;
        ctx->stats.exh_passes = 1;
    }
    fleet_weights_release(ctx, w);
    PT_CK(cudaStreamSynchronize(ctx->stream));
    const int nf = (sv[0] < INFINITY) + (sv[1] < INFINITY);
    if (n_found) *n_found = nf;
    for (int u = 0; u < k; u++) {
        best[u] = t[u];
        if (runner) runner[u] = t[k + u];
    }
    cost_out[0] = sv[0];
    cost_out[1] = sv[1];
    R_out[0] = nf >= 1 ? 1.0 / sv[0] : NAN;
    R_out[1] = nf >= 2 ? 1.0 / sv[1] : NAN;
    return PT_OK;
}
