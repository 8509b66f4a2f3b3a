// score.cu -- pt_score_sets: Eq. 1 fitness of arbitrary candidate sets.
//
// One warp per set; lanes stride over the environments; the per-environment
// best member is a running min of log-slowdowns held in registers (P:L222:
// "the performance for each environment is that of the best-performing of
// the ... variants"); the across-environment sum (Eq. 1) is a
// fixed xor-shuffle tree, so the result is deterministic.  fp64 throughout
// (this call is the exact scorer, not the throughput path).
#include "pt_internal.cuh"

__global__ void k_score_sets(const double *__restrict__ l64, int64_t E_pad, int64_t C,
                             const int32_t *__restrict__ sets, int64_t n_sets, int k,
                             double *__restrict__ out_s, int *__restrict__ bad)
{
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= n_sets) return;
    const int32_t *set = sets + w * k;
    bool ok = true;
    for (int u = 0; u < k; u++) ok = ok && set[u] >= 0 && set[u] < C;
    if (!ok) {
        if (lane == 0) {
            atomicExch(bad, 1);
            out_s[w] = NAN;
        }
        return;
    }
    double acc = 0.0;
    for (int64_t e = lane; e < E_pad; e += 32) {
        double m = l64[(int64_t)set[0] * E_pad + e];
        for (int u = 1; u < k; u++) m = fmin(m, l64[(int64_t)set[u] * E_pad + e]);
        acc += m;
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out_s[w] = acc;
}

// s -> G = exp(-s / E) in place
__global__ void k_s_to_G(double *__restrict__ v, int64_t n, double inv_E)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = exp(-v[i] * inv_E);
}

pt_status pt_score_view(pt_ctx *ctx, const pt_view *v, const int32_t *d_sets, int64_t n_sets,
                        int32_t k, double *d_s)
{
    if (n_sets == 0) return PT_OK;
    int *d_bad = nullptr;
    PT_CK(cudaMallocAsync((void **)&d_bad, sizeof(int), ctx->stream));
    PT_CK(cudaMemsetAsync(d_bad, 0, sizeof(int), ctx->stream));
    const int64_t threads = n_sets * 32;
    k_score_sets<<<(unsigned)((threads + 255) / 256), 256, 0, ctx->stream>>>(
        v->l64, v->E_pad, v->C, d_sets, n_sets, k, d_s, d_bad);
    ctx->stats.launches++;
    int bad = 0;
    PT_CK(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    PT_CK(cudaFreeAsync(d_bad, ctx->stream));
    PT_CK(cudaStreamSynchronize(ctx->stream));
    if (bad) return pt_fail(PT_EINVAL, "a set holds a configuration index outside [0, %lld)",
                            (long long)v->C);
    return PT_OK;
}

extern "C" pt_status pt_score_sets(pt_ctx *ctx, const int32_t *sets, int64_t n_sets, int32_t k,
                                   const uint8_t *env_mask, int32_t objective, double *out_G)
{
    PT_NVTX();
    if (!ctx || (!sets && n_sets > 0) || (!out_G && n_sets > 0) || n_sets < 0)
        return pt_fail(PT_EINVAL, "NULL argument");
    if (objective != PT_OBJ_GEOMEAN && objective != PT_OBJ_FLEET)
        return pt_fail(PT_EINVAL, "unknown objective %d", objective);
    if (k < 1) return pt_fail(PT_EEMPTY, "empty set (k < 1)");
    PT_CK(cudaSetDevice(ctx->dev));
    const pt_view *v = nullptr;
    if (objective == PT_OBJ_GEOMEAN) PT_TRY(pt_get_view(ctx, env_mask, &v));
    if (n_sets == 0) return PT_OK;
    const bool sets_dev = pt_is_device_ptr(sets), out_dev = pt_is_device_ptr(out_G);
    const size_t set_bytes = sizeof(int32_t) * (size_t)n_sets * k;
    const size_t out_bytes = sizeof(double) * (size_t)n_sets;
    void *scr = nullptr;
    PT_TRY(pt_scratch(ctx, set_bytes + out_bytes + 256, &scr));
    double *d_s = out_dev ? out_G : (double *)scr;
    const int32_t *d_sets = sets;
    if (!sets_dev) {
        int32_t *tmp = (int32_t *)((char *)scr + pt_round_up(out_bytes, 256));
        PT_CK(cudaMemcpyAsync(tmp, sets, set_bytes, cudaMemcpyHostToDevice, ctx->stream));
        d_sets = tmp;
    }
    if (objective == PT_OBJ_FLEET) {
        PT_TRY(pt_fleet_score(ctx, d_sets, n_sets, k, env_mask, d_s));
    } else {
        PT_TRY(pt_score_view(ctx, v, d_sets, n_sets, k, d_s));
        k_s_to_G<<<(unsigned)((n_sets + 255) / 256), 256, 0, ctx->stream>>>(d_s, n_sets,
                                                                           1.0 / (double)v->E);
        ctx->stats.launches++;
    }
    if (!out_dev)
        PT_CK(cudaMemcpyAsync(out_G, d_s, out_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    PT_CK(cudaStreamSynchronize(ctx->stream));
    return PT_OK;
}
