// TMA probe variants: which bulk-copy forms run on this B200 (development aid).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// V: 0 = tensor 2d .shared::cluster, 1 = tensor 2d .shared::cta, 2 = plain bulk 1d
template <int V>
__global__ void probe(const CUtensorMap *tmG, const float *src, float *out, int x, int y)
{
    __shared__ __align__(1024) float buf[32 * 64];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(8192) : "memory");
        if (V == 0)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(su32(buf)), "l"((uint64_t)tmG), "r"(x), "r"(y), "r"(su32(&bar)) : "memory");
#if V_CTA
        if (V == 1)
            asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(su32(buf)), "l"((uint64_t)tmG), "r"(x), "r"(y), "r"(su32(&bar)) : "memory");
#endif
        if (V == 2)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su32(buf)), "l"(src), "r"(8192), "r"(su32(&bar)) : "memory");
    }
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(su32(&bar)) : "memory");
    for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char **argv)
{
    int V = atoi(argv[1]);
    int cluster = argc > 2 ? atoi(argv[2]) : 0;
    int bx = argc > 3 ? atoi(argv[3]) : 64;
    const int C_pad = 128, E_pad = 64;
    float *g, *out;
    cudaMalloc(&g, sizeof(float) * C_pad * E_pad);
    cudaMalloc(&out, sizeof(float) * 32 * 64);
    static float h[128 * 64];
    for (int i = 0; i < C_pad * E_pad; i++) h[i] = (float)i;
    cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice);
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t ge = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    printf("entry %d q=%d p=%p\n", (int)ge, (int)q, p);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
    if (getenv("DIRECT")) { enc = cuTensorMapEncodeTiled; printf("direct\n"); }
    alignas(64) CUtensorMap tm;
    cuuint64_t gdim[2] = {(cuuint64_t)C_pad, (cuuint64_t)E_pad};
    cuuint64_t gstr[1] = {(cuuint64_t)C_pad * 4};
    cuuint32_t box[2] = {(cuuint32_t)bx, 32}, es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    {
        const unsigned char *b = (const unsigned char *)&tm;
        for (int i = 0; i < 128; i++) printf("%02x%s", b[i], (i % 32 == 31) ? "\n" : "");
    }
    CUtensorMap *dtm;
    cudaMalloc(&dtm, sizeof(CUtensorMap));
    cudaMemcpy(dtm, &tm, sizeof tm, cudaMemcpyHostToDevice);
    void (*kern)(const CUtensorMap *, const float *, float *, int, int) =
        V == 0 ? probe<0> : V == 1 ? probe<1> : probe<2>;
    if (cluster) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(1);
        cfg.blockDim = dim3(128);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 1;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kern, (const CUtensorMap *)dtm, (const float *)g, out, 3, 5);
    } else {
        kern<<<1, 128>>>(dtm, g, out, 3, 5);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("V=%d cluster=%d bx=%d: %s\n", V, cluster, bx, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    static float o[32 * 64];
    cudaMemcpy(o, out, sizeof o, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int yy = 0; yy < 32; yy++)
        for (int xx = 0; xx < bx; xx++)
            if (V != 2 && o[yy * bx + xx] != h[(5 + yy) * C_pad + 3 + xx]) bad++;
    printf("bad=%d o[0]=%g\n", bad, o[0]);
    return 0;
}
