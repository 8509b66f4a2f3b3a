// Probe: 2D TMA load of a 64x32 fp32 box, tensor map in param space vs global memory.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void probe(const __grid_constant__ CUtensorMap tmP, const CUtensorMap *tmG, float *out, int x, int y)
{
    __shared__ __align__(128) float buf[32 * 64];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const CUtensorMap *tm = MODE == 0 ? &tmP : tmG;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(8192) : "memory");
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(su32(buf)), "l"((uint64_t)tm), "r"(x), "r"(y), "r"(su32(&bar)) : "memory");
    }
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(su32(&bar)) : "memory");
    for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) out[i] = buf[i];
}

int g_mode = 0;
int main(int argc, char **argv)
{
    g_mode = argc > 1 ? atoi(argv[1]) : 0;
    const int C_pad = 128, E_pad = 64;
    float *g, *out;
    cudaMalloc(&g, sizeof(float) * C_pad * E_pad);
    cudaMalloc(&out, sizeof(float) * 32 * 64);
    float h[128 * 64];
    for (int i = 0; i < C_pad * E_pad; i++) h[i] = (float)i;
    cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice);
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
    CUtensorMap tm;
    cuuint64_t gdim[2] = {(cuuint64_t)C_pad, (cuuint64_t)E_pad};
    cuuint64_t gstr[1] = {(cuuint64_t)C_pad * 4};
    cuuint32_t box[2] = {64, 32}, es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    CUtensorMap *dtm;
    cudaMalloc(&dtm, sizeof(CUtensorMap));
    cudaMemcpy(dtm, &tm, sizeof tm, cudaMemcpyHostToDevice);
    float o[32 * 64];
    int m0 = 0; (void)m0;
    extern int g_mode; 
    for (int mode = g_mode; mode < g_mode + 1; mode++) {
        if (mode == 0) probe<0><<<1, 128>>>(tm, dtm, out, 3, 5);
        else probe<1><<<1, 128>>>(tm, dtm, out, 3, 5);
        cudaError_t e = cudaDeviceSynchronize();
        printf("mode %d: %s\n", mode, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
        cudaMemcpy(o, out, sizeof o, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int yy = 0; yy < 32; yy++)
            for (int xx = 0; xx < 64; xx++)
                if (o[yy * 64 + xx] != h[(5 + yy) * C_pad + 3 + xx]) bad++;
        printf("mode %d bad=%d o[0]=%g\n", mode, bad, o[0]);
    }
    // OOB box
    probe<1><<<1, 128>>>(tm, dtm, out, 100, 40);
    printf("oob: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    cudaMemcpy(o, out, sizeof o, cudaMemcpyDeviceToHost);
    printf("oob o[0]=%g (want %g) o[27]=%g (want 0) o[63+64*23]=%g\n", o[0], h[40 * 128 + 100], o[27], o[63 + 64 * 23]);
    return 0;
}
