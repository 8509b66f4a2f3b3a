// Instruction-mix ceiling of k_exh_tiled's inner loop (development aid): the exact
// HMNMX2 / HADD2 / FHADD tree of a thread's 8 rows x 4 columns over 16-env groups,
// operands re-read from shared memory each group as the kernel does, 16 warps per SM
// (2 CTAs x 8 warps, no ring, no barriers, no epilogue, no staging).  Prints (set, env)
// evaluations per clock per SM; the full kernel reaches ~85 at the paper shape.
// (A register-operand variant is not reported: the compiler folds its work away.)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hmin2(uint32_t a, uint32_t b) { uint32_t r; asm("min.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r; }
__device__ __forceinline__ uint32_t hadd2(uint32_t a, uint32_t b) { uint32_t r; asm("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r; }
__device__ __forceinline__ uint32_t blo(uint32_t w) { uint32_t r; asm("{ .reg .b16 l, h; mov.b32 {l, h}, %1; mov.b32 %0, {l, l}; }" : "=r"(r) : "r"(w)); return r; }
__device__ __forceinline__ uint32_t bhi(uint32_t w) { uint32_t r; asm("{ .reg .b16 l, h; mov.b32 {l, h}, %1; mov.b32 %0, {h, h}; }" : "=r"(r) : "r"(w)); return r; }
__device__ __forceinline__ void fhadd2(float &lo, float &hi, uint32_t p) {
    unsigned short a, b; asm("mov.b32 {%0, %1}, %2;" : "=h"(a), "=h"(b) : "r"(p));
    asm("add.rn.f32.f16 %0, %1, %0;" : "+f"(lo) : "h"(a)); asm("add.rn.f32.f16 %0, %1, %0;" : "+f"(hi) : "h"(b)); }

template <int SMEM>
__global__ void __launch_bounds__(256, 2) k(int iters, float *out)
{
    __shared__ __align__(16) uint16_t As[64 * 128];
    __shared__ __align__(16) uint32_t Bs[64 * 32];
    for (int i = threadIdx.x; i < 64 * 128; i += 256) As[i] = (uint16_t)(0x3000 + (i & 255));
    for (int i = threadIdx.x; i < 64 * 32; i += 256) Bs[i] = 0x34003400u + (i & 63);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tx = lane & 7, ty = lane >> 3;
    const int r0 = 32 * (warp >> 1) + 8 * ty, c0 = 32 * (warp & 1) + 4 * tx;
    float acc[8][4] = {};
    uint4 ar[4]; uint2 bc[4];
    for (int t = 0; t < 4; t++) { ar[t] = *(const uint4 *)(As + t * 128 + r0); bc[t] = *(const uint2 *)(Bs + t * 32 + c0 / 2); }
    for (int it = 0; it < iters; it++) {
#pragma unroll 1
        for (int e = 0; e < 64; e += 16) {
            uint32_t pp[8][2];
#pragma unroll
            for (int gq = 0; gq < 4; gq++) {
                if (SMEM) {
#pragma unroll
                    for (int t = 0; t < 4; t++) {
                        ar[t] = *(const uint4 *)(As + (e + 4 * gq + t) * 128 + r0);
                        bc[t] = *(const uint2 *)(Bs + (e + 4 * gq + t) * 32 + c0 / 2);
                    }
                } else {
                    // no instruction: the compiler must assume new operand values each group
#pragma unroll
                    for (int t = 0; t < 4; t++)
                        asm volatile("" : "+r"(ar[t].x), "+r"(ar[t].y), "+r"(ar[t].z), "+r"(ar[t].w),
                                     "+r"(bc[t].x), "+r"(bc[t].y));
                }
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    uint32_t av[4];
#pragma unroll
                    for (int t = 0; t < 4; t++) {
                        const uint32_t w = (i >> 1) == 0 ? ar[t].x : (i >> 1) == 1 ? ar[t].y : (i >> 1) == 2 ? ar[t].z : ar[t].w;
                        av[t] = (i & 1) ? bhi(w) : blo(w);
                    }
                    const uint32_t sx = hadd2(hadd2(hmin2(av[0], bc[0].x), hmin2(av[1], bc[1].x)), hadd2(hmin2(av[2], bc[2].x), hmin2(av[3], bc[3].x)));
                    const uint32_t sy = hadd2(hadd2(hmin2(av[0], bc[0].y), hmin2(av[1], bc[1].y)), hadd2(hmin2(av[2], bc[2].y), hmin2(av[3], bc[3].y)));
                    if (gq == 0) { pp[i][0] = sx; pp[i][1] = sy; }
                    else if (gq < 3) { pp[i][0] = hadd2(pp[i][0], sx); pp[i][1] = hadd2(pp[i][1], sy); }
                    else { fhadd2(acc[i][0], acc[i][1], hadd2(pp[i][0], sx)); fhadd2(acc[i][2], acc[i][3], hadd2(pp[i][1], sy)); }
                }
            }
        }
    }
    float s = 0; for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) s += acc[i][j];
    if (s == 1234.5f) out[0] = s;
}
int main()
{
    int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0); cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float *o; cudaMalloc(&o, 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 2000, blocks = sms * 2;
    for (int v = 1; v < 2; v++) {
        float best = 1e9;
        for (int r = 0; r < 5; r++) {
            cudaEventRecord(a);
            if (v == 0) k<0><<<blocks, 256>>>(iters, o); else k<1><<<blocks, 256>>>(iters, o);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best;
        }
        const double evals = (double)blocks * 256 * iters * 64 * 32;   // 64 envs x 32 sets per thread per iter
        printf("%s operands: %.3f ms, %.1f (set,env)/clk/SM (f16x2 ALU ceiling 128)\n", v ? "smem" : "register", best,
               evals / (best * 1e-3) / sms / (clk * 1e3));
    }
    return 0;
}
