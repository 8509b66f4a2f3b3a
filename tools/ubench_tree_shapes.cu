// loop-shape exploration: 8x4 (NG), 4x8 thread tiles; smem operands; 16 warps/SM
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

// R rows x CP column pairs per thread; NG 4-env groups chained
template <int R, int CP, int NG>
__global__ void __launch_bounds__(256, 2) k(int iters, float *out)
{
    __shared__ __align__(16) uint16_t As[64 * 128];
    __shared__ __align__(16) uint32_t Bs[64 * 64];
    for (int i = threadIdx.x; i < 64 * 128; i += 256) As[i] = (uint16_t)(0x3000 + (i & 255));
    for (int i = threadIdx.x; i < 64 * 64; i += 256) Bs[i] = 0x34003400u + (i & 63);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // rows per warp = 32*R/8... simple mapping: thread rows r0..r0+R-1, col pairs c0..c0+CP-1
    const int r0 = ((warp * 32 + lane) * R) & 127, c0 = (lane * CP) & 31;
    float acc[R][2 * CP] = {};
    for (int it = 0; it < iters; it++) {
#pragma unroll 1
        for (int e = 0; e < 64; e += 4 * NG) {
            uint32_t pp[R][CP];
#pragma unroll
            for (int gq = 0; gq < NG; gq++) {
                uint32_t a[4][R / 2];
                uint32_t b[4][CP];
#pragma unroll
                for (int t = 0; t < 4; t++) {
                    const int env = e + 4 * gq + t;
                    if (R == 8) { uint4 v = *(const uint4 *)(As + env * 128 + r0); a[t][0] = v.x; a[t][1] = v.y; a[t][2] = v.z; a[t][3] = v.w; }
                    else if (R == 4) { uint2 v = *(const uint2 *)(As + env * 128 + r0); a[t][0] = v.x; a[t][1] = v.y; }
                    if (CP == 2) { uint2 v = *(const uint2 *)(Bs + env * 64 + c0); b[t][0] = v.x; b[t][1] = v.y; }
                    else if (CP == 4) { uint4 v = *(const uint4 *)(Bs + env * 64 + c0); b[t][0] = v.x; b[t][1] = v.y; b[t][2] = v.z; b[t][3] = v.w; }
                }
#pragma unroll
                for (int i = 0; i < R; i++)
#pragma unroll
                    for (int j = 0; j < CP; j++) {
                        uint32_t av[4];
#pragma unroll
                        for (int t = 0; t < 4; t++) av[t] = (i & 1) ? bhi(a[t][i >> 1]) : blo(a[t][i >> 1]);
                        const uint32_t sx = hadd2(hadd2(hmin2(av[0], b[0][j]), hmin2(av[1], b[1][j])), hadd2(hmin2(av[2], b[2][j]), hmin2(av[3], b[3][j])));
                        if (gq == 0) pp[i][j] = sx;
                        else if (gq < NG - 1) pp[i][j] = hadd2(pp[i][j], sx);
                        else fhadd2(acc[i][2 * j], acc[i][2 * j + 1], NG == 1 ? sx : hadd2(pp[i][j], sx));
                    }
            }
        }
    }
    float s = 0; for (int i = 0; i < R; i++) for (int j = 0; j < 2 * CP; j++) s += acc[i][j];
    if (s == 1234.5f) out[0] = s;
}
template <int R, int CP, int NG> void run(const char *name, int sms, int clk, float *o)
{
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 2000, blocks = sms * 2;
    float best = 1e9;
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(a); k<R, CP, NG><<<blocks, 256>>>(iters, o); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best;
    }
    const double evals = (double)blocks * 256 * iters * 64 * R * 2 * CP;
    printf("%-22s %.3f ms, %.1f (set,env)/clk/SM\n", name, best, evals / (best * 1e-3) / sms / (clk * 1e3));
}
int main()
{
    int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0); cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float *o; cudaMalloc(&o, 4);
    run<8, 2, 4>("8 rows x 4 cols NG4", sms, clk, o);
    run<8, 2, 2>("8 rows x 4 cols NG2", sms, clk, o);
    run<8, 2, 1>("8 rows x 4 cols NG1", sms, clk, o);
    run<4, 4, 4>("4 rows x 8 cols NG4", sms, clk, o);
    run<4, 4, 2>("4 rows x 8 cols NG2", sms, clk, o);
    run<8, 4, 2>("8 rows x 8 cols NG2", sms, clk, o);
    return 0;
}
