// ubench_sad.cu -- the u8 |a-b| inner loop alone: a CTA of 256 threads holds a
// 128-row x 64-column tile; each thread 8 rows x 4 columns, one VABSDIFF4.U8.ACC per
// (row, column, 4 envs).  Operands re-read from shared memory (A [env-group][row],
// B [env-group][column], one 32-bit word = 4 envs), no staging / barriers / epilogue.
// Prints (set, env) evaluations per SM clock for 1..3 CTAs per SM.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/ubench_sad tools/ubench_sad.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define G 40          // env groups (160 envs; static smem <= 48 KB)
#define REPS 64

__global__ void __launch_bounds__(256) kern(uint32_t *out, unsigned long long *clk)
{
    __shared__ __align__(16) uint32_t As[G][128];
    __shared__ __align__(16) uint32_t Bs[G][64];
    for (int i = threadIdx.x; i < G * 128; i += 256) (&As[0][0])[i] = i * 2654435761u;
    for (int i = threadIdx.x; i < G * 64; i += 256) (&Bs[0][0])[i] = i * 40503u;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rg = warp * 2 + (lane >> 4);   // 16 row groups of 8
    const int cg = lane & 15;                // 16 column groups of 4
    uint32_t acc[8][4];
#pragma unroll
    for (int r = 0; r < 8; r++)
#pragma unroll
        for (int c = 0; c < 4; c++) acc[r][c] = 0;
    unsigned long long t0 = clock64();
    for (int rep = 0; rep < REPS; rep++) {
#pragma unroll 4
        for (int g = 0; g < G; g++) {
            const uint4 a0 = *(const uint4 *)&As[g][rg * 8];
            const uint4 a1 = *(const uint4 *)&As[g][rg * 8 + 4];
            const uint4 b = *(const uint4 *)&Bs[g][cg * 4];
            const uint32_t av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const uint32_t bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int r = 0; r < 8; r++)
#pragma unroll
                for (int c = 0; c < 4; c++)
                    asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(acc[r][c]) : "r"(av[r]), "r"(bv[c]));
        }
    }
    unsigned long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int r = 0; r < 8; r++)
#pragma unroll
        for (int c = 0; c < 4; c++) s += acc[r][c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) atomicMax(clk, t1 - t0);
}

int main()
{
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    uint32_t *out;
    unsigned long long *clk;
    cudaMalloc(&out, sizeof(uint32_t) * nsm * 4 * 256);
    cudaMalloc(&clk, 8);
    for (int per = 1; per <= 3; per++) {
        const int blocks = nsm * per;
        kern<<<blocks, 256>>>(out, clk);
        cudaMemset(clk, 0, 8);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        kern<<<blocks, 256>>>(out, clk);
        cudaEventRecord(e1);
        cudaDeviceSynchronize();
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long c;
        cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
        const double evals = (double)blocks * 128 * 64 * G * 4 * REPS;
        printf("%d CTA/SM: %.1f (set, env)/clk/SM  (%.3f ms, %s)\n", per, evals / ((double)c * nsm), ms,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
