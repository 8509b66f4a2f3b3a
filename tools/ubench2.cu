// ubench2.cu -- instruction-mix throughput for the (min,+) inner loop, timed with
// CUDA events (pipe attribution via ncu --metrics sm__inst_executed_pipe_*).
// Each thread: 8 accumulators x (one min + one add per "eval"); inputs from
// registers refreshed every iteration so nothing folds.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define ITERS 2048

// V0: FMNMX + FADD           (fp32)
// V1: HMNMX2 + 2x FHADD      (f16x2 mins, fp32 accumulate)
// V2: VIMNMX + IADD3 (pair)  (int32)
// V3: FMNMX + FFMA(x,1,acc)
template <int V>
__global__ void __launch_bounds__(256) kern(const uint32_t *in, float *out)
{
    __shared__ uint32_t sm[64 * 64];
    for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) sm[i] = in[i & 1023] + i;
    __syncthreads();
    float acc[8][4];
    uint32_t iacc[8][4];
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = 0.f, iacc[i][j] = 0;
    for (int it = 0; it < ITERS; it++) {
        const uint32_t *row = sm + (it & 63) * 64;
        const uint4 a0 = *reinterpret_cast<const uint4 *>(row + (threadIdx.x & 7) * 4);
        const uint4 a1 = *reinterpret_cast<const uint4 *>(row + 32 + (threadIdx.x & 7) * 4);
        const uint4 bb = *reinterpret_cast<const uint4 *>(row + ((threadIdx.x >> 3) & 15) * 4);
        const uint32_t a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const uint32_t b[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
        for (int i = 0; i < 8; i++) {
#pragma unroll
            for (int j = 0; j < 4; j++) {
                if (V == 0) acc[i][j] += fminf(__uint_as_float(a[i]), __uint_as_float(b[j]));
                if (V == 3) {
                    float m = fminf(__uint_as_float(a[i]), __uint_as_float(b[j]));
                    asm("fma.rn.f32 %0, %1, 0f3F800000, %0;" : "+f"(acc[i][j]) : "f"(m));
                }
                if (V == 2 && (j & 1) == 0) {
                    uint32_t m0 = min(a[i], b[j]), m1 = min(a[i], b[j + 1]);
                    iacc[i][j] = iacc[i][j] + m0 + m1;
                }
                if (V == 1 && (j & 1) == 0) {   // one HMNMX2 = 2 evals
                    uint32_t m;
                    asm("min.f16x2 %0, %1, %2;" : "=r"(m) : "r"(a[i]), "r"(b[j]));
                    unsigned short lo, hi;
                    asm("mov.b32 {%0, %1}, %2;" : "=h"(lo), "=h"(hi) : "r"(m));
                    asm("add.rn.f32.f16 %0, %1, %0;" : "+f"(acc[i][j]) : "h"(lo));
                    asm("add.rn.f32.f16 %0, %1, %0;" : "+f"(acc[i][j + 1]) : "h"(hi));
                }
            }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) s += acc[i][j] + (float)iacc[i][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int V>
void run(const char *name, int nsm, const uint32_t *in, float *out)
{
    const int blocks = nsm * 2;
    kern<V><<<blocks, 256>>>(in, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<V><<<blocks, 256>>>(in, out);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int mhz;
    cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, 0);
    const double evals = (double)blocks * 256 * ITERS * 32;
    printf("%-26s %8.3f ms  %7.2f Tevals/s  %6.1f evals/clk/SM @ max clock %d MHz\n", name, ms,
           evals / ms / 1e9, evals / (ms * 1e-3) / (nsm * mhz * 1e3), mhz / 1000);
}

int main()
{
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    uint32_t *in;
    float *out;
    cudaMalloc(&in, 4096);
    cudaMemset(in, 0x3c, 4096);
    cudaMalloc(&out, sizeof(float) * nsm * 512);
    run<0>("FMNMX+FADD", nsm, in, out);
    run<3>("FMNMX+FFMA(imm1)", nsm, in, out);
    run<2>("VIMNMX+IADD3", nsm, in, out);
    run<1>("HMNMX2+2xFHADD", nsm, in, out);
    return 0;
}
