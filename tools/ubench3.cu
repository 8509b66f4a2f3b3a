// ubench3.cu -- can the legacy tensor path (mma.sync, SASS HMMA) do the
// across-environment sum of the (min,+) product?  Measures on the whole chip:
//   op 0: mma.sync.m16n8k16 f16 -> f32, 8 independent accumulators per warp
//   op 1: mma.sync.m16n8k8  f16 -> f32
//   op 2: the candidate inner loop without loads: per MMA 4 HMNMX2 (the mins of
//         4 sets x 2 envs per thread) feeding one m16n8k16 (B = 0/1 selector)
//   op 3: op 2 with 8 HMNMX2 + 2 HMMA(k8) variant
// Rate = (set,env) evaluations per SM per clock (op 2/3), HMMA per SM per clock.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/ubench3 tools/ubench3.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define ITERS 2048
#define NACC 8

__device__ __forceinline__ void mma16(float *c, const uint32_t *a, uint32_t b0, uint32_t b1)
{
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma8(float *c, const uint32_t *a, uint32_t b0)
{
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(b0));
}
__device__ __forceinline__ uint32_t hmin2(uint32_t a, uint32_t b)
{
    uint32_t r;
    asm volatile("min.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

template <int OP>
__global__ void __launch_bounds__(256) kern(float *out, const uint32_t *in, unsigned long long *clk)
{
    float c[NACC][4];
    uint32_t a[8], b[4];
#pragma unroll
    for (int i = 0; i < 8; i++) a[i] = __ldcg(in + (threadIdx.x * 13 + i) % 4096);
#pragma unroll
    for (int i = 0; i < 4; i++) b[i] = __ldcg(in + (threadIdx.x * 7 + 100 + i) % 4096);
#pragma unroll
    for (int i = 0; i < NACC; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) c[i][j] = 0.f;
    const uint32_t one = 0x3C003C00u;
    unsigned long long t0 = clock64();
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int i = 0; i < NACC; i++) {
            if (OP == 0) {
                uint32_t f[4] = {a[i & 7], a[(i + 1) & 7], a[(i + 2) & 7], a[(i + 3) & 7]};
                mma16(c[i], f, one, one);
            }
            if (OP == 1) {
                uint32_t f[2] = {a[i & 7], a[(i + 1) & 7]};
                mma8(c[i], f, one);
            }
            if (OP == 2) {   // 4 sets (rows i>>1.., cols) x 1 env pair per thread per MMA
                uint32_t f[4];
                f[0] = hmin2(a[(i & 3) * 2], b[0]);
                f[1] = hmin2(a[(i & 3) * 2 + 1], b[0]);
                f[2] = hmin2(a[(i & 3) * 2], b[1]);
                f[3] = hmin2(a[(i & 3) * 2 + 1], b[1]);
                mma16(c[i], f, one, one);
            }
            if (OP == 3) {
                uint32_t f[2], g[2];
                f[0] = hmin2(a[(i & 3) * 2], b[0]);
                f[1] = hmin2(a[(i & 3) * 2 + 1], b[0]);
                g[0] = hmin2(a[(i & 3) * 2], b[1]);
                g[1] = hmin2(a[(i & 3) * 2 + 1], b[1]);
                mma8(c[i], f, one);
                mma8(c[i], g, one);
            }
        }
        // perturb operands so nothing is loop-invariant
#pragma unroll
        for (int i = 0; i < 4; i++) b[i] ^= (uint32_t)it & 1u;
    }
    unsigned long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NACC; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) s += c[i][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char *name, int nsm, int bps, float *out, const uint32_t *in, unsigned long long *clk,
         double per_mma_pairs, int mma_per_acc)
{
    const int grid = nsm * bps;
    kern<OP><<<grid, 256>>>(out, in, clk);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<OP><<<grid, 256>>>(out, in, clk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[4096];
    cudaMemcpy(h, clk, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < grid; i++) mx = h[i] > mx ? h[i] : mx;
    const double warps = grid * 8.0;
    const double mmas = warps * ITERS * NACC * mma_per_acc;
    const double clocks_per_sm = mx;   // all blocks co-resident
    printf("%-28s blocks/SM=%d  HMMA/SM/clk=%.3f  (set,env)/SM/clk=%.1f  ms=%.3f  TFLOP/s=%.1f\n", name, bps,
           mmas / nsm / clocks_per_sm, mmas * per_mma_pairs / nsm / clocks_per_sm, ms,
           mmas * (mma_per_acc == 1 ? 4096.0 : 2048.0) / (ms * 1e-3) / 1e12);
}

int main()
{
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float *out;
    uint32_t *in;
    unsigned long long *clk;
    cudaMalloc(&out, sizeof(float) * 4096 * 256);
    cudaMalloc(&in, sizeof(uint32_t) * 4096);
    cudaMemset(in, 0x31, sizeof(uint32_t) * 4096);
    cudaMalloc(&clk, sizeof(unsigned long long) * 4096);
    for (int bps : {1, 2, 4}) {
        run<0>("mma m16n8k16 f16->f32", nsm, bps, out, in, clk, 0.0, 1);
        run<1>("mma m16n8k8 f16->f32", nsm, bps, out, in, clk, 0.0, 1);
        run<2>("4xHMNMX2 + mma k16", nsm, bps, out, in, clk, 256.0, 1);
        run<3>("4xHMNMX2 + 2 mma k8", nsm, bps, out, in, clk, 128.0, 2);
    }
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
