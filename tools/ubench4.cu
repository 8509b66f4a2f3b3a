// ubench4.cu -- the k_exh_mma inner loop in isolation (operands from shared
// memory exactly as the kernel reads them), to separate the loop's own
// throughput from the kernel's pipeline / epilogue overheads.
//   v0: per env pair 2 LDS.128 (A: 8 rows) + 1 LDS.128 (B: 4 cols), 32 HMNMX2, 8 HMMA
//   v1: operands in registers (no LDS), same math
//   v2: v0 with 2 independent accumulator sets alternating (16 acc)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/ubench4 tools/ubench4.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define ITERS 512
__device__ __forceinline__ uint32_t hmin2(uint32_t a, uint32_t b)
{
    uint32_t r;
    asm("min.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ void mma_sum(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                        uint32_t b0, uint32_t b1)
{
    asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint4 lds128(const uint32_t *p)
{
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "r"((uint32_t)__cvta_generic_to_shared(p)));
    return r;
}

template <int V>
__global__ void __launch_bounds__(256, 3) kern(float *out, int n_warps_active)
{
    __shared__ __align__(16) uint32_t As[32 * 36];
    __shared__ __align__(16) uint32_t Bs[32 * 64];
    for (int i = threadIdx.x; i < 32 * 36; i += blockDim.x) As[i] = 0x3C003C00u ^ (i * 2654435761u & 0x03ff03ffu);
    for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) Bs[i] = 0x3C003C00u ^ (i * 40503u & 0x03ff03ffu);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, q = lane & 3;
    const int r0 = 8 * (warp >> 1), c0 = 32 * (warp & 1) + 4 * g;
    const uint32_t one2 = 0x3C003C00u;
    const uint32_t sel0 = (g & 1) ? 0u : one2, sel1 = (g & 1) ? one2 : 0u;
    float acc[4][2][4] = {};
    const uint32_t *A = As + q * 36 + r0;
    const uint32_t *B = Bs + q * 64 + 4 * ((c0 >> 2) ^ (q << 1));
    uint4 al0 = *reinterpret_cast<const uint4 *>(A), ah0 = *reinterpret_cast<const uint4 *>(A + 4),
          bv0 = *reinterpret_cast<const uint4 *>(B);
    uint32_t dummy = 0;
    if (V >= 7) {   // software-pipelined: operands of kk+1 loaded (volatile asm) before kk's math
        uint4 nal = lds128(A), nah = lds128(A + 4), nbv = lds128(B);
        for (int it = 0; it < ITERS; it++) {
#pragma unroll
            for (int kk = 0; kk < 8; kk++) {
                const uint32_t a[8] = {nal.x, nal.y, nal.z, nal.w, nah.x, nah.y, nah.z, nah.w};
                const uint32_t b[4] = {nbv.x, nbv.y, nbv.z, nbv.w};
                const int kn = (kk + 1) & 7;
                nal = lds128(A + 4 * kn * 36);
                nah = lds128(A + 4 * kn * 36 + 4);
                nbv = lds128(B + 4 * kn * 64);
#pragma unroll
                for (int i = 0; i < 4; i++)
#pragma unroll
                    for (int j = 0; j < 2; j++)
                        mma_sum(acc[i][j], hmin2(a[2 * i], b[2 * j]), hmin2(a[2 * i + 1], b[2 * j]),
                                hmin2(a[2 * i], b[2 * j + 1]), hmin2(a[2 * i + 1], b[2 * j + 1]), sel0, sel1);
            }
        }
    } else
    for (int it = 0; it < ITERS; it++) {
#pragma unroll 2
        for (int kk = 0; kk < 8; kk++) {
            uint4 al, ah, bv;
            if (V == 1) {
                al = al0;
                ah = ah0;
                bv = bv0;
                bv.x ^= kk;
            } else if (V == 2) {   // A from smem, B registers
                al = *reinterpret_cast<const uint4 *>(A + 4 * kk * 36);
                ah = *reinterpret_cast<const uint4 *>(A + 4 * kk * 36 + 4);
                bv = bv0;
                bv.x ^= kk;
            } else if (V == 3) {   // B from smem, A registers
                al = al0;
                ah = ah0;
                al.x ^= kk;
                bv = *reinterpret_cast<const uint4 *>(B + 4 * kk * 64);
            } else if (V == 5 || V == 6) {   // register math + an unrelated LDS.128 (V5) / LDS.32 (V6)
                al = al0;
                ah = ah0;
                bv = bv0;
                bv.x ^= kk;
                if (V == 5) {
                    const uint4 t = *reinterpret_cast<const uint4 *>(B + 4 * kk * 64);
                    dummy ^= t.x ^ t.y ^ t.z ^ t.w;
                } else {
                    dummy ^= *(const volatile uint32_t *)(B + 4 * kk * 64);
                }
            } else if (V == 4) {   // A via 8 x LDS.32
                const volatile uint32_t *Av = A + 4 * kk * 36;
                al = make_uint4(Av[0], Av[1], Av[2], Av[3]);
                ah = make_uint4(Av[4], Av[5], Av[6], Av[7]);
                bv = *reinterpret_cast<const uint4 *>(B + 4 * kk * 64);
            } else {
                al = *reinterpret_cast<const uint4 *>(A + 4 * kk * 36);
                ah = *reinterpret_cast<const uint4 *>(A + 4 * kk * 36 + 4);
                bv = *reinterpret_cast<const uint4 *>(B + 4 * kk * 64);
            }
            const uint32_t a[8] = {al.x, al.y, al.z, al.w, ah.x, ah.y, ah.z, ah.w};
            const uint32_t b[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 2; j++)
                    mma_sum(acc[i][j], hmin2(a[2 * i], b[2 * j]), hmin2(a[2 * i + 1], b[2 * j]),
                            hmin2(a[2 * i], b[2 * j + 1]), hmin2(a[2 * i + 1], b[2 * j + 1]), sel0, sel1);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 2; j++)
#pragma unroll
            for (int t = 0; t < 4; t++) s += acc[i][j][t];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)(dummy & 1);
}

template <int V>
void run(const char *name, int nsm, int bps, float *out)
{
    const int grid = nsm * bps;
    kern<V><<<grid, 256>>>(out, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<V><<<grid, 256>>>(out, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    // (set, env) per launch: warps x ITERS x 8 kk x 8 MMA x 256
    const double se = (double)grid * 8 * ITERS * 8 * 8 * 256;
    printf("%-34s blocks/SM=%d  %.3f ms  %.2f T(set,env)/s  (%.1f%% of 37.2)\n", name, bps, ms, se / (ms * 1e-3) / 1e12,
           se / (ms * 1e-3) / 1e12 / 37.22 * 100);
}

int main()
{
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float *out;
    cudaMalloc(&out, sizeof(float) * nsm * 4 * 256);
    for (int bps : {2, 3}) {
        run<0>("v0 LDS operands (kernel loop)", nsm, bps, out);
        run<1>("v1 register operands", nsm, bps, out);
        run<2>("v2 A smem, B regs", nsm, bps, out);
        run<3>("v3 B smem, A regs", nsm, bps, out);
        run<4>("v4 A 8xLDS.32, B LDS.128", nsm, bps, out);
        run<5>("v5 regs + unrelated LDS.128", nsm, bps, out);
        run<6>("v6 regs + unrelated LDS.32", nsm, bps, out);
        run<7>("v7 prefetch (volatile lds, unroll 8)", nsm, bps, out);
    }
    printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
