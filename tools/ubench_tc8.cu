// ubench_tc8.cu -- probe for the threshold-count tier: one CTA runs
// D[128 x 256] = A[128 x K] . B[256 x K]^T with tcgen05.mma kind::f8f6f4 (E4M3 0/1/2
// values, both operands K-major in shared memory, no swizzle) in the exact layouts of
// k_exh_tc, and checks every element against the host; then times a long MMA chain.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/ubench_tc8 tools/ubench_tc8.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define K 64
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
constexpr uint32_t kIdesc = (1u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);

__global__ void k_probe(const uint8_t *Ag, const uint8_t *Bg, float *D, int swapLS, int reps, long long *cyc)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *As = sm, *Bs = sm + 128 * K;
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    // A: offset(r,k) = (k/16)*2048 + (r/8)*128 + (r%8)*16 + k%16 ; B: (n/8)*(8K) + (k/16)*128 + (n%8)*16 + k%16
    for (int i = tid; i < 128 * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        As[(k / 16) * 2048 + (r / 8) * 128 + (r % 8) * 16 + k % 16] = Ag[i];
    }
    for (int i = tid; i < 256 * K; i += blockDim.x) {
        const int n = i / K, k = i % K;
        Bs[(n / 8) * (8 * K) + (k / 16) * 128 + (n % 8) * 16 + k % 16] = Bg[i];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    long long t0 = clock64();
    if (tid == 0) {
        for (int rep = 0; rep < reps; rep++)
            for (int i = 0; i < K / 32; i++) {
                const uint32_t aL = swapLS ? 128 : 2048, aS = swapLS ? 2048 : 128;
                const uint32_t bL = swapLS ? 8 * K : 128, bS = swapLS ? 128 : 8 * K;
                const uint64_t ad = sdesc(su32(As) + i * 2 * 2048, aL, aS);
                const uint64_t bd = sdesc(su32(Bs) + i * 2 * 128, bL, bS);
                const uint32_t acc = (rep > 0 || i > 0) ? 1u : 0u;
                asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p; }"
                             ::"r"(tm), "l"(ad), "l"(bd), "r"(kIdesc), "r"(acc) : "memory");
            }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    }
    {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                         : "=r"(ok) : "r"(su32(&bar)) : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    long long t1 = clock64();
    if (tid == 0) *cyc = t1 - t0;
    if (warp < 4) {
        for (int c = 0; c < 256; c += 32) {
            uint32_t v[32];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
                "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                  "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                  "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(tm + ((uint32_t)(32 * warp) << 16) + c));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const int r = 32 * warp + (tid & 31);
            for (int j = 0; j < 32; j++) D[r * 256 + c + j] = __uint_as_float(v[j]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

int main()
{
    std::vector<uint8_t> A(128 * K), B(256 * K);
    std::vector<int> a(128 * K), b(256 * K);
    srand(7);
    const uint8_t code[3] = {0x00, 0x38, 0x40};   // e4m3 0, 1, 2
    for (int i = 0; i < 128 * K; i++) { a[i] = rand() % 2; A[i] = code[a[i]]; }
    for (int i = 0; i < 256 * K; i++) { b[i] = rand() % 3; B[i] = code[b[i]]; }
    uint8_t *dA, *dB;
    float *dD;
    long long *dc;
    cudaMalloc(&dA, A.size());
    cudaMalloc(&dB, B.size());
    cudaMalloc(&dD, 128 * 256 * 4);
    cudaMalloc(&dc, 8);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
    const int smem = 128 * K + 256 * K;
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    std::vector<float> D(128 * 256);
    for (int sw = 0; sw < 1; sw++) {   // (LBO/SBO swapped faults: illegal address)
        cudaMemset(dD, 0, 128 * 256 * 4);
        k_probe<<<1, 128, smem>>>(dA, dB, dD, sw, 1, dc);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("swap=%d error %s\n", sw, cudaGetErrorString(e)); return 1; }
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int r = 0; r < 128; r++)
            for (int n = 0; n < 256; n++) {
                int ref = 0;
                for (int k = 0; k < K; k++) ref += a[r * K + k] * b[n * K + k];
                if (D[r * 256 + n] != (float)ref) {
                    if (bad < 4) printf("  swap=%d (%d,%d) got %g want %d\n", sw, r, n, D[r * 256 + n], ref);
                    bad++;
                }
            }
        printf("layout %s: %d mismatches of %d\n", sw ? "LBO/SBO swapped" : "LBO=K-step SBO=8-row-step", bad, 128 * 256);
    }
    for (int reps : {64, 1024}) {
        k_probe<<<1, 128, smem>>>(dA, dB, dD, 0, reps, dc);
        cudaDeviceSynchronize();
        long long c;
        cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
        printf("reps %d: %lld cycles, %.1f cycles per 128x256x32 MMA (%.0f MAC/clk)\n", reps, c,
               (double)c / (reps * (K / 32)), 128.0 * 256 * 32 * reps * (K / 32) / c);
    }
    return 0;
}
