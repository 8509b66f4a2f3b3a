// tcgen05 feasibility probe for a tensor-summed (min,+) inner loop (development aid).
//   ./ubench_tc check N      : one M=128 x N x K=16 f16 MMA, A from TMEM (tcgen05.st), B = 0/1
//                              selector in smem; prints D vs the host product (layout check)
//   ./ubench_tc sttm W X     : tcgen05.st.32x32b.x{X} throughput with W warps per CTA, 148 CTAs
//   ./ubench_tc mma M N      : back-to-back tcgen05.mma (A in TMEM) issue rate, cycles per MMA
// Every mbarrier wait is bounded (a stuck wait writes a flag and exits the loop).
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cmath>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tm_alloc(uint32_t *dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(su32(dst)), "r"(ncols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tm_free(uint32_t a, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(a), "r"(ncols) : "memory");
}
__device__ __forceinline__ void st8(uint32_t a, const uint32_t *v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "r"(a), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
}
__device__ __forceinline__ void st16(uint32_t a, const uint32_t *v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 :: "r"(a), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                    "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
}
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void ld8(uint32_t a, uint32_t *v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) : "r"(a) : "memory");
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                 :: "r"(d), "r"(a), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void bar_init(uint64_t *bar, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ bool bar_wait(uint64_t *bar, uint32_t parity) {
    for (long long spin = 0; spin < 200000000LL; spin++) {
        uint32_t ok;
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(su32(bar)), "r"(parity) : "memory");
        if (ok) return true;
    }
    return false;
}
// K-major, no swizzle: core matrix = 8 rows x 16 B contiguous; LBO = K-direction step, SBO = N-direction step
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
    return (1u << 4) /* D f32 */ | (0u << 7) /* A f16 */ | (0u << 10) /* B f16 */ |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// ---------------------------------------------------------------- check
__global__ void k_check(int N, const uint16_t *A /*[128][16]*/, const uint16_t *B /*[16][N]*/, float *D /*[128][N]*/,
                        int n_mma, int *flag)
{
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(128) uint16_t Bs[16 * 32];
    const int t = threadIdx.x, w = t >> 5;
    if (w == 0) tm_alloc(&tbase, 64);
    if (t == 0) bar_init(&bar, 1);
    for (int i = t; i < 16 * N; i += 128) {
        const int k = i / N, n = i % N;
        Bs[((n >> 3) * 256 + (k >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2) / 2] = B[k * N + n];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    fence_before(); __syncthreads(); fence_after();
    const uint32_t tb = tbase, lane_off = (uint32_t)(32 * (w & 3)) << 16;
    uint32_t v[8];
    for (int j = 0; j < 8; j++) v[j] = (uint32_t)A[t * 16 + 2 * j] | ((uint32_t)A[t * 16 + 2 * j + 1] << 16);
    st8(tb + lane_off + 32, v);   // A at columns 32..39
    wait_st();
    fence_before(); __syncthreads(); fence_after();
    if (t == 0) {
        const uint64_t bd = sdesc(su32(Bs), 128, 256);
        for (int q = 0; q < n_mma; q++) mma_ts(tb, tb + 32, bd, idesc_f16(128, N), q > 0);
        commit(&bar);
    }
    __syncwarp();
    if (!bar_wait(&bar, 0)) atomicExch(flag, 1);
    fence_after();
    for (int c = 0; c < N; c += 8) {
        uint32_t r[8];
        ld8(tb + lane_off + c, r);
        wait_ld();
        for (int j = 0; j < 8; j++) D[t * N + c + j] = __uint_as_float(r[j]);
    }
    fence_before(); __syncthreads();
    if (w == 0) tm_free(tb, 64);
}

static uint16_t h(float x) { __half y = __float2half(x); uint16_t r; memcpy(&r, &y, 2); return r; }

static int run_check(int N)
{
    uint16_t hA[128 * 16], hB[16 * 32];
    float Af[128 * 16], Bf[16 * 32], want[128 * 32], got[128 * 32];
    for (int m = 0; m < 128; m++) for (int k = 0; k < 16; k++) { Af[m * 16 + k] = (float)((m * 3 + k * 5) % 17) + 0.25f * k; hA[m * 16 + k] = h(Af[m * 16 + k]); }
    for (int k = 0; k < 16; k++) for (int n = 0; n < N; n++) { Bf[k * N + n] = (N == 8 ? (k % 8 == n) : (k == n)) ? 1.f : 0.f; if (k == 3 && n == (3 % N)) Bf[k * N + n] = -1.f; hB[k * N + n] = h(Bf[k * N + n]); }
    const int n_mma = 3;
    for (int m = 0; m < 128; m++) for (int n = 0; n < N; n++) { double s = 0; for (int k = 0; k < 16; k++) s += (double)Af[m * 16 + k] * Bf[k * N + n]; want[m * N + n] = (float)(s * n_mma); }
    uint16_t *dA, *dB; float *dD; int *flag;
    CK(cudaMalloc(&dA, sizeof hA)); CK(cudaMalloc(&dB, sizeof hB)); CK(cudaMalloc(&dD, sizeof got)); CK(cudaMalloc(&flag, 4));
    CK(cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice));
    CK(cudaMemset(flag, 0, 4)); CK(cudaMemset(dD, 0xFF, sizeof got));
    k_check<<<1, 128>>>(N, dA, dB, dD, n_mma, flag);
    CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
    int f; CK(cudaMemcpy(&f, flag, 4, cudaMemcpyDeviceToHost)); CK(cudaMemcpy(got, dD, 4 * 128 * N, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int i = 0; i < 128 * N; i++) if (got[i] != want[i]) { if (bad < 12) printf("  D[%d][%d] = %g want %g\n", i / N, i % N, got[i], want[i]); bad++; }
    printf("check N=%d: timeout=%d mismatches=%d of %d\n", N, f, bad, 128 * N);
    return bad != 0 || f;
}

// ---------------------------------------------------------------- sttm throughput
template <int X>
__global__ void k_sttm(int iters, long long *cyc, uint32_t seed)
{
    __shared__ uint32_t tbase;
    const int t = threadIdx.x, w = t >> 5, nw = blockDim.x >> 5;
    if (w == 0) tm_alloc(&tbase, 512);
    fence_before(); __syncthreads(); fence_after();
    const uint32_t tb = tbase, lane_off = (uint32_t)(32 * (w & 3)) << 16;
    const uint32_t colbase = (uint32_t)((w >> 2) * (512 / ((nw + 3) / 4)));
    uint32_t v[16];
    for (int j = 0; j < 16; j++) v[j] = seed * (j + 1) + t;
    __syncthreads();
    long long c0 = clock64();
    for (int i = 0; i < iters; i++) {
        const uint32_t a = tb + lane_off + colbase + (uint32_t)((i & 1) * X);
        if (X == 8) st8(a, v); else st16(a, v);
        v[0] += 1;
    }
    wait_st();
    __syncthreads();
    long long c1 = clock64();
    if (t == 0) cyc[blockIdx.x] = c1 - c0;
    fence_before(); __syncthreads();
    if (w == 0) tm_free(tb, 512);
}

static void run_sttm(int W, int X)
{
    const int iters = 20000, grid = 148;
    long long *dc, hc[148];
    CK(cudaMalloc(&dc, sizeof hc));
    for (int rep = 0; rep < 2; rep++) {
        if (X == 8) k_sttm<8><<<grid, 32 * W>>>(iters, dc, 7); else k_sttm<16><<<grid, 32 * W>>>(iters, dc, 7);
        CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
    }
    CK(cudaMemcpy(hc, dc, sizeof hc, cudaMemcpyDeviceToHost));
    long long mx = 0; for (int i = 0; i < grid; i++) mx = hc[i] > mx ? hc[i] : mx;
    const double bytes = (double)W * iters * 32 * X * 4;
    printf("sttm W=%d x%d: %.1f B/clk/SM (%lld cycles, %d st per warp)\n", W, X, bytes / mx, mx, iters);
}

// ---------------------------------------------------------------- mma issue rate
__global__ void k_mma(int M, int N, int nacc, int n_mma, long long *cyc, int *flag)
{
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(128) uint16_t Bs[16 * 256];
    const int t = threadIdx.x, w = t >> 5;
    if (w == 0) tm_alloc(&tbase, 512);
    if (t == 0) bar_init(&bar, 1);
    for (int i = t; i < 16 * 256; i += blockDim.x) Bs[i] = 0x3C00;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    fence_before(); __syncthreads(); fence_after();
    const uint32_t tb = tbase;
    long long c0 = clock64();
    if (t == 0) {
        const uint64_t bd = sdesc(su32(Bs), 128, 256);
        const uint32_t id = idesc_f16(M, N);
        for (int q = 0; q < n_mma; q++) mma_ts(tb + (uint32_t)((q % nacc) * N), tb + 256 + (uint32_t)((q & 3) * 8), bd, id, 1);
        commit(&bar);
    }
    __syncwarp();
    if (!bar_wait(&bar, 0)) atomicExch(flag, 1);
    long long c1 = clock64();
    if (t == 0) cyc[blockIdx.x] = c1 - c0;
    fence_after();
    fence_before(); __syncthreads();
    if (w == 0) tm_free(tb, 512);
}

static void run_mma(int M, int N, int nacc)
{
    const int n_mma = 20000, grid = 148;
    long long *dc, hc[148]; int *flag, f;
    CK(cudaMalloc(&dc, sizeof hc)); CK(cudaMalloc(&flag, 4)); CK(cudaMemset(flag, 0, 4));
    for (int rep = 0; rep < 2; rep++) { k_mma<<<grid, 128>>>(M, N, nacc, n_mma, dc, flag); CK(cudaGetLastError()); CK(cudaDeviceSynchronize()); }
    CK(cudaMemcpy(hc, dc, sizeof hc, cudaMemcpyDeviceToHost)); CK(cudaMemcpy(&f, flag, 4, cudaMemcpyDeviceToHost));
    long long mx = 0; for (int i = 0; i < grid; i++) mx = hc[i] > mx ? hc[i] : mx;
    printf("mma M=%d N=%d nacc=%d: %.2f cycles per MMA (timeout=%d) -> %.0f useful adds/clk/SM for a %d x 16 A tile\n",
           M, N, nacc, (double)mx / n_mma, f, (double)M * 16 * n_mma / mx, M);
}


__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 :: "r"(d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
__global__ void k_mmass(int M, int N, int nacc, int n_mma, long long *cyc, int *flag)
{
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(128) uint16_t Bs[16 * 256];
    __shared__ __align__(128) uint16_t As[16 * 128 * 4];
    const int t = threadIdx.x, w = t >> 5;
    if (w == 0) tm_alloc(&tbase, 512);
    if (t == 0) bar_init(&bar, 1);
    for (int i = t; i < 16 * 256; i += blockDim.x) Bs[i] = 0x3C00;
    for (int i = t; i < 16 * 128 * 4; i += blockDim.x) As[i] = 0x3C00;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    fence_before(); __syncthreads(); fence_after();
    const uint32_t tb = tbase;
    long long c0 = clock64();
    if (t == 0) {
        const uint64_t bd = sdesc(su32(Bs), 128, 256);
        const uint32_t id = idesc_f16(M, N);
        for (int q = 0; q < n_mma; q++)
            mma_ss(tb + (uint32_t)((q % nacc) * N), sdesc(su32(As) + (uint32_t)((q & 3) * 4096), 128, 256), bd, id, 1);
        commit(&bar);
    }
    __syncwarp();
    if (!bar_wait(&bar, 0)) atomicExch(flag, 1);
    long long c1 = clock64();
    if (t == 0) cyc[blockIdx.x] = c1 - c0;
    fence_after();
    fence_before(); __syncthreads();
    if (w == 0) tm_free(tb, 512);
}
static void run_mmass(int M, int N, int nacc)
{
    const int n_mma = 20000, grid = 148;
    long long *dc, hc[148]; int *flag, f;
    CK(cudaMalloc(&dc, sizeof hc)); CK(cudaMalloc(&flag, 4)); CK(cudaMemset(flag, 0, 4));
    for (int rep = 0; rep < 2; rep++) { k_mmass<<<grid, 128>>>(M, N, nacc, n_mma, dc, flag); CK(cudaGetLastError()); CK(cudaDeviceSynchronize()); }
    CK(cudaMemcpy(hc, dc, sizeof hc, cudaMemcpyDeviceToHost)); CK(cudaMemcpy(&f, flag, 4, cudaMemcpyDeviceToHost));
    long long mx = 0; for (int i = 0; i < grid; i++) mx = hc[i] > mx ? hc[i] : mx;
    printf("mmass M=%d N=%d nacc=%d: %.2f cycles per MMA (timeout=%d)\n", M, N, nacc, (double)mx / n_mma, f);
}

// issue-rate probe with a warp-uniform, unrolled issue loop (one elected lane issues)
__device__ __forceinline__ void mma_ts_elect(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc) {
    asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                 :: "r"(d), "r"(a), "l"(bdesc), "r"(idesc) : "memory");
}
template <int M, int N, int NACC>
__global__ void k_mma2(int n_iter, long long *cyc, int *flag)
{
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(128) uint16_t Bs[16 * 256];
    const int t = threadIdx.x, w = t >> 5;
    if (w == 0) tm_alloc(&tbase, 512);
    if (t == 0) bar_init(&bar, 1);
    for (int i = t; i < 16 * 256; i += blockDim.x) Bs[i] = 0x3C00;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    fence_before(); __syncthreads(); fence_after();
    const uint32_t tb = __shfl_sync(0xffffffffu, tbase, 0);
    long long c0 = clock64();
    if (w == 0) {
        const uint64_t bd = sdesc(su32(Bs), 128, 256);
        constexpr uint32_t id = idesc_f16(M, N);
        for (int q = 0; q < n_iter; q++) {
#pragma unroll
            for (int u = 0; u < 8; u++) mma_ts_elect(tb + (uint32_t)((u % NACC) * N), tb + 256 + (uint32_t)((u & 3) * 8), bd, id);
        }
        if (t == 0) commit(&bar);
        __syncwarp();
    }
    if (!bar_wait(&bar, 0)) atomicExch(flag, 1);
    long long c1 = clock64();
    if (t == 0) cyc[blockIdx.x] = c1 - c0;
    fence_after();
    fence_before(); __syncthreads();
    if (w == 0) tm_free(tb, 512);
}
template <int M, int N, int NACC>
static void run_mma2()
{
    const int n_iter = 2500, grid = 148;
    long long *dc, hc[148]; int *flag, f;
    CK(cudaMalloc(&dc, sizeof hc)); CK(cudaMalloc(&flag, 4)); CK(cudaMemset(flag, 0, 4));
    for (int rep = 0; rep < 2; rep++) { k_mma2<M, N, NACC><<<grid, 128>>>(n_iter, dc, flag); CK(cudaGetLastError()); CK(cudaDeviceSynchronize()); }
    CK(cudaMemcpy(hc, dc, sizeof hc, cudaMemcpyDeviceToHost)); CK(cudaMemcpy(&f, flag, 4, cudaMemcpyDeviceToHost));
    long long mx = 0; for (int i = 0; i < grid; i++) mx = hc[i] > mx ? hc[i] : mx;
    printf("mma2 M=%d N=%d nacc=%d: %.2f cycles per MMA (timeout=%d) -> %.0f useful adds/clk/SM (%d x 16 A)\n",
           M, N, NACC, (double)mx / (8.0 * n_iter), f, (double)M * 16 * 8.0 * n_iter / mx, M);
}

// two issuing warps (warps 0 and 1), each to its own accumulators
template <int M, int N, int NW>
__global__ void k_mma3(int n_iter, long long *cyc, int *flag)
{
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(128) uint16_t Bs[16 * 256];
    const int t = threadIdx.x, w = t >> 5;
    if (w == 0) tm_alloc(&tbase, 512);
    if (t == 0) bar_init(&bar, NW);
    for (int i = t; i < 16 * 256; i += blockDim.x) Bs[i] = 0x3C00;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    fence_before(); __syncthreads(); fence_after();
    const uint32_t tb = __shfl_sync(0xffffffffu, tbase, 0);
    long long c0 = clock64();
    if (w < NW) {
        const uint64_t bd = sdesc(su32(Bs), 128, 256);
        constexpr uint32_t id = idesc_f16(M, N);
        const uint32_t dcol = tb + (uint32_t)(w * 64), acol = tb + 256 + (uint32_t)(w * 64);
        for (int q = 0; q < n_iter; q++) {
#pragma unroll
            for (int u = 0; u < 8; u++) mma_ts_elect(dcol + (uint32_t)((u & 3) * N), acol + (uint32_t)((u & 3) * 8), bd, id);
        }
        if ((t & 31) == 0) commit(&bar);
        __syncwarp();
    }
    if (!bar_wait(&bar, 0)) atomicExch(flag, 1);
    long long c1 = clock64();
    if (t == 0) cyc[blockIdx.x] = c1 - c0;
    fence_after();
    fence_before(); __syncthreads();
    if (w == 0) tm_free(tb, 512);
}
template <int M, int N, int NW>
static void run_mma3()
{
    const int n_iter = 2500, grid = 148;
    long long *dc, hc[148]; int *flag, f;
    CK(cudaMalloc(&dc, sizeof hc)); CK(cudaMalloc(&flag, 4)); CK(cudaMemset(flag, 0, 4));
    for (int rep = 0; rep < 2; rep++) { k_mma3<M, N, NW><<<grid, 128>>>(n_iter, dc, flag); CK(cudaGetLastError()); CK(cudaDeviceSynchronize()); }
    CK(cudaMemcpy(hc, dc, sizeof hc, cudaMemcpyDeviceToHost)); CK(cudaMemcpy(&f, flag, 4, cudaMemcpyDeviceToHost));
    long long mx = 0; for (int i = 0; i < grid; i++) mx = hc[i] > mx ? hc[i] : mx;
    printf("mma3 M=%d N=%d issuers=%d: %.2f cycles per MMA (timeout=%d) -> %.0f useful adds/clk/SM\n",
           M, N, NW, (double)mx / (8.0 * n_iter * NW), f, (double)M * 16 * 8.0 * n_iter * NW / mx);
}

// ---------------------------------------------------------------- accumulation accuracy
// 160 chained M=128 N=8 K=16 MMAs (A from TMEM, f16 inputs, f32 accumulate, B = pair
// selector B[k][n] = (k/2 == n)): D[m][n] = sum over steps of A[m][2n] + A[m][2n+1].
// Host compares with the exact (double) sums.
__global__ void k_acc(const uint16_t *A /*[steps][128][16]*/, int steps, float *D /*[128][8]*/, int *flag)
{
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(128) uint16_t Bs[16 * 8];
    const int t = threadIdx.x, w = t >> 5;
    if (w == 0) tm_alloc(&tbase, 32);
    if (t == 0) bar_init(&bar, 1);
    for (int i = t; i < 16 * 8; i += 128) {
        const int k = i / 8, n = i % 8;
        Bs[((k >> 3) * 128 + n * 16 + (k & 7) * 2) / 2] = (k / 2 == n) ? 0x3C00 : 0;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    fence_before(); __syncthreads(); fence_after();
    const uint32_t tb = tbase, lane_off = (uint32_t)(32 * (w & 3)) << 16;
    const uint64_t bd = sdesc(su32(Bs), 128, 256);
    for (int q = 0; q < steps; q++) {
        uint32_t v[8];
        for (int j = 0; j < 8; j++) v[j] = (uint32_t)A[(q * 128 + t) * 16 + 2 * j] | ((uint32_t)A[(q * 128 + t) * 16 + 2 * j + 1] << 16);
        st8(tb + lane_off + 16, v);
        wait_st();
        fence_before(); __syncthreads(); fence_after();
        if (t == 0) { mma_ts(tb, tb + 16, bd, idesc_f16(128, 8), q > 0); commit(&bar); }
        __syncwarp();
        if (!bar_wait(&bar, q & 1)) atomicExch(flag, 1);
        fence_after();
    }
    uint32_t r[8];
    ld8(tb + lane_off, r);
    wait_ld();
    for (int j = 0; j < 8; j++) D[t * 8 + j] = __uint_as_float(r[j]);
    fence_before(); __syncthreads();
    if (w == 0) tm_free(tb, 32);
}

static int run_acc()
{
    const int steps = 160;
    std::vector<uint16_t> hA((size_t)steps * 128 * 16);
    std::vector<double> exact(128 * 8, 0.0);
    uint64_t x = 88172645463325252ull;
    auto rnd = [&]() { x ^= x << 13; x ^= x >> 7; x ^= x << 17; return x; };
    for (int q = 0; q < steps; q++)
        for (int m = 0; m < 128; m++)
            for (int k = 0; k < 16; k++) {
                // log-uniform magnitudes over 2^-16 .. 2^4 (fp16 subnormals included)
                const double u = (double)(rnd() >> 11) / 9007199254740992.0;
                float f = (float)std::exp2(-16.0 + 20.0 * u);
                uint16_t hb = h(f);
                __half hh; memcpy(&hh, &hb, 2);
                hA[((size_t)q * 128 + m) * 16 + k] = hb;
                exact[m * 8 + k / 2] += (double)__half2float(hh);
            }
    uint16_t *dA; float *dD; int *flag, f;
    float got[128 * 8];
    CK(cudaMalloc(&dA, hA.size() * 2)); CK(cudaMalloc(&dD, sizeof got)); CK(cudaMalloc(&flag, 4));
    CK(cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice)); CK(cudaMemset(flag, 0, 4));
    k_acc<<<1, 128>>>(dA, steps, dD, flag);
    CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(got, dD, sizeof got, cudaMemcpyDeviceToHost)); CK(cudaMemcpy(&f, flag, 4, cudaMemcpyDeviceToHost));
    double worst = 0, bias = 0;
    for (int i = 0; i < 128 * 8; i++) {
        const double rel = ((double)got[i] - exact[i]) / exact[i];
        worst = std::max(worst, std::fabs(rel));
        bias += rel;
    }
    printf("acc: %d chained MMAs, worst relative error %.3e (= %.2f x 2^-24 per step), mean %.3e, timeout=%d\n",
           steps, worst, worst / steps / std::ldexp(1.0, -24), bias / (128 * 8), f);
    return 0;
}

int main(int argc, char **argv)
{
    if (argc < 2) { printf("usage: check N | sttm W X | mma M N\n"); return 2; }
    if (!strcmp(argv[1], "check")) return run_check(atoi(argv[2]));
    if (!strcmp(argv[1], "sttm")) { run_sttm(atoi(argv[2]), atoi(argv[3])); return 0; }
    if (!strcmp(argv[1], "mma")) { run_mma(atoi(argv[2]), atoi(argv[3]), argc > 4 ? atoi(argv[4]) : 1); return 0; }
    if (!strcmp(argv[1], "mmass")) { run_mmass(atoi(argv[2]), atoi(argv[3]), argc > 4 ? atoi(argv[4]) : 1); return 0; }
    if (!strcmp(argv[1], "mma2")) {
        run_mma2<128, 8, 1>(); run_mma2<128, 8, 4>(); run_mma2<128, 8, 8>(); run_mma2<128, 16, 1>(); run_mma2<128, 16, 4>();
        run_mma2<128, 64, 4>(); run_mma2<128, 256, 1>(); run_mma2<64, 8, 8>(); run_mma2<64, 16, 8>(); return 0; }
    if (!strcmp(argv[1], "mma3")) { run_mma3<128, 8, 1>(); run_mma3<128, 8, 2>(); run_mma3<128, 8, 4>(); run_mma3<128, 16, 2>(); run_mma3<128, 32, 2>(); return 0; }
    if (!strcmp(argv[1], "acc")) return run_acc();
    return 2;
}
