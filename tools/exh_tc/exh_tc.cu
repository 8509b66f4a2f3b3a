// ARCHIVE (not built into libpt.so): the tcgen05-summed exhaustive kernel of round 2,
// measured 3.2x SLOWER than k_exh_tiled (TMEM traffic per evaluation).
// Needs the removed driver hooks to run; kept compiling (tests/test_variants_build.py).
// exh_tc.cu -- exhaustive k-subset search (Sec. 4.3.1), fp16 filter tier
// with the across-environment SUM on the 5th-generation tensor cores.
//
// A k-subset = a (k-1)-subset "row" rho (colex rank) + a larger column l; Eq. 1 with
// the best member per environment needs, per set,
//     s(rho u {l}) = sum_e min(A_rho[e], l[l][e]),   A_rho[e] = min_{c in rho} l[c][e].
// The mins are CUDA-core work (packed f16x2 HMNMX2, exact on the fp16 values); the sum
// is a contraction with a constant 0/1 selector, so it runs on tcgen05:
//   * thread = TMEM lane = one row of the 128-row task tile; per env pair (e, e+1) it
//     forms f16x2 min(A_rho[e,e+1], B_l[e,e+1]) for the tile's 64 columns and stores the
//     64 words into a TMEM staging buffer (tcgen05.st);
//   * after a 128-thread barrier, 8 MMAs (M=128, N=8, K=16, A from TMEM, B = the
//     selector S[k][n] = (k/2 == n) in shared memory) add each set's two env terms into
//     its fp32 accumulator D[row][l] in TMEM -- one MMA row holds 8 sets x 2 envs;
//   * after the last env pair of a column tile every thread reads its 64 sums back
//     (tcgen05.ld) and runs the rigorous window test of the fp16 tier.
// B column tiles (64 envs x 64 configs, env pairs packed) stream through a 3-stage
// ring of bulk copies (TMA engine, UBLKCP); A rows are staged from a config-major fp16
// copy with 16-byte loads.  TMEM: 64 accumulator columns + 3 x 64 staging columns =
// 256 per CTA, two CTAs per SM.
#include <cuda_fp16.h>

#include <cmath>
#include <cstdint>
#include <cstdio>

#include "exh_tc.cuh"

#define KEY_BITS_TC 21   // candidate key: (row rank << 21) | column  (as exhaustive.cu)
#ifndef TC_PROBE
#define TC_PROBE 0       // debug build: per-phase clock64 totals of warp 0 of CTA 0 -> printed by the host
#endif
#if TC_PROBE
__device__ unsigned long long g_tc_probe[8];
#define TC_T(i) do { if (probe) { const long long t_ = clock64(); ph[i] += t_ - tprev; tprev = t_; } } while (0)
#else
#define TC_T(i) do { } while (0)
#endif

namespace {

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t n)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity)
{
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok)
                     : "r"(su32(b)), "r"(parity), "r"(1000000u)
                     : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void bar_sync_cta() { asm volatile("bar.sync 1, %0;" ::"n"(TC_R) : "memory"); }
__device__ __forceinline__ uint32_t hmin2(uint32_t a, uint32_t b)
{
    uint32_t r;
    asm("min.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
// ---- tcgen05 ----
__device__ __forceinline__ void tm_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tm_st32(uint32_t a, const uint32_t (&v)[32])
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(a),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]),
        "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]),
        "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
__device__ __forceinline__ void tm_ld32(uint32_t a, uint32_t (&v)[32])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(a)
        : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// D[tmem d] (+)= A[tmem a] . B[smem desc]; kind::f16, one CTA
__device__ __forceinline__ void tm_mma(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc)
{
    asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }"
                 ::"r"(d), "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
                 : "memory");
}
__device__ __forceinline__ void tm_commit(uint64_t *bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ bool elect_one()
{
    uint32_t p;
    asm volatile("{ .reg .pred e; .reg .b32 r; elect.sync r|e, 0xffffffff; selp.u32 %0, 1, 0, e; }" : "=r"(p));
    return p != 0;
}
// shared-memory matrix descriptor, K-major, no swizzle: core matrix = 8 rows x 16 B,
// LBO = byte step between the two K halves, SBO = byte step between 8-row groups
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
// instruction descriptor: D f32, A/B f16, both K-major, N = 8, M = 128
constexpr uint32_t kIdesc = (1u << 4) | ((uint32_t)(8 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);

}  // namespace

// ---------------------------------------------------------------------------
// operand layouts (built once per view)
// ---------------------------------------------------------------------------
// hC[c][e] = hT[e][c]: the SAME fp16 values, config-major (zero past C / E)
__global__ void k_cfg_major_half(const uint16_t *__restrict__ hT, int64_t E_pad, int64_t C_pad,
                                 uint16_t *__restrict__ hC)
{
    __shared__ uint16_t t[32][33];
    const int64_t c0 = (int64_t)blockIdx.x * 32, e0 = (int64_t)blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += 8) t[r][threadIdx.x] = hT[(e0 + r) * C_pad + c0 + threadIdx.x];
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += 8) hC[(c0 + r) * E_pad + e0 + threadIdx.x] = t[threadIdx.x][r];
}

// hTileP[sh][ct][pp][j] = f16x2(hT[2pp][c], hT[2pp+1][c]), c = 64 ct + 8 sh + j (zero past
// C_pad): the column tile starting at any 8-aligned config, env pairs packed, so one
// 32-pair stage is one contiguous 8 KB block
__global__ void __launch_bounds__(256) k_tile_pairs_nat(const uint16_t *__restrict__ hT, int64_t E_pad, int64_t C_pad,
                                                        int64_t n_ct, uint32_t *__restrict__ hTileP)
{
    const int64_t sct = blockIdx.x, ct = sct % n_ct, sh = sct / n_ct;
    const int64_t c0 = 64 * ct + 8 * sh;
    uint32_t *dst = hTileP + sct * (E_pad / 2) * 64;
    for (int64_t i = threadIdx.x; i < (E_pad / 2) * 64; i += blockDim.x) {
        const int64_t pp = i >> 6, c = c0 + (i & 63);
        uint32_t w = 0;
        if (c < C_pad) w = (uint32_t)hT[(2 * pp) * C_pad + c] | ((uint32_t)hT[(2 * pp + 1) * C_pad + c] << 16);
        dst[i] = w;
    }
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(TC_R, 2) k_exh_tc(const TcParams p)
{
    extern __shared__ __align__(1024) unsigned char smem[];
    uint32_t *Bs = reinterpret_cast<uint32_t *>(smem);                          // [S][32 pairs][64] f16x2
    uint4 *As = reinterpret_cast<uint4 *>(Bs + TC_S * (TC_K / 2) * TC_C);       // [pairs/4][128] (4 pairs each)
    uint16_t *Sel = reinterpret_cast<uint16_t *>(As + (p.E_pad / 8) * TC_R);    // selector, 256 B
    int *last_s = reinterpret_cast<int *>(Sel + 128);                           // [128]
    uint64_t *full = reinterpret_cast<uint64_t *>(last_s + TC_R);               // [S]
    uint64_t *mma_done = full + TC_S;                                           // [NB]
    int4 *task_s = reinterpret_cast<int4 *>(full + ((TC_S + TC_NB + 1) & ~1));   // 16-byte aligned
    int *relcnt = reinterpret_cast<int *>(task_s + 1);                          // [S]
    uint32_t *tbase_s = reinterpret_cast<uint32_t *>(relcnt + TC_S);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nkc = (int)(p.E_pad / TC_K);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(tbase_s))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int s = 0; s < TC_S; s++) {
            mbar_init(&full[s], 1);
            relcnt[s] = 0;
        }
        for (int b = 0; b < TC_NB; b++) mbar_init(&mma_done[b], TC_R / 32);   // one commit per warp
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // selector S[k][n] = (k/2 == n), stored K-major: element (n, k) at (k/8)*128 + n*16 + (k%8)*2
    {
        const int k = tid >> 3, n = tid & 7;   // 128 threads = 16 k x 8 n
        Sel[((k >> 3) * 128 + n * 16 + (k & 7) * 2) / 2] = (k >> 1) == n ? (uint16_t)0x3C00 : (uint16_t)0;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // the selector is read by the tensor core
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    const uint32_t tmem = *tbase_s;
    const uint32_t lane_base = tmem + ((uint32_t)(32 * warp) << 16);   // this warp's 32 lanes
    const uint32_t d_col = 0, stg_col = 64;                             // accumulators, staging buffers
    const uint64_t bdesc = smem_desc(su32(Sel), 128, 256);

#if TC_PROBE
    const bool probe = blockIdx.x == 0 && tid == 0;
    long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tprev = clock64();
#endif
    uint32_t steps = 0;     // B stages of all previous tasks (ring phase)
    uint32_t npair = 0;     // env pairs issued so far (staging buffer + mma_done phase)
    float bA = INFINITY, bB = INFINITY, published = INFINITY;   // group minima for U

    for (;;) {
        if (tid == 0) {
            const int ti = atomicAdd(p.task_ctr, 1);
            *task_s = ti < p.task_hi ? p.tasks[ti] : make_int4(-1, 0, 0, 0);
        }
        __syncthreads();
        const int4 tk = *task_s;
        if (tk.x < 0) break;
        const int64_t R0 = (int64_t)tk.x * TC_R;
        int32_t mem0[PT_MAXK];
        pt_unrank_colex(R0, p.m, p.C, mem0);
        const int64_t lo = tile_lo(mem0[p.m - 1]);
        const int nsteps = (tk.z - tk.y) * nkc;
        // stage g of this task (column tile tk.y + g / nkc, env chunk g % nkc): one bulk copy
        auto issue = [&](int g) {
            const int sl = (int)((steps + (uint32_t)g) % TC_S);
            const int64_t col = lo + (int64_t)(tk.y + g / nkc) * TC_C;
            const int64_t sh = (col >> 3) & 7, ct = (col - 8 * sh) >> 6;
            const uint32_t *src = p.hTileP + ((sh * p.n_ct + ct) * (p.E_pad / 2) + (int64_t)(g % nkc) * (TC_K / 2)) * TC_C;
            mbar_expect_tx(&full[sl], (TC_K / 2) * TC_C * 4);
            bulk_g2s(Bs + sl * (TC_K / 2) * TC_C, src, (TC_K / 2) * TC_C * 4, &full[sl]);
        };
        if (tid == 0)   // every thread has left the previous task: the ring is free
            for (int g = 0; g < TC_S && g < nsteps; g++) issue(g);

        // ---- A: the task's 128 rows, A_rho[e] = min over the row's members, env pairs
        //      packed (f16x2), 4 pairs per 16-byte word: As[pq][r] ----
        const int r = tid;
        {
            const int64_t R = R0 + r;
            int32_t mem[PT_MAXK];
            const bool valid = R < p.n_rows;
            if (valid) pt_unrank_colex(R, p.m, p.C, mem);
            else
                for (int u = 0; u < p.m; u++) mem[u] = 0;
            last_s[r] = valid ? mem[p.m - 1] : 0x7fffffff;
            const int64_t npq = p.E_pad / 8;
            for (int64_t pq0 = 0; pq0 < npq; pq0 += 8) {
                uint4 v[8];
#pragma unroll
                for (int t = 0; t < 8; t++)
                    v[t] = pq0 + t < npq ? *reinterpret_cast<const uint4 *>(p.hC + (int64_t)mem[0] * p.E_pad + 8 * (pq0 + t))
                                         : make_uint4(0, 0, 0, 0);
                for (int u = 1; u < p.m; u++) {
#pragma unroll
                    for (int t = 0; t < 8; t++) {
                        if (pq0 + t >= npq) continue;
                        const uint4 w = *reinterpret_cast<const uint4 *>(p.hC + (int64_t)mem[u] * p.E_pad + 8 * (pq0 + t));
                        v[t] = make_uint4(hmin2(v[t].x, w.x), hmin2(v[t].y, w.y), hmin2(v[t].z, w.z), hmin2(v[t].w, w.w));
                    }
                }
#pragma unroll
                for (int t = 0; t < 8; t++)
                    if (pq0 + t < npq) As[(pq0 + t) * TC_R + r] = valid ? v[t] : make_uint4(0, 0, 0, 0);
            }
        }
        __syncthreads();
        const int last = last_s[r];

        uint32_t slot = steps % TC_S, phase = (steps / TC_S) & 1u;
        int64_t ltile = lo + (int64_t)tk.y * TC_C;   // first column of the current tile
        for (int ct = tk.y; ct < tk.z; ct++, ltile += TC_C) {
            const unsigned Ubits = *(volatile unsigned *)p.U;   // (a stale value is a looser bound)
            for (int q = 0; q < nkc; q++) {
                TC_T(7);
                mbar_wait(&full[slot], phase);
                TC_T(0);
                const uint32_t *B = Bs + slot * (TC_K / 2) * TC_C;
                uint4 a4 = make_uint4(0, 0, 0, 0);
#pragma unroll 1
                for (int pp = 0; pp < TC_K / 2; pp++) {
                    const uint32_t b = npair % TC_NB;
                    if (npair >= TC_NB) mbar_wait(&mma_done[b], ((npair / TC_NB) - 1) & 1u);   // buffer b free
                    tm_fence_after();
                    TC_T(1);
                    if ((pp & 3) == 0) a4 = As[((int64_t)q * (TC_K / 2) / 4 + pp / 4) * TC_R + r];
                    const uint32_t a2 = (pp & 3) == 0 ? a4.x : (pp & 3) == 1 ? a4.y : (pp & 3) == 2 ? a4.z : a4.w;
                    const uint32_t *Bp = B + pp * TC_C;
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        uint32_t st[32];
#pragma unroll
                        for (int t = 0; t < 8; t++) {
                            const uint4 bv = *reinterpret_cast<const uint4 *>(Bp + 32 * h + 4 * t);   // broadcast
                            st[4 * t + 0] = hmin2(a2, bv.x);
                            st[4 * t + 1] = hmin2(a2, bv.y);
                            st[4 * t + 2] = hmin2(a2, bv.z);
                            st[4 * t + 3] = hmin2(a2, bv.w);
                        }
                        tm_st32(lane_base + stg_col + 64 * b + 32 * h, st);
                    }
                    TC_T(2);
                    tm_wait_st();
                    TC_T(3);
                    tm_fence_before();
                    bar_sync_cta();   // all 128 lanes of this env pair are in TMEM
                    tm_fence_after();
                    TC_T(4);
                    if (elect_one()) {
                        const uint32_t acc = (q | pp) != 0;
#pragma unroll
                        for (int g = 2 * warp; g < 2 * warp + 2; g++)
                            tm_mma(tmem + d_col + 8 * g, tmem + stg_col + 64 * b + 8 * g, bdesc, kIdesc, acc);
                        tm_commit(&mma_done[b]);
                    }
                    __syncwarp();
                    TC_T(5);
                    npair++;
                }
                // release the stage: the last warp to finish refills it with stage g + S
                if (lane == 0) {
                    __threadfence_block();
                    if (atomicAdd(&relcnt[slot], 1) == TC_R / 32 - 1) {
                        relcnt[slot] = 0;
                        __threadfence_block();
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        const int gn = (ct - tk.y) * nkc + q + TC_S;
                        if (gn < nsteps) issue(gn);
                    }
                }
                __syncwarp();
                if (++slot == TC_S) {
                    slot = 0;
                    phase ^= 1u;
                }
            }
            // ---- epilogue of one column tile: the last env pair's MMAs (and with them all
            //      earlier ones of every warp) complete -> 64 sums of this thread's row ----
            {
                const uint32_t lp = npair - 1;
                mbar_wait(&mma_done[lp % TC_NB], (lp / TC_NB) & 1u);
            }
            tm_fence_after();
            float acc[64];
            {
                uint32_t v[32];
                tm_ld32(lane_base + d_col, v);
                tm_wait_ld();
#pragma unroll
                for (int j = 0; j < 32; j++) acc[j] = __uint_as_float(v[j]);
                tm_ld32(lane_base + d_col + 32, v);
                tm_wait_ld();
#pragma unroll
                for (int j = 0; j < 32; j++) acc[32 + j] = __uint_as_float(v[j]);
            }
            tm_fence_before();   // the next tile's first MMA overwrites D after the next barrier
            // invalid sets (past C, or a column not above the row's largest member) -> +inf
            if (!(ltile > last && ltile + TC_C - 1 < p.C)) {
#pragma unroll
                for (int j = 0; j < 64; j++) {
                    const int64_t l = ltile + j;
                    if (!(l < p.C && l > last)) acc[j] = INFINITY;
                }
            }
            // minima of two disjoint groups (columns 0-31, 32-63) for U
            float tA = INFINITY, tB = INFINITY;
#pragma unroll
            for (int j = 0; j < 32; j++) {
                tA = fminf(tA, acc[j]);
                tB = fminf(tB, acc[32 + j]);
            }
            bA = fminf(bA, tA);
            bB = fminf(bB, tB);
            const float tau = fminf(p.tau_seed, __uint_as_float(Ubits));
            if (__fmaf_rd(fminf(tA, tB), p.c1, -p.c2) <= tau) {   // rare: some set is in the window
#pragma unroll
                for (int j = 0; j < 64; j++) {
                    const float lb = __fmaf_rd(acc[j], p.c1, -p.c2);
                    if (acc[j] < INFINITY && lb <= tau) {
                        const unsigned idx = atomicAdd(p.cand_n, 1u);
                        if (idx < p.cap) {
                            p.cand_key[idx] = ((unsigned long long)(R0 + r) << KEY_BITS_TC) |
                                              (unsigned long long)(ltile + j);
                            p.cand_s[idx] = lb;
                        }
                    }
                }
            }
            // U: the warp's 2nd-smallest group minimum (minima of disjoint set groups, so
            // the two smallest belong to distinct sets and UB(2nd) >= s_(2))
            float x1 = fminf(bA, bB), x2 = fmaxf(bA, bB);
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const float y1 = __shfl_xor_sync(0xffffffffu, x1, o);
                const float y2 = __shfl_xor_sync(0xffffffffu, x2, o);
                x2 = fminf(fmaxf(x1, y1), fminf(x2, y2));
                x1 = fminf(x1, y1);
            }
            if (lane == 0) {
                const float ub = __fmaf_ru(x2, p.c3, p.c4);
                if (ub < published) {
                    atomicMin(p.U, __float_as_uint(ub));
                    published = ub;
                }
            }
        }
        steps += nsteps;
    }
#if TC_PROBE
    if (probe)
        for (int i = 0; i < 8; i++) g_tc_probe[i] = ph[i];
#endif
    tm_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
size_t pt_exh_tc_smem(int64_t E_pad)
{
    return sizeof(uint32_t) * TC_S * (TC_K / 2) * TC_C + sizeof(uint4) * (E_pad / 8) * TC_R + 256 +
           sizeof(int) * TC_R + sizeof(uint64_t) * ((TC_S + TC_NB + 1) & ~1) + sizeof(int4) + sizeof(int) * TC_S + 16;
}

const void *pt_exh_tc_kernel() { return (const void *)k_exh_tc; }

pt_status pt_exh_tc_launch(const TcParams &p, int grid, size_t smem, cudaStream_t s)
{
    k_exh_tc<<<grid, TC_R, smem, s>>>(p);
    PT_CK(cudaGetLastError());
#if TC_PROBE
    unsigned long long h[8];
    cudaMemcpyFromSymbolAsync(h, g_tc_probe, sizeof h, 0, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    fprintf(stderr, "TC_PROBE cycles: stage-wait %llu, buf-wait %llu, min+st %llu, wait::st %llu, barrier %llu, "
                    "mma-issue %llu, epilogue/other %llu\n", h[0], h[1], h[2], h[3], h[4], h[5], h[7]);
#endif
    return PT_OK;
}

pt_status pt_exh_tc_prepare(pt_ctx *ctx, const pt_view *v)
{
    pt_view *mv = const_cast<pt_view *>(v);
    cudaStream_t s = ctx->stream;
    if (!v->hC) {
        PT_TRY(pt_dalloc(ctx, (void **)&mv->hC, sizeof(uint16_t) * v->E_pad * v->C_pad));
        k_cfg_major_half<<<dim3((unsigned)(v->C_pad / 32), (unsigned)(v->E_pad / 32)), dim3(32, 8), 0, s>>>(
            v->hT, v->E_pad, v->C_pad, mv->hC);
        ctx->stats.launches++;
        PT_CK(cudaGetLastError());
    }
    if (!v->hPair) {
        mv->n_ct = (v->C_pad + TC_C - 1) / TC_C + 1;
        PT_TRY(pt_dalloc(ctx, (void **)&mv->hPair, sizeof(uint32_t) * 8 * mv->n_ct * (v->E_pad / 2) * TC_C));
        k_tile_pairs_nat<<<(unsigned)(8 * mv->n_ct), 256, 0, s>>>(v->hT, v->E_pad, v->C_pad, mv->n_ct, mv->hPair);
        ctx->stats.launches++;
        PT_CK(cudaGetLastError());
    }
    return PT_OK;
}
