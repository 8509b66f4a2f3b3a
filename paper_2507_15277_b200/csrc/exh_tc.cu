// exh_tc.cu -- the threshold-count filter tier of the tiled exhaustive search
// (k_exh_tc): the (min,+) filter of P:L271-276 / Eq. 1
// rewritten as a dense 0/1 contraction on the 5th-generation tensor cores.
//
// Floor quantisation with nt uniform levels below a cap.  With thresholds
// t_j = j u (j = 1..nt) and Q(x) = u #{j : x >= t_j}:  0 <= Q(x) <= x, Q is
// non-decreasing, so Q(min_c l_c) = min_c Q(l_c), and [min_c l_c >= t] is the AND of
// the members' [l_c >= t].  For a set S = rho u {l} (rho = a (k-1)-subset "row",
// l a larger "column" index, as in k_exh_tiled):
//     s(S) = sum_e min_{c in S} l[c][e]  >=  u P(S),
//     P(S) = sum_e sum_j [A_rho[e] >= t_j] [l[l][e] >= t_j]
// a dot product of two 0/1 vectors of length K = nt E_pad.  Over a task (128 rows x
// every column above the rows) that is a GEMM: E4M3 0/1 operands (exact), fp32
// accumulation of integers (exact below 2^24), tcgen05.mma kind::f8f6f4 into tensor
// memory.  A set survives iff u P - slack <= tau, tau = an upper bound of the second
// best score (two distinct k-sets scored exactly: the local optimum of a device-side
// swap search started from greedy's k-set and its best neighbour);
// survivors are re-scored in fp64 by the common refine (k_exh_refine_top2).  u is
// chosen from tau (u = 1.5 tau / E): the filter's strength is a property of the data,
// its correctness is not -- a weak filter overflows the candidate buffer and the
// search falls back to the u8 tier.
//
// k_exh_tc: one CTA per SM (persistent, dynamic task queue), 10 warps:
//   warps 0-3  epilogue: TMEM lane quarter w, thread = row; tcgen05.ld 32 columns at
//              a time, keep the (row, column) pairs with P <= Pthr, l > last member of
//              the row, l < C (the rare survivor path appends (key, lower bound));
//   warps 4-7  A builders: row r of the task = AND of its members' bit rows (16-byte
//              loads from tcA), stored in the UMMA K-major core-matrix layout of one
//              of two A buffers (the next task's A is built during this task's MMAs);
//   warp 8     B producer: 256-column x 64-byte K stages of tcB, one 16 KB bulk copy
//              (cp.async.bulk, the TMA engine) per stage into an S-deep ring;
//   warp 9     MMA issuer (one thread): per 256-column tile, K/32 MMAs of 128 x 256 x 32
//              into one of two TMEM accumulators (2 x 256 of the 512 columns), so the
//              epilogue of a tile overlaps the MMAs of the next.
// Shared-memory layouts (no swizzle; core matrix = 8 rows x 16 bytes):
//   A: offset(r, k) = (k/16) 2048 + (r/8) 128 + (r%8) 16 + k%16   (LBO 2048, SBO 128)
//   B stage: offset(n, kk) = (n/8) 512 + (kk/16) 128 + (n%8) 16 + kk%16 (LBO 128, SBO 512)
// (layouts and the instruction descriptor verified by tools/ubench_tc8.cu).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>

#include <cooperative_groups.h>

#include "pt_internal.cuh"

namespace cgt = cooperative_groups;

#define TC_R 128        // rows per task (TMEM lanes)
#define TC_N 256        // columns per accumulator tile
#define TC_KC 64        // K bytes per B stage
#define TC_KMAX 1024    // widest K (nt E_pad): the A buffer (128 K bytes) + a ring of >= 4 B stages
#define TC_THREADS 576
// TC_DIAG=1 (build flag) compiles the PT_TC_DBG ablations and the clock64 phase profile
// into the MMA thread's loop; without it that loop carries none of their branches (the
// single issuing thread is latency-bound: two extra branches per K chunk cost 4 %)
#ifndef TC_DIAG
#define TC_DIAG 0
#endif
#define TC_FAM2 (1 << 30)   // tinfo.w: family-2 task (columns a < b, lo = 0)
#define TC_LOMASK (TC_FAM2 - 1)

namespace {

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t *b, uint32_t n)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t *b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint64_t *b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
// try_wait without a suspend-time hint: with one, the wait compiles to a NANOSLEEP.SYNCS
// loop whose wake-up added ~1.5 us to every ring round trip (the single MMA thread and
// the producer ping-pong once per 64-byte K stage)
__device__ __forceinline__ void bar_wait(uint64_t *b, uint32_t parity)
{
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok)
                     : "r"(su32(b)), "r"(parity)
                     : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// shared-memory matrix descriptor: K-major, no swizzle, LBO = byte step between core
// matrices along K, SBO = byte step between 8-row groups, bit 46 = sm_100 version
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
// instruction descriptor (built per tile), kind::f8f6f4: D f32 (bits 4-5 = 1), A = B =
// E4M3 (0), both K-major, N >> 3 at bit 17, M >> 4 at bit 24
__device__ __forceinline__ void tc_mma(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc)
{
    asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p; }" ::"r"(d),
                 "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
                 : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t *bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void tc_ld32(uint32_t a, uint32_t (&v)[32])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
        "tcgen05.wait::ld.sync.aligned;"   // same asm: no use of v[] can be scheduled before the wait
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(a)
        : "memory");
}

}  // namespace

// device constants of one search (k_tc_const)
struct TcConst {
    double u;            // threshold step (a float value: j u is exact in fp64)
    double tau;          // upper bound of s_(2) (fp64, exact scores of two distinct sets)
    float pthr;          // survivor iff P <= pthr
    float u_dn;          // u as a float
    float slack;         // fp64 rounding slack of the refine's sums (rounded up)
    int ok;              // 0: tau is not finite / u underflows -> the caller falls back
    unsigned long long lmax_bits;   // scope max of l (atomicMax on the bit pattern)
};

// ---------------------------------------------------------------------------
// tau: best-improvement swap search from greedy's k-set, entirely on the device (one
// cooperative launch, one grid barrier per move).  Every move scores all k (C - k)
// neighbours S - S[a] + b exactly in fp64 (leave-one-out minima, as swap.cu); the
// larger score of two distinct sets bounds s_(2) from above, so
//     tau = min( greedy's runner-up at step k, min over moves max(s(S), s(best neighbour)) ).
// Every CTA merges the per-CTA bests itself (same order: same move everywhere), so the
// loop needs one grid barrier per move.  Ties and the move rule only affect tau's
// tightness, never correctness.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_swap_tau(const double *__restrict__ l64, int64_t C, int64_t E_pad, int k,
                                                  const int32_t *__restrict__ S0, const double *__restrict__ seed_s2,
                                                  int iters, double *__restrict__ rs, long long *__restrict__ rw,
                                                  double *__restrict__ tau_out)
{
    cgt::grid_group grid = cgt::this_grid();
    extern __shared__ double M[];   // [k][E_pad] leave-one-out minima
    __shared__ int32_t S[PT_MAXK];
    __shared__ double red[8];
    __shared__ long long redw[8];
    __shared__ double tau_s;
    __shared__ int stop_s;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < k) S[tid] = S0[tid];
    if (tid == 0) {
        tau_s = seed_s2 ? *seed_s2 : INFINITY;
        stop_s = 0;
    }
    __syncthreads();
    for (int it = 0; it < iters; it++) {
        // leave-one-out minima and the current score (same order in every CTA)
        double part = 0.0;
        for (int64_t e = tid; e < E_pad; e += blockDim.x) {
            double v[PT_MAXK], suf[PT_MAXK + 1];
            for (int u = 0; u < k; u++) v[u] = l64[(int64_t)S[u] * E_pad + e];
            suf[k] = INFINITY;
            for (int u = k - 1; u >= 0; u--) suf[u] = fmin(suf[u + 1], v[u]);
            double pre = INFINITY;
            for (int a = 0; a < k; a++) {
                M[(int64_t)a * E_pad + e] = fmin(pre, suf[a + 1]);
                pre = fmin(pre, v[a]);
            }
            part += pre;
        }
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) red[warp] = part;
        __syncthreads();
        double cur = 0.0;
        for (int w = 0; w < 8; w++) cur += red[w];
        // this CTA's best neighbour (warp per (a, b); ties -> smallest a C + b)
        double bs = INFINITY;
        long long bw = LLONG_MAX;
        const int64_t nw = (int64_t)k * C;
        for (int64_t w = (int64_t)blockIdx.x * 8 + warp; w < nw; w += (int64_t)gridDim.x * 8) {
            const int a = (int)(w / C);
            const int64_t b = w - (int64_t)a * C;
            bool in = false;
            for (int u = 0; u < k; u++) in |= (S[u] == b);
            if (in) continue;
            const double *mr = M + (int64_t)a * E_pad, *col = l64 + b * E_pad;
            double acc = 0.0;
#pragma unroll 8
            for (int64_t e = lane; e < E_pad; e += 32) acc += fmin(mr[e], __ldg(col + e));   // loads in flight
            for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (acc < bs) {
                bs = acc;
                bw = w;
            }
        }
        __syncthreads();   // red[] reused below
        if (lane == 0) {
            red[warp] = bs;
            redw[warp] = bw;
        }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < 8; w++)
                if (red[w] < bs || (red[w] == bs && redw[w] < bw)) {
                    bs = red[w];
                    bw = redw[w];
                }
            rs[(it & 1) * gridDim.x + blockIdx.x] = bs;
            rw[(it & 1) * gridDim.x + blockIdx.x] = bw;
        }
        grid.sync();
        // merge every CTA's record (identically in every CTA) and apply the move
        double ms = INFINITY;
        long long mw = LLONG_MAX;
        for (int b = tid; b < (int)gridDim.x; b += blockDim.x) {
            const double x = __ldcg(&rs[(it & 1) * gridDim.x + b]);
            const long long y = __ldcg(&rw[(it & 1) * gridDim.x + b]);
            if (x < ms || (x == ms && y < mw)) {
                ms = x;
                mw = y;
            }
        }
        for (int o = 16; o; o >>= 1) {
            const double x = __shfl_xor_sync(0xffffffffu, ms, o);
            const long long y = __shfl_xor_sync(0xffffffffu, mw, o);
            if (x < ms || (x == ms && y < mw)) {
                ms = x;
                mw = y;
            }
        }
        __syncthreads();
        if (lane == 0) {
            red[warp] = ms;
            redw[warp] = mw;
        }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < 8; w++)
                if (red[w] < ms || (red[w] == ms && redw[w] < mw)) {
                    ms = red[w];
                    mw = redw[w];
                }
            if (ms < INFINITY) tau_s = fmin(tau_s, fmax(cur, ms));
            if (ms < cur) {
                S[mw / C] = (int32_t)(mw % C);
            } else {
                stop_s = 1;
            }
        }
        __syncthreads();
        if (stop_s) break;
    }
    if (blockIdx.x == 0 && tid == 0) *tau_out = tau_s;
}

// scope max of l (non-negative doubles order as their bit patterns)
__global__ void __launch_bounds__(256) k_tc_lmax(const double *__restrict__ l64, int64_t C, int64_t E, int64_t E_pad,
                                                TcConst *__restrict__ cst)
{
    double m = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < C * E; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i / E, e = i - c * E;
        m = fmax(m, l64[c * E_pad + e]);
    }
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(&cst->lmax_bits, (unsigned long long)__double_as_longlong(m));
}

// u, the survivor threshold and the refine's tau (one thread, no host round trip).
// The refine's fp64 sum of E_pad terms in [0, lmax] differs from the exact score by
// <= E_pad^2 lmax 2^-53 (any order); two such sums (tau's sets and the refine's) and the
// lower bound give 3 of them: slack = 4 E_pad^2 lmax 2^-52.
__global__ void k_tc_const(const double *__restrict__ tau_dev, int64_t E, int64_t E_pad, double alpha,
                           TcConst *__restrict__ cst, unsigned *__restrict__ U, unsigned long long *__restrict__ cand_n)
{
    const double tau = *tau_dev;
    const double lmax = __longlong_as_double((long long)cst->lmax_bits);
    const double slack = 4.0 * (double)E_pad * (double)E_pad * lmax * 0x1p-52 + 1e-300;
    const float uf = (float)(alpha * tau / (double)E);
    const double u = (double)uf;
    const bool ok = isfinite(tau) && u > 1e-30 && isfinite(u);
    cst->u = u;
    cst->tau = tau;
    cst->ok = ok ? 1 : 0;
    cst->u_dn = uf;
    cst->slack = __double2float_ru(slack);
    cst->pthr = ok ? __double2float_ru((tau + slack) / u * (1.0 + 1e-12)) : -1.0f;
    *U = __float_as_uint(ok ? __double2float_ru(tau + slack) : 0.0f);
    if (!ok) *cand_n = 1ull << 63;   // "not run": the refine skips, the host falls back
}

// the bit operands, k = j E_pad + e, bit = [l[c][e] >= (j+1) u] for real configs and
// environments (0 elsewhere): tcA[c][k/32] packed bits (the builders AND and expand them),
// tcB bytes (E4M3 1.0 = 0x38) in the B-stage layout.  Thread = (config, k): a warp holds 32
// consecutive k of one threshold (E_pad % 64 == 0), its ballot is the packed word.
__global__ void __launch_bounds__(256) k_tc_build(const double *__restrict__ l64, int64_t C, int64_t E, int64_t E_pad,
                                                 int K, int64_t n_cfg, const TcConst *__restrict__ cst,
                                                 uint32_t *__restrict__ A, uint8_t *__restrict__ B)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // n_cfg K is a multiple of 32
    const int64_t c = i / K;
    const int k = (int)(i - c * K);
    const int j = k / (int)E_pad, e = k - j * (int)E_pad;
    const bool on = i < n_cfg * K && cst->ok && c < C && e < E && l64[c * E_pad + e] >= (double)(j + 1) * cst->u;
    const uint32_t word = __ballot_sync(0xffffffffu, on);
    if (i >= n_cfg * K) return;
    if ((threadIdx.x & 31) == 0) A[i >> 5] = word;
    const int64_t n_grp = n_cfg / 8;
    const int kc = k / TC_KC, kk = k % TC_KC;
    B[((int64_t)kc * n_grp + c / 8) * (8 * TC_KC) + (kk / 16) * 128 + (c % 8) * 16 + kk % 16] = on ? 0x38 : 0;
}

// 8 packed bits -> 8 bytes of E4M3 (1.0 = 0x38 where the bit is set): per nibble, the
// multiply by 0x00204081 places bit j at bit 8j with no overlapping partial products
__device__ __forceinline__ uint32_t expand4(uint32_t nib)
{
    return ((nib * 0x00204081u) & 0x01010101u) * 0x38u;
}
// colex unranking for the builders (pt_unrank_colex's answer; its binary searches cost
// ~7 K cycles per 256-row task on the critical path of short tasks): the largest c with
// C(c, u+1) <= r from a float estimate (sqrt / cbrt), corrected exactly in int64
__device__ __forceinline__ void unrank_fast(int64_t R, int m, int64_t n, int32_t *out)
{
    int64_t r = R;
    for (int u = m - 1; u >= 0; u--) {
        int64_t c;
        if (u == 0) c = r;
        else if (u == 1) c = (int64_t)((1.0f + sqrtf(1.0f + 8.0f * (float)r)) * 0.5f);
        else if (u == 2) c = (int64_t)cbrtf(6.0f * (float)r) + 1;
        else c = n - 1;
        c = min(max(c, (int64_t)u), n - 1);
        while (c > u && pt_binom(c, u + 1) > r) c--;
        while (c + 1 <= n - 1 && pt_binom(c + 1, u + 1) <= r) c++;
        out[u] = (int32_t)c;
        r -= pt_binom(c, u + 1);
    }
}

__device__ __forceinline__ uint4 expand16(uint32_t bits16)
{
    return make_uint4(expand4(bits16 & 15u), expand4((bits16 >> 4) & 15u), expand4((bits16 >> 8) & 15u),
                      expand4((bits16 >> 12) & 15u));
}

struct TcParams {
    int64_t C, n_rows, n_grp;
    int m, K, S, AB;   // S = B stages, AB = A buffers (1 or 2)
    int split;         // k = 3 two-family task list: task .w = family (1: rows (a,b) b < h, 2: rows (b,c) b >= h)
    int64_t n_rows2;   // family-2 rows (the family-1 row count is n_rows)
    const int4 *tasks;
    int task_hi;
    int *task_ctr;
    const uint32_t *A;   // packed bits [n_cfg][K/32]
    const uint8_t *B;
    const TcConst *cst;
    unsigned long long *cand_key;
    float *cand_s;
    unsigned long long *cand_n;
    unsigned cap;
    int dbg;   // development knob PT_TC_DBG, diagnostics only -- results may be wrong with bits
               // 0-4, 6 set (bit 0: the epilogue skips its TMEM reads, 1: no MMAs, 2: the MMA
               // thread does not wait for A, 3: the builders skip their stores, 4: no B copies,
               // 5: clock64 phase profile of CTA 0, 6: no tcgen05 fence after the B wait)
};

// warp roles (TC_THREADS = 18 warps)
#define TC_EPI_WARPS 8      // 0-7: epilogue
#define TC_BLD_WARPS 8      // 8-15: A builders
#define TC_PROD_WARP 16
#define TC_MMA_WARP 17

// One CTA per SM (persistent, dynamic task queue).  H = row halves per task: a task is
// 128 H rows x its column tiles of N = 256 / H columns; every B stage (N columns x 64 K
// bytes) feeds H MMAs of 128 x N x 32 per 32 K bytes, one per row half, so the B bytes
// streamed per MMA flop shrink by H (H = 2 is the default: the bulk-copy stream of B,
// not the tensor core, bounds H = 1).  Tensor memory: two accumulator buffers x H halves
// x N columns = 512 columns.  The A operand is ONE buffer (128 H rows x K) cut into
// K-chunks of 64 bytes: chunk kc of task t+1 is built as soon as the last tile of task t
// has consumed chunk kc, so the next task's A streams in behind the current task's last
// tile and the rest of shared memory goes to a deep B ring.  The last tile of a task is
// trimmed to N = round_up(columns, 16).
template <int H>
__global__ void __launch_bounds__(TC_THREADS, 1) k_exh_tc(const TcParams p)
{
    constexpr int N = TC_N / H;                 // columns per tile
    constexpr int ROWS = TC_R * H;              // rows per task
    constexpr int BSUB = N * TC_KC;             // one 64-byte K chunk of a B tile
    constexpr int BST = BSUB;                   // one B stage
    constexpr int ACH = ROWS * TC_KC;           // one A chunk (all rows, 64 K bytes)
    extern __shared__ __align__(128) uint8_t smem[];
    const int K = p.K, S = p.S, AB = p.AB, nkc = K / TC_KC;
    // builder groups: with H = 1 and two A buffers, two groups of 4 warps build alternate
    // tasks (group g: tasks t = g mod 2, A buffer g), so each has two tasks' time per task
    const int G = (H == 1 && AB == 2) ? 2 : 1;
    uint8_t *Abuf = smem;                                           // A [AB][nkc][ACH]
    uint8_t *Bbuf = smem + (size_t)AB * nkc * ACH;                  // B ring [S][BST]
    int4 *tinfo = reinterpret_cast<int4 *>(Bbuf + (size_t)S * BST);   // [2] (first row / 128, u0, u1, lo | family)
    uint64_t *bars = reinterpret_cast<uint64_t *>(tinfo + 2);
    uint64_t *t_full = bars, *t_empty = bars + 2, *acc_full = bars + 4, *acc_empty = bars + 6;
    uint64_t *a_full = bars + 8, *a_empty = a_full + AB * nkc;     // [AB][nkc] each
    uint64_t *b_full = a_empty + AB * nkc, *b_empty = b_full + S;
    uint32_t *tmem_s = reinterpret_cast<uint32_t *>(b_empty + S);
    int *bcast = reinterpret_cast<int *>(tmem_s + 1);               // [2] + each group's prefetched next index

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (!p.cst->ok) return;   // tau unusable (k_tc_const flagged the search as not run)
    if (tid == 0) {
        for (int i = 0; i < 2; i++) {
            bar_init(&t_full[i], TC_BLD_WARPS * 32 / G);
            bar_init(&t_empty[i], 1 + 1 + TC_EPI_WARPS);   // producer, MMA, epilogue warps
            bar_init(&acc_full[i], 1);
            bar_init(&acc_empty[i], TC_EPI_WARPS);
        }
        for (int c = 0; c < AB * nkc; c++) {
            bar_init(&a_full[c], TC_BLD_WARPS * 32 / G);
            bar_init(&a_empty[c], 1);
        }
        for (int q = 0; q < S; q++) {
            bar_init(&b_full[q], 1);
            bar_init(&b_empty[q], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tmem_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_s;
    const int m = p.m;

    if (warp < TC_EPI_WARPS) {
        // ---------------- epilogue: warp = (lane quarter, row half or column half) ----------------
        const int quarter = warp & 3, sel = warp >> 2;
        const int h = H == 2 ? sel : 0;                   // row half whose accumulator it reads
        const int q0 = H == 2 ? 0 : sel * 4;              // first 32-column chunk
        const int r = 128 * h + 32 * quarter + lane;      // row within the task
        const float pthr = p.cst->pthr, u_dn = p.cst->u_dn, slk = p.cst->slack;
        const uint32_t lane_base = tmem + ((uint32_t)(32 * quarter) << 16) + h * N;
        uint32_t tcnt = 0;
        int done = 0;   // bit g: builder group g posted its last task
        for (int t = 0;; t++) {
            const int slot = t & 1;
            if (done >> slot & 1) continue;
            bar_wait(&t_full[slot], (t >> 1) & 1);
            const int4 ti = tinfo[slot];
            __syncwarp();
            if (lane == 0) bar_arrive(&t_empty[slot]);
            if (ti.x < 0) {   // this builder group is done (with one group: every group)
                done |= 1 << slot;
                if (G == 1 || done == 3) break;
                continue;
            }
            const int64_t R = (int64_t)ti.x * TC_R + r;
            // the row's own members (decoded here: no per-row smem table).  Family 1 (and
            // the single decomposition): columns l in (lastr, C), key (R, l).  Family 2: row
            // (bb, cc), columns a in [0, bb), key (colex rank of (a, bb), cc).
            const bool fam2 = (ti.w & TC_FAM2) != 0;
            int lastr = 0x7fffffff, bb = 0, cc = 0;
            if (R < (fam2 ? p.n_rows2 : p.n_rows)) {
                int32_t mem[PT_MAXK];
                unrank_fast(R, m, p.C, mem);
                if (fam2) {
                    bb = (int)(p.C - 1 - mem[1]);
                    cc = (int)(p.C - 1 - mem[0]);
                } else {
                    lastr = mem[m - 1];
                }
            }
            const int64_t cmin = fam2 ? -1 : lastr, cend = fam2 ? bb : p.C;   // valid: cmin < l < cend
            for (int u = ti.y; u < ti.z; u++, tcnt++) {
                const int buf = tcnt & 1;
                const int64_t col0 = (int64_t)(ti.w & TC_LOMASK) + (int64_t)u * N;
                const int ncols = (int)min((int64_t)N, p.C - col0);
                bar_wait(&acc_full[buf], (tcnt >> 1) & 1);
                tc_fence_after();
#pragma unroll 1
                for (int q = q0; q < q0 + 4 && q * 32 < ncols && !(p.dbg & 1); q++) {
                    uint32_t v[32];
                    tc_ld32(lane_base + buf * 256 + q * 32, v);
                    const int64_t cb = col0 + q * 32;
                    float w[16];
                    if (cb > cmin && cb + 31 < cend) {   // every column valid: a 32-wide min tree
#pragma unroll
                        for (int j = 0; j < 16; j++) w[j] = fminf(__uint_as_float(v[j]), __uint_as_float(v[j + 16]));
                    } else {                             // row start / range end: mask first
#pragma unroll
                        for (int j = 0; j < 16; j++) {
                            const float a = (cb + j > cmin && cb + j < cend) ? __uint_as_float(v[j]) : INFINITY;
                            const float b = (cb + j + 16 > cmin && cb + j + 16 < cend) ? __uint_as_float(v[j + 16]) : INFINITY;
                            w[j] = fminf(a, b);
                        }
                    }
#pragma unroll
                    for (int j = 0; j < 8; j++) w[j] = fminf(w[j], w[j + 8]);
#pragma unroll
                    for (int j = 0; j < 4; j++) w[j] = fminf(w[j], w[j + 4]);
                    const float mn = fminf(fminf(w[0], w[2]), fminf(w[1], w[3]));
                    if (mn <= pthr) {   // rare: the window, then validity
                        for (int j = 0; j < 32; j++) {
                            const float P = __uint_as_float(v[j]);
                            const int64_t l = cb + j;
                            if (P <= pthr && l > cmin && l < cend) {
                                const unsigned long long idx = atomicAdd(p.cand_n, 1ull);
                                if (idx < p.cap) {
                                    // family 2: the set {l, bb, cc} as (colex rank of (l, bb), cc)
                                    const unsigned long long rk = fam2 ? (unsigned long long)bb * (bb - 1) / 2 + l
                                                                       : (unsigned long long)R;
                                    const unsigned long long col = fam2 ? (unsigned long long)cc : (unsigned long long)l;
                                    p.cand_key[idx] = (rk << KEY_BITS) | col;
                                    p.cand_s[idx] = __fmaf_rd(P, u_dn, -slk);
                                }
                            }
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) bar_arrive(&acc_empty[buf]);
            }
        }
    } else if (warp < TC_EPI_WARPS + TC_BLD_WARPS) {
        // ---------------- A builders: thread = (row, share of each chunk) ----------------
        const int nthr = TC_BLD_WARPS * 32 / G;                   // threads per group
        const int g = (tid - TC_EPI_WARPS * 32) / nthr;           // this thread's group
        const int bt = tid - TC_EPI_WARPS * 32 - g * nthr;        // thread within the group
        const int row = bt % ROWS, part = bt / ROWS;               // part: the thread's share of a row
        const int wpc = 2 * ROWS / nthr;                           // words of a chunk per thread (1 or 2)
        const bool prof = (p.dbg & 32) && blockIdx.x == 0 && bt == 0 && g == 0;
        long long bc[6] = {0, 0, 0, 0, 0, 0};   // t_empty, fetch, unrank, loads, a_empty waits, stores
        long long b0 = clock64();
        auto blap = [&](int i) {
            if (prof) {
                const long long b1 = clock64();
                bc[i] += b1 - b0;
                b0 = b1;
            }
        };
        for (int n = 0;; n++) {
            const int t = n * G + g;
            const int slot = t & 1;
            bar_wait(&t_empty[slot], ((t >> 1) & 1) ^ 1);
            blap(0);
            if (bt == 0) {   // this task's index was fetched one task ahead (off the critical path)
                bcast[slot] = n == 0 ? atomicAdd(p.task_ctr, 1) : bcast[2 + g];
                bcast[2 + g] = atomicAdd(p.task_ctr, 1);
            }
            named_sync(1 + g, nthr);
            const int ti = bcast[slot];
            blap(1);
            if (ti >= p.task_hi) {
                if (bt == 0) tinfo[slot] = make_int4(-1, 0, 0, 0);
                bar_arrive(&t_full[slot]);
                if (prof)
                    printf("[k_exh_tc builder 0, CTA 0] %d tasks, cycles: t_empty %lld fetch %lld unrank %lld loads %lld "
                           "a_empty %lld stores %lld\n", t, bc[0], bc[1], bc[2], bc[3], bc[4], bc[5]);
                break;
            }
            const int4 tk = p.tasks[ti];
            const bool fam2 = p.split && tk.w == 2;
            const int64_t R0 = (int64_t)tk.x * ROWS;
            const int64_t R = R0 + row;
            const bool valid = R < (fam2 ? p.n_rows2 : p.n_rows);
            int32_t mem[PT_MAXK];
            if (valid) unrank_fast(R, m, p.C, mem);
            else for (int u = 0; u < m; u++) mem[u] = 0;
            if (bt == 0)   // row 0 = R0; family 2 starts at column 0
                tinfo[slot] = make_int4((int)(R0 / TC_R), tk.y, tk.z, fam2 ? TC_FAM2 : (int)tile_lo(mem[m - 1]));
            if (fam2 && valid) {   // rows (x, y) stand for the pair (b, c) = (C-1-y, C-1-x)
                const int32_t x = mem[0];
                mem[0] = (int32_t)(p.C - 1 - mem[1]);
                mem[1] = (int32_t)(p.C - 1 - x);
            }
            bar_arrive(&t_full[slot]);
            blap(2);
            // the row's packed bits: per chunk c, words 2c and 2c+1 (H = 2: this thread both;
            // H = 1: word 2c + part), ANDed over the members (= the bits of the row's min)
            const int W = K / 32;
            const uint32_t *r0 = p.A + (int64_t)mem[0] * W;
            const uint32_t *r1 = p.A + (int64_t)mem[m > 1 ? 1 : 0] * W;
            const uint32_t *r2 = p.A + (int64_t)mem[m > 2 ? 2 : 0] * W;
            uint32_t wv[TC_KMAX / TC_KC][2];
#pragma unroll
            for (int c = 0; c < TC_KMAX / TC_KC; c++) {
                if (c < nkc) {
#pragma unroll
                    for (int i = 0; i < 2; i++) {
                        if (i >= wpc) break;
                        const int wi = 2 * c + (wpc == 2 ? i : part);
                        uint32_t x = __ldg(r0 + wi);
                        if (m > 1) x &= __ldg(r1 + wi);
                        if (m > 2) x &= __ldg(r2 + wi);
                        wv[c][i] = valid ? x : 0u;
                    }
                }
            }
            if (prof) {   // force the loads to complete before the lap (profiling only)
                uint32_t z = 0;
                for (int c = 0; c < TC_KMAX / TC_KC; c++)
                    if (c < nkc) z ^= wv[c][0];
                if (z == 0x12345678u) bcast[slot] = 0;
            }
            blap(3);
            const int hr = row >> 7, rr = row & 127;     // row half, row within it
            uint8_t *dst = Abuf + (size_t)hr * (TC_R * TC_KC) + (rr >> 3) * 128 + (rr & 7) * 16;
            // A buffer t % AB: with two, task t+1's A is built while task t's tiles run
            const int ab = AB == 2 ? (t & 1) : 0;
            const uint32_t aph = (uint32_t)((AB == 2 ? t >> 1 : t) & 1);   // this buffer's use parity
#pragma unroll
            for (int c = 0; c < TC_KMAX / TC_KC; c++) {
                if (c >= nkc) break;
                bar_wait(&a_empty[ab * nkc + c], aph ^ 1);   // the buffer's previous task is done with chunk c
                blap(4);
                uint8_t *cd = dst + (size_t)(ab * nkc + c) * ACH;
#pragma unroll
                for (int i = 0; i < 2; i++) {
                    if (i >= wpc || (p.dbg & 8)) break;
                    const int piece = 2 * (wpc == 2 ? i : part);   // 16-byte K piece within the chunk
                    *reinterpret_cast<uint4 *>(cd + piece * (TC_R * 16)) = expand16(wv[c][i] & 0xffffu);
                    *reinterpret_cast<uint4 *>(cd + (piece + 1) * (TC_R * 16)) = expand16(wv[c][i] >> 16);
                }
                if (AB == 1) {   // single buffer: hand each chunk over as soon as it is written
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor core
                    bar_arrive(&a_full[ab * nkc + c]);
                }
                blap(5);
            }
            if (AB == 2) {   // the buffer is built a task ahead: one proxy fence for all chunks
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                for (int c = 0; c < nkc; c++) bar_arrive(&a_full[ab * nkc + c]);
            }
        }
    } else if (warp == TC_PROD_WARP) {
        // ---------------- B producer ----------------
        if (lane == 0) {
            int st = 0;
            uint32_t ph = 0;   // ring position and the phase parity of its current lap
            const int64_t kstride = p.n_grp * (8 * TC_KC);
            int done = 0;   // bit g: builder group g posted its last task
            for (int t = 0;; t++) {
                const int slot = t & 1;
                if (done >> slot & 1) continue;
                bar_wait(&t_full[slot], (t >> 1) & 1);
                const int4 ti = tinfo[slot];
                bar_arrive(&t_empty[slot]);
                if (ti.x < 0) {
                    done |= 1 << slot;
                    if (G == 1 || done == 3) break;
                    continue;
                }
                for (int u = ti.y; u < ti.z; u++) {
                    const int64_t col0 = (int64_t)(ti.w & TC_LOMASK) + (int64_t)u * N;
                    const int n_eff = (int)min((int64_t)N, (p.C - col0 + 15) & ~(int64_t)15);
                    const uint32_t bytes = (uint32_t)n_eff * TC_KC;
                    const uint8_t *src = p.B + (col0 >> 3) * (8 * TC_KC);
                    for (int kc = 0; kc < nkc; kc++, src += kstride) {
                        bar_wait(&b_empty[st], ph ^ 1);
                        if (p.dbg & 16) {
                            bar_arrive(&b_full[st]);
                        } else {
                            bar_expect_tx(&b_full[st], bytes);
                            bulk_g2s(Bbuf + (size_t)st * BST, src, bytes, &b_full[st]);
                        }
                        if (++st == S) {
                            st = 0;
                            ph ^= 1;
                        }
                    }
                }
            }
        }
        __syncwarp();
    } else {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            // one thread issues everything: keep its loop lean (no division, descriptors
            // advanced by adding (byte offset >> 4) to their 14-bit address field)
            int st = 0;
            uint32_t ph = 0, tcnt = 0;
            const uint64_t adesc0 = sdesc(su32(Abuf), TC_R * 16, 128);
            const uint64_t bdesc0 = sdesc(su32(Bbuf), 128, 8 * TC_KC);
            constexpr uint64_t A_HALF = (uint64_t)TC_R * TC_KC >> 4;   // the second row half of a chunk
            constexpr uint64_t A_CH = (uint64_t)ACH >> 4;                // one A chunk
            constexpr uint64_t A_K32 = (uint64_t)2 * TC_R * 16 >> 4;     // 32 bytes of K in A
            constexpr uint64_t B_ST = (uint64_t)BST >> 4;                // one B stage
            constexpr uint64_t B_K32 = 256 >> 4;                         // 32 bytes of K in B
            const bool prof = TC_DIAG && (p.dbg & 32) && blockIdx.x == 0;
            const int dbg = TC_DIAG ? p.dbg : 0;
            long long cyc[6] = {0, 0, 0, 0, 0, 0};   // t_full, acc_empty, a_full, b_full, mma, commit
            long long c0 = clock64();
            auto lap = [&](int i) {
                if (prof) {
                    const long long c1 = clock64();
                    cyc[i] += c1 - c0;
                    c0 = c1;
                }
            };
            int done = 0;   // bit g: builder group g posted its last task
            for (int t = 0;; t++) {
                const int slot = t & 1;
                if (done >> slot & 1) continue;
                bar_wait(&t_full[slot], (t >> 1) & 1);
                lap(0);
                const int4 ti = tinfo[slot];
                bar_arrive(&t_empty[slot]);
                if (ti.x < 0) {
                    done |= 1 << slot;
                    if (G == 1 || done == 3) break;
                    continue;
                }
                for (int u = ti.y; u < ti.z; u++, tcnt++) {
                    const int buf = tcnt & 1;
                    const int64_t col0 = (int64_t)(ti.w & TC_LOMASK) + (int64_t)u * N;
                    const int n_eff = (int)min((int64_t)N, (p.C - col0 + 15) & ~(int64_t)15);
                    const uint32_t idesc = (1u << 4) | ((uint32_t)(n_eff >> 3) << 17) | ((uint32_t)(TC_R >> 4) << 24);
                    const bool first = u == ti.y, lastu = u == ti.z - 1;
                    bar_wait(&acc_empty[buf], ((tcnt >> 1) & 1) ^ 1);
                    tc_fence_after();
                    lap(1);
                    const uint32_t d = tmem + buf * 256;
                    const int ab = AB == 2 ? (t & 1) : 0;
                    const uint32_t aph = (uint32_t)((AB == 2 ? t >> 1 : t) & 1);
                    // the K loop, specialised on (first tile of the task, last tile of the task):
                    // the single issuing thread is latency-bound, so no per-chunk branches on them
                    auto kloop = [&](auto FIRST, auto LAST) {
                        uint64_t ad = adesc0 + (uint64_t)ab * nkc * A_CH;
                        uint64_t bd = bdesc0 + (uint64_t)st * B_ST;
                        for (int kc = 0; kc < nkc; kc++, ad += A_CH) {
                            if (decltype(FIRST)::value && !(dbg & 4)) bar_wait(&a_full[ab * nkc + kc], aph);
                            lap(2);
                            bar_wait(&b_full[st], ph);
                            if (!(dbg & 64)) tc_fence_after();   // (bit 6: diagnostics only)
                            lap(3);
                            if (!(dbg & 2)) {
#pragma unroll
                                for (int hh = 0; hh < H; hh++) {
                                    tc_mma(d + hh * N, ad + hh * A_HALF, bd, idesc, kc ? 1u : 0u);
                                    tc_mma(d + hh * N, ad + hh * A_HALF + A_K32, bd + B_K32, idesc, 1u);
                                }
                            }
                            lap(4);
                            tc_commit(&b_empty[st]);
                            if (decltype(LAST)::value) tc_commit(&a_empty[ab * nkc + kc]);   // the task's last use of chunk kc
                            lap(5);
                            if (++st == S) {
                                st = 0;
                                ph ^= 1;
                                bd = bdesc0;
                            } else {
                                bd += B_ST;
                            }
                        }
                    };
                    if (first && lastu) kloop(std::true_type(), std::true_type());
                    else if (first) kloop(std::true_type(), std::false_type());
                    else if (lastu) kloop(std::false_type(), std::true_type());
                    else kloop(std::false_type(), std::false_type());
                    tc_commit(&acc_full[buf]);
                    lap(5);
                }
            }
            if (prof)
                printf("[k_exh_tc MMA thread, CTA 0] cycles: t_full %lld acc_empty %lld a_full %lld b_full %lld mma %lld commit %lld\n",
                       cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cyc[5]);
        }
        __syncwarp();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static size_t tc_smem(int K, int S, int H, int AB)
{
    return (size_t)AB * TC_R * H * K + (size_t)S * (TC_N / H) * TC_KC + sizeof(int4) * 2 +
           sizeof(uint64_t) * (8 + 2 * AB * (K / TC_KC) + 2 * S) + 48;
}

// row halves per task (PT_TC_H = 1 or 2, default 1); the caller's task list has 128 H rows
// and 256 / H columns per tile
int pt_tc_halves()
{
    const char *e = getenv("PT_TC_H");
    return (e && atoi(e) == 2) ? 2 : 1;
}

pt_status pt_exh_tc_enqueue(pt_ctx *ctx, const pt_view *v, const pt_tc_args &a, int *nt_out)
{
    cudaStream_t s = ctx->stream;
    const int m = a.k - 1;
    if (m < 1 || m > 3 || v->C >= (1 << KEY_BITS) || v->E_pad % TC_KC != 0) return PT_EINVAL;
    // nt thresholds (PT_TC_NT, default 2), as many as fit TC_KMAX
    // (read per call: the tests vary them in one process)
    const int nt_env = getenv("PT_TC_NT") ? atoi(getenv("PT_TC_NT")) : 2;
    const double alpha = getenv("PT_TC_ALPHA") ? atof(getenv("PT_TC_ALPHA")) : 1.5;
    const int nt = (int)std::min<int64_t>(std::max(nt_env, 1), TC_KMAX / v->E_pad);
    if (nt < 1) return PT_EINVAL;
    const int K = nt * (int)v->E_pad;
    const size_t smem_limit = 227 * 1024 - 1024;   // margin for static shared memory
    const int H = a.halves;
    // two A buffers when they fit beside a B ring of >= 4 stages (PT_TC_AB=1 forces one);
    // then as many 64-byte K stages as fit (up to 16)
    int AB = (getenv("PT_TC_AB") && atoi(getenv("PT_TC_AB")) == 1) ? 1 : 2;
    if (AB == 2 && tc_smem(K, 4, H, 2) > smem_limit) AB = 1;
    int S = 16;
    while (S > 2 && tc_smem(K, S, H, AB) > smem_limit) S--;
    if (tc_smem(K, S, H, AB) > smem_limit) return PT_EINVAL;
    // per-call operands (the thresholds follow tau)
    pt_view *mv = const_cast<pt_view *>(v);
    const int64_t n_cfg = pt_round_up(v->C + TC_N + 8, 8);
    if (!mv->tcConst) PT_TRY(pt_dalloc(ctx, &mv->tcConst, sizeof(TcConst)));
    if (mv->tc_ncfg != n_cfg || mv->tc_K != K) {
        pt_dfree(ctx, mv->tcA);
        pt_dfree(ctx, mv->tcB);
        mv->tcA = mv->tcB = nullptr;
        PT_TRY(pt_dalloc(ctx, (void **)&mv->tcA, (size_t)n_cfg * K / 8));
        PT_TRY(pt_dalloc(ctx, (void **)&mv->tcB, (size_t)n_cfg * K));
        mv->tc_ncfg = n_cfg;
        mv->tc_K = K;
    }
    TcConst *cst = (TcConst *)mv->tcConst;
    // tau: device swap search from greedy's k-set
    static std::mutex mu;
    static std::map<std::tuple<int, size_t>, int> occ_cache;
    const size_t sw_smem = sizeof(double) * a.k * v->E_pad;
    int occ = 0;
    {
        std::lock_guard<std::mutex> g(mu);
        auto key = std::make_tuple(ctx->dev, sw_smem);
        auto it = occ_cache.find(key);
        if (it == occ_cache.end()) {
            PT_TRY(pt_smem_optin(ctx, (const void *)k_swap_tau));
            PT_TRY(pt_smem_optin(ctx, (const void *)k_exh_tc<1>));
            PT_TRY(pt_smem_optin(ctx, (const void *)k_exh_tc<2>));
            PT_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_swap_tau, 256, sw_smem));
            occ_cache[key] = occ;
        } else {
            occ = it->second;
        }
    }
    if (occ < 1) return PT_EINVAL;
    const int nblk = ctx->num_sms;
    double *rs = a.swap_rs;
    long long *rw = a.swap_rw;
    double *tau_dev = a.tau_dev;
    {
        const double *l64 = v->l64;
        int64_t CC = v->C, EE = v->E_pad;
        int kk = a.k, iters = getenv("PT_TC_SWAP_ITERS") ? std::max(1, atoi(getenv("PT_TC_SWAP_ITERS"))) : 16;
        const int32_t *S0 = a.d_S0;
        const double *seed = a.d_seed_s2;
        void *args[] = {(void *)&l64, (void *)&CC, (void *)&EE, (void *)&kk, (void *)&S0, (void *)&seed,
                        (void *)&iters, (void *)&rs, (void *)&rw, (void *)&tau_dev};
        PT_CK(cudaLaunchCooperativeKernel((void *)k_swap_tau, dim3(nblk), dim3(256), args, sw_smem, s));
    }
    PT_CK(cudaMemsetAsync(&cst->lmax_bits, 0, sizeof(unsigned long long), s));
    const int64_t ne = v->C * v->E;
    const unsigned gmax = (unsigned)std::max<int64_t>(1, std::min<int64_t>((ne + 255) / 256, 4L * ctx->num_sms));
    k_tc_lmax<<<gmax, 256, 0, s>>>(v->l64, v->C, v->E, v->E_pad, cst);
    k_tc_const<<<1, 1, 0, s>>>(tau_dev, v->E, v->E_pad, alpha, cst, a.U, a.cand_n);
    const int64_t nb = n_cfg * K;
    k_tc_build<<<(unsigned)((nb + 255) / 256), 256, 0, s>>>(v->l64, v->C, v->E, v->E_pad, K, n_cfg, cst,
                                                             (uint32_t *)mv->tcA, mv->tcB);
    ctx->stats.launches += 4;
    PT_CK(cudaGetLastError());
    TcParams p;
    p.C = v->C;
    p.n_rows = a.split ? pt_binom(v->C / 2, 2) : pt_binom(v->C, m);   // (split: the family-1 rows)
    p.n_grp = n_cfg / 8;
    p.m = m;
    p.K = K;
    p.S = S;
    p.AB = AB;
    p.split = a.split ? 1 : 0;
    p.n_rows2 = a.split ? pt_binom(v->C - v->C / 2, 2) : 0;
    p.tasks = a.tasks;
    p.task_hi = a.tb;
    p.task_ctr = a.ctr;
    p.A = (const uint32_t *)mv->tcA;
    p.B = mv->tcB;
    p.cst = cst;
    p.cand_key = a.cand_key;
    p.cand_s = a.cand_s;
    p.cand_n = a.cand_n;
    p.cap = a.cap;
    p.dbg = getenv("PT_TC_DBG") ? atoi(getenv("PT_TC_DBG")) : 0;
    const size_t smem = tc_smem(K, S, H, AB);
    // an empty shard still runs (one CTA that finds no task): whether the tc tier answers or
    // falls back is decided on the device from tau, identically on every rank, and all
    // ranks must scan the same tier's task list
    const int grid = std::max(1, std::min(ctx->num_sms, a.tb - a.ta));
    PT_CK(cudaEventRecord(ctx->ev0, s));
    if (H == 2) k_exh_tc<2><<<grid, TC_THREADS, smem, s>>>(p);
    else k_exh_tc<1><<<grid, TC_THREADS, smem, s>>>(p);
    PT_CK(cudaEventRecord(ctx->ev1, s));
    ctx->stats.launches++;
    PT_CK(cudaGetLastError());
    if (nt_out) *nt_out = nt;
    return PT_OK;
}

