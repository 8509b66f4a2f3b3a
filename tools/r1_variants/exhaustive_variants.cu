// ARCHIVE (not built into libpt.so): the round-1 exhaustive.cu with every measured
// variant (XT_TC, XT_MMA, XW_ENABLE, XT_HALF, XT_SHAPE48, XT_PROBE, ...), for
// tools/build_variants.sh A/B builds; DESIGN.md 6.2-6.3 has the measurements.
// exhaustive.cu -- exhaustive k-subset search (Sec. 4.3.1):
// "search through the space of variant combinations ... determine the fitness
// of the kernel combination ... returns the variant combination with the
// highest ranking".
//
// (min,+) structure.  Write a k-subset as a (k-1)-subset "row" rho (colex rank
// R) plus a larger index l ("column").  With A_rho[e] = min_{c in rho} l[c][e]
//     s(rho u {l}) = sum_e min(A_rho[e], l[l][e])
// which is a (min,+) product of the row matrix A and the column matrix l over
// the environment axis.  k_exh_tiled computes it on 128-row x 64-column tiles:
//   * rows are 128 consecutive colex ranks (the combinatorial-rank decoder maps
//     each thread's rows to their subsets); A for ALL environments stays
//     resident in shared memory for every column tile of the row tile;
//   * column tiles (64 configs x 32 envs, fp32) stream from the env-major copy
//     l32T through the TMA engine (cp.async.bulk, one 256-byte row copy per
//     env, completion on an mbarrier) into a 4-stage ring;
//   * every thread holds an 8x4 block of running sums in registers; each env
//     costs one FMNMX + one FADD per (set, env) -- the per-environment best
//     member and the across-environment reduction of Eq. 1;
//   * fp32 is a FILTER: a set survives only if its fp32 score is inside a
//     rigorous error window of the best two; survivors
//     are re-scored in fp64 (k_exh_refine) and the exact top-2 is taken in
//     (s asc, sorted tuple asc) order (k_top2) -- indices bit-exact.
// k_exh_generic is the plain thread-per-subset fp64 kernel (k = 1, k > 4,
// scopes wider than 384 envs, and the PT_EXACT_FP64 debug mode).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include <cuda_fp16.h>

#include "pt_internal.cuh"

#ifndef XT_R
#define XT_R 128    // rows per CTA tile (k_exh_tiled); its consumer warps = XT_R / 16
#endif
#ifndef XT_SB
#define XT_SB 32    // k_exh_tiled A staging: loads in flight per member (E_pad % (2 XT_SB) == 0)
#endif
#ifndef XT_MINB
#define XT_MINB 2   // k_exh_tiled CTAs per SM the register budget is sized for
#endif
#ifndef XM_TC
#define XM_TC 4     // k_exh_mma: columns per thread (4: 8x4 sets per thread, 32x64 CTA tile; 8: 8x8, 64x64)
#endif
#define XM_R (XM_TC == 8 ? 64 : 32)   // rows per CTA tile (k_exh_mma)
#define XT_C 64     // columns per CTA tile
// Kernel choice.  Measured on B200 at the paper shape (k=3, 1775 x 320):
//   XT_MMA=0  k_exh_tiled (packed-fp16 tree)      13.66 ms   (default)
//   XT_MMA=1  k_exh_mma   (HMNMX2 + HMMA sum)      17.7 ms  (XM_TC=4), 21.9 ms (XM_TC=8)
// The HMMA kernel issues 0.67 instructions per (set, env) instead of 1.19 and its
// window is ~3x tighter (49 vs 184 survivors), but a shared-memory load feeding
// HMNMX2 -> HMMA stalls the loop (tools/ubench4.cu: 87% of the ALU ceiling with
// register operands, 60% with the operands from shared memory), so it stays opt-in.
#ifndef XT_MMA
#define XT_MMA 0    // 1: tensor-summed kernel k_exh_mma, 0: packed-fp16 tree kernel k_exh_tiled
#endif
// pipeline stage = XT_K envs x 64 configs (fp16); measured on B200 at the paper
// shape: K=32/S=4 13.94 ms, K=32/S=3 14.00, K=64/S=2 13.70, K=64/S=3 13.67,
// K=160/S=2 15.77 (only 1 CTA/SM fits beyond ~113 KB of smem per CTA)
#ifndef XT_K
#define XT_K 64     // environments per pipeline stage (E_pad is a multiple of 64)
#endif
#ifndef XT_S
#define XT_S 3      // pipeline stages
#endif
#ifndef XT_G8
#define XT_G8 2     // 0: one 4-env fp16 tree per FHADD; 1: one 8-env tree; 2: XT_NG 4-env trees chained in fp16
// measured (k=3, paper shape): 0 -> 13.67 ms, 2/NG=2 -> 13.48, 2/NG=4 -> 13.37 (unroll 2), 2/NG=8 -> 13.42
#endif
#ifndef XT_PUNROLL
#define XT_PUNROLL 2  // unroll of the 4*XT_NG-env loop for XT_G8 == 2
#endif
[[maybe_unused]] static constexpr int kXtPUnroll = XT_PUNROLL;
#ifndef XT_NG
#define XT_NG 4       // XT_G8 == 2: 4-env tree results summed in fp16 per FHADD (XT_K % (4 NG) == 0)
#endif
static_assert(XT_K % (4 * XT_NG) == 0, "a pipeline stage must hold whole fp16 chains");
#define XT_EMAX 768 // widest scope the resident-A kernel takes (smem)
#define XT_UMAX 1024 // column tiles per task (a whole row tile: A staged once)

// ---------------------------------------------------------------------------
// work list
// ---------------------------------------------------------------------------
// first column of a row tile whose first row's largest member is j0: j0 + 1
// rounded down to 8 configs (16-byte aligned fp16 rows); the extra columns are
// <= every row's largest member and masked.  Used by the task builder AND the
// kernel so both cover exactly [tile_lo, tile_lo + 64 * n_ct) >= [j0+1, C).
// (tile_lo and KEY_BITS: pt_internal.cuh)

struct pt_tasks {
    int m = 0;
    int64_t C = 0;
    std::vector<int4> h;              // (row tile, u0, u1, 0)
    std::vector<int64_t> slot_pre;    // prefix sums of slots per task
    std::vector<int64_t> set_pre;     // prefix sums of useful sets per task
    int4 *d = nullptr;                // device copy (lives for the process)
    // multi-GPU shard plans, keyed by shard count: the tasks dealt to shards in snake
    // order (0..N-1, N-1..0, ...) down the decreasing-size list, so every shard gets
    // the same mix of large and small tasks and ends on small ones (a contiguous cut
    // would hand shard 0 all of the largest tasks: a long tail at 8 GPUs)
    struct plan {
        int4 *d = nullptr;
        std::vector<int> off;          // shard r owns d[off[r], off[r+1])
        std::vector<int64_t> sets, slots;
    };
    std::map<std::vector<double>, plan> plans;   // key: {N} or {N, w_0 .. w_N-1}
};

// w: empty = equal shares (snake deal); else per-shard weights (weighted greedy deal:
// each task, largest first, to the shard whose load / weight would stay smallest)
static pt_status shard_plan(pt_tasks *T, int N, const std::vector<double> &w, const pt_tasks::plan **out)
{
    static std::mutex mu;
    std::lock_guard<std::mutex> g(mu);
    std::vector<double> key{(double)N};
    key.insert(key.end(), w.begin(), w.end());
    auto it = T->plans.find(key);
    if (it != T->plans.end()) {
        *out = &it->second;
        return PT_OK;
    }
    const int n = (int)T->h.size();
    std::vector<std::vector<int>> per(N);
    if (w.empty()) {
        for (int i = 0; i < n; i++) {
            const int rnd = i / N, pos = i % N;
            per[(rnd & 1) ? N - 1 - pos : pos].push_back(i);
        }
    } else {
        std::vector<double> load(N, 0.0);
        for (int i = 0; i < n; i++) {
            const double sz = (double)(T->slot_pre[i + 1] - T->slot_pre[i]);
            int best = 0;
            for (int r = 1; r < N; r++)
                if ((load[r] + sz) / w[r] < (load[best] + sz) / w[best]) best = r;
            load[best] += sz;
            per[best].push_back(i);
        }
    }
    pt_tasks::plan P;
    std::vector<int4> h;
    h.reserve(n);
    P.off.push_back(0);
    for (int r = 0; r < N; r++) {
        int64_t se = 0, sl = 0;
        for (int i : per[r]) {
            h.push_back(T->h[i]);
            se += T->set_pre[i + 1] - T->set_pre[i];
            sl += T->slot_pre[i + 1] - T->slot_pre[i];
        }
        P.off.push_back((int)h.size());
        P.sets.push_back(se);
        P.slots.push_back(sl);
    }
    if (n > 0) {
        if (cudaMalloc(&P.d, sizeof(int4) * n) != cudaSuccess) {
            cudaGetLastError();
            return pt_fail(PT_ENOMEM, "shard plan allocation failed");
        }
        cudaMemcpy(P.d, h.data(), sizeof(int4) * n, cudaMemcpyHostToDevice);
    }
    *out = &(T->plans[key] = std::move(P));
    return PT_OK;
}

extern "C" pt_status pt_set_shard_weights(pt_ctx *ctx, const double *weights, int32_t n)
{
    PT_NVTX();
    if (!ctx || n < 0) return pt_fail(PT_EINVAL, "bad argument");
    if (!weights || n == 0) {
        ctx->shard_w.clear();
        return PT_OK;
    }
    for (int r = 0; r < n; r++)
        if (!(weights[r] > 0.0) || !std::isfinite(weights[r]))
            return pt_fail(PT_EINVAL, "shard weight %d is %g (must be > 0 and finite)", r, weights[r]);
    ctx->shard_w.assign(weights, weights + n);
    return PT_OK;
}

// The work list depends only on (C, m, tile shape): built once per process and
// shared by every context (a fresh pt_load_perf does not rebuild it).  It must not
// depend on the local GPU: the ranks of a sharded search each deal the SAME list
// (ADVICE r1), so the task granularity is sized for a 148-SM B200 on every device.
static pt_status build_tasks(pt_ctx *ctx, const pt_view *v, int m, int rows, int cols, pt_tasks **out)
{
    static std::mutex mu;
    static std::map<std::tuple<int, int64_t, int, int, int, int>, pt_tasks *> cache;
    std::lock_guard<std::mutex> g(mu);
    const auto key = std::make_tuple(ctx->dev, v->C, m, ctx->num_sms, rows, cols);
    auto it = cache.find(key);
    if (it != cache.end()) {
        *out = it->second;
        return PT_OK;
    }
    pt_tasks *T = new pt_tasks();
    T->m = m;
    T->C = v->C;
    const int64_t C = v->C;
    const int64_t n_rows = pt_binom(C, m);
    const int64_t n_rt = (n_rows + rows - 1) / rows;
    T->slot_pre.push_back(0);
    T->set_pre.push_back(0);
    // task granularity: whole row tiles (A staged once) unless that leaves too
    // few tasks for the SMs (small problems, e.g. k=2)
    int64_t total_ct = 0;
    for (int64_t t = 0; t < n_rt; t++) {
        int32_t mem[PT_MAXK];
        pt_unrank_colex(t * rows, m, C, mem);
        if (mem[m - 1] + 1 >= C) continue;
        total_ct += (C - tile_lo(mem[m - 1]) + cols - 1) / cols;
    }
    const int64_t umax = std::max<int64_t>(1, std::min<int64_t>(XT_UMAX, total_ct / (8 * 148)));
    for (int64_t t = 0; t < n_rt; t++) {
        const int64_t R0 = t * rows, R1 = std::min(n_rows, R0 + rows);
        int32_t mem[PT_MAXK];
        pt_unrank_colex(R0, m, C, mem);
        const int64_t j0 = mem[m - 1];
        if (j0 + 1 >= C) continue;                    // no column l > j0
        const int64_t lo = tile_lo(j0);
        const int64_t n_ct = (C - lo + cols - 1) / cols;
        for (int64_t u0 = 0; u0 < n_ct; u0 += umax) {
            const int64_t u1 = std::min(n_ct, u0 + umax);
            const int64_t clo = lo + u0 * cols, chi = std::min(C, lo + u1 * cols);
            // useful sets: rows grouped by their largest element j (colex)
            int64_t useful = 0;
            for (int64_t j = j0; j < C; j++) {
                const int64_t a = std::max(R0, pt_binom(j, m)), b = std::min(R1, pt_binom(j + 1, m));
                if (a >= R1) break;
                if (b <= a) continue;
                const int64_t first = std::max(clo, j + 1);
                if (chi > first) useful += (b - a) * (chi - first);
            }
            T->h.push_back(make_int4((int)t, (int)u0, (int)u1, 0));
            T->slot_pre.push_back(T->slot_pre.back() + (u1 - u0) * rows * cols);
            T->set_pre.push_back(T->set_pre.back() + useful);
        }
    }
    if (!T->h.empty()) {
        if (cudaMalloc(&T->d, sizeof(int4) * T->h.size()) != cudaSuccess) {
            cudaGetLastError();
            delete T;
            return pt_fail(PT_ENOMEM, "task list allocation failed");
        }
        cudaMemcpy(T->d, T->h.data(), sizeof(int4) * T->h.size(), cudaMemcpyHostToDevice);
    }
    cache[key] = T;
    *out = T;
    return PT_OK;
}

// ---------------------------------------------------------------------------
// PTX helpers: mbarrier + TMA
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t *b, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
// try_wait with a suspend-time hint: the warp sleeps in hardware until the phase
// completes (or the hint expires) instead of spinning through issue slots
__device__ __forceinline__ bool mbar_try_sleep(uint64_t *b, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity), "r"(1000000u)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity)
{
    while (!mbar_try_sleep(b, parity)) {
    }
}
// non-blocking test of a phase
__device__ __forceinline__ bool mbar_test(uint64_t *b, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
#ifndef XT_WAITNS
#define XT_WAITNS 0   // > 0: consumers poll a B stage with test_wait + nanosleep backoff (cap in ns)
#endif
// wait for a B stage: with XT_WAITNS the warp sleeps between polls (exponential
// backoff up to XT_WAITNS ns) instead of being woken by every barrier event of
// the CTA -- fewer polling instructions competing for issue slots
__device__ __forceinline__ void mbar_wait_stage(uint64_t *b, uint32_t parity)
{
#if XT_WAITNS > 0
    if (mbar_test(b, parity)) return;
    unsigned ns = 32;
    while (!mbar_test(b, parity)) {
        __nanosleep(ns);
        ns = ns * 2 < XT_WAITNS ? ns * 2 : XT_WAITNS;
    }
#else
    mbar_wait(b, parity);
#endif
}
// bulk async copy global -> shared on the TMA engine (SASS UBLKCP), completion
// counted on an mbarrier.  src/dst 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// packed-fp16 helpers (values are non-negative log-slowdowns)
__device__ __forceinline__ uint32_t hmin2(uint32_t a, uint32_t b)
{
    uint32_t r;
    asm("min.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t hadd2(uint32_t a, uint32_t b)
{
    uint32_t r;
    asm("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
// relu(a - b) per half on the FMA pipe (HFMA2.RELU b * -1 + a): with it
// sum_e min(a, b) = sum_e a - sum_e relu(a - b)
__device__ __forceinline__ uint32_t hrelu_sub2(uint32_t a, uint32_t b)
{
    uint32_t r;
    asm("fma.rn.relu.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(b), "r"(0xBC00BC00u), "r"(a));
    return r;
}
// (acc_lo, acc_hi) += (f32(p.lo), f32(p.hi)): two FHADD (fp32 += fp16)
__device__ __forceinline__ void fhadd2(float &lo_acc, float &hi_acc, uint32_t p)
{
    unsigned short lo, hi;
    asm("mov.b32 {%0, %1}, %2;" : "=h"(lo), "=h"(hi) : "r"(p));
    asm("add.rn.f32.f16 %0, %1, %0;" : "+f"(lo_acc) : "h"(lo));
    asm("add.rn.f32.f16 %0, %1, %0;" : "+f"(hi_acc) : "h"(hi));
}

// ---------------------------------------------------------------------------
// the tiled (min,+) kernel -- packed-fp16 filter tier
//
// Fast score of a set = sum over env pairs of fp16(min(a,b)_e + min(a,b)_e+1)
// accumulated in fp32: per (set, env pair) HMNMX2 (two mins for two columns)
// is shared by two sets, one HADD2 adds the two envs of both sets, two FHADD
// accumulate into fp32 -- 1.25 issue slots per (set, env) instead of 2 for
// FMNMX+FADD, with the mins on the (half-rate) ALU pipe and the adds on the
// FMA pipe.  Every error is bounded:
//     |s_hat - s| <= eta_rel * s + eta_abs
// so the filter keeps every set that could be one of the exact best two and
// the fp64 refine decides.
//
// Warps (256 threads, 2 CTAs per SM): 8 warps compute (8 rows x 4 columns per
// thread, 128x64 per CTA).  64-env x 64-config fp16 column stages come from the
// pre-tiled hTile through the TMA engine (cp.async.bulk, one 8 KB copy per
// stage) into an XT_S-deep ring: full[] mbarriers count the bytes, and the
// last warp to release a stage (shared-memory counter) issues its refill, so no
// warp is spent on production and the SM keeps 16 warps at <= 128 registers
// (with a 9th producer warp, 18 warps per SM cap the registers at 96: a
// sub-partition's 16 K registers hold 5 warps of 96).  XT_NOPROD=0 restores
// the producer warp.  Consumers never wait for each other inside a task.
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// XT_TC=1: tensor-summed variant of k_exh_tiled.  The mins stay on the ALU pipe
// (HMNMX2: one set at two envs per instruction); the across-environment sum runs
// on the tensor pipe as m16n8k16 HMMA (f16 in, f32 accumulate) with the 0/1
// selector  B[k][n] = 1 iff floor(k/2) == n,  so C[m][n] += A[m][2n] + A[m][2n+1]:
// one MMA tile is 16 x 8 = 128 distinct sets at one env pair, no accumulator is
// duplicated.  Warp tile 32 rows x 32 columns = 8 MMA tiles (2 row blocks rb x 4
// column blocks cb).  Thread (g = lane/4, q = lane%4) feeds rows {g, g+8, g+16,
// g+24} x columns {q + 4j, j < 8} of the warp tile (one LDS.128 of A and two of B
// per env pair: the smem layouts are permuted so they are contiguous) and holds
// the sums of rows 16 rb + {g, g+8} x columns 8 cb + {2q, 2q+1} of tile (rb, cb).
// Per env pair and thread: 3 LDS + 32 HMNMX2 + 8 HMMA for 64 (set, env)
// evaluations = 0.67 issue slots per evaluation (tree: 1.09); the ALU (HMNMX2,
// half rate) and the tensor pipe (HMMA.16816, 0.5 / SM / clk) both cap at 128
// evaluations / clk / SM.
// ---------------------------------------------------------------------------
#ifndef XT_TC
#define XT_TC 0
#endif
#ifndef XT_HALF
#define XT_HALF 0   // 1 (with XT_NOPROD, not XT_TC): one B ring per 32-column half, 4 warps each
#endif              //   (measured 12.08 vs 12.04 ms: the stage misses are not warp coupling)
#define XT_BSTR (XT_HALF ? XT_C / 4 : XT_C / 2)   // u32 per env row of a warp's B stage
#ifndef XT_SHAPE48
#define XT_SHAPE48 0   // 1: 4 rows x 8 columns per thread (tree path)
#endif
#ifndef XT_PROBE
#define XT_PROBE 0    // debug build: wait statistics in the tail of the candidate score buffer
#endif
#ifndef XT_TCU
#define XT_TCU (XT_TC >= 2 ? 32 : 4)   // XT_TC: unroll of the env-pair loop (the hybrid needs it whole)
#endif
[[maybe_unused]] static constexpr int kXtTcUnroll = XT_TCU;
// row position inside a 32-row block: rows g, g+8, g+16, g+24 -> 4g .. 4g+3
__host__ __device__ __forceinline__ int tc_rpos(int r) { return (r & ~31) | ((r & 7) << 2) | ((r >> 3) & 3); }
// column position inside a 32-column half: columns q, q+4, ..., q+28 -> 8q .. 8q+7
__host__ __device__ __forceinline__ int tc_cpos(int c) { return (c & ~31) | ((c & 3) << 3) | ((c >> 2) & 7); }
__device__ __forceinline__ void tc_mma(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                       uint32_t b0, uint32_t b1)
{
    asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

struct XParams {
    int64_t C, C_pad, E_pad, n_rows;
    int m;
    const int4 *tasks;
    int task_hi;              // end of this shard's task range
    int *task_ctr;            // dynamic scheduler (starts at the shard's first task)
    float tau_seed;           // upper bound of s_(2): greedy's exact runner-up score (rounded up)
    float c1, c2, c3, c4;     // min form: LB = RD(s*c1 - c2), UB = RU(s*c3 + c4)
    float eta_A, eta_abs_r;   // relu form: |s_hat - s| <= eta_A * sumA_row + eta_abs_r
    unsigned *U;              // float bits: min over warps of their 2nd-smallest upper bound
    unsigned long long *cand_key;
    float *cand_s;
    unsigned *cand_n;
    unsigned cap;
    const uint16_t *hT;
    const uint16_t *hTile;
    int64_t n_ct;
    const uint16_t *hC;       // k_exh_mma: config-major fp16 (A staging)
    const uint32_t *hPair;    // k_exh_mma: env-pair column tiles
};

// Rows (of a thread's 8) whose 2nd column pair uses the relu form on the FMA pipe
// instead of HMNMX2 on the ALU pipe.  Measured on B200 (k=3 paper shape): 0 ->
// 14.02 ms, 1 -> 14.12, 2 -> 14.12, 4 -> 14.85, 8 -> 16.3 -- the FMA pipe is as
// loaded as the ALU pipe (FHADD), so the default keeps every unit on HMNMX2.
#ifndef RELU_ROWS
#define RELU_ROWS 0
#endif
#define XT_THREADS 288      // k_exh_mma
#define XT_CONS 256
#define XT_TCONS (2 * XT_R)  // k_exh_tiled consumers: 2 warps (column halves) per 32 rows
#ifndef XT_NOPROD
#define XT_NOPROD 1   // 1: no producer warp; the last consumer warp to release a stage refills it (0: producer warp)
#endif
#define XT_TTHREADS (XT_TCONS + (XT_NOPROD ? 0 : 32))
#define XT_BROW (XT_C * 2)     // bytes of one env row of a column tile

// broadcast one fp16 lane of a word to both halves (ptxas folds this into the
// .H0_H0 / .H1_H1 operand selector of the HMNMX2 that consumes it)
__device__ __forceinline__ uint32_t bcast_lo(uint32_t w)
{
    uint32_t r;
    asm("{ .reg .b16 l, h; mov.b32 {l, h}, %1; mov.b32 %0, {l, l}; }" : "=r"(r) : "r"(w));
    return r;
}
__device__ __forceinline__ uint32_t bcast_hi(uint32_t w)
{
    uint32_t r;
    asm("{ .reg .b16 l, h; mov.b32 {l, h}, %1; mov.b32 %0, {h, h}; }" : "=r"(r) : "r"(w));
    return r;
}

#ifndef XT_MAXREG
#define XT_MAXREG 0   // 0: __launch_bounds__(288, 2) (ptxas picks 96); else __maxnreg__(XT_MAXREG)
#endif
#if XT_MAXREG
__global__ void __maxnreg__(XT_MAXREG) k_exh_tiled(const XParams p)
#else
__global__ void __launch_bounds__(XT_TTHREADS, XT_MINB) k_exh_tiled(const XParams p)
#endif
{
    extern __shared__ __align__(128) unsigned char smem[];
    uint32_t *Bs = reinterpret_cast<uint32_t *>(smem);                        // [S][K][32] half2
    uint16_t *As = reinterpret_cast<uint16_t *>(Bs + XT_S * XT_K * (XT_C / 2)); // [E_pad][128] fp16
    int *last_s = reinterpret_cast<int *>(As + p.E_pad * XT_R);                // [128]
    float *sumA_s = reinterpret_cast<float *>(last_s + XT_R);                  // [128] (XT_TC == 3 only)
    [[maybe_unused]] float *bndA_s = sumA_s + XT_R;                            // [128] (XT_TC == 3 only)
    // B ring: XT_HALF ? [2 halves][S] stages of [K][32 cols] : [S] stages of [K][64 cols]
    uint64_t *full = reinterpret_cast<uint64_t *>(sumA_s + (XT_TC == 3 ? 2 * XT_R : 0));   // [2S]
    uint64_t *empty = full + 2 * XT_S;                                         // [2S] (keeps task_s 16-aligned)
    int4 *task_s = reinterpret_cast<int4 *>(empty + 2 * XT_S);
    int *relcnt = reinterpret_cast<int *>(task_s + 1);                         // [2S] (XT_NOPROD)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nkc = (int)(p.E_pad / XT_K);
    if (tid == 0) {
        for (int s = 0; s < XT_S; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&full[XT_S + s], 1);
            mbar_init(&empty[s], XT_TCONS / 32);
            relcnt[s] = relcnt[XT_S + s] = 0;
        }
        mbar_fence_init();
    }
    __syncthreads();

    uint32_t steps = 0;   // pipeline steps of all previous tasks (same in every thread)
    [[maybe_unused]] const int tx = lane & 7, ty = lane >> 3;
    float bA = INFINITY, bB = INFINITY, published = INFINITY;   // acc-domain group minima (window U)

    for (;;) {
        if (tid == 0) {
            int ti = atomicAdd(p.task_ctr, 1);
            *task_s = ti < p.task_hi ? p.tasks[ti] : make_int4(-1, 0, 0, 0);
        }
        __syncthreads();
        const int4 tk = *task_s;
        if (tk.x < 0) break;
        const int64_t R0 = (int64_t)tk.x * XT_R;
        int32_t mem0[PT_MAXK];
        pt_unrank_colex(R0, p.m, p.C, mem0);
        const int64_t lo = tile_lo(mem0[p.m - 1]);
        const int nsteps = (tk.z - tk.y) * nkc;
#if XT_NOPROD
        // stage g of this task (column tile tk.y + g / nkc, env chunk g % nkc) into its ring
        // slot: one bulk copy, completion counted on full[slot]
        auto issue = [&](int g, int h) {
            const int sl = (int)((steps + (uint32_t)g) % XT_S);
            const int64_t col = lo + (int64_t)(tk.y + g / nkc) * XT_C;
            const int64_t sh = (col >> 3) & 7, ct = (col - 8 * sh) >> 6;
#if XT_HALF
            // half h of the stage: hTile is stored [sh][ct][half][e][32]
            const uint16_t *src = p.hTile + (((sh * p.n_ct + ct) * 2 + h) * p.E_pad + (int64_t)(g % nkc) * XT_K) * 32;
            mbar_expect_tx(&full[h * XT_S + sl], XT_K * 64);
            bulk_g2s(Bs + (h * XT_S + sl) * XT_K * 16, src, XT_K * 64, &full[h * XT_S + sl]);
#else
            const uint16_t *src = p.hTile + ((sh * p.n_ct + ct) * p.E_pad + (int64_t)(g % nkc) * XT_K) * XT_C;
            mbar_expect_tx(&full[sl], XT_K * XT_BROW);
            bulk_g2s(Bs + sl * XT_K * (XT_C / 2), src, XT_K * XT_BROW, &full[sl]);
#endif
        };
        // every warp has left the previous task (barrier above): the whole ring is free
        if (tid == 0)
            for (int g = 0; g < XT_S && g < nsteps; g++) {
                issue(g, 0);
                if (XT_HALF) issue(g, 1);
            }
#endif

        if (!XT_NOPROD && warp == XT_TCONS / 32) {
            // ---------------- producer warp ----------------
            // column tile starting at config `col` (8-aligned) = shift s, tile ct
            // of hTile; each stage is one contiguous 32-env x 64-config block
            if (lane == 0) {
                int q = 0;
                int64_t col = lo + (int64_t)tk.y * XT_C;
                uint32_t G = steps;
                for (int g = 0; g < nsteps; g++, G++) {
                    const int slot = G % XT_S;
                    const uint32_t par = ((G / XT_S) & 1u) ^ 1u;
                    mbar_wait(&empty[slot], par);
                    const int64_t sh = (col >> 3) & 7, ct = (col - 8 * sh) >> 6;
                    const uint16_t *src = p.hTile + ((sh * p.n_ct + ct) * p.E_pad + (int64_t)q * XT_K) * XT_C;
                    mbar_expect_tx(&full[slot], XT_K * XT_BROW);
                    bulk_g2s(Bs + slot * XT_K * (XT_C / 2), src, XT_K * XT_BROW, &full[slot]);
                    if (++q == nkc) {
                        q = 0;
                        col += XT_C;
                    }
                }
            }
            __syncwarp();
        } else {
            // ---------------- consumers ----------------
            // stage A for the whole task: A[e][r] = min over the row's members
            // (fp16, non-negative: integer order).  Loads are batched XT_SB deep per member.
            {
                const int r = tid & (XT_R - 1);
                const int64_t R = R0 + r;
                int32_t mem[PT_MAXK];
                const bool valid = R < p.n_rows;
                if (valid) pt_unrank_colex(R, p.m, p.C, mem);
                else for (int u = 0; u < p.m; u++) mem[u] = 0;
                if (tid < XT_R) last_s[r] = valid ? mem[p.m - 1] : 0x7fffffff;
                const int64_t e0 = tid / XT_R;
#if XT_TC
                // env pairs (2 pp, 2 pp + 1) packed into one f16x2 word, row at tc_rpos(r)
                uint32_t *Aw = reinterpret_cast<uint32_t *>(As);
                const int rp = tc_rpos(r);
                for (int64_t pb = e0; pb < p.E_pad / 2; pb += XT_SB) {
                    uint16_t v[XT_SB];   // v[2t + h] = env 2 (pb + 2t) + h
#pragma unroll
                    for (int t = 0; t < XT_SB; t++) v[t] = p.hT[(2 * (pb + 2 * (t >> 1)) + (t & 1)) * p.C_pad + mem[0]];
                    for (int u = 1; u < p.m; u++) {
                        uint16_t w[XT_SB];
#pragma unroll
                        for (int t = 0; t < XT_SB; t++)
                            w[t] = p.hT[(2 * (pb + 2 * (t >> 1)) + (t & 1)) * p.C_pad + mem[u]];
#pragma unroll
                        for (int t = 0; t < XT_SB; t++) v[t] = v[t] < w[t] ? v[t] : w[t];
                    }
#pragma unroll
                    for (int t = 0; t < XT_SB / 2; t++)
                        Aw[(pb + 2 * t) * XT_R + rp] = valid ? ((uint32_t)v[2 * t] | ((uint32_t)v[2 * t + 1] << 16)) : 0u;
                }
#else
                for (int64_t eb = e0; eb < p.E_pad; eb += 2 * XT_SB) {
                    uint16_t v[XT_SB];
#pragma unroll
                    for (int t = 0; t < XT_SB; t++) v[t] = p.hT[(eb + 2 * t) * p.C_pad + mem[0]];
                    for (int u = 1; u < p.m; u++) {
                        uint16_t w[XT_SB];
#pragma unroll
                        for (int t = 0; t < XT_SB; t++) w[t] = p.hT[(eb + 2 * t) * p.C_pad + mem[u]];
#pragma unroll
                        for (int t = 0; t < XT_SB; t++) v[t] = v[t] < w[t] ? v[t] : w[t];
                    }
#pragma unroll
                    for (int t = 0; t < XT_SB; t++) As[(eb + 2 * t) * XT_R + r] = valid ? v[t] : (uint16_t)0;
                }
#endif
            }
            named_sync(1, XT_TCONS);
#if XT_TC == 3
            // relu-form sets need their row's sum_e A (fp32, pairs ascending) and its error
            // bound eta_A * sumA + eta_abs_r (rounded up)
            if (tid < XT_R) {
                const uint32_t *Aw = reinterpret_cast<const uint32_t *>(As);
                const int rp = tc_rpos(tid);
                float sa = 0.0f;
                for (int64_t pp = 0; pp < p.E_pad / 2; pp++) {
                    const uint32_t w = Aw[pp * XT_R + rp];
                    sa += __half2float(__ushort_as_half((unsigned short)(w & 0xffffu)));
                    sa += __half2float(__ushort_as_half((unsigned short)(w >> 16)));
                }
                sumA_s[tid] = sa;
                bndA_s[tid] = __fmaf_ru(p.eta_A, sa, p.eta_abs_r);
            }
            named_sync(1, XT_TCONS);
#endif

            float acc[8][4];
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) acc[i][j] = 0.0f;

            // warp w covers rows 32*(w>>1) .. +31 and columns 32*(w&1) .. +31 of the
            // 128x64 tile; a thread holds 8 consecutive rows (one 16-byte LDS) x 4
            // consecutive columns (one 8-byte LDS)
#if XT_TC
            // warp tile rows r0 .. r0+31, columns cw .. cw+31; acc[4 rb + cb][t] is the set
            // (row r0 + 16 rb + g + 8 (t>>1), column cw + 8 cb + 2 qd + (t&1))
            const int gq = lane >> 2, qd = lane & 3;
            const int r0 = 32 * (warp >> 1);
            const int cw = 32 * (warp & 1);
            const int c0 = cw + (XT_TC >= 2 ? qd : 2 * qd);  // the thread's first column
            const int last7 = last_s[r0 + 24 + gq];          // its last row (colex: largest last member)
            const uint32_t one2 = 0x3C003C00u;               // f16x2 (1, 1)
            const uint32_t sel0 = gq == qd ? one2 : 0u, sel1 = gq == qd + 4 ? one2 : 0u;
#if XT_TC >= 2
            // hybrid, split by sets: the warp tile's columns 0-15 (MMA tiles cb = 0, 1) are
            // summed on the tensor pipe into accm[2 rb + cb][t], columns 16-31 by fp16 chains
            // on the FMA pipe into acc[2 i' + 1][jj] (the thread's own input sets: row
            // r0 + gq + 8 i', column cw + qd + 16 + 4 jj); at each epilogue the MMA sums move
            // to their owners' acc[2 i'][j'] (row r0 + gq + 8 i', column cw + qd + 4 j')
            float accm[4][4];
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) accm[i][j] = 0.0f;
            uint32_t hp[4][4];                               // fp16 chains of the tree sets
#define XT_ROW(i, j) (r0 + gq + 8 * ((i) >> 1))
#define XT_COL(i, j) (cw + qd + 4 * (((i) & 1) * 4 + (j)))
#define XT_GRPB(i, j) ((i) & 1)
#define XT_SPAN 28
#else
#define XT_ROW(i, j) (r0 + 16 * ((i) >> 2) + gq + 8 * ((j) >> 1))
#define XT_COL(i, j) (cw + 8 * ((i) & 3) + 2 * qd + ((j) & 1))
#define XT_GRPB(i, j) (((i) & 3) >= 2)
#define XT_SPAN 25                                       // thread's last column - first column
#endif
#else
#if XT_SHAPE48
            // 4 rows x 8 columns per thread (one 8-byte A LDS, one 16-byte B LDS per env);
            // acc[i][j] is row r0 + (i>>1), column c0 + 4 (i&1) + j
            const int r0 = 32 * (warp >> 1) + 4 * (lane >> 2);
            const int c0 = 32 * (warp & 1) + 8 * (lane & 3);
            const int last7 = last_s[r0 + 3];
#define XT_ROW(i, j) (r0 + ((i) >> 1))
#define XT_COL(i, j) (c0 + 4 * ((i) & 1) + (j))
#define XT_GRPB(i, j) ((i) & 1)
#define XT_SPAN 7
#else
            const int r0 = 32 * (warp >> 1) + 8 * ty;
            const int c0 = 32 * (warp & 1) + 4 * tx;
            // colex order: a row's largest member is non-decreasing in its rank (padding
            // rows hold INT_MAX), so the thread's last row bounds all eight
            const int last7 = last_s[r0 + 7];
#define XT_ROW(i, j) (r0 + (i))
#define XT_COL(i, j) (c0 + (j))
#define XT_GRPB(i, j) ((j) >= 2)
#define XT_SPAN 3
#endif
#endif
            uint32_t slot = steps % XT_S, phase = (steps / XT_S) & 1u;
            int64_t ltile = lo + (int64_t)tk.y * XT_C;     // first column of the current tile
            for (int ct = tk.y; ct < tk.z; ct++, ltile += XT_C) {
                // the whole warp's column half lies past the last config: skip the math
                const bool skip = ltile + 32 * (warp & 1) >= p.C;
                // window threshold for this tile's epilogue, loaded before the math so the
                // L2 latency hides behind it (a stale value is only a looser bound)
                const unsigned Ubits = *(volatile unsigned *)p.U;
                for (int q = 0; q < nkc; q++) {
#if XT_PROBE
                    // debug: count stage waits that find the data missing, split into the first
                    // stage of a task, the first stage of a later column tile, and the rest
                    if (!mbar_test(&full[(XT_HALF ? (warp & 1) * XT_S : 0) + slot], phase) && lane == 0) {
#if XT_PROBE == 2
                        // breakdown: kind 0 = skipping warp, 1 = warp parity 0, 2 = parity 1
                        const int kind = skip ? 0 : 1 + (warp & 1);
#else
                        const int kind = (ct == tk.y && q == 0) ? 0 : (q == 0 ? 1 : 2);
#endif
                        atomicAdd(reinterpret_cast<unsigned long long *>(p.cand_s) + (p.cap / 2 - 4 + kind), 1ull);
                    }
                    if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long *>(p.cand_s) + (p.cap / 2 - 1), 1ull);
#endif
                    mbar_wait_stage(&full[(XT_HALF ? (warp & 1) * XT_S : 0) + slot], phase);
                    if (!skip) {
#if XT_TC
                        const uint32_t *Bw = Bs + slot * XT_K * (XT_C / 2) + cw + 8 * qd;
                        const uint32_t *Aw = reinterpret_cast<const uint32_t *>(As) +
                                             (int64_t)q * (XT_K / 2) * XT_R + r0 + 4 * gq;
#pragma unroll kXtTcUnroll
                        for (int pp = 0; pp < XT_K / 2; pp++) {
                            const uint4 av = *reinterpret_cast<const uint4 *>(Aw + pp * XT_R);
                            const uint4 b0 = *reinterpret_cast<const uint4 *>(Bw + pp * XT_C);
                            const uint4 b1 = *reinterpret_cast<const uint4 *>(Bw + pp * XT_C + 4);
                            const uint32_t rv[4] = {av.x, av.y, av.z, av.w};
                            const uint32_t cv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#if XT_TC >= 2
#pragma unroll
                            for (int rb = 0; rb < 2; rb++)
#pragma unroll
                                for (int cb = 0; cb < 2; cb++)
                                    tc_mma(accm[2 * rb + cb], hmin2(rv[2 * rb], cv[2 * cb]),
                                           hmin2(rv[2 * rb + 1], cv[2 * cb]), hmin2(rv[2 * rb], cv[2 * cb + 1]),
                                           hmin2(rv[2 * rb + 1], cv[2 * cb + 1]), sel0, sel1);
                            // tree sets: a set's two envs stay in the two lanes; 8 pairs (16 envs)
                            // are chained in fp16, then both halves go to fp32
                            const int u = pp & 7;   // position in the chain
#pragma unroll
                            for (int i = 0; i < 4; i++)
#pragma unroll
                                for (int jj = 0; jj < 4; jj++) {
#if XT_TC == 3
                                    // columns 24-31: relu(a - b) on the FMA pipe instead of the min
                                    const uint32_t m = jj >= 2 ? hrelu_sub2(rv[i], cv[4 + jj]) : hmin2(rv[i], cv[4 + jj]);
#else
                                    const uint32_t m = hmin2(rv[i], cv[4 + jj]);
#endif
                                    if (u == 0) hp[i][jj] = m;
                                    else hp[i][jj] = hadd2(hp[i][jj], m);
                                    if (u == 7) {
                                        float &a = acc[2 * i + 1][jj];
                                        fhadd2(a, a, hp[i][jj]);
                                    }
                                }
#else
#pragma unroll
                            for (int rb = 0; rb < 2; rb++)
#pragma unroll
                                for (int cb = 0; cb < 4; cb++)
                                    tc_mma(acc[4 * rb + cb], hmin2(rv[2 * rb], cv[2 * cb]),
                                           hmin2(rv[2 * rb + 1], cv[2 * cb]), hmin2(rv[2 * rb], cv[2 * cb + 1]),
                                           hmin2(rv[2 * rb + 1], cv[2 * cb + 1]), sel0, sel1);
#endif
                        }
#else
#if XT_HALF
                        const uint32_t *B = Bs + ((warp & 1) * XT_S + slot) * XT_K * 16 + (c0 & 31) / 2;
#else
                        const uint32_t *B = Bs + slot * XT_K * (XT_C / 2) + c0 / 2;
#endif
                        const uint16_t *A = As + (int64_t)q * XT_K * XT_R + r0;
#if XT_SHAPE48
#pragma unroll kXtPUnroll
                        for (int e = 0; e < XT_K; e += 4 * XT_NG) {
                            uint32_t pp[4][4];
#pragma unroll
                            for (int gq = 0; gq < XT_NG; gq++) {
                                uint2 ar[4];
                                uint4 bc[4];
#pragma unroll
                                for (int t = 0; t < 4; t++) {
                                    ar[t] = *reinterpret_cast<const uint2 *>(A + (e + 4 * gq + t) * XT_R);
                                    bc[t] = *reinterpret_cast<const uint4 *>(B + (e + 4 * gq + t) * XT_BSTR);
                                }
#pragma unroll
                                for (int i = 0; i < 4; i++) {
                                    uint32_t av[4];
#pragma unroll
                                    for (int t = 0; t < 4; t++) {
                                        const uint32_t w = (i >> 1) == 0 ? ar[t].x : ar[t].y;
                                        av[t] = (i & 1) ? bcast_hi(w) : bcast_lo(w);
                                    }
#pragma unroll
                                    for (int j = 0; j < 4; j++) {
                                        const uint32_t b0 = j == 0 ? bc[0].x : j == 1 ? bc[0].y : j == 2 ? bc[0].z : bc[0].w;
                                        const uint32_t b1 = j == 0 ? bc[1].x : j == 1 ? bc[1].y : j == 2 ? bc[1].z : bc[1].w;
                                        const uint32_t b2 = j == 0 ? bc[2].x : j == 1 ? bc[2].y : j == 2 ? bc[2].z : bc[2].w;
                                        const uint32_t b3 = j == 0 ? bc[3].x : j == 1 ? bc[3].y : j == 2 ? bc[3].z : bc[3].w;
                                        const uint32_t sx = hadd2(hadd2(hmin2(av[0], b0), hmin2(av[1], b1)),
                                                                  hadd2(hmin2(av[2], b2), hmin2(av[3], b3)));
                                        float *a2 = &acc[2 * i + (j >> 1)][2 * (j & 1)];
                                        if (gq == 0) pp[i][j] = sx;
                                        else if (gq < XT_NG - 1) pp[i][j] = hadd2(pp[i][j], sx);
                                        else fhadd2(a2[0], a2[1], XT_NG == 1 ? sx : hadd2(pp[i][j], sx));
                                    }
                                }
                            }
                        }
#elif XT_G8 == 2
                        // XT_NG 4-env fp16 trees per unit summed in fp16 (one HADD2 each) before
                        // the two FHADD: (8 NG + 1) slots per 8 NG (set, env) pairs of columns
                        // instead of 9 NG; the running fp16 partial waits in pp[][] (16 registers)
                        // while the next group loads
#pragma unroll kXtPUnroll
                        for (int e = 0; e < XT_K; e += 4 * XT_NG) {
                            uint32_t pp[8][2];
#pragma unroll
                            for (int gq = 0; gq < XT_NG; gq++) {
                                uint4 ar[4];
                                uint2 bc[4];
#pragma unroll
                                for (int t = 0; t < 4; t++) {
                                    ar[t] = *reinterpret_cast<const uint4 *>(A + (e + 4 * gq + t) * XT_R);
                                    bc[t] = *reinterpret_cast<const uint2 *>(B + (e + 4 * gq + t) * XT_BSTR);
                                }
#pragma unroll
                                for (int i = 0; i < 8; i++) {
                                    uint32_t av[4];
#pragma unroll
                                    for (int t = 0; t < 4; t++) {
                                        const uint32_t w = (i >> 1) == 0 ? ar[t].x : (i >> 1) == 1 ? ar[t].y
                                                                         : (i >> 1) == 2 ? ar[t].z : ar[t].w;
                                        av[t] = (i & 1) ? bcast_hi(w) : bcast_lo(w);
                                    }
                                    const uint32_t tx = hadd2(hadd2(hmin2(av[0], bc[0].x), hmin2(av[1], bc[1].x)),
                                                              hadd2(hmin2(av[2], bc[2].x), hmin2(av[3], bc[3].x)));
                                    const uint32_t ty = hadd2(hadd2(hmin2(av[0], bc[0].y), hmin2(av[1], bc[1].y)),
                                                              hadd2(hmin2(av[2], bc[2].y), hmin2(av[3], bc[3].y)));
                                    if (gq == 0) {
                                        pp[i][0] = tx;
                                        pp[i][1] = ty;
                                    } else if (gq < XT_NG - 1) {
                                        pp[i][0] = hadd2(pp[i][0], tx);
                                        pp[i][1] = hadd2(pp[i][1], ty);
                                    } else {
                                        fhadd2(acc[i][0], acc[i][1], hadd2(pp[i][0], tx));
                                        fhadd2(acc[i][2], acc[i][3], hadd2(pp[i][1], ty));
                                    }
                                }
                            }
                        }
#elif XT_G8
#pragma unroll 1
                        for (int e = 0; e < XT_K; e += 8) {
                            uint4 ar[8];
                            uint2 bc[8];
#pragma unroll
                            for (int t = 0; t < 8; t++) {
                                ar[t] = *reinterpret_cast<const uint4 *>(A + (e + t) * XT_R);
                                bc[t] = *reinterpret_cast<const uint2 *>(B + (e + t) * XT_BSTR);
                            }
#pragma unroll
                            for (int i = 0; i < 8; i++) {
                                uint32_t av[8];
#pragma unroll
                                for (int t = 0; t < 8; t++) {
                                    const uint32_t w = (i >> 1) == 0 ? ar[t].x : (i >> 1) == 1 ? ar[t].y
                                                                     : (i >> 1) == 2 ? ar[t].z : ar[t].w;
                                    av[t] = (i & 1) ? bcast_hi(w) : bcast_lo(w);
                                }
                                fhadd2(acc[i][0], acc[i][1],
                                       hadd2(hadd2(hadd2(hmin2(av[0], bc[0].x), hmin2(av[1], bc[1].x)),
                                                   hadd2(hmin2(av[2], bc[2].x), hmin2(av[3], bc[3].x))),
                                             hadd2(hadd2(hmin2(av[4], bc[4].x), hmin2(av[5], bc[5].x)),
                                                   hadd2(hmin2(av[6], bc[6].x), hmin2(av[7], bc[7].x)))));
                                fhadd2(acc[i][2], acc[i][3],
                                       hadd2(hadd2(hadd2(hmin2(av[0], bc[0].y), hmin2(av[1], bc[1].y)),
                                                   hadd2(hmin2(av[2], bc[2].y), hmin2(av[3], bc[3].y))),
                                             hadd2(hadd2(hmin2(av[4], bc[4].y), hmin2(av[5], bc[5].y)),
                                                   hadd2(hmin2(av[6], bc[6].y), hmin2(av[7], bc[7].y)))));
                            }
                        }
#else
#pragma unroll 2
                        for (int e = 0; e < XT_K; e += 4) {
                            uint4 ar[4];
                            uint2 bc[4];
#pragma unroll
                            for (int t = 0; t < 4; t++) {
                                ar[t] = *reinterpret_cast<const uint4 *>(A + (e + t) * XT_R);
                                bc[t] = *reinterpret_cast<const uint2 *>(B + (e + t) * XT_BSTR);
                            }
#pragma unroll
                            for (int i = 0; i < 8; i++) {
                                uint32_t av[4];
#pragma unroll
                                for (int t = 0; t < 4; t++) {
                                    const uint32_t w = (i >> 1) == 0 ? ar[t].x : (i >> 1) == 1 ? ar[t].y
                                                                     : (i >> 1) == 2 ? ar[t].z : ar[t].w;
                                    av[t] = (i & 1) ? bcast_hi(w) : bcast_lo(w);
                                }
                                // fp16 tree over the 4 envs, then 2 FHADD into fp32
                                fhadd2(acc[i][0], acc[i][1],
                                       hadd2(hadd2(hmin2(av[0], bc[0].x), hmin2(av[1], bc[1].x)),
                                             hadd2(hmin2(av[2], bc[2].x), hmin2(av[3], bc[3].x))));
                                fhadd2(acc[i][2], acc[i][3],
                                       hadd2(hadd2(hmin2(av[0], bc[0].y), hmin2(av[1], bc[1].y)),
                                             hadd2(hmin2(av[2], bc[2].y), hmin2(av[3], bc[3].y))));
                            }
                        }
#endif
#endif
                    }
                    __syncwarp();
#if XT_NOPROD
                    if (lane == 0) {
                        // release: the last of the consumer warps to finish this stage refills
                        // the slot with stage g + S of the task
                        __threadfence_block();
                        const int h = XT_HALF ? (warp & 1) : 0;
                        if (atomicAdd(&relcnt[h * XT_S + slot], 1) == XT_TCONS / (XT_HALF ? 64 : 32) - 1) {
                            relcnt[h * XT_S + slot] = 0;
                            __threadfence_block();
                            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                            const int gn = (ct - tk.y) * nkc + q + XT_S;
                            if (gn < nsteps) issue(gn, h);
                        }
                    }
#else
                    if (lane == 0) mbar_arrive(&empty[slot]);
#endif
                    if (++slot == XT_S) {
                        slot = 0;
                        phase ^= 1u;
                    }
                }
                if (skip) continue;
#if XT_TC >= 2
                // move the MMA sums to their owners: own set (row g + 8 i', column qd + 4 j'),
                // j' < 4, is C-fragment element (rb = i'>>1, cb = j'>>1, t = 2 (i'&1) + (qd&1))
                // of quad lane (qd>>1) + 2 (j'&1); two shuffles (t even / odd) and a select
#pragma unroll
                for (int ip = 0; ip < 4; ip++)
#pragma unroll
                    for (int jp = 0; jp < 4; jp++) {
                        const int src = (lane & ~3) | ((qd >> 1) + 2 * (jp & 1));
                        const int reg = 2 * (ip >> 1) + (jp >> 1), th = ip & 1;
                        const float v0 = __shfl_sync(0xffffffffu, accm[reg][2 * th], src);
                        const float v1 = __shfl_sync(0xffffffffu, accm[reg][2 * th + 1], src);
                        acc[2 * ip][jp] = (qd & 1) ? v1 : v0;
                    }
#pragma unroll
                for (int i = 0; i < 4; i++)
#pragma unroll
                    for (int j = 0; j < 4; j++) accm[i][j] = 0.0f;
#endif
                // ---- epilogue of one column tile ----
                // LB = RD(acc*c1 - c2) and UB = RU(acc*c3 + c4) are non-decreasing in acc, so
                // order statistics and the window test are taken on acc itself and mapped
                // once.  Padding / ragged sets become +inf.
                const int64_t l0 = ltile + c0;
                if (!(l0 + XT_SPAN < p.C && l0 > last7)) {
#pragma unroll
                    for (int i = 0; i < 8; i++)
#pragma unroll
                        for (int j = 0; j < 4; j++) {
                            const int64_t l = ltile + XT_COL(i, j);
                            if (!(l < p.C && l > last_s[XT_ROW(i, j)])) acc[i][j] = INFINITY;
                        }
                }
#if XT_TC == 3
                // relu sets (odd i, j >= 2): acc holds sum relu(a - b); bounds from the row sum.
                // Bounds are computed explicitly (LB, UB) and the U minima kept in UB terms.
                float lbv[8][4], tA = INFINITY, tB = INFINITY, tL = INFINITY;
#pragma unroll
                for (int i = 0; i < 8; i++)
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        float lb, ub;
                        if (!(acc[i][j] < INFINITY)) {
                            lb = ub = INFINITY;
                        } else if ((i & 1) && j >= 2) {
                            const int r = XT_ROW(i, j);
                            const float sh = sumA_s[r] - acc[i][j];
                            lb = __fsub_rd(sh, bndA_s[r]);
                            ub = __fadd_ru(sh, bndA_s[r]);
                        } else {
                            lb = __fmaf_rd(acc[i][j], p.c1, -p.c2);
                            ub = __fmaf_ru(acc[i][j], p.c3, p.c4);
                        }
                        lbv[i][j] = lb;
                        tL = fminf(tL, lb);
                        if (XT_GRPB(i, j)) tB = fminf(tB, ub);
                        else tA = fminf(tA, ub);
                    }
                bA = fminf(bA, tA);
                bB = fminf(bB, tB);
                const float tau = fminf(p.tau_seed, __uint_as_float(Ubits));
                if (tL <= tau) {
#pragma unroll
                    for (int i = 0; i < 8; i++)
#pragma unroll
                        for (int j = 0; j < 4; j++) {
                            const float lb = lbv[i][j];
                            if (lb < INFINITY && lb <= tau) {
#else
                // tile minima of two disjoint groups of the thread's sets
                float tA = INFINITY, tB = INFINITY;
#pragma unroll
                for (int i = 0; i < 8; i++)
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        if (XT_GRPB(i, j)) tB = fminf(tB, acc[i][j]);
                        else tA = fminf(tA, acc[i][j]);
                    }
                bA = fminf(bA, tA);
                bB = fminf(bB, tB);
                const float tau = fminf(p.tau_seed, __uint_as_float(Ubits));
                if (__fmaf_rd(fminf(tA, tB), p.c1, -p.c2) <= tau) {   // rare: some set is in the window
#pragma unroll
                    for (int i = 0; i < 8; i++)
#pragma unroll
                        for (int j = 0; j < 4; j++) {
                            const float lb = __fmaf_rd(acc[i][j], p.c1, -p.c2);
                            if (acc[i][j] < INFINITY && lb <= tau) {
#endif
                                const unsigned idx = atomicAdd(p.cand_n, 1u);
                                if (idx < p.cap) {
                                    p.cand_key[idx] = ((unsigned long long)(R0 + XT_ROW(i, j)) << KEY_BITS) |
                                                      (unsigned long long)(ltile + XT_COL(i, j));
                                    p.cand_s[idx] = lb;
                                }
                            }
                        }
                }
#pragma unroll
                for (int i = 0; i < 8; i++)
#pragma unroll
                    for (int j = 0; j < 4; j++) acc[i][j] = 0.0f;
                // U: the warp's 2nd-smallest group minimum.  bA and bB of all lanes are
                // minima over disjoint sets of sets, so the two smallest belong to two
                // distinct sets and UB(2nd) >= s_(2)
                float x1 = fminf(bA, bB), x2 = fmaxf(bA, bB);
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    const float y1 = __shfl_xor_sync(0xffffffffu, x1, o);
                    const float y2 = __shfl_xor_sync(0xffffffffu, x2, o);
                    x2 = fminf(fmaxf(x1, y1), fminf(x2, y2));
                    x1 = fminf(x1, y1);
                }
                if (lane == 0) {
                    const float ub = XT_TC == 3 ? x2 : __fmaf_ru(x2, p.c3, p.c4);   // (TC 3: already UB)
                    if (ub < published) {
                        atomicMin(p.U, __float_as_uint(ub));
                        published = ub;
                    }
                }
            }
        }
        steps += nsteps;
    }
#undef XT_ROW
#undef XT_COL
#undef XT_GRPB
#undef XT_SPAN
}

// ---------------------------------------------------------------------------
// k_exh_ws: warp-specialised persistent variant of k_exh_tiled (one CTA per
// SM) for scopes where the double-buffered A tile fits (E_pad <= XW_EMAX).
// Opt-in (XW_ENABLE=1): measured 13.54 ms vs 12.33 ms for k_exh_tiled at k=3 --
// 18 warps cap the registers at 96 (spills), and one stager warp gathering
// 82 K fp16 values per task cannot keep up with the small tasks at the end of
// the decreasing-size queue.
//   warps 0-15 : consumers; CTA tile 128 rows x 128 columns (warp w: rows
//                32*(w>>2) + 8*ty, columns 32*(w&3) + 4*tx); the inner loop and
//                the epilogue are k_exh_tiled's
//   warp 16    : producer; streams 64-env x 128-config stages (two 8 KB bulk
//                copies from hTile) through the XT_S-deep B ring
//   warp 17    : stager; takes tasks from the dynamic queue and builds the NEXT
//                task's A tile into the other half of a double buffer
// The roles meet only on mbarriers -- B ring full/empty, A buffer full
// (stager -> consumers, producer) and empty (consumers -> stager) -- so there
// is no CTA-wide barrier between tasks: the A gather overlaps the math and a
// fast warp runs on into the next task.
// ---------------------------------------------------------------------------
#ifndef XW_ENABLE
#define XW_ENABLE 0                 // 1: k_exh_ws where it fits (measured slower)
#endif
#define XW_C 128                    // columns per CTA tile
#define XW_CONS 512                 // consumer threads (16 warps)
#define XW_THREADS (XW_CONS + 64)   // + producer + stager
#define XW_EMAX 320                 // widest scope: 2 A buffers + the B ring fit 227 KB
#ifndef XW_MAXREG
#define XW_MAXREG 96   // 18 warps put 5 on one SM sub-partition: 5 x 32 x 104 > its 16 K registers
#endif
#define XW_SE 8                     // stager: envs per batch (4 rows x 8 envs x members in flight)

__global__ void __maxnreg__(XW_MAXREG) k_exh_ws(const XParams p)
{
    extern __shared__ __align__(128) unsigned char smem[];
    uint32_t *Bs = reinterpret_cast<uint32_t *>(smem);                        // [S][2][K][32] half2
    uint16_t *As0 = reinterpret_cast<uint16_t *>(Bs + XT_S * 2 * XT_K * 32);  // [2][E_pad][128] fp16
    int *last_s0 = reinterpret_cast<int *>(As0 + 2 * p.E_pad * XT_R);         // [2][128]
    int4 *task_s = reinterpret_cast<int4 *>(last_s0 + 2 * XT_R);              // [2]
    uint64_t *full = reinterpret_cast<uint64_t *>(task_s + 2);                // [S]
    uint64_t *empty = full + XT_S;                                            // [S]
    uint64_t *afull = empty + XT_S;                                           // [2]
    uint64_t *aempty = afull + 2;                                             // [2]

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nkc = (int)(p.E_pad / XT_K);
    if (tid == 0) {
        for (int s = 0; s < XT_S; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], XW_CONS / 32);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(&afull[b], 1);
            mbar_init(&aempty[b], XW_CONS / 32);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == XW_CONS / 32 + 1) {
        // ---------------- stager ----------------
        for (uint32_t n = 0;; n++) {
            const int b = n & 1;
            mbar_wait(&aempty[b], ((n >> 1) & 1u) ^ 1u);
            int ti = 0;
            if (lane == 0) ti = atomicAdd(p.task_ctr, 1);
            ti = __shfl_sync(0xffffffffu, ti, 0);
            const int4 tk = ti < p.task_hi ? p.tasks[ti] : make_int4(-1, 0, 0, 0);
            if (tk.x >= 0) {
                // A[e][r] = min over row r's members (fp16 bits, non-negative: integer
                // order); lane owns rows lane + 32 i
                uint16_t *As = As0 + (int64_t)b * p.E_pad * XT_R;
                int *last_s = last_s0 + b * XT_R;
                const int64_t R0 = (int64_t)tk.x * XT_R;
                int32_t mem[4][PT_MAXK];
                bool valid[4];
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const int64_t R = R0 + lane + 32 * i;
                    valid[i] = R < p.n_rows;
                    if (valid[i]) pt_unrank_colex(R, p.m, p.C, mem[i]);
                    else for (int u = 0; u < p.m; u++) mem[i][u] = 0;
                    last_s[lane + 32 * i] = valid[i] ? mem[i][p.m - 1] : 0x7fffffff;
                }
                for (int64_t e0 = 0; e0 < p.E_pad; e0 += XW_SE) {
                    uint16_t v[4][XW_SE];
#pragma unroll
                    for (int i = 0; i < 4; i++)
#pragma unroll
                        for (int t = 0; t < XW_SE; t++) v[i][t] = p.hT[(e0 + t) * p.C_pad + mem[i][0]];
                    for (int u = 1; u < p.m; u++) {
                        uint16_t w[4][XW_SE];
#pragma unroll
                        for (int i = 0; i < 4; i++)
#pragma unroll
                            for (int t = 0; t < XW_SE; t++) w[i][t] = p.hT[(e0 + t) * p.C_pad + mem[i][u]];
#pragma unroll
                        for (int i = 0; i < 4; i++)
#pragma unroll
                            for (int t = 0; t < XW_SE; t++) v[i][t] = v[i][t] < w[i][t] ? v[i][t] : w[i][t];
                    }
#pragma unroll
                    for (int i = 0; i < 4; i++)
#pragma unroll
                        for (int t = 0; t < XW_SE; t++)
                            As[(e0 + t) * XT_R + lane + 32 * i] = valid[i] ? v[i][t] : (uint16_t)0;
                }
            }
            if (lane == 0) task_s[b] = tk;
            __threadfence_block();
            __syncwarp();                        // every lane's A writes precede the release
            if (lane == 0) mbar_arrive(&afull[b]);
            if (tk.x < 0) break;
        }
    } else if (warp == XW_CONS / 32) {
        // ---------------- producer ----------------
        uint32_t G = 0;   // B-ring stages issued (lane 0)
        for (uint32_t n = 0;; n++) {
            const int b = n & 1;
            mbar_wait(&afull[b], (n >> 1) & 1u);
            const int4 tk = task_s[b];
            if (tk.x < 0) break;
            if (lane == 0) {
                int32_t mem0[PT_MAXK];
                pt_unrank_colex((int64_t)tk.x * XT_R, p.m, p.C, mem0);
                int64_t col = tile_lo(mem0[p.m - 1]) + (int64_t)tk.y * XW_C;
                for (int ct = tk.y; ct < tk.z; ct++, col += XW_C) {
                    // 128 configs from `col` (8-aligned) = 64-config tiles c64 and c64 + 1 of
                    // shift sh (hTile carries one zero tile of padding past the last)
                    const int64_t sh = (col >> 3) & 7, c64 = (col - 8 * sh) >> 6;
                    const uint16_t *src = p.hTile + (sh * p.n_ct + c64) * p.E_pad * 64;
                    for (int q = 0; q < nkc; q++, G++) {
                        const int slot = G % XT_S;
                        mbar_wait(&empty[slot], ((G / XT_S) & 1u) ^ 1u);
                        mbar_expect_tx(&full[slot], 2 * XT_K * 128);
                        bulk_g2s(Bs + slot * 2 * XT_K * 32, src + (int64_t)q * XT_K * 64, XT_K * 128, &full[slot]);
                        bulk_g2s(Bs + (slot * 2 + 1) * XT_K * 32, src + (p.E_pad + (int64_t)q * XT_K) * 64,
                                 XT_K * 128, &full[slot]);
                    }
                }
            }
            __syncwarp();
        }
    } else {
        // ---------------- consumers ----------------
        const int tx = lane & 7, ty = lane >> 3;
        const int r0 = 32 * (warp >> 2) + 8 * ty;
        const int cq = warp & 3;                         // 32-column quarter of the tile
        const int c0 = 32 * cq + 4 * tx;                 // first of the thread's 4 columns
        const int c0h = c0 - 64 * (cq >> 1);             // ... within its 64-column half
        float bA = INFINITY, bB = INFINITY, published = INFINITY;   // acc-domain group minima (window U)
        uint32_t slot = 0, phase = 0;
        for (uint32_t n = 0;; n++) {
            const int b = n & 1;
            mbar_wait(&afull[b], (n >> 1) & 1u);
            const int4 tk = task_s[b];
            if (tk.x < 0) break;
            const int64_t R0 = (int64_t)tk.x * XT_R;
            const uint16_t *As = As0 + (int64_t)b * p.E_pad * XT_R;
            const int *last_s = last_s0 + b * XT_R;
            int32_t mem0[PT_MAXK];
            pt_unrank_colex(R0, p.m, p.C, mem0);
            // colex order: a row's largest member is non-decreasing in its rank (padding
            // rows hold INT_MAX), so the thread's last row bounds all eight
            const int last7 = last_s[r0 + 7];
            float acc[8][4];
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) acc[i][j] = 0.0f;
            int64_t ltile = tile_lo(mem0[p.m - 1]) + (int64_t)tk.y * XW_C;
            for (int ct = tk.y; ct < tk.z; ct++, ltile += XW_C) {
                const bool skip = ltile + 32 * cq >= p.C;   // the warp's quarter lies past the last config
                const unsigned Ubits = *(volatile unsigned *)p.U;
                for (int q = 0; q < nkc; q++) {
                    mbar_wait(&full[slot], phase);
                    if (!skip) {
                        const uint32_t *B = Bs + (slot * 2 + (cq >> 1)) * XT_K * 32 + c0h / 2;
                        const uint16_t *A = As + (int64_t)q * XT_K * XT_R + r0;
#pragma unroll kXtPUnroll
                        for (int e = 0; e < XT_K; e += 4 * XT_NG) {
                            uint32_t pp[8][2];
#pragma unroll
                            for (int gq = 0; gq < XT_NG; gq++) {
                                uint4 ar[4];
                                uint2 bc[4];
#pragma unroll
                                for (int t = 0; t < 4; t++) {
                                    ar[t] = *reinterpret_cast<const uint4 *>(A + (e + 4 * gq + t) * XT_R);
                                    bc[t] = *reinterpret_cast<const uint2 *>(B + (e + 4 * gq + t) * 32);
                                }
#pragma unroll
                                for (int i = 0; i < 8; i++) {
                                    uint32_t av[4];
#pragma unroll
                                    for (int t = 0; t < 4; t++) {
                                        const uint32_t w = (i >> 1) == 0 ? ar[t].x : (i >> 1) == 1 ? ar[t].y
                                                                         : (i >> 1) == 2 ? ar[t].z : ar[t].w;
                                        av[t] = (i & 1) ? bcast_hi(w) : bcast_lo(w);
                                    }
                                    const uint32_t sx = hadd2(hadd2(hmin2(av[0], bc[0].x), hmin2(av[1], bc[1].x)),
                                                              hadd2(hmin2(av[2], bc[2].x), hmin2(av[3], bc[3].x)));
                                    const uint32_t sy = hadd2(hadd2(hmin2(av[0], bc[0].y), hmin2(av[1], bc[1].y)),
                                                              hadd2(hmin2(av[2], bc[2].y), hmin2(av[3], bc[3].y)));
                                    if (gq == 0) {
                                        pp[i][0] = sx;
                                        pp[i][1] = sy;
                                    } else if (gq < XT_NG - 1) {
                                        pp[i][0] = hadd2(pp[i][0], sx);
                                        pp[i][1] = hadd2(pp[i][1], sy);
                                    } else {
                                        fhadd2(acc[i][0], acc[i][1], hadd2(pp[i][0], sx));
                                        fhadd2(acc[i][2], acc[i][3], hadd2(pp[i][1], sy));
                                    }
                                }
                            }
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[slot]);
                    if (++slot == XT_S) {
                        slot = 0;
                        phase ^= 1u;
                    }
                }
                if (skip) continue;
                // ---- epilogue of one column tile (as k_exh_tiled) ----
                const int64_t l0 = ltile + c0;
                if (!(l0 + 3 < p.C && l0 > last7)) {
#pragma unroll
                    for (int i = 0; i < 8; i++) {
                        const int last = last_s[r0 + i];
#pragma unroll
                        for (int j = 0; j < 4; j++)
                            if (!(l0 + j < p.C && l0 + j > last)) acc[i][j] = INFINITY;
                    }
                }
                float tA = fminf(acc[0][0], acc[0][1]), tB = fminf(acc[0][2], acc[0][3]);
#pragma unroll
                for (int i = 1; i < 8; i++) {
                    tA = fminf(tA, fminf(acc[i][0], acc[i][1]));
                    tB = fminf(tB, fminf(acc[i][2], acc[i][3]));
                }
                bA = fminf(bA, tA);
                bB = fminf(bB, tB);
                const float tau = fminf(p.tau_seed, __uint_as_float(Ubits));
                if (__fmaf_rd(fminf(tA, tB), p.c1, -p.c2) <= tau) {
#pragma unroll
                    for (int i = 0; i < 8; i++)
#pragma unroll
                        for (int j = 0; j < 4; j++) {
                            const float lb = __fmaf_rd(acc[i][j], p.c1, -p.c2);
                            if (acc[i][j] < INFINITY && lb <= tau) {
                                const unsigned idx = atomicAdd(p.cand_n, 1u);
                                if (idx < p.cap) {
                                    p.cand_key[idx] = ((unsigned long long)(R0 + r0 + i) << KEY_BITS) |
                                                      (unsigned long long)(l0 + j);
                                    p.cand_s[idx] = lb;
                                }
                            }
                        }
                }
#pragma unroll
                for (int i = 0; i < 8; i++)
#pragma unroll
                    for (int j = 0; j < 4; j++) acc[i][j] = 0.0f;
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
            __syncwarp();
            if (lane == 0) mbar_arrive(&aempty[b]);
        }
    }
}

// ---------------------------------------------------------------------------
// the tensor-summed (min,+) kernel (default)
//
// The mins stay on the ALU pipe (HMNMX2, two environments of one set per
// instruction); the across-environment sum of Eq. 1 moves to the legacy tensor
// path: the mins are laid out as the A fragment of mma.sync.m16n8k16 (f16 in,
// f32 accumulate, SASS HMMA.16816.F32) and B is a 0/1 selector,
//     B[k][n] = 1 iff (k < 8) == (n even),
// so output column n even accumulates A[m][0..7] and n odd A[m][8..15]: each
// MMA row carries TWO sets (its k < 8 and k >= 8 halves), and every thread's
// four accumulator registers are four different sets -- no wasted registers.
// Per thread and MMA: 4 HMNMX2 (4 sets x 1 env pair) + 1 HMMA; the 4 lanes of
// a quad hold the same 4 sets at 4 different env pairs (the MMA adds them).
// Measured (tools/ubench3.cu): HMMA.16816 issues at 0.5 per SM per clock, i.e.
// 256 mins / 8 cycles / SMSP -- exactly the HMNMX2 rate, so the two pipes are
// balanced and the issue port carries 0.67 instructions per (set, env) instead
// of 1.19 for the HADD2/FHADD tree.
// Numerics: the mins are exact fp16 values (min commutes with RN16), products
// by the selector's 1.0 are exact, and the only extra error is the tensor
// accumulation (measured <= 2.2 ulp per MMA, tools/mma_acc_probe.cu; the
// window assumes 2^-18 relative per MMA -- DESIGN.md "Numerics").
//
// CTA tile 32 rows x 64 columns; warp w: rows 8*(w>>1) .. +7 (shared by the
// warp's 8 quads: one broadcast LDS), columns 32*(w&1) + 4*quad .. +3.
// smem A: [E_pad/2][XM_R + 4] u32 env pairs (the +4 spreads the 4 lanes of a
// quad over distinct banks); B ring: XT_S stages of [XT_K/2][64] u32.
// ---------------------------------------------------------------------------
#define XM_AST (XM_R + 4)
#ifndef XM_VOL
#define XM_VOL 0    // 1: mma asm volatile (pins the MMA order)
#endif
#ifndef XM_UNROLL
#define XM_UNROLL 2
#endif
[[maybe_unused]] static constexpr int kXmUnroll = XM_UNROLL;
// bank swizzle of hPair: 16-byte chunk ch of env pair pp is stored at chunk
// ch ^ pair_swz(pp & 3) (see the B loads in k_exh_mma)
__host__ __device__ __forceinline__ int pair_swz(int q)
{
    return XM_TC == 8 ? ((q & 1) | ((q & 2) << 1)) : (q << 1);
}

__device__ __forceinline__ void mma_sum(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                        uint32_t b0, uint32_t b1)
{
#if XM_VOL
    asm volatile(
#else
    asm(
#endif
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

#ifndef XM_MAXREG
#define XM_MAXREG (XM_TC == 8 ? 112 : 96)   // 2 CTAs x 288 threads x 112 = 64,512 of 65,536 registers
#endif
__global__ void __maxnreg__(XM_MAXREG) k_exh_mma(const XParams p)
{
    extern __shared__ __align__(128) unsigned char smem[];
    uint32_t *Bs = reinterpret_cast<uint32_t *>(smem);                  // [S][XT_K/2][64]
    uint32_t *As = Bs + XT_S * (XT_K / 2) * XT_C;                       // [E_pad/2][XM_AST]
    int *last_s = reinterpret_cast<int *>(As + (p.E_pad / 2) * XM_AST);  // [XM_R]
    uint64_t *full = reinterpret_cast<uint64_t *>(last_s + XM_R);        // [S]
    uint64_t *empty = full + XT_S;                                       // [S]
    int4 *task_s = reinterpret_cast<int4 *>(empty + XT_S);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nkc = (int)(p.E_pad / XT_K);
    if (tid == 0) {
        for (int s = 0; s < XT_S; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], XT_CONS / 32);
        }
        mbar_fence_init();
    }
    __syncthreads();

    uint32_t steps = 0;
    const int g = lane >> 2, q = lane & 3;
    const int r0 = XM_TC == 8 ? 8 * warp : 8 * (warp >> 1);
    const int c0 = XM_TC == 8 ? 8 * g : 32 * (warp & 1) + 4 * g;
    const uint32_t one2 = 0x3C003C00u;
    const uint32_t sel0 = (g & 1) ? 0u : one2, sel1 = (g & 1) ? one2 : 0u;
    float b1 = INFINITY, published = INFINITY;

    for (;;) {
        if (tid == 0) {
            int ti = atomicAdd(p.task_ctr, 1);
            *task_s = ti < p.task_hi ? p.tasks[ti] : make_int4(-1, 0, 0, 0);
        }
        __syncthreads();
        const int4 tk = *task_s;
        if (tk.x < 0) break;
        const int64_t R0 = (int64_t)tk.x * XM_R;
        int32_t mem0[PT_MAXK];
        pt_unrank_colex(R0, p.m, p.C, mem0);
        const int64_t lo = tile_lo(mem0[p.m - 1]);
        const int nsteps = (tk.z - tk.y) * nkc;

        if (warp == XT_CONS / 32) {
            // ---------------- producer warp: one 8 KB bulk copy per stage ----------------
            if (lane == 0) {
                int qs = 0;
                int64_t col = lo + (int64_t)tk.y * XT_C;
                uint32_t G = steps;
                for (int gs = 0; gs < nsteps; gs++, G++) {
                    const int slot = G % XT_S;
                    const uint32_t par = ((G / XT_S) & 1u) ^ 1u;
                    mbar_wait(&empty[slot], par);
                    const int64_t sh = (col >> 3) & 7, ct = (col - 8 * sh) >> 6;
                    const uint32_t *src =
                        p.hPair + ((sh * p.n_ct + ct) * (p.E_pad / 2) + (int64_t)qs * (XT_K / 2)) * XT_C;
                    mbar_expect_tx(&full[slot], XT_K * XT_BROW);
                    bulk_g2s(Bs + slot * (XT_K / 2) * XT_C, src, XT_K * XT_BROW, &full[slot]);
                    if (++qs == nkc) {
                        qs = 0;
                        col += XT_C;
                    }
                }
            }
            __syncwarp();
        } else {
            // ---------------- consumers ----------------
            // stage A pairs: As[pp][r] = min over the row's members of (env 2pp, 2pp+1)
            {
                constexpr int TPR = XT_CONS / XM_R;   // staging threads per row
                const int r = tid / TPR, sub = tid % TPR;
                const int64_t R = R0 + r;
                int32_t mem[PT_MAXK];
                const bool valid = R < p.n_rows;
                if (valid) pt_unrank_colex(R, p.m, p.C, mem);
                else for (int u = 0; u < p.m; u++) mem[u] = 0;
                if (sub == 0) last_s[r] = valid ? mem[p.m - 1] : 0x7fffffff;
                for (int64_t ch = sub; ch < p.E_pad / 8; ch += TPR) {
                    uint4 v = __ldg(reinterpret_cast<const uint4 *>(p.hC + (int64_t)mem[0] * p.E_pad) + ch);
                    for (int u = 1; u < p.m; u++) {
                        const uint4 w =
                            __ldg(reinterpret_cast<const uint4 *>(p.hC + (int64_t)mem[u] * p.E_pad) + ch);
                        v.x = hmin2(v.x, w.x);
                        v.y = hmin2(v.y, w.y);
                        v.z = hmin2(v.z, w.z);
                        v.w = hmin2(v.w, w.w);
                    }
                    if (!valid) v = make_uint4(0, 0, 0, 0);
                    uint32_t *dst = As + 4 * ch * XM_AST + r;
                    dst[0] = v.x;
                    dst[XM_AST] = v.y;
                    dst[2 * XM_AST] = v.z;
                    dst[3 * XM_AST] = v.w;
                }
            }
            named_sync(1, XT_CONS);

            float acc[4][XM_TC / 2][4];
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < XM_TC / 2; j++)
#pragma unroll
                    for (int t = 0; t < 4; t++) acc[i][j][t] = 0.0f;

            int qs = 0;
            int64_t ltile = lo + (int64_t)tk.y * XT_C;
            uint32_t G = steps;
            for (int gs = 0; gs < nsteps; gs++, G++) {
                const int slot = G % XT_S;
                mbar_wait(&full[slot], (G / XT_S) & 1u);
                const bool skip = ltile + (XM_TC == 8 ? 0 : 32 * (warp & 1)) >= p.C;
                if (!skip) {
                    // hPair is stored swizzled (pair_swz): the 8 lanes of a quarter-warp
                    // phase (2 quads x 4 env pairs) hit 8 distinct bank groups
                    const uint32_t *B = Bs + slot * (XT_K / 2) * XT_C + q * XT_C +
                                        4 * ((c0 >> 2) ^ pair_swz(q));
#if XM_TC == 8
                    const uint32_t *B2 = Bs + slot * (XT_K / 2) * XT_C + q * XT_C +
                                         4 * (((c0 >> 2) + 1) ^ pair_swz(q));
#endif
                    const uint32_t *A = As + ((int64_t)qs * (XT_K / 2) + q) * XM_AST + r0;
#pragma unroll kXmUnroll
                    for (int kk = 0; kk < XT_K / 8; kk++) {
                        const uint4 al = *reinterpret_cast<const uint4 *>(A + 4 * kk * XM_AST);
                        const uint4 ah = *reinterpret_cast<const uint4 *>(A + 4 * kk * XM_AST + 4);
                        const uint4 bv = *reinterpret_cast<const uint4 *>(B + 4 * kk * XT_C);
                        const uint32_t a[8] = {al.x, al.y, al.z, al.w, ah.x, ah.y, ah.z, ah.w};
#if XM_TC == 8
                        const uint4 bw = *reinterpret_cast<const uint4 *>(B2 + 4 * kk * XT_C);
                        const uint32_t b[8] = {bv.x, bv.y, bv.z, bv.w, bw.x, bw.y, bw.z, bw.w};
#else
                        const uint32_t b[4] = {bv.x, bv.y, bv.z, bv.w};
#endif
#pragma unroll
                        for (int i = 0; i < 4; i++)
#pragma unroll
                            for (int j = 0; j < XM_TC / 2; j++)
                                mma_sum(acc[i][j], hmin2(a[2 * i], b[2 * j]), hmin2(a[2 * i + 1], b[2 * j]),
                                        hmin2(a[2 * i], b[2 * j + 1]), hmin2(a[2 * i + 1], b[2 * j + 1]),
                                        sel0, sel1);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[slot]);
                if (++qs == nkc) {
                    qs = 0;
                    if (!skip) {
                        // epilogue of one column tile.  The 4 lanes of a quad hold the same
                        // 32 sums; lane q takes row pair i = q (selected without branching,
                        // so all 32 lanes work on distinct sets).  Each lane tracks only its
                        // smallest upper bound b1; the warp's 2nd-smallest b1 bounds s_(2)
                        // (lanes own disjoint sets).
                        const float tau = fminf(p.tau_seed, __uint_as_float(*(volatile unsigned *)p.U));
                        const int lbase = (int)(ltile + c0);
                        const int last0 = last_s[r0 + 2 * q], last1 = last_s[r0 + 2 * q + 1];
#pragma unroll
                        for (int j = 0; j < XM_TC / 2; j++)
#pragma unroll
                            for (int t = 0; t < 4; t++) {
                                // acc[i][j]: {row 2i col 2j, row 2i col 2j+1, row 2i+1 col 2j, row 2i+1 col 2j+1}
                                const float sh = q == 0 ? acc[0][j][t] : q == 1 ? acc[1][j][t]
                                               : q == 2 ? acc[2][j][t] : acc[3][j][t];
                                const int l = lbase + 2 * j + (t & 1);
                                const int last = (t >> 1) ? last1 : last0;
                                if (l < (int)p.C && l > last) {
                                    b1 = fminf(b1, __fmaf_ru(sh, p.c3, p.c4));
                                    const float lb = __fmaf_rd(sh, p.c1, -p.c2);
                                    if (lb <= tau) {
                                        const unsigned idx = atomicAdd(p.cand_n, 1u);
                                        if (idx < p.cap) {
                                            const int r = r0 + 2 * q + (t >> 1);
                                            p.cand_key[idx] = ((unsigned long long)(R0 + r) << KEY_BITS) |
                                                              (unsigned long long)l;
                                            p.cand_s[idx] = lb;
                                        }
                                    }
                                }
                            }
#pragma unroll
                        for (int i = 0; i < 4; i++)
#pragma unroll
                            for (int j = 0; j < XM_TC / 2; j++)
#pragma unroll
                                for (int t = 0; t < 4; t++) acc[i][j][t] = 0.0f;
                        // warp: two smallest lane minima (merge of sorted pairs)
                        float m1 = b1, m2 = INFINITY;
                        for (int o = 16; o; o >>= 1) {
                            const float a1 = __shfl_xor_sync(0xffffffffu, m1, o);
                            const float a2 = __shfl_xor_sync(0xffffffffu, m2, o);
                            const float n1 = fminf(m1, a1);
                            m2 = fminf(fmaxf(m1, a1), fminf(m2, a2));
                            m1 = n1;
                        }
                        if (lane == 0 && m2 < published) {
                            atomicMin(p.U, __float_as_uint(m2));
                            published = m2;
                        }
                    }
                    ltile += XT_C;
                }
            }
        }
        steps += nsteps;
    }
}

// hC[c][e] = the same fp16(l64[c][e]) as hT, config-major (0 for padded configs)
__global__ void k_half_cfg(const double *__restrict__ l64, int64_t E, int64_t C, int64_t E_pad,
                           int64_t C_pad, uint16_t *__restrict__ hC)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= C_pad * E_pad) return;
    const int64_t c = i / E_pad, e = i % E_pad;
    hC[i] = (c < C && e < E) ? __half_as_ushort(__double2half(l64[c * E_pad + e])) : (uint16_t)0;
}

// hPair[s][ct][pp][j'] = hT[2pp][c] | hT[2pp+1][c] << 16, c = 64*ct + 8*s + j, stored at the
// swizzled position j' = 4*((j/4) ^ pair_swz(pp%4)) + j%4
__global__ void k_tile_pairs(const uint16_t *__restrict__ hT, int64_t E_pad, int64_t C_pad, int64_t n_ct,
                             uint32_t *__restrict__ hPair)
{
    const int64_t blk = blockIdx.x;                  // (s, ct, pp)
    const int64_t np = E_pad / 2;
    const int64_t pp = blk % np, sct = blk / np;
    const int64_t ct = sct % n_ct, sh = sct / n_ct;
    const int j = threadIdx.x;                       // 64 threads
    const int64_t c = 64 * ct + 8 * sh + j;
    uint32_t w = 0;
    if (c < C_pad) w = (uint32_t)hT[(2 * pp) * C_pad + c] | ((uint32_t)hT[(2 * pp + 1) * C_pad + c] << 16);
    hPair[blk * 64 + 4 * ((j >> 2) ^ pair_swz((int)(pp & 3))) + (j & 3)] = w;   // swizzled (see k_exh_mma)
}

// hTile[sh][ct][e][0..64) = hT[e][64 ct + 8 sh + 0..64) (zero past C_pad): one block
// per (sh, ct), 16-byte copies (C_pad and the 8-config shifts keep them aligned)
__global__ void __launch_bounds__(256) k_tile_hT(const uint16_t *__restrict__ hT, int64_t E_pad, int64_t C_pad,
                                                 int64_t n_ct, uint16_t *__restrict__ hTile)
{
    const int64_t sct = blockIdx.x, ct = sct % n_ct, sh = sct / n_ct;
    const int64_t c0 = 64 * ct + 8 * sh;
    uint4 *dst = reinterpret_cast<uint4 *>(hTile + sct * E_pad * 64);
    for (int64_t i = threadIdx.x; i < E_pad * 8; i += blockDim.x) {
        const int64_t e = i >> 3, c = c0 + 8 * (i & 7);
        const uint4 v = c < C_pad ? *reinterpret_cast<const uint4 *>(hT + e * C_pad + c) : make_uint4(0, 0, 0, 0);
#if XT_HALF
        dst[((i & 7) >> 2) * E_pad * 4 + e * 4 + (i & 3)] = v;   // [half][e][32]
#else
        dst[i] = v;
#endif
    }
}

// XT_TC layout of the same tiles: hTileP[sh][ct][pp][tc_cpos(j)] = f16x2(hT[2pp][c], hT[2pp+1][c]),
// c = 64 ct + 8 sh + j (zero past C_pad); same byte offsets per 64-env stage as hTile
__global__ void __launch_bounds__(256) k_tile_pp(const uint16_t *__restrict__ hT, int64_t E_pad, int64_t C_pad,
                                                 int64_t n_ct, uint32_t *__restrict__ hTileP)
{
    const int64_t sct = blockIdx.x, ct = sct % n_ct, sh = sct / n_ct;
    const int64_t c0 = 64 * ct + 8 * sh;
    uint32_t *dst = hTileP + sct * (E_pad / 2) * 64;
    for (int64_t i = threadIdx.x; i < (E_pad / 2) * 64; i += blockDim.x) {
        const int64_t pp = i >> 6;
        const int j = (int)(i & 63);
        const int64_t c = c0 + j;
        uint32_t w = 0;
        if (c < C_pad) w = (uint32_t)hT[(2 * pp) * C_pad + c] | ((uint32_t)hT[(2 * pp + 1) * C_pad + c] << 16);
        dst[pp * 64 + tc_cpos(j)] = w;
    }
}

// ---------------------------------------------------------------------------
// top-2 over (s, tuple) records -- one CTA
// ---------------------------------------------------------------------------
struct Rec2 {
    double s1, s2;
    int32_t t1[PT_MAXK], t2[PT_MAXK];
};

__device__ __forceinline__ void rec_offer(Rec2 &r, double s, const int32_t *t, int k)
{
    if (s == INFINITY) return;
    if (pt_key_less(s, t, r.s1, r.t1, k)) {
        r.s2 = r.s1;
        for (int u = 0; u < k; u++) r.t2[u] = r.t1[u];
        r.s1 = s;
        for (int u = 0; u < k; u++) r.t1[u] = t[u];
    } else if (pt_key_less(s, t, r.s2, r.t2, k)) {
        bool same = s == r.s1;
        for (int u = 0; u < k && same; u++) same = t[u] == r.t1[u];
        if (!same) {
            r.s2 = s;
            for (int u = 0; u < k; u++) r.t2[u] = t[u];
        }
    }
}

// n records, or min(*n_dev, cap) when n_dev is given (a device-side count)
__global__ void __launch_bounds__(256) k_top2(const double *__restrict__ s, const int32_t *__restrict__ t,
                                             int64_t n, const unsigned *__restrict__ n_dev, unsigned cap,
                                             int k, double *__restrict__ out_s, int32_t *__restrict__ out_t)
{
    if (n_dev) n = min(*n_dev, cap);
    __shared__ Rec2 sh[256];
    Rec2 r;
    r.s1 = r.s2 = INFINITY;
    for (int u = 0; u < PT_MAXK; u++) r.t1[u] = r.t2[u] = 0x7fffffff;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) rec_offer(r, s[i], t + i * k, k);
    sh[threadIdx.x] = r;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) {
            Rec2 o = sh[threadIdx.x + w];
            Rec2 me = sh[threadIdx.x];
            rec_offer(me, o.s1, o.t1, k);
            rec_offer(me, o.s2, o.t2, k);
            sh[threadIdx.x] = me;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out_s[0] = sh[0].s1;
        out_s[1] = sh[0].s2;
        for (int u = 0; u < k; u++) {
            out_t[u] = sh[0].t1[u];
            out_t[k + u] = sh[0].t2[u];
        }
    }
}

// fp64 refine of the survivors fused with their top-2: every block re-scores its
// share (warp per candidate, the same fixed shuffle tree as k_exh_refine), keeps a
// block top-2 and publishes it; the last block to finish (a counter it then resets)
// merges the block records.  One launch instead of refine + k_top2.
__global__ void __launch_bounds__(256) k_exh_refine_top2(
    const unsigned long long *__restrict__ key, const float *__restrict__ cs, const unsigned *__restrict__ n_dev,
    unsigned cap, float tau_pass, const unsigned *__restrict__ U, int m, int64_t C, const double *__restrict__ l64,
    int64_t E_pad, Rec2 *__restrict__ blk, unsigned *__restrict__ done, double *__restrict__ out_s,
    int32_t *__restrict__ out_t)
{
    const int64_t n = min(*n_dev, cap);
    const float tau = fminf(tau_pass, __uint_as_float(*U));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int k = m + 1;
    __shared__ Rec2 sh[256];
    Rec2 r;
    r.s1 = r.s2 = INFINITY;
    for (int u = 0; u < PT_MAXK; u++) r.t1[u] = r.t2[u] = 0x7fffffff;
    for (int64_t w = (int64_t)blockIdx.x * 8 + warp; w < n; w += (int64_t)gridDim.x * 8) {
        int32_t tup[PT_MAXK];
        const unsigned long long kv = key[w];
        pt_unrank_colex((int64_t)(kv >> KEY_BITS), m, C, tup);
        tup[m] = (int32_t)(kv & ((1ull << KEY_BITS) - 1));
        if (cs[w] > tau) continue;
        double acc = 0.0;
        for (int64_t e = lane; e < E_pad; e += 32) {
            double v = l64[(int64_t)tup[0] * E_pad + e];
            for (int u = 1; u < k; u++) v = fmin(v, l64[(int64_t)tup[u] * E_pad + e]);
            acc += v;
        }
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) rec_offer(r, acc, tup, k);
    }
    sh[threadIdx.x] = r;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) {
            Rec2 o = sh[threadIdx.x + w];
            Rec2 me = sh[threadIdx.x];
            rec_offer(me, o.s1, o.t1, k);
            rec_offer(me, o.s2, o.t2, k);
            sh[threadIdx.x] = me;
        }
        __syncthreads();
    }
    __shared__ bool last;
    if (threadIdx.x == 0) {
        blk[blockIdx.x] = sh[0];
        __threadfence();
        last = atomicAdd(done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    r.s1 = r.s2 = INFINITY;
    for (int u = 0; u < PT_MAXK; u++) r.t1[u] = r.t2[u] = 0x7fffffff;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
        Rec2 o;   // L2 reads (other blocks' records; L1 is not coherent)
        o.s1 = __ldcg(&blk[b].s1);
        o.s2 = __ldcg(&blk[b].s2);
        for (int u = 0; u < k; u++) {
            o.t1[u] = __ldcg(&blk[b].t1[u]);
            o.t2[u] = __ldcg(&blk[b].t2[u]);
        }
        rec_offer(r, o.s1, o.t1, k);
        rec_offer(r, o.s2, o.t2, k);
    }
    sh[threadIdx.x] = r;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) {
            Rec2 o = sh[threadIdx.x + w];
            Rec2 me = sh[threadIdx.x];
            rec_offer(me, o.s1, o.t1, k);
            rec_offer(me, o.s2, o.t2, k);
            sh[threadIdx.x] = me;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out_s[0] = sh[0].s1;
        out_s[1] = sh[0].s2;
        for (int u = 0; u < k; u++) {
            out_t[u] = sh[0].t1[u];
            out_t[k + u] = sh[0].t2[u];
        }
        *done = 0;   // ready for the next launch
    }
}

// ---------------------------------------------------------------------------
// generic fp64 thread-per-subset kernel: block -> its top-2 records
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_exh_generic(const double *__restrict__ l64, int64_t C,
                                                    int64_t E_pad, int k, int64_t r0, int64_t r1,
                                                    double *__restrict__ blk_s,
                                                    int32_t *__restrict__ blk_t)
{
    __shared__ Rec2 sh[256];
    Rec2 r;
    r.s1 = r.s2 = INFINITY;
    for (int u = 0; u < PT_MAXK; u++) r.t1[u] = r.t2[u] = 0x7fffffff;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t R = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; R < r1; R += stride) {
        int32_t tup[PT_MAXK];
        pt_unrank_colex(R, k, C, tup);
        double acc = 0.0;
        for (int64_t e = 0; e < E_pad; e++) {
            double v = l64[(int64_t)tup[0] * E_pad + e];
            for (int u = 1; u < k; u++) v = fmin(v, l64[(int64_t)tup[u] * E_pad + e]);
            acc += v;
        }
        rec_offer(r, acc, tup, k);
    }
    sh[threadIdx.x] = r;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) {
            Rec2 o = sh[threadIdx.x + w];
            Rec2 me = sh[threadIdx.x];
            rec_offer(me, o.s1, o.t1, k);
            rec_offer(me, o.s2, o.t2, k);
            sh[threadIdx.x] = me;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        blk_s[2 * blockIdx.x] = sh[0].s1;
        blk_s[2 * blockIdx.x + 1] = sh[0].s2;
        for (int u = 0; u < k; u++) {
            blk_t[(2 * blockIdx.x) * k + u] = sh[0].t1[u];
            blk_t[(2 * blockIdx.x + 1) * k + u] = sh[0].t2[u];
        }
    }
}

// the exhaustive search's threshold seeded from a device-resident greedy runner-up score
// (rounded up, as f_up on the host path)
__global__ void k_seed_U(const double *__restrict__ s2, unsigned *__restrict__ U)
{
    *U = __float_as_uint(__double2float_ru(*s2 * (1.0 + 1e-9) + 1e-30));
}

// one-CTA (s, tuple) top-2 over n records on the device -> host
pt_status pt_top2_records(pt_ctx *ctx, const double *d_s, const int32_t *d_t, int64_t n, int k,
                          double *s_out, int32_t *t_out)
{
    double *os = nullptr;
    int32_t *ot = nullptr;
    PT_TRY(pt_dalloc(ctx, (void **)&os, sizeof(double) * 2));
    PT_TRY(pt_dalloc(ctx, (void **)&ot, sizeof(int32_t) * 2 * k));
    k_top2<<<1, 256, 0, ctx->stream>>>(d_s, d_t, n, nullptr, 0, k, os, ot);
    ctx->stats.launches++;
    PT_CK(cudaGetLastError());
    pt_hostio io(ctx);
    PT_TRY(io.d2h(s_out, os, sizeof(double) * 2));
    PT_TRY(io.d2h(t_out, ot, sizeof(int32_t) * 2 * k));
    pt_dfree(ctx, os);
    pt_dfree(ctx, ot);
    PT_TRY(io.finish());
    return PT_OK;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static pt_status run_generic(pt_ctx *ctx, const pt_view *v, int k, int64_t r0, int64_t r1,
                             double *s_out, int32_t *t_out)
{
    cudaStream_t s = ctx->stream;
    const int64_t n = r1 - r0;
    const int nblk = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 8));
    size_t off = 0;
    auto take = [&](size_t b) { size_t o = off; off += pt_round_up(b, 256); return o; };
    const size_t o_bs = take(sizeof(double) * 2 * nblk), o_bt = take(sizeof(int32_t) * 2 * nblk * k),
                 o_os = take(sizeof(double) * 2), o_ot = take(sizeof(int32_t) * 2 * k);
    void *scr = nullptr;
    PT_TRY(pt_scratch(ctx, off, &scr));
    char *b = (char *)scr;
    double *bs = (double *)(b + o_bs), *os = (double *)(b + o_os);
    int32_t *bt = (int32_t *)(b + o_bt), *ot = (int32_t *)(b + o_ot);
    PT_CK(cudaEventRecord(ctx->ev0, s));
    k_exh_generic<<<nblk, 256, 0, s>>>(v->l64, v->C, v->E_pad, k, r0, r1, bs, bt);
    PT_CK(cudaEventRecord(ctx->ev1, s));
    k_top2<<<1, 256, 0, s>>>(bs, bt, 2 * nblk, nullptr, 0, k, os, ot);
    ctx->stats.launches += 2;
    pt_pack_record(ctx, os, ot, k);
    PT_CK(cudaGetLastError());
    pt_hostio io(ctx);
    PT_TRY(io.d2h(s_out, os, sizeof(double) * 2));
    PT_TRY(io.d2h(t_out, ot, sizeof(int32_t) * 2 * k));
    PT_TRY(io.finish());
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    ctx->stats.exh_main_ms = ms;
    ctx->stats.exh_kernel = 1;
    ctx->stats.exh_sets = n;
    ctx->stats.exh_slots = n;
    ctx->stats.exh_env_pad = v->E_pad;
    ctx->stats.exh_candidates = 0;
    ctx->stats.exh_passes = 1;
    return PT_OK;
}

static pt_status run_tiled(pt_ctx *ctx, const pt_view *v, int k, int32_t shard_rank,
                           int32_t shard_count, double *s_out, int32_t *t_out)
{
    // PT_TRACE=1 (development): host timestamps of the call's phases on stderr
    static const bool trace = getenv("PT_TRACE") != nullptr;
    const auto t_entry = std::chrono::steady_clock::now();
    auto mark = [&](const char *what) {
        if (trace)
            fprintf(stderr, "[pt k=%d] %-12s %8.1f us\n", k, what,
                    std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_entry).count());
    };
    cudaStream_t s = ctx->stream;
    const int m = k - 1;
    pt_tasks *T = nullptr;
    const bool ws = XW_ENABLE && !XT_MMA && v->E_pad <= XW_EMAX;   // warp-specialised kernel (A double-buffered)
    PT_TRY(build_tasks(ctx, v, m, XT_MMA ? XM_R : XT_R, ws ? XW_C : XT_C, &T));
    const int n_tasks = (int)T->h.size();
    // this shard's tasks: the whole list, or its snake-dealt part (shard_plan)
    const int4 *task_list = T->d;
    int ta = 0, tb = n_tasks;
    ctx->stats.exh_sets = T->set_pre.back();
    ctx->stats.exh_slots = T->slot_pre.back();
    if (shard_count > 1) {
        const pt_tasks::plan *P = nullptr;
        static const std::vector<double> equal;
        PT_TRY(shard_plan(T, shard_count, (int)ctx->shard_w.size() == shard_count ? ctx->shard_w : equal, &P));
        task_list = P->d;
        ta = P->off[shard_rank];
        tb = P->off[shard_rank + 1];
        ctx->stats.exh_sets = P->sets[shard_rank];
        ctx->stats.exh_slots = P->slots[shard_rank];
    }
    ctx->stats.exh_kernel = 0;   // (2 below for the tcgen05 kernel)
    ctx->stats.exh_env_pad = v->E_pad;
    ctx->stats.exh_candidates = 0;
    ctx->stats.exh_passes = 0;
    ctx->stats.exh_main_ms = 0.0;
    s_out[0] = s_out[1] = INFINITY;
    if (ta >= tb) return PT_OK;

    // error model of the fp16 tier; per set:
    //   min form : |s_hat - s| <= eta_rel * s + eta_abs
    //              (fp16 terms u16, 2-level fp16 tree 2 u16, fp32 sum of E_pad/4 groups)
    //   relu form: s_hat = sum_e a - sum_e relu(a-b): |s_hat - s| <= eta_A * sumA + eta_abs_r
    //              (u16 quantisation + relu rounding u16 + tree 2 u16 + fp32 sums + the
    //              final subtraction, all relative to sumA >= s)
    // The kernel turns them into a lower bound LB <= s <= UB per set (directed rounding)
    // and keeps every set with LB <= min(tau_seed, U), U = smallest 2nd-best UB seen.
    const double u16 = std::ldexp(1.0, -11), u32 = std::ldexp(1.0, -24);
    // envs per fp32 addition and fp16 rounding levels per term (quantisation + tree + fp16 chain)
    const double env_per_add = XT_G8 == 2 ? 4.0 * XT_NG : XT_G8 ? 8.0 : 4.0;
    const double lv16 = XT_G8 == 2 ? 2.0 + XT_NG : XT_G8 ? 4.0 : 3.0;
    const double ngrp = (double)v->E_pad / env_per_add + 2.0;
    const double gam = ngrp * u32 / (1.0 - ngrp * u32);
    const double gamE = ((double)v->E_pad + 2.0) * u32 / (1.0 - ((double)v->E_pad + 2.0) * u32);
    // quantisation u16 + a (2 or 3)-level fp16 tree
    const double eta_rel16 = (lv16 * u16 + lv16 * lv16 * u16 * u16 + gam) * 1.01;
    const double eta_abs16 = 3.0 * (double)v->E_pad * std::ldexp(1.0, -25) * 1.01;
    // relu form: quantisation of A and B (2 u16 sumA: relu is 1-Lipschitz and nonzero only
    // where b < a), sumA's own quantisation (u16), and L16 + 1 fp16 roundings on the relu
    // terms (HFMA2 + tree + chain), all relative to sumA >= s; plus the fp32 sums
#if XT_TC == 3
    // relu sets of the hybrid: quantisation of a and b (2 u16, relu is 1-Lipschitz), the
    // HFMA2.RELU rounding and the 7 HADD2 of the 8-pair chain (8 u16), all relative to
    // sumA >= s; the FHADD sums (E_pad/16 adds) and sumA's own fp32 sum and quantisation
    const double lvr = 11.0;
    const double n32r = (double)v->E_pad / 16.0 + 3.0;
    const double gamr = n32r * u32 / (1.0 - n32r * u32);
    const double eta_A = (lvr * u16 + lvr * lvr * u16 * u16 + u16 + gamr + 2.0 * gamE + 4.0 * u32) * 1.05;
#else
    const double lvr = lv16 + 3.0;
    const double eta_A = (lvr * u16 + lvr * lvr * u16 * u16 + gam + 2.0 * gamE + 4.0 * u32) * 1.02;
#endif
    const double eta_abs_r = 4.0 * (double)v->E_pad * std::ldexp(1.0, -25) * 1.01;
    auto f_up = [](double x) -> float {
        if (!(x < 3.0e38)) return INFINITY;
        float f = (float)x;
        if ((double)f < x) f = nextafterf(f, INFINITY);
        return f;
    };
    auto f_dn = [](double x) -> float {
        float f = (float)x;
        if ((double)f > x) f = nextafterf(f, -INFINITY);
        return f;
    };
    // seed: exact score of greedy's runner-up set at its last step (>= s_(2))
    // (reused from an earlier greedy run of >= k steps on this view when there is one)
    // (a missing trace is computed for 4 steps -- the tiled kernel's largest k -- at once,
    // so a k=2 search followed by a k=3 one seeds both from one cooperative greedy launch)
    // (development knob PT_EXH_SEED=none: no seed, the window starts at +inf and
    // tightens only through the kernel's own U)
    // Without a host trace the seed greedy is only enqueued: its runner-up trace stays on
    // the device and a one-thread kernel writes the rounded-up seed into U before the
    // search (U is itself an upper bound of s_(2), so min(seed, U) is one), no host
    // round trip between the two.
    static const bool no_seed = getenv("PT_EXH_SEED") && !strcmp(getenv("PT_EXH_SEED"), "none");
    float tau_seed = INFINITY;
    const double *seed_dev = nullptr;
    if (!no_seed) {
        if (v->greedy_s2.size() >= (size_t)k) {
            tau_seed = f_up(v->greedy_s2[k - 1] * (1.0 + 1e-9) + 1e-30);
        } else {
            const int kg = (int)std::min<int64_t>(std::max(k, 3), v->C);   // a k=2 search leaves k=3's seed
            if (v->d_seed_k < k && pt_greedy_seed_enqueue(ctx, v, kg) != PT_OK) {
                std::vector<int32_t> gidx(kg);
                std::vector<double> gs1(kg), gs2(kg);
                PT_TRY(pt_greedy_view(ctx, v, kg, gidx.data(), gs1.data(), gs2.data()));
                tau_seed = f_up(v->greedy_s2[k - 1] * (1.0 + 1e-9) + 1e-30);
            } else {
                seed_dev = v->d_seed_s2 + (k - 1);
            }
        }
    }
#if XT_MMA
    // tensor-summed kernel: fp16 terms u16 (the mins are exact fp16 values), then
    // E_pad/8 chained MMA accumulations, each assumed within 2^-18 relative of
    // its exact result (measured worst 2^-22.1, tools/mma_acc_probe.cu)
    const double n_mma = (double)v->E_pad / 8.0, d_mma = std::ldexp(1.0, -18);
    const double gam_mma = n_mma * d_mma / (1.0 - n_mma * d_mma);
    const double eta_rel = (u16 + gam_mma + u16 * gam_mma) * 1.01;
    const double eta_abs = (double)v->E_pad * std::ldexp(1.0, -25) * (1.0 + gam_mma) * 1.01;
#elif XT_TC >= 2
    // hybrid: a set is summed either by MMA (E_pad/2 chained MMAs, 2^-18 each, as below)
    // or by fp16 chains of 8 pairs (quantisation + 7 HADD2 = 8 roundings per term) into
    // fp32 (E_pad/16 FHADD per set); bounded by the sum of both relative terms
    const double n_mma = (double)v->E_pad / 2.0, d_mma = std::ldexp(1.0, -18);
    const double gam_mma = n_mma * d_mma / (1.0 - n_mma * d_mma);
    const double n32 = (double)v->E_pad / 16.0 + 3.0;
    const double gam32 = n32 * u32 / (1.0 - n32 * u32);
    const double eta_rel = (8.0 * u16 + 64.0 * u16 * u16 + gam32 + gam_mma + u16 * gam_mma) * 1.02;
    const double eta_abs = 3.0 * (double)v->E_pad * std::ldexp(1.0, -25) * (1.0 + gam_mma) * 1.02;
#elif XT_TC
    // tensor-summed tiled kernel: fp16 terms u16 (the mins are exact fp16 values), then
    // E_pad/2 chained MMA accumulations of one env pair each, each assumed within 2^-18
    // relative of its exact result (as k_exh_mma; measured worst 2^-22.1)
    const double n_mma = (double)v->E_pad / 2.0, d_mma = std::ldexp(1.0, -18);
    const double gam_mma = n_mma * d_mma / (1.0 - n_mma * d_mma);
    const double eta_rel = (u16 + gam_mma + u16 * gam_mma) * 1.01;
    const double eta_abs = (double)v->E_pad * std::ldexp(1.0, -25) * (1.0 + gam_mma) * 1.01;
#else
    const double eta_rel = eta_rel16, eta_abs = eta_abs16;
#endif
    const double eta_rel_k = eta_rel, eta_abs_k = eta_abs;
    const double c1d = 1.0 / (1.0 + eta_rel_k), c3d = 1.0 / (1.0 - eta_rel_k);
    const float c1 = f_dn(c1d), c2 = f_up(eta_abs_k), c3 = f_up(c3d), c4 = f_up(eta_abs_k * c3d * (1.0 + 1e-6));

    if (v->E_pad % XT_K != 0)   // a stage must not straddle the padded env range
        return pt_fail(PT_EINVAL, "E_pad=%lld is not a multiple of the stage depth %d", (long long)v->E_pad, XT_K);
    mark("seeded");
    PT_TRY(pt_view_fp16(ctx, v));
    if (!v->hTile) {
        pt_view *mv = const_cast<pt_view *>(v);
        // 64-config tiles, plus one zero tile so a 128-config stage (k_exh_ws) never
        // reads past the end
        mv->n_ct = (v->C_pad + XT_C - 1) / XT_C + 1;
        PT_TRY(pt_dalloc(ctx, (void **)&mv->hTile, sizeof(uint16_t) * 8 * mv->n_ct * v->E_pad * XT_C));
#if XT_TC
        k_tile_pp<<<(unsigned)(8 * mv->n_ct), 256, 0, s>>>(v->hT, v->E_pad, v->C_pad, mv->n_ct,
                                                           reinterpret_cast<uint32_t *>(mv->hTile));
#else
        k_tile_hT<<<(unsigned)(8 * mv->n_ct), 256, 0, s>>>(v->hT, v->E_pad, v->C_pad, mv->n_ct, mv->hTile);
#endif
        ctx->stats.launches++;
        PT_CK(cudaGetLastError());
    }
#if XT_MMA
    if (!v->hC) {
        pt_view *mv = const_cast<pt_view *>(v);
        PT_TRY(pt_dalloc(ctx, (void **)&mv->hC, sizeof(uint16_t) * v->E_pad * v->C_pad));
        k_half_cfg<<<(unsigned)((v->C_pad * v->E_pad + 255) / 256), 256, 0, s>>>(v->l64, v->E, v->C, v->E_pad,
                                                                                v->C_pad, mv->hC);
        ctx->stats.launches++;
    }
    if (!v->hPair) {
        pt_view *mv = const_cast<pt_view *>(v);
        PT_TRY(pt_dalloc(ctx, (void **)&mv->hPair, sizeof(uint32_t) * 8 * mv->n_ct * (v->E_pad / 2) * XT_C));
        k_tile_pairs<<<(unsigned)(8 * mv->n_ct * (v->E_pad / 2)), 64, 0, s>>>(v->hT, v->E_pad, v->C_pad,
                                                                            mv->n_ct, mv->hPair);
        ctx->stats.launches++;
        PT_CK(cudaGetLastError());
    }
    auto kern = k_exh_mma;
    const size_t smem = sizeof(uint32_t) * XT_S * (XT_K / 2) * XT_C + sizeof(uint32_t) * (v->E_pad / 2) * XM_AST +
                        sizeof(int) * XM_R + 2 * sizeof(uint64_t) * XT_S + sizeof(int4);
#else
    auto kern = ws ? k_exh_ws : k_exh_tiled;
    const size_t smem =
        ws ? sizeof(uint32_t) * XT_S * 2 * XT_K * 32 + 2 * sizeof(uint16_t) * v->E_pad * XT_R +
                 2 * sizeof(int) * XT_R + 2 * sizeof(int4) + 2 * sizeof(uint64_t) * (XT_S + 2)
           : sizeof(uint32_t) * XT_S * XT_K * (XT_C / 2) + sizeof(uint16_t) * v->E_pad * XT_R +
                 sizeof(int) * XT_R + (XT_TC == 3 ? 2 * sizeof(float) * XT_R : 0) + 4 * sizeof(uint64_t) * XT_S +
                 sizeof(int4) + 2 * sizeof(int) * XT_S;
#endif
    const void *kfn = (const void *)kern;
    const size_t smem_k = smem;
    const int threads = XT_MMA ? XT_THREADS : ws ? XW_THREADS : XT_TTHREADS;
    // per (kernel, smem) once per process: the attribute and the occupancy query
    static std::mutex attr_mu;
    static std::map<std::pair<const void *, size_t>, int> attr_occ;
    int occ = 1;
    {
        std::lock_guard<std::mutex> g(attr_mu);
        auto key = std::make_pair(kfn, smem_k);
        auto it = attr_occ.find(key);
        if (it == attr_occ.end()) {
            PT_CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_k));
            PT_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, threads, smem_k));
            attr_occ[key] = occ;
        } else {
            occ = it->second;
        }
    }

    unsigned cap = 1u << 20;
    unsigned n_cand = 0;
    float tau_pass = tau_seed;
    for (int pass = 0; pass < 2; pass++) {
        size_t off = 0;
        auto take = [&](size_t b) { size_t o = off; off += pt_round_up(b, 256); return o; };
        const size_t o_ctr = take(sizeof(int)), o_U = take(sizeof(unsigned)),
                     o_n = take(sizeof(unsigned)), o_key = take(sizeof(unsigned long long) * cap),
                     o_cq = take(sizeof(float) * cap),
                     o_os = take(sizeof(double) * 2), o_ot = take(sizeof(int32_t) * 2 * k),
                     o_blk = take(sizeof(Rec2) * (size_t)ctx->num_sms * 2), o_done = take(sizeof(unsigned));
        void *scr = nullptr;
        PT_TRY(pt_scratch(ctx, off, &scr));
        char *b = (char *)scr;
        int *ctr = (int *)(b + o_ctr);
        unsigned *U = (unsigned *)(b + o_U), *cn = (unsigned *)(b + o_n);
        unsigned long long *ckey = (unsigned long long *)(b + o_key);
        float *cq = (float *)(b + o_cq);
        double *os = (double *)(b + o_os);
        int32_t *ot = (int32_t *)(b + o_ot);
        Rec2 *blk = (Rec2 *)(b + o_blk);
        unsigned *done = (unsigned *)(b + o_done);
        const unsigned u_init = 0x7f800000u;   // +inf
        pt_hostio io(ctx);
        PT_TRY(io.h2d(ctr, &ta, sizeof(int)));
        if (seed_dev) {
            k_seed_U<<<1, 1, 0, s>>>(seed_dev, U);
            ctx->stats.launches++;
        } else {
            PT_TRY(io.h2d(U, &u_init, sizeof(unsigned)));
        }
        PT_CK(cudaMemsetAsync(cn, 0, sizeof(unsigned), s));
        PT_CK(cudaMemsetAsync(done, 0, sizeof(unsigned), s));
        XParams p;
        p.C = v->C;
        p.C_pad = v->C_pad;
        p.E_pad = v->E_pad;
        p.n_rows = pt_binom(v->C, m);
        p.m = m;
        p.tasks = task_list;
        p.task_hi = tb;
        p.task_ctr = ctr;
        p.tau_seed = tau_pass;
        p.c1 = c1;
        p.c2 = c2;
        p.c3 = c3;
        p.c4 = c4;
        p.eta_A = f_up(eta_A);
        p.eta_abs_r = f_up(eta_abs_r);
        p.U = U;
        p.cand_key = ckey;
        p.cand_s = cq;
        p.cand_n = cn;
        p.cap = cap;
        p.hT = v->hT;
        p.hTile = v->hTile;
        p.n_ct = v->n_ct;
        p.hC = v->hC;
        p.hPair = v->hPair;
        const int grid = std::min(ctx->num_sms * std::max(occ, 1), tb - ta);
#if XT_PROBE
        PT_CK(cudaMemsetAsync(cq + cap - 8, 0, 32, s));
#endif
        mark("pre-launch");
        PT_CK(cudaEventRecord(ctx->ev0, s));
        kern<<<grid, threads, smem, s>>>(p);
        PT_CK(cudaEventRecord(ctx->ev1, s));
        ctx->stats.launches++;
        PT_CK(cudaGetLastError());
        // refine + top-2 run on the device-side survivor count (no host round trip);
        // one synchronisation returns the count, U and the exact top-2
        k_exh_refine_top2<<<(unsigned)(ctx->num_sms * 2), 256, 0, s>>>(ckey, cq, cn, cap, tau_pass, U, m, v->C,
                                                                        v->l64, v->E_pad, blk, done, os, ot);
        ctx->stats.launches++;
        mark("launched");
        pt_pack_record(ctx, os, ot, k);   // sharded search: this rank's record stays on the device
        PT_CK(cudaGetLastError());
        unsigned hU = 0;
        PT_TRY(io.d2h(&n_cand, cn, sizeof(unsigned)));
        PT_TRY(io.d2h(&hU, U, sizeof(unsigned)));
        PT_TRY(io.d2h(s_out, os, sizeof(double) * 2));
        PT_TRY(io.d2h(t_out, ot, sizeof(int32_t) * 2 * k));
        PT_TRY(io.finish());
        mark("synced");
#if XT_PROBE
        {
            unsigned long long w[4];
            cudaMemcpy(w, cq + cap - 8, 32, cudaMemcpyDeviceToHost);
            fprintf(stderr, "XT_PROBE k=%d waits: task-first %llu tile-first %llu other %llu of %llu stage waits\n", k,
                    w[0], w[1], w[2], w[3]);
        }
#endif
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        if (pass == 0) ctx->stats.exh_main_ms = ms;
        ctx->stats.exh_passes = pass + 1;
        float Uf;
        memcpy(&Uf, &hU, sizeof Uf);
        if (n_cand > cap) {
            // overflow: rerun with the final threshold and room for every survivor
            cap = n_cand;
            tau_pass = std::min(tau_pass, Uf);
            continue;
        }
        ctx->stats.exh_candidates = n_cand;
        if (n_cand == 0) {
            s_out[0] = s_out[1] = INFINITY;
            for (int u = 0; u < 2 * k; u++) t_out[u] = 0;
        }
        return PT_OK;
    }
    return pt_fail(PT_ECUDA, "candidate buffer overflowed twice (internal error)");
}

pt_status pt_exhaustive_view(pt_ctx *ctx, const pt_view *v, int32_t k, int32_t shard_rank,
                             int32_t shard_count, int32_t *best, int32_t *runner, double *s_out,
                             int *n_found)
{
    if (k < 1 || k > v->C) return pt_fail(PT_EINVAL, "k=%d outside [1, %lld]", k, (long long)v->C);
    if (shard_count < 1 || shard_rank < 0 || shard_rank >= shard_count)
        return pt_fail(PT_EINVAL, "bad shard %d of %d", shard_rank, shard_count);
    if (k == v->C) {
        // the only k-subset is every configuration
        std::vector<int32_t> all(k);
        for (int u = 0; u < k; u++) all[u] = u;
        int32_t *d_set = nullptr;
        double *d_s = nullptr;
        PT_CK(cudaMallocAsync((void **)&d_set, sizeof(int32_t) * k, ctx->stream));
        PT_CK(cudaMallocAsync((void **)&d_s, sizeof(double), ctx->stream));
        PT_CK(cudaMemcpyAsync(d_set, all.data(), sizeof(int32_t) * k, cudaMemcpyHostToDevice, ctx->stream));
        PT_TRY(pt_score_view(ctx, v, d_set, 1, k, d_s));
        PT_CK(cudaMemcpyAsync(s_out, d_s, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        PT_CK(cudaFreeAsync(d_set, ctx->stream));
        PT_CK(cudaFreeAsync(d_s, ctx->stream));
        PT_CK(cudaStreamSynchronize(ctx->stream));
        s_out[1] = INFINITY;
        for (int u = 0; u < k; u++) {
            best[u] = u;
            if (runner) runner[u] = -1;
        }
        if (n_found) *n_found = shard_rank == 0 ? 1 : 0;
        if (shard_rank != 0) s_out[0] = INFINITY;
        return PT_OK;
    }
    if (k > PT_MAXK) return pt_fail(PT_EINVAL, "k=%d above the supported maximum %d", k, PT_MAXK);
    const double nsets = std::exp(std::lgamma((double)v->C + 1) - std::lgamma((double)k + 1) -
                                  std::lgamma((double)(v->C - k) + 1));
    if (nsets > 1e13) return pt_fail(PT_ECAP, "C(%lld,%d) = %.3g exceeds the cap 1e13", (long long)v->C, k, nsets);
    std::vector<int32_t> t(2 * k, 0);
    double sv[2] = {INFINITY, INFINITY};
    const bool tiled = !(ctx->flags & PT_EXACT_FP64) && k >= 2 && k <= 4 && v->E_pad <= XT_EMAX &&
                       v->C > k;
    if (tiled) {
        PT_TRY(run_tiled(ctx, v, k, shard_rank, shard_count, sv, t.data()));
    } else {
        const int64_t n = pt_binom(v->C, k);
        const int64_t r0 = n * shard_rank / shard_count, r1 = n * (shard_rank + 1) / shard_count;
        if (r1 > r0) PT_TRY(run_generic(ctx, v, k, r0, r1, sv, t.data()));
    }
    int nf = (sv[0] != INFINITY) + (sv[1] != INFINITY);
    if (n_found) *n_found = nf;
    for (int u = 0; u < k; u++) {
        best[u] = t[u];
        if (runner) runner[u] = t[k + u];
    }
    s_out[0] = sv[0];
    s_out[1] = sv[1];
    return PT_OK;
}

extern "C" pt_status pt_exhaustive_best(pt_ctx *ctx, int32_t k, const uint8_t *env_mask,
                                        int32_t objective, int32_t shard_rank, int32_t shard_count,
                                        int32_t *out_idx, double *out_G, int32_t *out_runner_idx,
                                        double *out_G_runner, double *out_s)
{
    PT_NVTX();
    if (!ctx || !out_idx || !out_G) return pt_fail(PT_EINVAL, "NULL argument");
    if (objective != PT_OBJ_GEOMEAN && objective != PT_OBJ_FLEET)
        return pt_fail(PT_EINVAL, "unknown objective %d", objective);
    PT_CK(cudaSetDevice(ctx->dev));
    if (objective == PT_OBJ_FLEET) {
        std::vector<int32_t> runner(k > 0 ? k : 1);
        double R[2], cost[2];
        int nf = 0;
        PT_TRY(pt_fleet_exhaustive(ctx, k, env_mask, shard_rank, shard_count, out_idx, runner.data(),
                                   R, cost, &nf));
        *out_G = R[0];
        if (out_runner_idx)
            for (int u = 0; u < k; u++) out_runner_idx[u] = runner[u];
        if (out_G_runner) *out_G_runner = R[1];
        if (out_s) {
            out_s[0] = cost[0];
            out_s[1] = cost[1];
        }
        return PT_OK;
    }
    const pt_view *v = nullptr;
    PT_TRY(pt_get_view(ctx, env_mask, &v));
    std::vector<int32_t> runner(k > 0 ? k : 1);
    double sv[2];
    int nf = 0;
    PT_TRY(pt_exhaustive_view(ctx, v, k, shard_rank, shard_count, out_idx, runner.data(), sv, &nf));
    const double invE = 1.0 / (double)v->E;
    *out_G = nf >= 1 ? std::exp(-sv[0] * invE) : NAN;
    if (out_runner_idx)
        for (int u = 0; u < k; u++) out_runner_idx[u] = runner[u];
    if (out_G_runner) *out_G_runner = nf >= 2 ? std::exp(-sv[1] * invE) : NAN;
    if (out_s) {
        out_s[0] = sv[0];
        out_s[1] = sv[1];
    }
    return PT_OK;
}

extern "C" pt_status pt_merge_top2(const double *s, const int32_t *tuples, int32_t n_rec, int32_t k,
                                   int32_t *out_idx, int32_t *out_runner_idx, double *out_s)
{
    PT_NVTX();
    if (!s || !tuples || !out_idx || !out_s || k < 1 || k > PT_MAXK || n_rec < 0)
        return pt_fail(PT_EINVAL, "bad argument");
    double s1 = INFINITY, s2 = INFINITY;
    int i1 = -1, i2 = -1;
    for (int r = 0; r < n_rec; r++) {
        if (!(s[r] < INFINITY)) continue;
        const int32_t *t = tuples + (int64_t)r * k;
        if (i1 < 0 || pt_key_less(s[r], t, s1, tuples + (int64_t)i1 * k, k)) {
            s2 = s1;
            i2 = i1;
            s1 = s[r];
            i1 = r;
        } else if (i2 < 0 || pt_key_less(s[r], t, s2, tuples + (int64_t)i2 * k, k)) {
            bool same = s[r] == s1;
            for (int u = 0; u < k && same; u++) same = t[u] == tuples[(int64_t)i1 * k + u];
            if (!same) {
                s2 = s[r];
                i2 = r;
            }
        }
    }
    if (i1 < 0) return pt_fail(PT_EEMPTY, "no record present");
    for (int u = 0; u < k; u++) {
        out_idx[u] = tuples[(int64_t)i1 * k + u];
        if (out_runner_idx) out_runner_idx[u] = i2 >= 0 ? tuples[(int64_t)i2 * k + u] : -1;
    }
    out_s[0] = s1;
    out_s[1] = i2 >= 0 ? s2 : INFINITY;
    return PT_OK;
}
