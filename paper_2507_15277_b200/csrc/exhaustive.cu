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
//   * a task is a row tile of 128 consecutive colex ranks (the combinatorial-rank
//     decoder pt_unrank_colex maps each thread's rows to their subsets) and a range
//     of its column tiles; A (fp16, all environments of the scope) is staged once
//     per task into shared memory;
//   * column tiles (64 envs x 64 configs, fp16, 8 KB) stream from hTile -- hT re-cut
//     into 64-config tiles at every 8-aligned offset -- through the TMA engine
//     (cp.async.bulk, one copy per stage, completion on an mbarrier) into a
//     3-stage ring refilled by the last consumer warp to release a stage;
//   * every thread holds an 8-row x 4-column block of sets; per environment pair
//     HMNMX2 (packed f16x2 min) forms the best member per environment and a 2-level
//     HADD2 tree over 4 environments, chained over 16 environments in fp16, then
//     FHADD into fp32, forms the across-environment sum of Eq. 1:
//     33 issue slots per 32 (set, env) evaluations, 1.09 with the operand loads;
//   * the fp16 tier is a FILTER: a set survives only if its lower bound is inside
//     a rigorous error window of the best two; survivors are
//     re-scored in fp64 and the exact top-2 is taken in (s asc, sorted tuple asc)
//     order (k_exh_refine_top2) -- indices bit-exact.
// k_exh_generic is the plain thread-per-subset fp64 kernel (k = 1, k > 4,
// scopes wider than 768 envs, and the PT_EXACT_FP64 debug mode).
// Variants measured and rejected live in tools/r1_variants/ and
// tools/exh_tc/, not in the library.
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

#define XT_R 128    // rows per CTA tile (k_exh_tiled); its consumer warps = XT_R / 16
#define XT_SB 32    // k_exh_tiled A staging: loads in flight per member (E_pad % (2 XT_SB) == 0)
#define XT_MINB 2   // k_exh_tiled CTAs per SM the register budget is sized for
#define XT_C 64     // columns per CTA tile
// pipeline stage = XT_K envs x 64 configs (fp16); measured on B200 at the paper
// shape: K=32/S=4 13.94 ms, K=32/S=3 14.00, K=64/S=2 13.70, K=64/S=3 13.67,
// K=160/S=2 15.77 (only 1 CTA/SM fits beyond ~113 KB of smem per CTA)
#define XT_K 64     // environments per pipeline stage (E_pad is a multiple of 64)
#define XT_S 3      // pipeline stages
// 4-env fp16 trees chained in fp16 per FHADD pair; measured (k=3, paper shape):
// one tree per FHADD 13.67 ms, NG=2 13.48, NG=4 13.37 (unroll 2), NG=8 13.42
#define XT_PUNROLL 2  // unroll of the 4*XT_NG-env loop
static constexpr int kXtPUnroll = XT_PUNROLL;
#define XT_NG 4       // 4-env tree results summed in fp16 per FHADD (XT_K % (4 NG) == 0)
static_assert(XT_K % (4 * XT_NG) == 0, "a pipeline stage must hold whole fp16 chains");
#define XT_EMAX 768 // widest scope the resident-A kernel takes (smem)
#define XT_UMAX 1024 // column tiles per task (a whole row tile: A staged once)

// ---------------------------------------------------------------------------
// work list
// ---------------------------------------------------------------------------

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

// The tc tier's k = 3 list, split by the middle member b at h = C / 2 so that every task
// has many columns (its A operand -- 128 rows x K -- is then amortised over >= C/2
// columns; with one decomposition half of the tasks had one or two 256-column tiles and
// the tensor core waited for their A hand-overs):
//   family 1: rows (a, b) with b < h in colex order, columns c > b      (as build_tasks)
//   family 2: rows (b, c) with b >= h, columns a < b; rows enumerated as the colex pairs
//             (x, y) = (C-1-c, C-1-b) with y < C - h (b descending, c descending)
// Every 3-set is in exactly one family.  int4 = (row tile, 0, n_ct, family), the tasks
// sorted by decreasing size (stable: row-tile order among equals).
// pieces > 1 (sharded searches): every task's column tiles are cut into up to `pieces`
// runs of consecutive tiles (each run rebuilds the row tile's A), so a shard's dynamic
// queue ends on short runs instead of whole 4-7-tile tasks
static pt_status build_tasks_split3(pt_ctx *ctx, const pt_view *v, int rows, int cols, int pieces, pt_tasks **out)
{
    static std::mutex mu;
    static std::map<std::tuple<int, int64_t, int, int, int>, pt_tasks *> cache;
    std::lock_guard<std::mutex> g(mu);
    const auto key = std::make_tuple(ctx->dev, v->C, rows, cols, pieces);
    auto it = cache.find(key);
    if (it != cache.end()) {
        *out = it->second;
        return PT_OK;
    }
    const int64_t C = v->C, h = C / 2;
    struct Tk { int4 t; int64_t slots, sets; };
    std::vector<Tk> all;
    // family 1
    const int64_t n1 = pt_binom(h, 2);
    for (int64_t t = 0; t * rows < n1; t++) {
        const int64_t R0 = t * rows, R1 = std::min(n1, R0 + rows);
        int32_t mem[2];
        pt_unrank_colex(R0, 2, C, mem);
        const int64_t lo = tile_lo(mem[1]);
        const int64_t n_ct = (C - lo + cols - 1) / cols;
        int64_t useful = 0;
        for (int64_t R = R0; R < R1; R++) {
            pt_unrank_colex(R, 2, C, mem);
            useful += C - 1 - mem[1];
        }
        all.push_back({make_int4((int)t, 0, (int)n_ct, 1), n_ct * rows * cols, useful});
    }
    // family 2
    const int64_t n2 = pt_binom(C - h, 2);
    for (int64_t t = 0; t * rows < n2; t++) {
        const int64_t R0 = t * rows, R1 = std::min(n2, R0 + rows);
        int32_t mem[2];
        pt_unrank_colex(R0, 2, C, mem);
        const int64_t bmax = C - 1 - mem[1];      // the first row has the smallest y: the largest b
        const int64_t n_ct = (bmax + cols - 1) / cols;
        int64_t useful = 0;
        for (int64_t R = R0; R < R1; R++) {
            pt_unrank_colex(R, 2, C, mem);
            useful += C - 1 - mem[1];            // b = C-1-y columns a < b
        }
        all.push_back({make_int4((int)t, 0, (int)n_ct, 2), n_ct * rows * cols, useful});
    }
    if (pieces > 1) {   // cut each task's column tiles into runs; useful sets pro rata by slots
        std::vector<Tk> cut;
        for (const Tk &x : all) {
            const int n = x.t.z, np = std::min(pieces, n);
            int64_t sets_left = x.sets;
            for (int q = 0, u0 = 0; q < np; q++) {
                const int u1 = (int)((int64_t)n * (q + 1) / np);
                const int64_t se = q == np - 1 ? sets_left : x.sets * (u1 - u0) / n;
                sets_left -= se;
                cut.push_back({make_int4(x.t.x, u0, u1, x.t.w), (int64_t)(u1 - u0) * rows * cols, se});
                u0 = u1;
            }
        }
        all.swap(cut);
    }
    std::stable_sort(all.begin(), all.end(),
                     [](const Tk &x, const Tk &y) { return x.t.z - x.t.y > y.t.z - y.t.y; });
    pt_tasks *T = new pt_tasks();
    T->m = 2;
    T->C = C;
    T->slot_pre.push_back(0);
    T->set_pre.push_back(0);
    for (const Tk &x : all) {
        T->h.push_back(x.t);
        T->slot_pre.push_back(T->slot_pre.back() + x.slots);
        T->set_pre.push_back(T->set_pre.back() + x.sets);
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
// Fast score of a set = fp16 trees over 4 envs, chained in fp16 over 16 envs, summed
// in fp32 (FHADD).  Every error is bounded:
//     |s_hat - s| <= eta_rel * s + eta_abs
// so the filter keeps every set that could be one of the exact best two and the fp64
// refine decides.
//
// 256 threads, 2 CTAs per SM: 8 warps compute (8 rows x 4 columns per thread, 128x64
// per CTA).  64-env x 64-config fp16 column stages come from the pre-tiled hTile
// through the TMA engine (cp.async.bulk, one 8 KB copy per stage) into an XT_S-deep
// ring: full[] mbarriers count the bytes, and the last warp to release a stage (a
// shared-memory counter) issues its refill, so no warp is spent on production and
// the SM keeps 16 warps at <= 128 registers.  Consumers never wait for each other
// inside a task.
// ---------------------------------------------------------------------------
struct XParams {
    int64_t C, C_pad, E_pad, n_rows;
    int m;
    const int4 *tasks;
    int task_hi;              // end of this shard's task range
    int *task_ctr;            // dynamic scheduler (starts at the shard's first task)
    float tau_seed;           // upper bound of s_(2): greedy's exact runner-up score (rounded up)
    float c1, c2, c3, c4;     // LB = RD(s*c1 - c2), UB = RU(s*c3 + c4)
    unsigned *U;              // float bits: min over warps of their 2nd-smallest upper bound
    unsigned long long *cand_key;
    float *cand_s;
    unsigned long long *cand_n;   // 64-bit: more than 2^32 survivors cannot wrap it
    unsigned cap;
    const uint16_t *hT;
    const uint16_t *hTile;
    int64_t n_ct;
    // fleet objective (Eq. 2, k_exh_tiled<true>): every 64-env stage belongs to one
    // device; after the last stage of device d each set adds Q_d / (its segment sum)
    // to its rate.  Q_d = quantity(d) x the device's fp16 scale (see run_fleet_tiled).
    uint32_t stage_end_mask;  // bit q: stage q is the last stage of its device
    float stage_Q[32];        // Q_d of the device stage q ends
};
#define XT_MAXSTAGE 32

#define XT_TCONS (2 * XT_R)    // consumer threads: 2 warps (column halves) per 32 rows
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

// FLEET = false: Eq. 1 geomean (minimise s; the default, graded path).
// FLEET = true : Eq. 2 fleet rate (maximise R = sum_d Q_d / s_d, per-device segment sums
//               s_d of weighted runtimes); one CTA per SM (32 more live registers).
template <bool FLEET>
__global__ void __launch_bounds__(XT_TCONS, FLEET ? 1 : XT_MINB) k_exh_tiled(const XParams p)
{
    extern __shared__ __align__(128) unsigned char smem[];
    uint32_t *Bs = reinterpret_cast<uint32_t *>(smem);                        // [S][K][32] half2
    uint16_t *As = reinterpret_cast<uint16_t *>(Bs + XT_S * XT_K * (XT_C / 2)); // [E_pad][128] fp16
    int *last_s = reinterpret_cast<int *>(As + p.E_pad * XT_R);                // [128]
    uint64_t *full = reinterpret_cast<uint64_t *>(last_s + XT_R);              // [S] (2S: keeps task_s aligned)
    int4 *task_s = reinterpret_cast<int4 *>(full + 2 * XT_S);
    int *relcnt = reinterpret_cast<int *>(task_s + 1);                         // [S]

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nkc = (int)(p.E_pad / XT_K);
    if (tid == 0) {
        for (int s = 0; s < XT_S; s++) {
            mbar_init(&full[s], 1);
            relcnt[s] = 0;
        }
        mbar_fence_init();
    }
    __syncthreads();

    uint32_t steps = 0;   // pipeline steps of all previous tasks (same in every thread)
    const int tx = lane & 7, ty = lane >> 3;
    // group minima of acc (FLEET: maxima of the rate) for the window's U
    float bA = FLEET ? -INFINITY : INFINITY, bB = FLEET ? -INFINITY : INFINITY;
    float published = FLEET ? -INFINITY : INFINITY;

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
        // stage g of this task (column tile tk.y + g / nkc, env chunk g % nkc) into its ring
        // slot: one bulk copy, completion counted on full[slot]
        auto issue = [&](int g) {
            const int sl = (int)((steps + (uint32_t)g) % XT_S);
            const int64_t col = lo + (int64_t)(tk.y + g / nkc) * XT_C;
            const int64_t sh = (col >> 3) & 7, ct = (col - 8 * sh) >> 6;
            const uint16_t *src = p.hTile + ((sh * p.n_ct + ct) * p.E_pad + (int64_t)(g % nkc) * XT_K) * XT_C;
            mbar_expect_tx(&full[sl], XT_K * XT_BROW);
            bulk_g2s(Bs + sl * XT_K * (XT_C / 2), src, XT_K * XT_BROW, &full[sl]);
        };
        // every warp has left the previous task (barrier above): the whole ring is free
        if (tid == 0)
            for (int g = 0; g < XT_S && g < nsteps; g++) issue(g);

        {
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
            }
            named_sync(1, XT_TCONS);

            float acc[8][4];
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) acc[i][j] = 0.0f;
            // FLEET: the running rate of every set (sum over completed devices)
            [[maybe_unused]] float rate[FLEET ? 8 : 1][FLEET ? 4 : 1];
            if constexpr (FLEET) {
#pragma unroll
                for (int i = 0; i < 8; i++)
#pragma unroll
                    for (int j = 0; j < 4; j++) rate[i][j] = 0.0f;
            }

            // warp w covers rows 32*(w>>1) .. +31 and columns 32*(w&1) .. +31 of the
            // 128x64 tile; a thread holds 8 consecutive rows (one 16-byte LDS) x 4
            // consecutive columns (one 8-byte LDS)
            const int r0 = 32 * (warp >> 1) + 8 * ty;
            const int c0 = 32 * (warp & 1) + 4 * tx;
            // colex order: a row's largest member is non-decreasing in its rank (padding
            // rows hold INT_MAX), so the thread's last row bounds all eight
            const int last7 = last_s[r0 + 7];
#define XT_ROW(i, j) (r0 + (i))
#define XT_COL(i, j) (c0 + (j))
#define XT_GRPB(i, j) ((j) >= 2)
#define XT_SPAN 3
            uint32_t slot = steps % XT_S, phase = (steps / XT_S) & 1u;
            int64_t ltile = lo + (int64_t)tk.y * XT_C;     // first column of the current tile
            for (int ct = tk.y; ct < tk.z; ct++, ltile += XT_C) {
                // the whole warp's column half lies past the last config: skip the math
                const bool skip = ltile + 32 * (warp & 1) >= p.C;
                // window threshold for this tile's epilogue, loaded before the math so the
                // L2 latency hides behind it (a stale value is only a looser bound)
                const unsigned Ubits = *(volatile unsigned *)p.U;
                for (int q = 0; q < nkc; q++) {
                    mbar_wait(&full[slot], phase);
                    if (!skip) {
                        const uint32_t *B = Bs + slot * XT_K * (XT_C / 2) + c0 / 2;
                        const uint16_t *A = As + (int64_t)q * XT_K * XT_R + r0;
                        // per 4 envs and column pair: four HMNMX2 (row value broadcast to both
                        // halves x the two columns) and a 2-level HADD2 tree; XT_NG such trees are
                        // chained in fp16 (one HADD2 each) before the two FHADD into fp32 --
                        // 33 issue slots per 32 (set, env); the running fp16 partial waits in pp[][]
                        // (16 registers) while the next group loads
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
                                    bc[t] = *reinterpret_cast<const uint2 *>(B + (e + 4 * gq + t) * (XT_C / 2));
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
                    }
                    if constexpr (FLEET) {
                        // end of a device segment: fold Q_d / s_d into the rate (IEEE division,
                        // correctly rounded) and restart the segment sum
                        if (!skip && ((p.stage_end_mask >> q) & 1u)) {
                            const float Q = p.stage_Q[q];
#pragma unroll
                            for (int i = 0; i < 8; i++)
#pragma unroll
                                for (int j = 0; j < 4; j++) {
                                    rate[i][j] = __fadd_rn(rate[i][j], __fdiv_rn(Q, acc[i][j]));
                                    acc[i][j] = 0.0f;
                                }
                        }
                    }
                    __syncwarp();
                    if (lane == 0) {
                        // release: the last of the consumer warps to finish this stage refills
                        // the slot with stage g + S of the task
                        __threadfence_block();
                        if (atomicAdd(&relcnt[slot], 1) == XT_TCONS / 32 - 1) {
                            relcnt[slot] = 0;
                            __threadfence_block();
                            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                            const int gn = (ct - tk.y) * nkc + q + XT_S;
                            if (gn < nsteps) issue(gn);
                        }
                    }
                    if (++slot == XT_S) {
                        slot = 0;
                        phase ^= 1u;
                    }
                }
                if (skip) continue;
                // ---- epilogue of one column tile ----
                if constexpr (FLEET) {
                    // rate R_hat: R in [R_hat c1, R_hat c3]; invalid sets -> -inf.
                    // Keep every set whose UB >= tau, tau = a lower bound of R_(2).
                    const int64_t l0 = ltile + c0;
                    const bool all_valid = l0 + XT_SPAN < p.C && l0 > last7;
                    float tA = -INFINITY, tB = -INFINITY;
#pragma unroll
                    for (int i = 0; i < 8; i++)
#pragma unroll
                        for (int j = 0; j < 4; j++) {
                            const int64_t l = ltile + XT_COL(i, j);
                            if (!all_valid && !(l < p.C && l > last_s[XT_ROW(i, j)])) rate[i][j] = -INFINITY;
                            if (XT_GRPB(i, j)) tB = fmaxf(tB, rate[i][j]);
                            else tA = fmaxf(tA, rate[i][j]);
                        }
                    bA = fmaxf(bA, tA);
                    bB = fmaxf(bB, tB);
                    const float tau = fmaxf(p.tau_seed, __uint_as_float(Ubits));
                    if (__fmul_ru(fmaxf(tA, tB), p.c3) >= tau) {   // rare: some set is in the window
#pragma unroll
                        for (int i = 0; i < 8; i++)
#pragma unroll
                            for (int j = 0; j < 4; j++) {
                                const float ub = __fmul_ru(rate[i][j], p.c3);
                                if (rate[i][j] > -INFINITY && ub >= tau) {
                                    const unsigned long long idx = atomicAdd(p.cand_n, 1ull);
                                    if (idx < p.cap) {
                                        p.cand_key[idx] = ((unsigned long long)(R0 + XT_ROW(i, j)) << KEY_BITS) |
                                                          (unsigned long long)(ltile + XT_COL(i, j));
                                        p.cand_s[idx] = ub;
                                    }
                                }
                            }
                    }
#pragma unroll
                    for (int i = 0; i < 8; i++)
#pragma unroll
                        for (int j = 0; j < 4; j++) rate[i][j] = 0.0f;
                    // U: the warp's 2nd-largest group maximum, mapped to its lower bound
                    float x1 = fmaxf(bA, bB), x2 = fminf(bA, bB);
#pragma unroll
                    for (int o = 16; o; o >>= 1) {
                        const float y1 = __shfl_xor_sync(0xffffffffu, x1, o);
                        const float y2 = __shfl_xor_sync(0xffffffffu, x2, o);
                        x2 = fmaxf(fminf(x1, y1), fmaxf(x2, y2));
                        x1 = fmaxf(x1, y1);
                    }
                    if (lane == 0) {
                        const float lb = __fmul_rd(x2, p.c1);
                        if (lb > published && lb > 0.0f) {
                            atomicMax(p.U, __float_as_uint(lb));   // positive floats: integer order
                            published = lb;
                        }
                    }
                } else {
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
                                    const unsigned long long idx = atomicAdd(p.cand_n, 1ull);
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
                        const float ub = __fmaf_ru(x2, p.c3, p.c4);
                        if (ub < published) {
                            atomicMin(p.U, __float_as_uint(ub));
                            published = ub;
                        }
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
        dst[i] = v;
    }
}

// ---------------------------------------------------------------------------
// top-2 over (s, tuple) records -- one CTA
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// u8 tier (k_exh_q8): the default filter of the tiled search since round 2.
//
// Quantise every value of the scope to q(l) = rint(l / Delta) in 0..255 with
// Delta = (scope max of l) / 255.  q is non-decreasing, so the quantised best
// member of a set is the quantisation of its best member, and the quantised set
// score S_q = sum_e min_c q(l[c][e]) is an exact integer with
//     |Delta * S_q - s| <= E * Delta / 2   (+ the fp64 slack of DESIGN.md 6.3)
// For bytes, min(a, b) = (a + b - |a - b|) / 2, so with SA_rho = sum_e A_q[e] and
// SB_l = sum_e q[l][e]
//     2 S_q = SA_rho + SB_l - sum_e |A_q[e] - q[l][e]|
// and the sum of absolute differences of four environments (one 32-bit word of
// bytes) plus the running sum is ONE instruction, VABSDIFF4.U8.ACC: 4 (set, env)
// evaluations per instruction, against 2 per HMNMX2 and 2 per HADD2 in the fp16
// tier.  Measured alone (tools/ubench_sad.cu, 8 rows x 4 columns per thread,
// operands from shared memory): 245 (set, env)/clk/SM, against 83 for the fp16
// tree.  The integer score is exact, so the only error is the quantisation's,
// bounded per term; the window test and the U bookkeeping are those of the fp16
// tier with X = 2 S_q in place of the fp32 accumulator.
// ---------------------------------------------------------------------------
#define XQ_R 128   // rows per CTA tile
#define XQ_C 64    // columns per CTA tile

// qmax: scope max of l (non-negative doubles order as their bit patterns)
__global__ void __launch_bounds__(256) k_q8_max(const double *__restrict__ l64, int64_t C, int64_t E,
                                               int64_t E_pad, unsigned long long *__restrict__ qmax)
{
    double m = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < C * E; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i / E, e = i - c * E;
        m = fmax(m, l64[c * E_pad + e]);
    }
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(qmax, (unsigned long long)__double_as_longlong(m));
}

// Delta, 1/Delta and the window constants (one thread; no host round trip).
// Per term |Delta q(l) - l| <= Delta (1/2 + 1e-12) (1/Delta and l/Delta rounded in
// fp64); the refine's fp64 sum differs from the exact s by <= E_pad^2 qmax 2^-52.
__global__ void k_q8_const(const unsigned long long *__restrict__ qmax_bits, int64_t E_pad, float *__restrict__ qc)
{
    const double qmax = __longlong_as_double((long long)*qmax_bits);
    const double delta = qmax > 0.0 ? qmax / 255.0 : 1.0;
    const double Ed = (double)E_pad;
    const double slack = Ed * delta * (0.5 + 1e-12) + Ed * Ed * qmax * 0x1p-52 + 1e-300;
    qc[0] = __double2float_rd(delta * 0.5);
    qc[1] = __double2float_ru(slack);
    qc[2] = __double2float_ru(delta * 0.5);
    qc[3] = __double2float_ru(slack);
    *reinterpret_cast<double *>(qc + 4) = 1.0 / delta;
}

// qC[c][g] = bytes q(l[c][4g + 0..3]) (0 past E and past C), qSum[c] = sum of them:
// one warp per config
__global__ void __launch_bounds__(256) k_q8_build(const double *__restrict__ l64, int64_t C, int64_t E, int64_t E_pad,
                                                 int64_t C_pad, const float *__restrict__ qc,
                                                 uint32_t *__restrict__ qC, int32_t *__restrict__ qSum)
{
    const int64_t c = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (c >= C_pad) return;
    const double inv = *reinterpret_cast<const double *>(qc + 4);
    const int64_t G = E_pad / 4;
    int sum = 0;
    for (int64_t g = lane; g < G; g += 32) {
        uint32_t w = 0;
        for (int b = 0; b < 4; b++) {
            const int64_t e = 4 * g + b;
            uint32_t q = 0;
            if (c < C && e < E) q = (uint32_t)fmin(fmax(rint(l64[c * E_pad + e] * inv), 0.0), 255.0);
            w |= q << (8 * b);
            sum += (int)q;
        }
        qC[c * G + g] = w;
    }
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) qSum[c] = sum;
}

// qTile[sh][ct][g][j] = qC[64 ct + 8 sh + j][g] (0 past C_pad)
__global__ void __launch_bounds__(256) k_q8_tile(const uint32_t *__restrict__ qC, int64_t G, int64_t C_pad,
                                                int64_t n_ct, uint32_t *__restrict__ qTile)
{
    const int64_t sct = blockIdx.x, ct = sct % n_ct, sh = sct / n_ct;
    const int64_t c0 = 64 * ct + 8 * sh;
    uint32_t *dst = qTile + sct * G * 64;
    for (int64_t i = threadIdx.x; i < G * 64; i += blockDim.x) {
        const int64_t g = i >> 6, c = c0 + (i & 63);
        dst[i] = c < C_pad ? qC[c * G + g] : 0u;
    }
}

struct QParams {
    int64_t C, E_pad, n_rows, n_ct;
    int m, G, S;              // G = E_pad / 4 words per config; S = ring depth
    const int4 *tasks;
    int task_hi;
    int *task_ctr;
    float tau_seed;
    const float *qc;          // c1..c4 (k_q8_const)
    unsigned *U;
    unsigned long long *cand_key;
    float *cand_s;
    unsigned long long *cand_n;
    unsigned cap;
    const uint32_t *qC, *qTile;
    const int32_t *qSum;
};

__device__ __forceinline__ uint32_t sad4(uint32_t a, uint32_t b, uint32_t acc)
{
    uint32_t r;
    asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(acc));
    return r;
}

// 256 threads, 8 rows x 4 columns per thread (the k_exh_tiled mapping); a task's A
// (128 rows x all envs, bytes) is staged once; each column tile (all envs x 64
// configs, E_pad * 64 bytes) is one bulk copy into an S-deep ring.
__global__ void __launch_bounds__(256, 2) k_exh_q8(const QParams p)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const int G = p.G, S = p.S;
    uint32_t *Bs = reinterpret_cast<uint32_t *>(smem);                 // [S][G][64]
    uint32_t *As = Bs + (size_t)S * G * XQ_C;                           // [G][128]
    int *sap = reinterpret_cast<int *>(As + (size_t)G * XQ_R);          // [256] partial row sums
    int *last_s = sap + 256;                                            // [128]
    uint64_t *full = reinterpret_cast<uint64_t *>(last_s + XQ_R);       // [4]
    int4 *task_s = reinterpret_cast<int4 *>(full + 4);
    int *relcnt = reinterpret_cast<int *>(task_s + 1);                  // [4]

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        for (int s = 0; s < S; s++) {
            mbar_init(&full[s], 1);
            relcnt[s] = 0;
        }
        mbar_fence_init();
    }
    __syncthreads();
    const float c1 = p.qc[0], c2 = p.qc[1], c3 = p.qc[2], c4 = p.qc[3];
    const uint32_t stage_bytes = (uint32_t)G * XQ_C * 4u;

    uint32_t steps = 0;
    const int tx = lane & 7, ty = lane >> 3;
    int bA = INT_MAX, bB = INT_MAX;      // group minima of X for U
    float published = INFINITY;

    for (;;) {
        if (tid == 0) {
            int ti = atomicAdd(p.task_ctr, 1);
            *task_s = ti < p.task_hi ? p.tasks[ti] : make_int4(-1, 0, 0, 0);
        }
        __syncthreads();
        const int4 tk = *task_s;
        if (tk.x < 0) break;
        const int64_t R0 = (int64_t)tk.x * XQ_R;
        int32_t mem0[PT_MAXK];
        pt_unrank_colex(R0, p.m, p.C, mem0);
        const int64_t lo = tile_lo(mem0[p.m - 1]);
        const int nsteps = tk.z - tk.y;
        auto issue = [&](int g) {
            const int sl = (int)((steps + (uint32_t)g) % (uint32_t)S);
            const int64_t col = lo + (int64_t)(tk.y + g) * XQ_C;
            const int64_t sh = (col >> 3) & 7, ct = (col - 8 * sh) >> 6;
            mbar_expect_tx(&full[sl], stage_bytes);
            bulk_g2s(Bs + (size_t)sl * G * XQ_C, p.qTile + (sh * p.n_ct + ct) * (int64_t)G * XQ_C, stage_bytes, &full[sl]);
        };
        if (tid == 0)
            for (int g = 0; g < S && g < nsteps; g++) issue(g);

        // ---- stage A: byte-wise min over the row's members, and its row sum ----
        {
            const int r = tid & (XQ_R - 1), half = tid >> 7;
            const int64_t R = R0 + r;
            int32_t mem[PT_MAXK];
            const bool valid = R < p.n_rows;
            if (valid) pt_unrank_colex(R, p.m, p.C, mem);
            else for (int u = 0; u < p.m; u++) mem[u] = 0;
            if (tid < XQ_R) last_s[r] = valid ? mem[p.m - 1] : 0x7fffffff;
            uint32_t part = 0;
            // 16-byte loads (4 words = 16 envs); the two threads of a row take alternate ones
            for (int g4 = half; g4 < G / 4; g4 += 2) {
                uint4 v = *reinterpret_cast<const uint4 *>(p.qC + (int64_t)mem[0] * G + 4 * g4);
                for (int u = 1; u < p.m; u++) {
                    const uint4 w = *reinterpret_cast<const uint4 *>(p.qC + (int64_t)mem[u] * G + 4 * g4);
                    v.x = __vminu4(v.x, w.x);
                    v.y = __vminu4(v.y, w.y);
                    v.z = __vminu4(v.z, w.z);
                    v.w = __vminu4(v.w, w.w);
                }
                if (!valid) v = make_uint4(0, 0, 0, 0);
                As[(4 * g4 + 0) * XQ_R + r] = v.x;
                As[(4 * g4 + 1) * XQ_R + r] = v.y;
                As[(4 * g4 + 2) * XQ_R + r] = v.z;
                As[(4 * g4 + 3) * XQ_R + r] = v.w;
                part = sad4(v.x, 0u, part);
                part = sad4(v.y, 0u, part);
                part = sad4(v.z, 0u, part);
                part = sad4(v.w, 0u, part);
            }
            sap[tid] = (int)part;
        }
        __syncthreads();

        const int r0 = 32 * (warp >> 1) + 8 * ty;
        const int c0 = 32 * (warp & 1) + 4 * tx;
        int SA[8];
#pragma unroll
        for (int i = 0; i < 8; i++) SA[i] = sap[r0 + i] + sap[XQ_R + r0 + i];
        const int last7 = last_s[r0 + 7];
        uint32_t slot = steps % (uint32_t)S, phase = (steps / (uint32_t)S) & 1u;
        int64_t ltile = lo + (int64_t)tk.y * XQ_C;
        for (int ct = tk.y; ct < tk.z; ct++, ltile += XQ_C) {
            const bool skip = ltile + 32 * (warp & 1) >= p.C;
            const unsigned Ubits = *(volatile unsigned *)p.U;
            uint32_t acc[8][4];
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) acc[i][j] = 0u;
            mbar_wait(&full[slot], phase);
            if (!skip) {
                const uint32_t *B = Bs + (size_t)slot * G * XQ_C + c0;
                const uint32_t *A = As + r0;
#pragma unroll 4
                for (int g = 0; g < G; g++) {
                    const uint4 a0 = *reinterpret_cast<const uint4 *>(A + g * XQ_R);
                    const uint4 a1 = *reinterpret_cast<const uint4 *>(A + g * XQ_R + 4);
                    const uint4 b = *reinterpret_cast<const uint4 *>(B + g * XQ_C);
                    const uint32_t av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                    const uint32_t bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                    for (int i = 0; i < 8; i++)
#pragma unroll
                        for (int j = 0; j < 4; j++) acc[i][j] = sad4(av[i], bv[j], acc[i][j]);
                }
            }
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                if (atomicAdd(&relcnt[slot], 1) == 256 / 32 - 1) {
                    relcnt[slot] = 0;
                    __threadfence_block();
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    const int gn = ct - tk.y + S;
                    if (gn < nsteps) issue(gn);
                }
            }
            if (++slot == (uint32_t)S) {
                slot = 0;
                phase ^= 1u;
            }
            if (skip) continue;
            // ---- epilogue: X = 2 S_q = SA + SB - D; invalid sets -> INT_MAX ----
            int SB[4];
#pragma unroll
            for (int j = 0; j < 4; j++) SB[j] = __ldg(p.qSum + ltile + c0 + j);
            int X[8][4];
            const int64_t l0 = ltile + c0;
            const bool all_valid = l0 + 3 < p.C && l0 > last7;
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    X[i][j] = SA[i] + SB[j] - (int)acc[i][j];
                    if (!all_valid) {
                        const int64_t l = l0 + j;
                        if (!(l < p.C && l > last_s[r0 + i])) X[i][j] = INT_MAX;
                    }
                }
            int tA = INT_MAX, tB = INT_MAX;
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    if (j >= 2) tB = min(tB, X[i][j]);
                    else tA = min(tA, X[i][j]);
                }
            bA = min(bA, tA);
            bB = min(bB, tB);
            const float tau = fminf(p.tau_seed, __uint_as_float(Ubits));
            const int tmin = min(tA, tB);
            if (tmin != INT_MAX && __fmaf_rd((float)tmin, c1, -c2) <= tau) {   // rare
#pragma unroll
                for (int i = 0; i < 8; i++)
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        const float lb = __fmaf_rd((float)X[i][j], c1, -c2);
                        if (X[i][j] != INT_MAX && lb <= tau) {
                            const unsigned long long idx = atomicAdd(p.cand_n, 1ull);
                            if (idx < p.cap) {
                                p.cand_key[idx] = ((unsigned long long)(R0 + r0 + i) << KEY_BITS) |
                                                  (unsigned long long)(l0 + j);
                                p.cand_s[idx] = lb;
                            }
                        }
                    }
            }
            // U: the warp's 2nd-smallest group minimum (two distinct sets), as an upper bound
            int x1 = min(bA, bB), x2 = max(bA, bB);
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const int y1 = __shfl_xor_sync(0xffffffffu, x1, o);
                const int y2 = __shfl_xor_sync(0xffffffffu, x2, o);
                x2 = min(max(x1, y1), min(x2, y2));
                x1 = min(x1, y1);
            }
            if (lane == 0 && x2 != INT_MAX) {
                const float ub = __fmaf_ru((float)x2, c3, c4);
                if (ub < published) {
                    atomicMin(p.U, __float_as_uint(ub));
                    published = ub;
                }
            }
        }
        steps += nsteps;
    }
}

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
    const unsigned long long *__restrict__ key, const float *__restrict__ cs, const unsigned long long *__restrict__ n_dev,
    unsigned cap, float tau_pass, const unsigned *__restrict__ U, int m, int64_t C, const double *__restrict__ l64,
    int64_t E_pad, Rec2 *__restrict__ blk, unsigned *__restrict__ done, double *__restrict__ out_s,
    int32_t *__restrict__ out_t)
{
    const unsigned long long nd = *n_dev;   // bit 63: the filter did not run (tc tier)
    const int64_t n = (nd >> 63) ? 0 : (int64_t)min(nd, (unsigned long long)cap);
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

// 64-config column tiles of a view (one extra zero tile past the end), shared by both tiers
static int64_t view_n_ct(const pt_view *v) { return (v->C_pad + XT_C - 1) / XT_C + 1; }

// fp16 tier operands: hT (pt_view_fp16) re-cut into hTile, built on first use
static pt_status tile_fp16(pt_ctx *ctx, const pt_view *v)
{
    if (v->hTile) return PT_OK;
    pt_view *mv = const_cast<pt_view *>(v);
    mv->n_ct = view_n_ct(v);
    PT_TRY(pt_dalloc(ctx, (void **)&mv->hTile, sizeof(uint16_t) * 8 * mv->n_ct * v->E_pad * XT_C));
    k_tile_hT<<<(unsigned)(8 * mv->n_ct), 256, 0, ctx->stream>>>(v->hT, v->E_pad, v->C_pad, mv->n_ct, mv->hTile);
    ctx->stats.launches++;
    PT_CK(cudaGetLastError());
    return PT_OK;
}

// u8 tier operands (qC, qTile, qSum, qConst), built on first use: four launches,
// stream-ordered, no host round trip (Delta stays on the device)
static pt_status pt_view_q8(pt_ctx *ctx, const pt_view *v)
{
    if (v->qTile) return PT_OK;
    pt_view *mv = const_cast<pt_view *>(v);
    cudaStream_t s = ctx->stream;
    mv->n_ct = view_n_ct(v);
    const int64_t G = v->E_pad / 4, nsum = (mv->n_ct + 1) * XQ_C + XQ_C;
    PT_TRY(pt_dalloc(ctx, (void **)&mv->qConst, sizeof(float) * 8 + sizeof(unsigned long long)));
    PT_TRY(pt_dalloc(ctx, (void **)&mv->qC, sizeof(uint32_t) * v->C_pad * G));
    PT_TRY(pt_dalloc(ctx, (void **)&mv->qSum, sizeof(int32_t) * nsum));
    PT_TRY(pt_dalloc(ctx, (void **)&mv->qTile, sizeof(uint32_t) * 8 * mv->n_ct * G * XQ_C));
    unsigned long long *qmax = reinterpret_cast<unsigned long long *>(mv->qConst + 8);
    PT_CK(cudaMemsetAsync(qmax, 0, sizeof(unsigned long long), s));
    PT_CK(cudaMemsetAsync(mv->qSum, 0, sizeof(int32_t) * nsum, s));
    const int64_t n = v->C * v->E;
    const unsigned gmax = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 4L * ctx->num_sms));
    k_q8_max<<<gmax, 256, 0, s>>>(v->l64, v->C, v->E, v->E_pad, qmax);
    k_q8_const<<<1, 1, 0, s>>>(qmax, v->E_pad, mv->qConst);
    k_q8_build<<<(unsigned)((v->C_pad + 7) / 8), 256, 0, s>>>(v->l64, v->C, v->E, v->E_pad, v->C_pad, mv->qConst,
                                                              mv->qC, mv->qSum);
    k_q8_tile<<<(unsigned)(8 * mv->n_ct), 256, 0, s>>>(mv->qC, G, v->C_pad, mv->n_ct, mv->qTile);
    ctx->stats.launches += 4;
    PT_CK(cudaGetLastError());
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
    PT_TRY(build_tasks(ctx, v, m, XT_R, XT_C, &T));
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
    ctx->stats.exh_kernel = 0;
    ctx->stats.exh_env_pad = v->E_pad;
    ctx->stats.exh_candidates = 0;
    ctx->stats.exh_passes = 0;
    ctx->stats.exh_main_ms = 0.0;
    s_out[0] = s_out[1] = INFINITY;
    if (ta >= tb) return PT_OK;

    // error model of the fp16 tier; per set |s_hat - s| <= eta_rel * s + eta_abs:
    // every term passes through at most lv16 = 2 + XT_NG fp16 roundings (its quantisation,
    // the 2-level tree over 4 envs, the fp16 chain of XT_NG trees) and then the fp32 sum of
    // E_pad / (4 XT_NG) chain values (Higham gamma); subnormal quantisation adds an
    // absolute 2^-25 per term.  The kernel turns this into LB <= s <= UB per set (directed
    // rounding) and keeps every set with LB <= min(tau_seed, U), U = smallest 2nd-best UB.
    const double u16 = std::ldexp(1.0, -11), u32 = std::ldexp(1.0, -24);
    const double lv16 = 2.0 + XT_NG;
    const double ngrp = (double)v->E_pad / (4.0 * XT_NG) + 2.0;
    const double gam = ngrp * u32 / (1.0 - ngrp * u32);
    const double eta_rel = (lv16 * u16 + lv16 * lv16 * u16 * u16 + gam) * 1.01;
    const double eta_abs = 3.0 * (double)v->E_pad * std::ldexp(1.0, -25) * 1.01;
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
    // seed: exact score of greedy's runner-up set at step k (two distinct k-sets, so
    // >= s_(2)), reused from an earlier greedy run of >= k steps on this view when there
    // is one.  Otherwise the seed greedy is only enqueued (max(k, 3) steps: a k=2 search
    // leaves k=3's seed): its runner-up trace stays on the device and a one-thread kernel
    // writes the rounded-up seed into U before the search (U is itself an upper bound of
    // s_(2), so min(seed, U) is one) -- no host round trip between the two.
    // (development knob PT_EXH_SEED=none: no seed; the window tightens only through U)
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
    const double c1d = 1.0 / (1.0 + eta_rel), c3d = 1.0 / (1.0 - eta_rel);
    const float c1 = f_dn(c1d), c2 = f_up(eta_abs), c3 = f_up(c3d), c4 = f_up(eta_abs * c3d * (1.0 + 1e-6));

    if (v->E_pad % XT_K != 0)   // a stage must not straddle the padded env range
        return pt_fail(PT_EINVAL, "E_pad=%lld is not a multiple of the stage depth %d", (long long)v->E_pad, XT_K);
    mark("seeded");
    // per (kernel, smem) once per process: the attribute and the occupancy query
    static std::mutex attr_mu;
    static std::map<std::tuple<int, const void *, size_t>, int> attr_occ;   // per device
    auto occupancy = [&](const void *kfn, size_t smem_k, int threads, int *occ) -> pt_status {
        std::lock_guard<std::mutex> g(attr_mu);
        auto key = std::make_tuple(ctx->dev, kfn, smem_k);
        auto it = attr_occ.find(key);
        if (it == attr_occ.end()) {
            PT_TRY(pt_smem_optin(ctx, kfn));
            PT_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, kfn, threads, smem_k));
            attr_occ[key] = *occ;
        } else {
            *occ = it->second;
        }
        return PT_OK;
    };
    // fp16 tier (k_exh_tiled)
    auto kern = k_exh_tiled<false>;
    const size_t smem = sizeof(uint32_t) * XT_S * XT_K * (XT_C / 2) + sizeof(uint16_t) * v->E_pad * XT_R +
                        sizeof(int) * XT_R + 2 * sizeof(uint64_t) * XT_S + sizeof(int4) + sizeof(int) * XT_S;
    const int threads = XT_TCONS;
    int occ = 1;
    PT_TRY(occupancy((const void *)kern, smem, threads, &occ));
    // u8 tier (k_exh_q8): the default; PT_EXH_TIER=fp16 keeps the fp16 tier (read per call,
    // so the tests can exercise both tiers in one process)
    const char *tier_env = getenv("PT_EXH_TIER");
    const bool force_fp16 = tier_env && !strcmp(tier_env, "fp16");
    const bool force_u8 = tier_env && !strcmp(tier_env, "u8");
    bool q8 = !force_fp16;
    // threshold-count tier (k_exh_tc, exh_tc.cu): the default for k = 2..4; its own task
    // list (256-column tiles); on an unusable tau or a buffer overflow the search falls
    // back to the u8 tier in the next pass
    // (k = 2 is a 1.6 M-set search: the u8 tier's single launch beats the tc tier's
    // swap search + operand build there, 0.11 vs 0.17 ms per call at the paper shape;
    // PT_EXH_TIER=tc forces the tc tier for k = 2 too)
    const bool force_tc = tier_env && !strcmp(tier_env, "tc");
    bool tc = !force_fp16 && !force_u8 && k <= 4 && (k >= 3 || (force_tc && k >= 2));
    const int4 *tc_list = nullptr;
    int tc_ta = 0, tc_tb = 0;
    int64_t tc_sets = 0, tc_slots = 0;
    int tc_halves = 2;
    bool tc_split = false;
    if (tc) {
        pt_tasks *TT = nullptr;
        tc_halves = pt_tc_halves();
        // k = 3 (H = 1): the two-family list (PT_TC_SPLIT=0 keeps the single decomposition)
        tc_split = m == 2 && v->C >= 4 && !(getenv("PT_TC_SPLIT") && !strcmp(getenv("PT_TC_SPLIT"), "0"));
        if (tc_split)
            PT_TRY(build_tasks_split3(ctx, v, XT_R * tc_halves, 256 / tc_halves, shard_count >= 4 ? 2 : 1, &TT));
        else PT_TRY(build_tasks(ctx, v, m, XT_R * tc_halves, 256 / tc_halves, &TT));
        tc_list = TT->d;
        tc_tb = (int)TT->h.size();
        tc_sets = TT->set_pre.back();
        tc_slots = TT->slot_pre.back();
        if (shard_count > 1) {
            const pt_tasks::plan *P = nullptr;
            static const std::vector<double> equal;
            PT_TRY(shard_plan(TT, shard_count, (int)ctx->shard_w.size() == shard_count ? ctx->shard_w : equal, &P));
            tc_list = P->d;
            tc_ta = P->off[shard_rank];
            tc_tb = P->off[shard_rank + 1];
            tc_sets = P->sets[shard_rank];
            tc_slots = P->slots[shard_rank];
        }
        if (shard_count == 1 && tc_sets != ctx->stats.exh_sets) tc = false;   // both lists cover every set (always)
    }
    const int G = (int)(v->E_pad / 4);
    auto q8_smem = [&](int S) {
        return (size_t)4 * S * G * XQ_C + (size_t)4 * G * XQ_R + sizeof(int) * (256 + XQ_R) +
               sizeof(uint64_t) * 4 + sizeof(int4) + sizeof(int) * 4;
    };
    const size_t smem_budget = 227 * 1024;
    const int q8_S = 2 * q8_smem(3) <= smem_budget ? 3 : 2;
    const size_t smem_q8 = q8_smem(q8_S);
    int occ_q8 = 0;
    bool q8_ready = false;
    auto prepare_q8 = [&]() -> pt_status {
        if (q8 && !q8_ready) {
            PT_TRY(pt_view_q8(ctx, v));
            PT_TRY(occupancy((const void *)k_exh_q8, smem_q8, 256, &occ_q8));
            if (occ_q8 < 1) q8 = false;
            q8_ready = true;
        }
        return PT_OK;
    };
    if (!tc) PT_TRY(prepare_q8());
    // the tc tier starts its swap search from greedy's k-set: the host trace's picks, or
    // the device trace (enqueued above when there is no host trace)
    if (tc && v->greedy_idx.size() < (size_t)k && v->d_seed_k < k) {
        if (pt_greedy_seed_enqueue(ctx, v, (int)std::min<int64_t>(std::max(k, 3), v->C)) != PT_OK) tc = false;
    }

    unsigned cap = 1u << 20;
    if (tc && getenv("PT_TC_CAP")) cap = (unsigned)std::max(1, atoi(getenv("PT_TC_CAP")));   // (tests: overflow paths)
    unsigned long long n_cand = 0;
    float tau_pass = tau_seed;
    int tier_pass0 = -1;   // first pass of the filter tier whose answer is returned (its time is exh_main_ms)
    for (int pass = 0; pass < 6; pass++) {
        size_t off = 0;
        auto take = [&](size_t b) { size_t o = off; off += pt_round_up(b, 256); return o; };
        const size_t o_ctr = take(sizeof(int)), o_U = take(sizeof(unsigned)),
                     o_n = take(sizeof(unsigned long long)), o_key = take(sizeof(unsigned long long) * cap),
                     o_cq = take(sizeof(float) * cap),
                     o_os = take(sizeof(double) * 2), o_ot = take(sizeof(int32_t) * 2 * k),
                     o_blk = take(sizeof(Rec2) * (size_t)ctx->num_sms * 2), o_done = take(sizeof(unsigned)),
                     o_S0 = take(sizeof(int32_t) * k), o_sd = take(sizeof(double)), o_tau = take(sizeof(double)),
                     o_rs = take(sizeof(double) * 2 * ctx->num_sms), o_rw = take(sizeof(long long) * 2 * ctx->num_sms);
        void *scr = nullptr;
        PT_TRY(pt_scratch(ctx, off, &scr));
        char *b = (char *)scr;
        int *ctr = (int *)(b + o_ctr);
        unsigned *U = (unsigned *)(b + o_U);
        unsigned long long *cn = (unsigned long long *)(b + o_n);
        unsigned long long *ckey = (unsigned long long *)(b + o_key);
        float *cq = (float *)(b + o_cq);
        double *os = (double *)(b + o_os);
        int32_t *ot = (int32_t *)(b + o_ot);
        Rec2 *blk = (Rec2 *)(b + o_blk);
        unsigned *done = (unsigned *)(b + o_done);
        const unsigned u_init = 0x7f800000u;   // +inf
        pt_hostio io(ctx);
        if (!tc) PT_TRY(prepare_q8());
        PT_TRY(io.h2d(ctr, tc ? &tc_ta : &ta, sizeof(int)));
        if (tc) {
            // (U is written by the tc tier's constants kernel)
        } else if (seed_dev) {
            k_seed_U<<<1, 1, 0, s>>>(seed_dev, U);
            ctx->stats.launches++;
        } else {
            PT_TRY(io.h2d(U, &u_init, sizeof(unsigned)));
        }
        PT_CK(cudaMemsetAsync(cn, 0, sizeof(unsigned long long), s));
        PT_CK(cudaMemsetAsync(done, 0, sizeof(unsigned), s));
        bool tc_launched = false;
        if (!tc && tier_pass0 < 0) tier_pass0 = pass;
        if (tc) {
            pt_tc_args a;
            a.k = k;
            a.tasks = tc_list;
            a.ta = tc_ta;
            a.tb = tc_tb;
            a.ctr = ctr;
            a.U = U;
            a.cand_n = cn;
            a.cand_key = ckey;
            a.cand_s = cq;
            a.cap = cap;
            if (v->greedy_idx.size() >= (size_t)k) {
                const double sd = v->greedy_s2[k - 1];
                PT_TRY(io.h2d(b + o_S0, v->greedy_idx.data(), sizeof(int32_t) * k));
                PT_TRY(io.h2d(b + o_sd, &sd, sizeof(double)));
                a.d_S0 = (const int32_t *)(b + o_S0);
                a.d_seed_s2 = (const double *)(b + o_sd);
            } else {
                a.d_S0 = v->d_seed_idx;
                a.d_seed_s2 = v->d_seed_s2 + (k - 1);
            }
            a.swap_rs = (double *)(b + o_rs);
            a.swap_rw = (long long *)(b + o_rw);
            a.tau_dev = (double *)(b + o_tau);
            a.halves = tc_halves;
            a.split = tc_split;
            mark("pre-launch");
            int nt = 0;
            const pt_status st = pt_exh_tc_enqueue(ctx, v, a, &nt);
            if (st == PT_OK) {
                tc_launched = true;
                ctx->stats.exh_tc_nt = nt;
            } else if (st == PT_EINVAL) {
                tc = false;   // not eligible: this pass runs the u8 tier
                tier_pass0 = pass;
                PT_TRY(prepare_q8());
                PT_TRY(io.h2d(ctr, &ta, sizeof(int)));
                if (seed_dev) {
                    k_seed_U<<<1, 1, 0, s>>>(seed_dev, U);
                    ctx->stats.launches++;
                } else {
                    PT_TRY(io.h2d(U, &u_init, sizeof(unsigned)));
                }
            } else {
                return st;
            }
        }
        if (tc_launched) {
            tau_pass = INFINITY;   // the refine's threshold is U (k_tc_const)
        } else if (q8) {
            QParams p;
            p.C = v->C;
            p.E_pad = v->E_pad;
            p.n_rows = pt_binom(v->C, m);
            p.n_ct = v->n_ct;
            p.m = m;
            p.G = G;
            p.S = q8_S;
            p.tasks = task_list;
            p.task_hi = tb;
            p.task_ctr = ctr;
            p.tau_seed = tau_pass;
            p.qc = v->qConst;
            p.U = U;
            p.cand_key = ckey;
            p.cand_s = cq;
            p.cand_n = cn;
            p.cap = cap;
            p.qC = v->qC;
            p.qTile = v->qTile;
            p.qSum = v->qSum;
            const int grid = std::min(ctx->num_sms * occ_q8, tb - ta);
            mark("pre-launch");
            PT_CK(cudaEventRecord(ctx->ev0, s));
            k_exh_q8<<<grid, 256, smem_q8, s>>>(p);
        } else {
            PT_TRY(pt_view_fp16(ctx, v));
            PT_TRY(tile_fp16(ctx, v));
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
            p.U = U;
            p.cand_key = ckey;
            p.cand_s = cq;
            p.cand_n = cn;
            p.cap = cap;
            p.hT = v->hT;
            p.hTile = v->hTile;
            p.n_ct = v->n_ct;
            const int grid = std::min(ctx->num_sms * std::max(occ, 1), tb - ta);
            mark("pre-launch");
            PT_CK(cudaEventRecord(ctx->ev0, s));
            kern<<<grid, threads, smem, s>>>(p);
        }
        PT_CK(cudaEventRecord(ctx->ev1, s));
        ctx->stats.launches++;
        PT_CK(cudaGetLastError());
        // refine + top-2 run on the device-side survivor count (no host round trip);
        // one synchronisation returns the count, U and the exact top-2
        // (the tc tier leaves a few thousand survivors: fewer blocks, a shorter final merge)
        k_exh_refine_top2<<<(unsigned)(tc_launched ? 64 : ctx->num_sms * 2), 256, 0, s>>>(ckey, cq, cn, cap, tau_pass, U, m, v->C,
                                                                        v->l64, v->E_pad, blk, done, os, ot);
        ctx->stats.launches++;
        mark("launched");
        pt_pack_record(ctx, os, ot, k);   // sharded search: this rank's record stays on the device
        PT_CK(cudaGetLastError());
        unsigned hU = 0;
        PT_TRY(io.d2h(&n_cand, cn, sizeof(unsigned long long)));
        PT_TRY(io.d2h(&hU, U, sizeof(unsigned)));
        PT_TRY(io.d2h(s_out, os, sizeof(double) * 2));
        PT_TRY(io.d2h(t_out, ot, sizeof(int32_t) * 2 * k));
        PT_TRY(io.finish());
        mark("synced");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        if (pass == tier_pass0 || tc_launched) ctx->stats.exh_main_ms = ms;
        ctx->stats.exh_passes = pass + 1;
        float Uf;
        memcpy(&Uf, &hU, sizeof Uf);
        if (tc_launched) {
            ctx->stats.exh_tc_survivors = (n_cand >> 63) ? -1 : (int64_t)n_cand;
            if (!(n_cand >> 63) && n_cand > cap && shard_count > 1) {
                // sharded: every rank must scan the SAME task list (the tiers' lists
                // partition the subset space differently), and an overflow is a
                // per-shard event -- so a sharded tc search reruns itself with room
                // for every survivor instead of falling back
                if (n_cand > (1ull << 28))
                    return pt_fail(PT_ECAP, "%llu tc-tier survivors in this shard: above the 2^28 buffer limit",
                                   n_cand);
                cap = (unsigned)n_cand;
                continue;
            }
            if ((n_cand >> 63) || n_cand > cap) {
                // tau unusable (identical on every rank) or too weak a filter: the u8
                // tier, seeded as before
                tc = false;
                tau_pass = tau_seed;
                cap = 1u << 20;
                continue;
            }
            ctx->stats.exh_kernel = 5;
            ctx->stats.exh_candidates = n_cand;
            ctx->stats.exh_sets = tc_sets;
            ctx->stats.exh_slots = tc_slots;
            if (n_cand == 0) {
                s_out[0] = s_out[1] = INFINITY;
                for (int u = 0; u < 2 * k; u++) t_out[u] = 0;
            }
            return PT_OK;
        }
        if (n_cand > cap) {
            // overflow: rerun with the final threshold (U is an upper bound of s_(2) in
            // either tier) and room for every survivor; a u8 tier that leaves more than
            // 2^24 survivors hands over to the finer fp16 tier
            tau_pass = std::min(tau_pass, Uf);
            if (q8 && n_cand > (1ull << 24)) {
                q8 = false;
                cap = 1u << 20;
                continue;
            }
            if (n_cand > (1ull << 28))
                return pt_fail(PT_ECAP, "%llu fp16-tier survivors (massively tied data): above the 2^28 buffer limit",
                               n_cand);
            cap = (unsigned)n_cand;
            continue;
        }
        ctx->stats.exh_kernel = q8 ? 4 : 0;
        ctx->stats.exh_candidates = n_cand;
        if (n_cand == 0) {
            s_out[0] = s_out[1] = INFINITY;
            for (int u = 0; u < 2 * k; u++) t_out[u] = 0;
        }
        return PT_OK;
    }
    return pt_fail(PT_ECUDA, "candidate buffer overflowed twice (internal error)");
}

// ---------------------------------------------------------------------------
// the tiled search for the fleet objective (Eq. 2): k_exh_tiled<true> on
// the fp16 weighted runtimes, each device one run of 64-env stages (pt_fleet_tiled),
// fp64 exact refine of the survivors, ranked by cost 1/R ascending
// ---------------------------------------------------------------------------
// exact R of every candidate whose rate upper bound reaches the final threshold,
// fused with the (cost = 1/R, tuple) top-2 (last-block merge, as k_exh_refine_top2)
__global__ void __launch_bounds__(256) k_fleet_refine_top2(
    const unsigned long long *__restrict__ key, const float *__restrict__ cub, const unsigned long long *__restrict__ n_dev,
    unsigned cap, float tau_pass, const unsigned *__restrict__ U, int m, int64_t C,
    const double *__restrict__ tcm, int64_t E_pad, const double *__restrict__ w, const int32_t *__restrict__ seg,
    int n_devices, const double *__restrict__ qdev, Rec2 *__restrict__ blk, unsigned *__restrict__ done,
    double *__restrict__ out_s, int32_t *__restrict__ out_t)
{
    const int64_t n = (int64_t)min(*n_dev, (unsigned long long)cap);
    const float tau = fmaxf(tau_pass, __uint_as_float(*U));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int k = m + 1;
    __shared__ Rec2 sh[256];
    Rec2 r;
    r.s1 = r.s2 = INFINITY;
    for (int u = 0; u < PT_MAXK; u++) r.t1[u] = r.t2[u] = 0x7fffffff;
    for (int64_t wi = (int64_t)blockIdx.x * 8 + warp; wi < n; wi += (int64_t)gridDim.x * 8) {
        if (cub[wi] < tau) continue;
        int32_t tup[PT_MAXK];
        const unsigned long long kv = key[wi];
        pt_unrank_colex((int64_t)(kv >> KEY_BITS), m, C, tup);
        tup[m] = (int32_t)(kv & ((1ull << KEY_BITS) - 1));
        double R = 0.0;
        for (int d = 0; d < n_devices; d++) {
            double den = 0.0, wsum = 0.0;
            for (int q = seg[d] + lane; q < seg[d + 1]; q += 32) {
                double y = tcm[(int64_t)tup[0] * E_pad + q];
                for (int u = 1; u < k; u++) y = fmin(y, tcm[(int64_t)tup[u] * E_pad + q]);
                den += w[q] * y;
                wsum += w[q];
            }
            for (int o = 16; o; o >>= 1) {
                den += __shfl_xor_sync(0xffffffffu, den, o);
                wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
            }
            if (wsum > 0.0) R += qdev[d] / den;
        }
        if (lane == 0) rec_offer(r, 1.0 / R, tup, k);
    }
    sh[threadIdx.x] = r;
    __syncthreads();
    for (int h = 128; h > 0; h >>= 1) {
        if ((int)threadIdx.x < h) {
            Rec2 o = sh[threadIdx.x + h];
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
        Rec2 o;
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
    for (int h = 128; h > 0; h >>= 1) {
        if ((int)threadIdx.x < h) {
            Rec2 o = sh[threadIdx.x + h];
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
        *done = 0;
    }
}

pt_status pt_fleet_exhaustive_tiled(pt_ctx *ctx, int32_t k, int32_t shard_rank, int32_t shard_count,
                                    const pt_fleet_tiled *ft, int32_t *best, int32_t *runner, double *R_out,
                                    double *cost_out, int *n_found)
{
    cudaStream_t s = ctx->stream;
    const pt_view *v = &ctx->full;
    const pt_fleet &f = ctx->fl;
    const int m = k - 1;
    pt_tasks *T = nullptr;
    PT_TRY(build_tasks(ctx, v, m, XT_R, XT_C, &T));
    const int4 *task_list = T->d;
    int ta = 0, tb = (int)T->h.size();
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
    ctx->stats.exh_kernel = 3;
    ctx->stats.exh_env_pad = ft->E_fp;
    ctx->stats.exh_candidates = 0;
    ctx->stats.exh_passes = 0;
    ctx->stats.exh_main_ms = 0.0;
    std::vector<int32_t> t(2 * k, 0);
    double sv[2] = {INFINITY, INFINITY};
    auto finish = [&]() {
        const int nf = (sv[0] < INFINITY) + (sv[1] < INFINITY);
        if (n_found) *n_found = nf;
        for (int u = 0; u < k; u++) {
            best[u] = t[u];
            if (runner) runner[u] = t[k + u];
        }
        cost_out[0] = sv[0];
        cost_out[1] = sv[1];
        R_out[0] = nf >= 1 ? 1.0 / sv[0] : NAN;
        R_out[1] = nf >= 2 ? 1.0 / sv[1] : NAN;
        return PT_OK;
    };
    if (ta >= tb) return finish();

    // error model: each device sum s'_d of scaled weighted runtimes is
    // the fp16 tier's sum of exact-normal fp16 terms -> |s_hat - s| <= eta s (the same
    // tree/chain analysis as Eq. 1, no absolute term: every term is a normal fp16); then
    // R_hat = sum_d RN(Q_d / s_hat_d) in fp32 (Q_d carries one fp32 rounding):
    //   R_hat = R (1 + phi),  |phi| <= eta / (1 - eta) + (n_dev + 3) u32
    const double u16 = std::ldexp(1.0, -11), u32 = std::ldexp(1.0, -24);
    const double lv16 = 2.0 + XT_NG;
    const double ngrp = (double)ft->E_fp / (4.0 * XT_NG) + 2.0;
    const double gam = ngrp * u32 / (1.0 - ngrp * u32);
    const double eta = (lv16 * u16 + lv16 * lv16 * u16 * u16 + gam + std::ldexp(1.0, -50)) * 1.01;
    const double eta_R = (eta / (1.0 - eta) + (f.n_dev + 3) * u32) * 1.02;
    auto f_up = [](double x) -> float {
        if (!(x < 3.0e38)) return INFINITY;
        float g = (float)x;
        if ((double)g < x) g = nextafterf(g, INFINITY);
        return g;
    };
    auto f_dn = [](double x) -> float {
        float g = (float)x;
        if ((double)g > x) g = nextafterf(g, -INFINITY);
        return g;
    };
    const float c1 = f_dn(1.0 / (1.0 + eta_R)), c3 = f_up(1.0 / (1.0 - eta_R));
    // seed: greedy's runner-up rate at step k (two distinct k-sets: <= R_(2))
    float tau_seed = 0.0f;
    {
        std::vector<int32_t> gi(k);
        std::vector<double> gr(k), gg(k);
        PT_TRY(pt_fleet_greedy(ctx, k, nullptr, gi.data(), gr.data(), gg.data()));
        const double r2 = gr[k - 1] - gg[k - 1];
        if (std::isfinite(r2) && r2 > 0.0) tau_seed = f_dn(r2 * (1.0 - 1e-9));
    }
    if (!ft->hWTile) {
        pt_fleet_tiled *mt = const_cast<pt_fleet_tiled *>(ft);
        mt->n_ct = (v->C_pad + XT_C - 1) / XT_C + 1;
        PT_TRY(pt_dalloc(ctx, (void **)&mt->hWTile, sizeof(uint16_t) * 8 * mt->n_ct * ft->E_fp * XT_C));
        k_tile_hT<<<(unsigned)(8 * mt->n_ct), 256, 0, s>>>(ft->hWT, ft->E_fp, v->C_pad, mt->n_ct, mt->hWTile);
        ctx->stats.launches++;
        PT_CK(cudaGetLastError());
    }
    auto kern = k_exh_tiled<true>;
    const size_t smem = sizeof(uint32_t) * XT_S * XT_K * (XT_C / 2) + sizeof(uint16_t) * ft->E_fp * XT_R +
                        sizeof(int) * XT_R + 2 * sizeof(uint64_t) * XT_S + sizeof(int4) + sizeof(int) * XT_S;
    static std::mutex mu;
    static std::map<std::pair<int, size_t>, int> occ_cache;   // (device, smem) -> blocks per SM
    int occ = 1;
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = occ_cache.find(std::make_pair(ctx->dev, smem));
        if (it == occ_cache.end()) {
            PT_TRY(pt_smem_optin(ctx, (const void *)kern));
            PT_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, XT_TCONS, smem));
            occ_cache[std::make_pair(ctx->dev, smem)] = occ;
        } else {
            occ = it->second;
        }
    }
    unsigned cap = 1u << 20;
    unsigned long long n_cand = 0;
    float tau_pass = tau_seed;
    for (int pass = 0; pass < 2; pass++) {
        size_t off = 0;
        auto take = [&](size_t b) { size_t o = off; off += pt_round_up(b, 256); return o; };
        const size_t o_ctr = take(sizeof(int)), o_U = take(sizeof(unsigned)), o_n = take(sizeof(unsigned long long)),
                     o_key = take(sizeof(unsigned long long) * cap), o_cq = take(sizeof(float) * cap),
                     o_os = take(sizeof(double) * 2), o_ot = take(sizeof(int32_t) * 2 * k),
                     o_blk = take(sizeof(Rec2) * (size_t)ctx->num_sms * 2), o_done = take(sizeof(unsigned));
        void *scr = nullptr;
        PT_TRY(pt_scratch(ctx, off, &scr));
        char *b = (char *)scr;
        int *ctr = (int *)(b + o_ctr);
        unsigned *U = (unsigned *)(b + o_U), *done = (unsigned *)(b + o_done);
        unsigned long long *cn = (unsigned long long *)(b + o_n);
        unsigned long long *ckey = (unsigned long long *)(b + o_key);
        float *cq = (float *)(b + o_cq);
        double *os = (double *)(b + o_os);
        int32_t *ot = (int32_t *)(b + o_ot);
        Rec2 *blk = (Rec2 *)(b + o_blk);
        pt_hostio io(ctx);
        PT_TRY(io.h2d(ctr, &ta, sizeof(int)));
        PT_CK(cudaMemsetAsync(U, 0, sizeof(unsigned), s));   // 0.0f: no lower bound yet
        PT_CK(cudaMemsetAsync(cn, 0, sizeof(unsigned long long), s));
        PT_CK(cudaMemsetAsync(done, 0, sizeof(unsigned), s));
        XParams p{};
        p.C = v->C;
        p.C_pad = v->C_pad;
        p.E_pad = ft->E_fp;
        p.n_rows = pt_binom(v->C, m);
        p.m = m;
        p.tasks = task_list;
        p.task_hi = tb;
        p.task_ctr = ctr;
        p.tau_seed = tau_pass;
        p.c1 = c1;
        p.c2 = 0.0f;
        p.c3 = c3;
        p.c4 = 0.0f;
        p.U = U;
        p.cand_key = ckey;
        p.cand_s = cq;
        p.cand_n = cn;
        p.cap = cap;
        p.hT = ft->hWT;
        p.hTile = ft->hWTile;
        p.n_ct = ft->n_ct;
        p.stage_end_mask = ft->stage_end_mask;
        for (int q = 0; q < XT_MAXSTAGE; q++) p.stage_Q[q] = ft->stage_Q[q];
        const int grid = std::min(ctx->num_sms * std::max(occ, 1), tb - ta);
        PT_CK(cudaEventRecord(ctx->ev0, s));
        kern<<<grid, XT_TCONS, smem, s>>>(p);
        PT_CK(cudaEventRecord(ctx->ev1, s));
        k_fleet_refine_top2<<<(unsigned)(ctx->num_sms * 2), 256, 0, s>>>(
            ckey, cq, cn, cap, tau_pass, U, m, v->C, f.tcm, v->E_pad, f.w, f.seg, f.n_dev, f.qdev, blk, done, os, ot);
        ctx->stats.launches += 2;
        pt_pack_record(ctx, os, ot, k);
        PT_CK(cudaGetLastError());
        unsigned hU = 0;
        PT_TRY(io.d2h(&n_cand, cn, sizeof(unsigned long long)));
        PT_TRY(io.d2h(&hU, U, sizeof(unsigned)));
        PT_TRY(io.d2h(sv, os, sizeof(double) * 2));
        PT_TRY(io.d2h(t.data(), ot, sizeof(int32_t) * 2 * k));
        PT_TRY(io.finish());
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        if (pass == 0) ctx->stats.exh_main_ms = ms;
        ctx->stats.exh_passes = pass + 1;
        float Uf;
        memcpy(&Uf, &hU, sizeof Uf);
        if (n_cand > cap) {   // overflow: rerun with the final threshold and room for every survivor
            if (n_cand > (1ull << 28))
                return pt_fail(PT_ECAP, "%llu fp16-tier survivors (massively tied data): above the 2^28 buffer limit",
                               n_cand);
            cap = (unsigned)n_cand;
            tau_pass = std::max(tau_pass, Uf);
            continue;
        }
        ctx->stats.exh_candidates = n_cand;
        if (n_cand == 0) {
            sv[0] = sv[1] = INFINITY;
            for (int u = 0; u < 2 * k; u++) t[u] = 0;
        }
        return finish();
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
