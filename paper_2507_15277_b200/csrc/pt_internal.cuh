// pt_internal.cuh -- context, error plumbing and small device helpers shared by
// the libpt.so translation units.  Nothing here is shared with oracle/.
#pragma once

#include <cuda.h>            // CUtensorMap (type only; entry point fetched at run time)
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "pt.h"

// NVTX ranges (header-only nvtx3; no-ops unless a tool is attached): every pt_* entry
// point opens one named range for its whole duration (nsys / ncu --nvtx)
#include <nvtx3/nvToolsExt.h>
struct pt_nvtx_range {
    explicit pt_nvtx_range(const char *name) { nvtxRangePushA(name); }
    ~pt_nvtx_range() { nvtxRangePop(); }
};
#define PT_NVTX() pt_nvtx_range pt_nvtx_range_(__func__)

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
pt_status pt_fail(pt_status st, const char *fmt, ...);

#define PT_CK(call)                                                                   \
    do {                                                                              \
        cudaError_t e_ = (call);                                                      \
        if (e_ != cudaSuccess)                                                        \
            return pt_fail(PT_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,       \
                           cudaGetErrorString(e_));                                   \
    } while (0)

#define PT_TRY(call)                                                                  \
    do {                                                                              \
        pt_status s_ = (call);                                                        \
        if (s_ != PT_OK) return s_;                                                   \
    } while (0)

// ---------------------------------------------------------------------------
// a scope = the environments in play, compacted to a dense matrix.
//   l32  [C][E_pad]  fp32 log-slowdowns, config-major (env fastest)
//   l64  [C][E_pad]  fp64 log-slowdowns, config-major
//   hT   [E_pad][C_pad] fp16 (raw bits), env-major (config fastest): l64
//        rounded to nearest fp16 -- the operand of the exhaustive kernel's
//        packed-fp16 filter tier (error window in DESIGN.md "Numerics").
// Padded environments hold 0 (adds nothing to any sum); padded configs of hT
// hold 0 and are never selectable (index-masked).
// ---------------------------------------------------------------------------
struct pt_view {
    int64_t E = 0, E_pad = 0, C = 0, C_pad = 0;
    float *l32 = nullptr;
    double *l64 = nullptr;
    uint16_t *hT = nullptr;
    // hTile[s][ct][e][64]: hT re-laid out in 64-config column tiles starting at
    // config 64*ct + 8*s (s = 0..7), so any 8-aligned 32-env x 64-config tile is
    // one contiguous 4 KB block (one bulk copy).  Built on first exhaustive use.
    uint16_t *hTile = nullptr;
    int64_t n_ct = 0;
    // u8 tier of the exhaustive search (k_exh_q8), built on first use: every value
    // quantised to q = rint(l / Delta) in 0..255, Delta = (scope max of l) / 255;
    //   qC    [C_pad][E_pad/4] u32, config-major, 4 consecutive envs per word (low byte first)
    //   qTile [8][n_ct][E_pad/4][64] u32: qC re-laid out in 64-config column tiles
    //         starting at config 64*ct + 8*s (one contiguous block per tile: one bulk copy)
    //   qSum  [(n_ct + 1) * 64] int32: sum over envs of q per config (0 past C)
    //   qConst[0..3] float: c1, c2, c3, c4 of the window (LB = RD(X c1 - c2), UB = RU(X c3 + c4),
    //         X = twice the quantised set score); qConst + 4 (as double): 1 / Delta
    uint32_t *qC = nullptr;
    uint32_t *qTile = nullptr;
    int32_t *qSum = nullptr;
    float *qConst = nullptr;
    // operands of the archived tensor-summed variants (tools/r1_variants, tools/exh_tc):
    //   hC [C_pad][E_pad] fp16 config-major; hPair [8][n_ct][E_pad/2][64] env-pair words
    uint16_t *hC = nullptr;
    uint32_t *hPair = nullptr;
    bool owned = false;
    // exact greedy trace of the longest greedy run on this view (greedy is
    // deterministic and prefix-consistent, so a k-step run answers every k' <= k):
    // the exhaustive search reads its seed (runner-up score at step k) from here
    mutable std::vector<double> greedy_s2;
    // the same runner-up trace left on the device by a seed-only greedy launch
    // (pt_greedy_seed_enqueue): the exhaustive search seeds its threshold from it
    // without a host round trip.  d_seed_k = steps it holds (0 = none).
    double *d_seed_s2 = nullptr;
    int32_t *d_seed_idx = nullptr;   // the picks of that run (the swap search's start)
    int d_seed_k = 0;
    mutable std::vector<int32_t> greedy_idx;   // picks of the host-traced greedy run
    // threshold-count tier (exh_tc.cu), rebuilt per search (the thresholds follow tau):
    //   tcA [tc_ncfg][tc_K] bytes, config-major: E4M3 1.0 where l[c][e] >= j u (k = j E_pad + e)
    //   tcB the same bits in the B-stage layout of k_exh_tc ([K/64][tc_ncfg/8][512 B])
    //   tcConst device constants (u, survivor threshold, slack, the scope max of l)
    uint8_t *tcA = nullptr, *tcB = nullptr;
    void *tcConst = nullptr;
    int64_t tc_ncfg = 0;
    int tc_K = 0;
};

struct pt_tasks;  // exhaustive work list (exhaustive.cu)

struct pt_scope {   // one cached compacted scope
    std::vector<uint8_t> mask;
    pt_view view;
    uint64_t last_use = 0;
};

// fp16 operands of the tiled fleet search (full scope, built on first use after
// pt_set_fleet): per device d the weighted runtimes W[q][c] = quantity(q) * T[q][c]
// of its environments, scaled by a power of two sigma_d (max of the segment -> 2^10,
// so a 16-env fp16 chain cannot overflow), rounded to fp16, each segment padded with
// zero rows to whole 64-env stages.  eligible = every scaled value is a normal fp16
// (>= 2^-14: pure relative rounding error) and there are at most 32 stages.
struct pt_fleet_tiled {
    bool built = false, eligible = false;
    int64_t E_fp = 0;            // padded env rows (sum of ceil64(E_d))
    int64_t n_ct = 0;
    uint16_t *hWT = nullptr;     // [E_fp][C_pad] fp16, env-major
    uint16_t *hWTile = nullptr;  // [8 shifts][n_ct][E_fp][64] (the hTile layout)
    uint32_t stage_end_mask = 0; // bit q: stage q ends a device segment
    float stage_Q[32] = {};      // quantity(d) * sigma_d at that stage
};

// fleet objective (Eq. 2) data, built by pt_set_fleet
struct pt_fleet {
    pt_fleet_tiled tiled;
    bool set = false;
    int32_t n_dev = 0;
    double *tcm = nullptr;    // [C][E_pad] runtimes (missing -> penalty*best), envs grouped by device
    double *tem = nullptr;    // [E_pad][C] the same values env-major (thread-per-subset exhaustive)
    double *w = nullptr;      // [E_pad] quantity(i) of each (permuted) env, 0 for padding
    double *qdev = nullptr;   // [n_dev] quantity(d)
    int32_t *seg = nullptr;   // [n_dev+1] env offsets of each device's segment
    std::vector<int32_t> perm;      // permuted position -> original env
    std::vector<int32_t> h_seg;
    std::vector<double> h_w, h_qdev;
};

struct pt_ctx {
    int dev = 0;
    cudaStream_t stream = nullptr;
    uint32_t flags = 0;
    int num_sms = 0;
    int64_t E = 0, C = 0;
    std::vector<int32_t> env_device;
    std::vector<double> shard_w;   // pt_set_shard_weights (empty = equal shares)
    bool have_device = false;
    double penalty = 1.0;
    double *best = nullptr;   // [E] fp64, each env's Oracle
    float *T32 = nullptr;     // [E][C] fp32 runtimes as loaded (NaN/inf = missing)
    pt_fleet fl;
    pt_view full;
    // scope cache (LRU of compacted scopes)
    std::vector<pt_scope> scopes;
    uint64_t tick = 0;
    // scratch reused across calls
    void *scratch = nullptr;
    size_t scratch_bytes = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    pt_stats stats{};
    // sharded search (dist.cu): where the exhaustive search packs this rank's record
    double *rec_out = nullptr;
    double rec_fp = 0.0;
    bool rec_written = false;
};

// Small host<->device transfers of one API call through a pinned staging buffer
// (thread-local, allocated once per thread): a pageable cudaMemcpyAsync is
// synchronous (~10 us each on B200), a pinned one is a queued DMA.  Transfers are
// stream-ordered on ctx->stream; finish() synchronises once and scatters the
// device->host results to their destinations.  Larger transfers fall back to a
// direct (pageable) copy.
struct pt_hostio {
    explicit pt_hostio(pt_ctx *c) : ctx(c) {}
    pt_status h2d(void *dev_dst, const void *host_src, size_t n);
    pt_status d2h(void *host_dst, const void *dev_src, size_t n);
    pt_status finish();
    pt_ctx *ctx;
    size_t off = 0;
    struct item { void *dst; size_t off, n; };
    std::vector<item> items;
};

// stream-ordered device allocation from the device's (cached) memory pool
pt_status pt_dalloc(pt_ctx *ctx, void **p, size_t bytes);
void pt_dfree(pt_ctx *ctx, void *p);
// scratch allocation (grows, never shrinks); returns PT_OK or PT_ENOMEM
pt_status pt_scratch(pt_ctx *ctx, size_t bytes, void **p);
// resolve a mask into a view (NULL -> full); E_scope returned in view->E
pt_status pt_get_view(pt_ctx *ctx, const uint8_t *env_mask, const pt_view **out);
void pt_view_free(pt_ctx *ctx, pt_view &v);
// build the view's fp16 tier (hT) if it does not exist yet
// raise a kernel's dynamic shared-memory limit to the device's opt-in maximum, once per
// (device, kernel).  A per-call limit cached by smem size can be left below a later
// launch's smem when a smaller size was set in between (a launch error).
pt_status pt_smem_optin(pt_ctx *ctx, const void *kfn);
pt_status pt_view_fp16(pt_ctx *ctx, const pt_view *v);
// true if p is device (or managed) memory
bool pt_is_device_ptr(const void *p);

// selection entry points used across files
pt_status pt_greedy_view(pt_ctx *ctx, const pt_view *v, int32_t k, int32_t *out_idx,
                         double *s1_trace, double *s2_trace);
// enqueue a resident greedy of k steps on ctx->stream whose runner-up trace stays on the
// device (v->d_seed_s2); PT_EINVAL if this view takes the streamed greedy instead
pt_status pt_greedy_seed_enqueue(pt_ctx *ctx, const pt_view *v, int32_t k);
pt_status pt_exhaustive_view(pt_ctx *ctx, const pt_view *v, int32_t k, int32_t shard_rank,
                             int32_t shard_count, int32_t *best, int32_t *runner,
                             double *s_out, int *n_found);
pt_status pt_score_view(pt_ctx *ctx, const pt_view *v, const int32_t *d_sets, int64_t n_sets,
                        int32_t k, double *d_s);
// threshold-count tier of the exhaustive search (exh_tc.cu): enqueue the device swap
// search for tau, the bit operands and k_exh_tc on ctx->stream (no host round trip).
// PT_EINVAL = not eligible for this view / k (the caller takes the u8 tier); a tau that
// turns out unusable on the device sets *cand_n = 2^63 (the refine then skips).
struct pt_tc_args {
    int k = 0;
    const int4 *tasks = nullptr;   // this shard's task list [ta, tb) (rows 128, columns 256)
    int ta = 0, tb = 0;
    int *ctr = nullptr;
    unsigned *U = nullptr;         // written: the refine's threshold (float bits)
    unsigned long long *cand_n = nullptr, *cand_key = nullptr;
    float *cand_s = nullptr;
    unsigned cap = 0;
    const int32_t *d_S0 = nullptr;     // greedy's k-set (device)
    const double *d_seed_s2 = nullptr; // greedy's runner-up score at step k (device) or NULL
    double *swap_rs = nullptr;         // [2 num_sms] scratch
    long long *swap_rw = nullptr;      // [2 num_sms] scratch
    double *tau_dev = nullptr;         // [1] scratch
    int halves = 2;                    // row halves per task: 128 halves rows x (256 / halves) columns
    bool split = false;                // k = 3 two-family task list (exhaustive.cu build_tasks_split3)
};
pt_status pt_exh_tc_enqueue(pt_ctx *ctx, const pt_view *v, const pt_tc_args &a, int *nt_out);
int pt_tc_halves();
// sharded search (dist.cu): pack the local top-2 (device os[2], ot[2k]) into ctx->rec_out
void pt_pack_record(pt_ctx *ctx, const double *d_os, const int32_t *d_ot, int k);
// fleet objective (fleet.cu): rates of sets / greedy / exhaustive, env_mask may be NULL
pt_status pt_fleet_score(pt_ctx *ctx, const int32_t *d_sets, int64_t n_sets, int32_t k,
                         const uint8_t *env_mask, double *d_R);
pt_status pt_fleet_greedy(pt_ctx *ctx, int32_t k, const uint8_t *env_mask, int32_t *out_idx,
                          double *R_trace, double *gap_trace);
pt_status pt_fleet_exhaustive(pt_ctx *ctx, int32_t k, const uint8_t *env_mask, int32_t shard_rank,
                              int32_t shard_count, int32_t *best, int32_t *runner, double *R_out,
                              double *cost_out, int *n_found);
// the tiled fleet search: operands (fleet.cu) and the search itself (exhaustive.cu)
pt_status pt_fleet_tiled_operands(pt_ctx *ctx, const pt_fleet_tiled **out);
void pt_fleet_tiled_free(pt_ctx *ctx);
pt_status pt_fleet_exhaustive_tiled(pt_ctx *ctx, int32_t k, int32_t shard_rank, int32_t shard_count,
                                    const pt_fleet_tiled *ft, int32_t *best, int32_t *runner, double *R_out,
                                    double *cost_out, int *n_found);


// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
static inline int64_t pt_round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// binomial coefficient C(n, r) for small r, exact in int64 for the sizes used
// here (n <= 2^21, r <= 4); returns 0 when n < r.
__host__ __device__ static inline int64_t pt_binom(int64_t n, int r)
{
    if (n < r || r < 0) return 0;
    switch (r) {   // constant divisors: no 64-bit division loop on the device
    case 0: return 1;
    case 1: return n;
    case 2: return n * (n - 1) / 2;
    case 3: return n * (n - 1) * (n - 2) / 6;
    case 4: return n * (n - 1) * (n - 2) / 6 * (n - 3) / 4;
    default: {
        int64_t v = 1;
        for (int q = 0; q < r; q++) v = v * (n - q) / (q + 1);
        return v;
    }
    }
}

// colex unranking of a (k-1)... generic m-subset: rank R -> ascending members.
// Largest c with C(c, u+1) <= R, for u = m-1 .. 0.  n = universe size.
__host__ __device__ static inline void pt_unrank_colex(int64_t R, int m, int64_t n, int32_t *out)
{
    for (int u = m - 1; u >= 0; u--) {
        // binary search c in [u, n-1]
        int64_t lo = u, hi = n - 1;
        while (lo < hi) {
            int64_t mid = (lo + hi + 1) >> 1;
            if (pt_binom(mid, u + 1) <= R) lo = mid; else hi = mid - 1;
        }
        out[u] = (int32_t)lo;
        R -= pt_binom(lo, u + 1);
    }
}

// lexicographic order on sorted tuples + score: returns true if (sa,a) < (sb,b)
__host__ __device__ static inline bool pt_key_less(double sa, const int32_t *a, double sb,
                                                   const int32_t *b, int k)
{
    if (sa < sb) return true;
    if (sa > sb) return false;
    for (int u = 0; u < k; u++) {
        if (a[u] < b[u]) return true;
        if (a[u] > b[u]) return false;
    }
    return false;
}

#define PT_MAXK 8

// exhaustive search (exhaustive.cu, exh_tc.cu): first column of a row tile whose first
// row's largest member is j0: j0 + 1 rounded down to 8 configs (16-byte aligned rows);
// the extra columns are <= every row's largest member and masked.  Used by the task
// builder AND every tiled kernel so all cover exactly [tile_lo, tile_lo + W * n_ct) >=
// [j0+1, C) for their column-tile width W.
__host__ __device__ static inline int64_t tile_lo(int64_t j0) { return (j0 + 1) & ~(int64_t)7; }
// survivor key = (row colex rank << KEY_BITS) | column
#define KEY_BITS 21
#define PT_SWAP_MAXK 32
