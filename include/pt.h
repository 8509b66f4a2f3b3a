/*
 * pt.h -- C ABI of the B200-native portability-tuning hot path
 * (arXiv 2507.15277, "portability tuning").  Implemented by libpt.so
 * (hand-written sm_100a CUDA, paper_2507_15277_b200/csrc/).
 *
 * Problem statement (Sec. 4.2):  kappa = PortabilityTune(iota,
 * delta, eps) returns a size-bounded SET of parameter configurations that is
 * best by a summary metric over the environments (device x GEMM input,
 * P:L151).  The summary metric is Eq. 1 (Sec. 4.4.1) read with
 * the best member per environment, reported as the geometric-mean
 * efficiency
 *
 *     G(S) = exp( -(1/|scope|) * sum_{e in scope} min_{c in S} l[c][e] ),
 *     l[c][e] = log( T[e][c] / best[e] ),   best[e] = min_c T[e][c]
 *
 * i.e. G = 1 / geomean(Slowdown over Oracle); G in (0, 1], maximised.
 * eps (OS, compiler, ...) has no data representation and is not modelled.
 *
 * Conventions (every function):
 *   - returns a pt_status; PT_OK = 0, errors < 0; never aborts; the message of
 *     the last error on the calling thread is pt_last_error().
 *   - the caller owns every input array (copied or read during the call) and
 *     every output array; scalar and small outputs are HOST pointers.
 *   - all device work is ordered on the CUDA stream given to pt_load_perf and
 *     each call returns after its results are on the host.
 *   - a pt_ctx is not thread-safe; use one per thread / per GPU.
 *   - "host or device" pointers are classified with cudaPointerGetAttributes.
 *   - ties between equal scores: exhaustive -> the lexicographically smallest
 *     sorted index tuple; greedy -> the lowest configuration index.
 */
#ifndef PT_H
#define PT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pt_ctx pt_ctx;   /* opaque; owns every device buffer it allocates */

typedef enum {
    PT_OK = 0,
    PT_EINVAL = -1,   /* bad argument (k < 1, k > #configs, bad index, bad shard) */
    PT_ENOMEM = -2,   /* host or device allocation failed */
    PT_ECUDA = -3,    /* CUDA runtime / driver error (message has details) */
    PT_ENCCL = -4,    /* collective failure (NCCL or the caller's exchange callback) */
    PT_ECAP = -5,     /* C(n,k) exceeds the enumeration cap (1e13) */
    PT_EEMPTY = -6,   /* empty scope (mask selects no environment) or empty set */
    PT_EDATA = -7     /* runtime <= 0, or an environment with no measured cell */
} pt_status;

typedef enum {
    PT_OBJ_GEOMEAN = 0,   /* Eq. 1 library objective: G = geomean efficiency (graded path) */
    PT_OBJ_FLEET = 1      /* Eq. 2 fleet rate R (tasks/ms); needs pt_set_fleet.
                             Reported in the out_G slots; sets are ranked by R desc
                             (the tuner minimises 1/R), ties as above */
} pt_objective;

/* pt_load_perf flags */
enum {
    PT_MISSING_PENALTY_MAX = 0x1, /* default: a missing cell (NaN/+inf) costs the
                                     dataset-max slowdown x best[e] */
    PT_EXACT_FP64 = 0x2,          /* debug: exhaustive search by the thread-per-subset
                                     fp64 kernel, no fp32 tier */
    PT_GREEDY_STREAM = 0x4,       /* force the streamed fp32-filter/fp64-refine greedy
                                     (default only when the matrix is large) */
    PT_GREEDY_LAZY = 0x8          /* streamed greedy, lazy from step 3 on: exact (Minoux)
                                     upper-bound pruning by submodularity of the gain; same
                                     picks, far fewer sets scored (gap trace: an upper bound) */
};

/*
 * pt_load_perf -- ingest + normalise (the post-processing pass, P:L392;
 * the Oracle best[e]).
 *   times_ms   host or device, fp32, env-major rows: times_ms[e*ld + c] is the
 *              runtime (ms) of configuration c in environment e.  NaN/+inf =
 *              missing.  Environments are device-major then input.
 *   n_env, n_cfg, ld   E >= 1, C >= 1, ld >= C (elements).
 *   env_device host, int32[n_env] device id per environment (>= 0, else
 *              PT_EINVAL), or NULL (then every env is device 0; pt_eval_holdout
 *              needs it).
 *   flags      PT_* flags above.
 *   cuda_device  device ordinal; cuda_stream: cudaStream_t borrowed (NULL =
 *              the legacy default stream), not owned.
 * On success *out receives a context owning the device copies:
 *   l32  [C][E_pad] fp32 and l64 [C][E_pad] fp64 (config-major), l32T
 *   [E_pad][C_pad] fp32 (env-major), best [E] fp64.
 * Errors: PT_EINVAL, PT_EDATA (runtime <= 0 / env with no measured cell),
 *         PT_ENOMEM, PT_ECUDA.
 */
pt_status pt_load_perf(pt_ctx **out, const float *times_ms, int64_t n_env, int64_t n_cfg,
                       int64_t ld, const int32_t *env_device, uint32_t flags,
                       int cuda_device, void *cuda_stream);

/*
 * pt_score_sets -- Eq. 1 fitness of a batch of candidate sets.
 *   sets       host or device, int32[n_sets][k] configuration indices
 *              (any order; duplicates allowed and harmless).
 *   env_mask   host, uint8[n_env] (nonzero = env in scope) or NULL = all.
 *   objective  PT_OBJ_GEOMEAN.
 *   out_G      host or device, double[n_sets]: G of every set (fp64, fixed
 *              summation order).
 * Errors: PT_EINVAL (index out of range, k < 1), PT_EEMPTY (empty scope).
 */
pt_status pt_score_sets(pt_ctx *ctx, const int32_t *sets, int64_t n_sets, int32_t k,
                        const uint8_t *env_mask, int32_t objective, double *out_G);

/*
 * pt_greedy_select -- greedy forward selection (north_star): k dependent steps,
 * each scores S u {c} for every unselected c in parallel and takes the argmax
 * (ties -> lowest c).  Exact in fp64 (or fp32 filter + fp64 refine, same
 * result).
 *   out_idx        host int32[k]: the picks in order.
 *   out_G_trace    host double[k] or NULL: G(S_t) after step t.
 *   out_gap_trace  host double[k] or NULL: G of the step's best minus G of its
 *                  second-best candidate (+inf if there was one candidate).
 * Errors: PT_EINVAL (k < 1 or k > C), PT_EEMPTY.
 */
pt_status pt_greedy_select(pt_ctx *ctx, int32_t k, const uint8_t *env_mask, int32_t objective,
                           int32_t *out_idx, double *out_G_trace, double *out_gap_trace);

/*
 * pt_exhaustive_best -- exhaustive search over every k-subset (P:L271-276,
 * Sec. 4.3.1; distinct unordered subsets of size exactly k).
 *   shard_rank, shard_count   this call searches shard `shard_rank` of
 *              `shard_count` equal-work pieces of the subset space (0, 1 =
 *              everything; the tiled search deals its decreasing-size task list
 *              to the shards in snake order, or by pt_set_shard_weights; the
 *              generic search (k > 4 or > 768 envs) cuts contiguous rank ranges).
 *              Results of all shards merged with pt_merge_top2 equal the
 *              unsharded result.
 *   out_idx        host int32[k]: best set, ascending.
 *   out_G          host: its G.
 *   out_runner_idx host int32[k] or NULL: the second set in (G desc, tuple asc)
 *                  order; out_G_runner host or NULL: its G (NaN if none).
 *   out_s          host double[2] or NULL: the exact fp64 log-slowdown sums
 *                  s = -|scope| log G of best and runner-up (+inf if absent) --
 *                  the keys pt_merge_top2 orders by.
 * Method (k = 2..4, scopes <= 768 envs): a filter scores every set, keeps every
 * set whose rigorous lower bound reaches the best two, and re-scores those in
 * fp64; the result is the same as scoring every set in fp64.  Filters: for k = 3, 4
 * (and k = 2 with environment PT_EXH_TIER=tc) the threshold-count lower bound on
 * the tcgen05 tensor cores against tau from a device-side swap search (DESIGN.md
 * 6.2c); for k = 2, and whenever that filter cannot run (tau not usable, more than
 * 2^20 survivors unsharded, > 1024 padded envs), the exact integer score of the
 * matrix quantised to bytes (q = rint(l / Delta), Delta = scope max / 255,
 * DESIGN.md 6.2b); PT_EXH_TIER=u8 / fp16 select those tiers.  Sharded searches
 * choose the tier identically on every rank (tau is computed from the whole scope)
 * and rerun a tc pass with a larger buffer rather than fall back, so all ranks
 * scan the same task list.
 * Errors: PT_EINVAL (k < 1, k > C, bad shard), PT_ECAP (C(n,k) > 1e13, or more
 *         than 2^28 fp16-tier or tc-shard survivors), PT_EEMPTY.
 */
pt_status pt_exhaustive_best(pt_ctx *ctx, int32_t k, const uint8_t *env_mask, int32_t objective,
                             int32_t shard_rank, int32_t shard_count,
                             int32_t *out_idx, double *out_G,
                             int32_t *out_runner_idx, double *out_G_runner, double *out_s);

/*
 * pt_set_shard_weights -- relative work shares of the shards for later sharded
 * exhaustive searches on this context with shard_count == n (heterogeneous
 * ranks: e.g. a rank that also runs the unsharded greedy takes a smaller share).
 * The tiled search deals its decreasing-size task list to the shard with the
 * smallest weighted load (each shard's list stays decreasing); results are exact
 * and identical for any weights.  weights: host double[n], each > 0 and finite,
 * copied (caller keeps ownership); n = 0 or weights = NULL restores equal shares.
 * Errors: PT_EINVAL (n < 0, a non-positive or non-finite weight).
 */
pt_status pt_set_shard_weights(pt_ctx *ctx, const double *weights, int32_t n);

/*
 * pt_greedy_sharded -- the greedy selection with the configurations sharded
 * across ranks: rank shard_rank streams only its
 * contiguous 1/shard_count of the configurations each step, finds its exact
 * local top-2 (s, config), and the ranks exchange those records through
 * `allgather` (the caller's collective, e.g. NCCL via torch.distributed); every
 * rank merges them identically (s asc, config asc) and commits the winner from
 * its own copy of the matrix.  Result identical to pt_greedy_select on every rank.
 *   allgather(user, mine, n, all): gather n doubles from every rank into
 *     all[rank * n ...] (rank order); return 0 on success.  Called k times, on
 *     the calling thread.
 * Errors: as pt_greedy_select; PT_ENCCL if the callback fails.
 */
typedef int (*pt_allgather_fn)(void *user, const double *mine, int32_t n, double *all);
pt_status pt_greedy_sharded(pt_ctx *ctx, int32_t k, const uint8_t *env_mask, int32_t shard_rank,
                            int32_t shard_count, pt_allgather_fn allgather, void *user,
                            int32_t *out_idx, double *out_G_trace, double *out_gap_trace);

/*
 * pt_greedy_sharded_dev -- pt_greedy_sharded with a STREAM-ORDERED exchange and
 * no host synchronisation inside the k-step loop: `mine` and `all` are DEVICE
 * pointers (4 doubles; shard_count * 4 doubles) and `stream` is the context's
 * cudaStream_t.  The callback must enqueue the all-gather so that `all` is
 * complete, in stream order, before any later work on `stream` (e.g. an NCCL
 * all-gather on that stream, or a wait on its completion event); the merge of
 * the records and the commit then run on the device.  Same results as
 * pt_greedy_sharded.
 * Errors: as pt_greedy_sharded.
 */
typedef int (*pt_dev_allgather_fn)(void *user, const double *mine, int32_t n, double *all, void *stream);
pt_status pt_greedy_sharded_dev(pt_ctx *ctx, int32_t k, const uint8_t *env_mask, int32_t shard_rank,
                                int32_t shard_count, pt_dev_allgather_fn allgather, void *user,
                                int32_t *out_idx, double *out_G_trace, double *out_gap_trace);

/*
 * ---- the cross-GPU reduction of the sharded exhaustive search ----
 * "returns the variant combination with the highest ranking" over ranks:
 * every rank searches shard `shard_rank` of `shard_count` (pt_exhaustive_best's
 * partition), the ranks all-gather one record each -- [plan fingerprint, s1, s2,
 * tuple1[k], tuple2[k]] as pt_record_len(k) doubles, on the device -- and every rank
 * merges them on the device in (s asc, tuple asc) order and maps s to the objective
 * (G = exp(-s/|scope|), Eq. 1; R = 1/cost, Eq. 2).  Identical results on every rank,
 * equal to the unsharded pt_exhaustive_best for any shard_count.
 *
 * The exchange is either an NCCL all-gather over a communicator the LIBRARY builds
 * (pt_comm_init; NVLink/NVSwitch between the GPUs of a node) or a caller's stream-
 * ordered all-gather (pt_dev_allgather_fn, e.g. gloo with host staging in tests).
 * NCCL is loaded at run time (libnccl.so.2; in a PyTorch process the one torch
 * loaded).  All ranks must load the same matrix and set the same shard weights; a
 * different shard plan on some rank is detected (the fingerprints disagree) and
 * reported as PT_EINVAL instead of a wrong answer.
 */
typedef struct pt_comm pt_comm;        /* opaque; owns an ncclComm_t */
#define PT_COMM_ID_BYTES 128           /* sizeof(ncclUniqueId) */

/* pt_comm_unique_id -- one rank (e.g. rank 0) creates the id (host buffer of
 * PT_COMM_ID_BYTES bytes) and broadcasts it to the others by any means.
 * Errors: PT_EINVAL (NULL), PT_ENCCL (NCCL missing or failing). */
pt_status pt_comm_unique_id(void *out_id);

/* pt_comm_init -- collective over `world` ranks: every rank calls it with the same id
 * and its own rank (0 <= rank < world); one GPU (cuda_device) per rank.
 * *out is freed with pt_comm_free.  Errors: PT_EINVAL, PT_ENCCL, PT_ECUDA. */
pt_status pt_comm_init(pt_comm **out, const void *id, int32_t rank, int32_t world, int cuda_device);
void pt_comm_free(pt_comm *comm);

/* pt_exhaustive_best_sharded -- the sharded search end to end.  Give exactly one of
 *   comm       a communicator whose (rank, world) is (shard_rank, shard_count) and
 *              whose device is the context's, or
 *   allgather  a stream-ordered all-gather (pt_dev_allgather_fn above): mine =
 *              pt_record_len(k) doubles on the device, all = shard_count times that,
 *              in rank order; called once, on the calling thread.
 * Outputs as pt_exhaustive_best (host).  Errors: those of pt_exhaustive_best,
 * PT_ENCCL (the exchange failed), PT_EINVAL (bad shard, mismatched communicator, or
 * ranks with different shard plans), PT_EEMPTY (no subset in any shard). */
pt_status pt_exhaustive_best_sharded(pt_ctx *ctx, int32_t k, const uint8_t *env_mask, int32_t objective,
                                     int32_t shard_rank, int32_t shard_count, pt_comm *comm,
                                     pt_dev_allgather_fn allgather, void *user, int32_t *out_idx,
                                     double *out_G, int32_t *out_runner_idx, double *out_G_runner,
                                     double *out_s);

/* pt_record_len -- doubles per rank record for k (3 + 2k), or -1 if k is out of range. */
int32_t pt_record_len(int32_t k);

/* pt_merge_records -- host-only form of the merge above over n_rank gathered records
 * (host double[n_rank * pt_record_len(k)]), for callers that exchange records
 * themselves; n_env = the scope size (|scope| of Eq. 1).  Same outputs and errors. */
pt_status pt_merge_records(const double *records, int32_t n_rank, int32_t k, int64_t n_env,
                           int32_t objective, int32_t *out_idx, double *out_G,
                           int32_t *out_runner_idx, double *out_G_runner, double *out_s);

/*
 * pt_merge_top2 -- host-only: merge n_rec (s, sorted k-tuple) records (e.g.
 * gathered from every shard/rank) into the best two in (s asc, tuple asc)
 * order.  s = +inf marks an absent record.
 *   s         host double[n_rec];  tuples host int32[n_rec][k]
 *   out_idx, out_runner_idx  host int32[k];  out_s host double[2]
 * Returns PT_EEMPTY if no record is present.
 */
pt_status pt_merge_top2(const double *s, const int32_t *tuples, int32_t n_rec, int32_t k,
                        int32_t *out_idx, int32_t *out_runner_idx, double *out_s);

/*
 * pt_eval_holdout -- leave-one-device-out generalization, the analogue of the
 * unseen-device experiment (Sec. 5.8).
 *   train scope = envs whose device != heldout_device; test = device ==.
 *   method 0 = greedy, 1 = exhaustive.
 *   out_idx        host int32[k]  set selected on the train scope
 *   out_G_train    G of out_idx on the train scope
 *   out_G_unseen   G of out_idx on the held-out device (each env normalised by
 *                  its own best[e])
 *   out_G_known    G of the set selected directly on the held-out envs
 *   out_known_idx  host int32[k] or NULL: that set
 * Errors: PT_EINVAL (no env_device given / bad method), PT_EEMPTY (a scope is
 * empty), plus those of the selection calls.
 */
pt_status pt_eval_holdout(pt_ctx *ctx, int32_t heldout_device, int32_t k, int32_t method,
                          int32_t *out_idx, double *out_G_train, double *out_G_unseen,
                          double *out_G_known, int32_t *out_known_idx);

/*
 * pt_eval_holdout_all -- pt_eval_holdout (method 0, greedy) for every device
 * d = 0..D-1 at once (D = 1 + the largest env_device id), computed in one
 * batched launch.  Outputs are [D][k] / [D] host arrays in the same meaning as
 * pt_eval_holdout, with room for n_device_cap devices (nothing is written past
 * it); *out_n_device (host, or NULL) receives D.
 * Errors: as pt_eval_holdout; PT_EINVAL if D > n_device_cap (*out_n_device
 * still set); PT_EEMPTY if some device has no environment.
 */
pt_status pt_eval_holdout_all(pt_ctx *ctx, int32_t k, int32_t n_device_cap, int32_t *out_idx, double *out_G_train,
                              double *out_G_unseen, double *out_G_known, int32_t *out_known_idx,
                              int32_t *out_n_device);

/*
 * pt_swap_search -- deterministic best-improvement swap local search over
 * k-sets (the stand-in for the paper's heuristic search over variant
 * combinations, Sec. 4.3.1).  From `init` (host
 * int32[k], distinct) or, if NULL, the greedy k-set, every move evaluates all
 * k*(C-k) swaps exactly (fp64) and applies the best if it strictly improves G
 * (ties -> lexicographically smallest resulting sorted tuple); stops at a local
 * optimum or after max_moves moves.
 *   out_idx   host int32[k], the final set ascending;  out_G its G;
 *   out_moves host or NULL: moves applied.
 * PT_OBJ_GEOMEAN only.  Errors: PT_EINVAL (k < 1, k >= C, k > 32, bad init).
 */
pt_status pt_swap_search(pt_ctx *ctx, int32_t k, const uint8_t *env_mask, int32_t objective,
                         int32_t max_moves, const int32_t *init, int32_t *out_idx, double *out_G,
                         int32_t *out_moves);

/*
 * pt_kmeans_select -- the paper's k-means selector (Sec. 4.3.2):
 * environments in scope are points of their slowdowns T/best over all
 * configurations; k centroids by Lloyd iterations from a deterministic maximin
 * initialisation (the point nearest the mean, then successive farthest points);
 * an emptied cluster is re-seeded with the point farthest from its centroid;
 * stops when no assignment changes or after max_iter passes.  Per centroid the
 * configuration with the smallest centroid slowdown is selected;
 * duplicates collapse.  fp64 in a fixed order (bit-identical to the oracle).
 *   out_idx host int32[k]: the selection ascending, *out_n (<= k) entries;
 *   out_G   host or NULL: its Eq. 1 G on the scope; out_iters host or NULL.
 * Errors: PT_EINVAL (k < 1, k > 32, k > #envs in scope), PT_EEMPTY.
 */
pt_status pt_kmeans_select(pt_ctx *ctx, int32_t k, const uint8_t *env_mask, int32_t max_iter,
                           int32_t *out_idx, int32_t *out_n, double *out_G, int32_t *out_iters);

/*
 * pt_kmeans_select_from -- pt_kmeans_select from a given start instead of the maximin
 * initialisation: init host double[k][C] (row j = centroid j in the slowdown space of
 * the points, T/best per configuration), copied.  Same Lloyd loop, re-seed rule and
 * selection; bit-identical to the oracle's or_kmeans_from.
 * Errors: as pt_kmeans_select; PT_EINVAL if init is NULL.
 */
pt_status pt_kmeans_select_from(pt_ctx *ctx, int32_t k, const uint8_t *env_mask, int32_t max_iter,
                                const double *init, int32_t *out_idx, int32_t *out_n, double *out_G,
                                int32_t *out_iters);

/*
 * pt_set_fleet -- quantities for the fleet objective, Eq. 2:
 *   R(S) = sum_d quantity(d) / sum_{i} y'_{d,i}(S) * quantity(i),
 *   y'_{d,i}(S) = min_{c in S} T[(d,i)][c]  (best member; a missing cell costs
 *   the dataset-max slowdown x best[e]).  The inner sum runs over the
 *   environments of device d in scope; a device with none does not contribute.
 *   q_device  host double[n_device], quantity(d) for device ids 0..n_device-1
 *   q_env     host double[n_env], quantity(i) of each environment's input
 * Copied; the context keeps them until the next call.
 * Errors: PT_EINVAL (an env's device id outside [0, n_device), q <= 0).
 */
pt_status pt_set_fleet(pt_ctx *ctx, const double *q_device, int32_t n_device,
                       const double *q_env);

/* Per-context counters (for bench.py's roofline and gpu_launches fields). */
typedef struct {
    int64_t launches;        /* kernels this context has launched so far */
    double exh_main_ms;      /* CUDA-event time of the last exhaustive main-kernel launch */
    int64_t exh_sets;        /* k-subsets that launch scored (its shard) */
    int64_t exh_slots;       /* (row, column) slots it computed, incl. masked waste */
    int64_t exh_env_pad;     /* padded env count of its scope (K-loop length) */
    int64_t exh_candidates;  /* filter-tier candidates re-scored in fp64 */
    int32_t exh_passes;      /* 1; +1 per candidate-buffer overflow rerun or u8 -> fp16 hand-over */
    int32_t exh_kernel;      /* 5 = tiled threshold-count filter on tcgen05 (k_exh_tc, the default
                                for k = 3, 4), 4 = tiled u8 filter (k_exh_q8; k = 2, PT_EXH_TIER=u8,
                                or the fall-back of the tc tier), 0 = tiled fp16 filter (k_exh_tiled;
                                PT_EXH_TIER=fp16, or the u8 tier left more than 2^24 candidates),
                                1 = generic fp64, 2 = fleet fp64, 3 = fleet tiled fp16 */
    double greedy_ms;        /* CUDA-event time of the last greedy selection */
    int64_t greedy_candidates; /* streamed greedy: configs re-scored in fp64 (all steps) */
    int32_t exh_tc_nt;       /* tc tier: thresholds per environment of the last search */
    int32_t exh_tc_pad;
    int64_t exh_tc_survivors; /* tc tier: survivors of its last pass (-1: tau unusable, fell back) */
} pt_stats;

pt_status pt_get_stats(const pt_ctx *ctx, pt_stats *out);

/* Frees every buffer of the context (NULL is a no-op). */
void pt_free(pt_ctx *ctx);

/* Message of the last non-OK status returned on this thread ("" if none). */
const char *pt_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* PT_H */
