/*
 * oracle.c -- CPU ORACLE for portability tuning (arXiv 2507.15277).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * The product path (paper_2507_15277_b200/, libpt.so) never calls it and
 * shares no code, header, table or helper with it.
 *
 * Plain, slow, obviously-correct definitions in fp64.  No blocking, no
 * fusion, no reordering beyond what the definitions state.  Citations are
 * PAPER.md line numbers (P:Ln) with the section they fall in.
 *
 * Data convention: T is the runtime matrix in milliseconds, env-major,
 * T[e*ld + c] for environment e (= device x GEMM input) and
 * parameter configuration c.  A non-finite entry (NaN, +inf)
 * is a missing measurement.
 *
 * Parity status of each function: see DESIGN.md "Oracle pins".  All
 * functions below are pinned (tests/test_oracle*.py, mutation-checked by
 * tools/oracle_mutants.py); none is "parity unpinned".  (The k-means re-seed
 * of an emptied cluster is pinned through or_kmeans_from: the maximin start
 * itself never empties a cluster on the inputs searched.)
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL -1
#define OR_ENOMEM -2
#define OR_EEMPTY -6
#define OR_EDATA -7

/*
 * or_normalize -- the paper's post-processing pass (Sec. 5.3
 * "relative to the best ... kernels for that device and input") and the
 * Oracle of Sec. 5.5 ("best-known configuration ... for every
 * ... device + input pair").
 *
 *   best[e]      = min_c T[e][c]
 *   slowdown     = T[e][c] / best[e]                   (S/O)
 *   penalty      = max over all measured cells of the slowdown
 *                  (reading c4 in DESIGN.md: missing cell -> penalty x best)
 *   logeff[e][c] = log(best[e] / T[e][c])  (<= 0; log of the relative
 *                  performance P/best of north_star, reading c11)
 *
 * logeff is written env-major, logeff[e*C + c].
 * Errors: OR_EDATA for a finite runtime <= 0, or an environment with no
 * measured cell.
 */
int or_normalize(const float *T, int64_t E, int64_t C, int64_t ld,
                 double *best, double *logeff, double *penalty_out)
{
    if (E <= 0 || C <= 0 || ld < C) return OR_EINVAL;
    for (int64_t e = 0; e < E; e++) {
        double b = INFINITY;
        for (int64_t c = 0; c < C; c++) {
            float t = T[e * ld + c];
            if (!isfinite(t)) continue;
            if (t <= 0.0f) return OR_EDATA;
            if ((double)t < b) b = (double)t;
        }
        if (!isfinite(b)) return OR_EDATA;
        best[e] = b;
    }
    double penalty = 1.0;
    for (int64_t e = 0; e < E; e++)
        for (int64_t c = 0; c < C; c++) {
            float t = T[e * ld + c];
            if (!isfinite(t)) continue;
            double s = (double)t / best[e];
            if (s > penalty) penalty = s;
        }
    for (int64_t e = 0; e < E; e++)
        for (int64_t c = 0; c < C; c++) {
            float t = T[e * ld + c];
            double tt = isfinite(t) ? (double)t : penalty * best[e];
            logeff[e * C + c] = log(best[e] / tt);
        }
    if (penalty_out) *penalty_out = penalty;
    return OR_OK;
}

/* The environments in scope, ascending (mask == NULL: all). */
static int64_t scope_list(const uint8_t *mask, int64_t E, int64_t *out)
{
    int64_t n = 0;
    for (int64_t e = 0; e < E; e++)
        if (!mask || mask[e]) out[n++] = e;
    return n;
}

/*
 * Sum over the scope, e ascending, of log(max_{c in S} eff[e][c]).
 * Eq. 1 (Sec. 4.4.1) under the best-member reading c1:
 * "the performance for each environment is that of the best-performing
 * of the ... variants on that environment".
 */
static double logsum(const double *logeff, int64_t C, const int64_t *envs,
                     int64_t ne, const int32_t *set, int k)
{
    double acc = 0.0;
    for (int64_t q = 0; q < ne; q++) {
        const double *row = logeff + envs[q] * C;
        double m = row[set[0]];
        for (int u = 1; u < k; u++)
            if (row[set[u]] > m) m = row[set[u]];
        acc += m;
    }
    return acc;
}

/*
 * or_score -- Eq. 1 as a maximised efficiency (reading c2):
 *   G(S) = exp( (1/|scope|) * sum_{e in scope} log max_{c in S} eff[e][c] )
 * = 1 / geomean(Slowdown over Oracle).  Writes G and the log-sum L.
 */
int or_score(const double *logeff, int64_t E, int64_t C, const uint8_t *mask,
             const int32_t *set, int k, double *G_out, double *L_out)
{
    if (k <= 0) return OR_EEMPTY;
    for (int u = 0; u < k; u++)
        if (set[u] < 0 || set[u] >= C) return OR_EINVAL;
    int64_t *envs = malloc(sizeof(int64_t) * (size_t)E);
    if (!envs) return OR_ENOMEM;
    int64_t ne = scope_list(mask, E, envs);
    if (ne == 0) { free(envs); return OR_EEMPTY; }
    double L = logsum(logeff, C, envs, ne, set, k);
    free(envs);
    if (L_out) *L_out = L;
    if (G_out) *G_out = exp(L / (double)ne);
    return OR_OK;
}

/* ---- exhaustive k-subset search (Sec. 4.3.1) ---------------- */

/* Total order of candidates: higher L first; ties -> lexicographically
 * smaller sorted tuple first (reading c5). Returns 1 if (La,a) precedes (Lb,b). */
static int precedes(double La, const int32_t *a, double Lb, const int32_t *b, int k)
{
    if (La > Lb) return 1;
    if (La < Lb) return 0;
    for (int u = 0; u < k; u++) {
        if (a[u] < b[u]) return 1;
        if (a[u] > b[u]) return 0;
    }
    return 0;
}

typedef struct {
    double L1, L2;          /* best and runner-up log-sums */
    int32_t s1[32], s2[32];   /* their tuples */
    int have;               /* number of valid entries (0..2) */
} top2;

static void top2_offer(top2 *t, double L, const int32_t *s, int k)
{
    if (t->have == 0 || precedes(L, s, t->L1, t->s1, k)) {
        if (t->have >= 1) { t->L2 = t->L1; memcpy(t->s2, t->s1, sizeof t->s1); }
        t->L1 = L; memcpy(t->s1, s, sizeof(int32_t) * (size_t)k);
        t->have = t->have < 2 ? t->have + 1 : 2;
    } else if (t->have == 1 || precedes(L, s, t->L2, t->s2, k)) {
        t->L2 = L; memcpy(t->s2, s, sizeof(int32_t) * (size_t)k);
        t->have = 2;
    }
}

typedef struct {
    const double *logeff;
    int64_t C;
    const int64_t *envs;
    int64_t ne;
    int k;
    int64_t lo, hi;     /* first-index range [lo, hi) */
    int tid, nth;
    top2 res;
} exh_job;

/* Enumerate every sorted k-tuple (a0 < a1 < ... < a_{k-1}) with
 * a0 in {lo + tid, lo + tid + nth, ...} in lexicographic order and offer
 * each to the thread-local top-2. */
static void *exh_worker(void *arg)
{
    exh_job *j = (exh_job *)arg;
    int k = j->k;
    int32_t s[32];
    memset(&j->res, 0, sizeof j->res);
    for (int64_t a0 = j->lo + j->tid; a0 < j->hi; a0 += j->nth) {
        if (a0 + k > j->C) break;
        s[0] = (int32_t)a0;
        for (int u = 1; u < k; u++) s[u] = s[u - 1] + 1;
        for (;;) {
            double L = logsum(j->logeff, j->C, j->envs, j->ne, s, k);
            top2_offer(&j->res, L, s, k);
            /* next combination with fixed s[0] (lexicographic) */
            int u = k - 1;
            while (u >= 1 && s[u] == (int32_t)(j->C - k + u)) u--;
            if (u < 1) break;
            s[u]++;
            for (int v = u + 1; v < k; v++) s[v] = s[v - 1] + 1;
        }
    }
    return NULL;
}

/*
 * or_exhaustive -- "search through the space of variant combinations ...
 * returns the variant combination with the highest ranking",
 * restricted to distinct unordered subsets of size exactly k (reading c8).
 * First indices restricted to [lo, hi) (pass 0, C for the full search;
 * a sub-range is how bench.py takes a bounded CPU sample).
 * Writes the best tuple + G and the runner-up (second in the total order)
 * tuple + G; *n_found = number of candidates (0, 1 or 2 reported).
 */
int or_exhaustive(const double *logeff, int64_t E, int64_t C, const uint8_t *mask,
                  int k, int64_t lo, int64_t hi, int nthreads,
                  int32_t *best_set, double *G_best, int32_t *runner_set,
                  double *G_runner, int *n_found)
{
    if (k <= 0 || k > 32) return OR_EINVAL;
    if (k > C) return OR_EINVAL;
    if (lo < 0) lo = 0;
    if (hi > C) hi = C;
    if (nthreads < 1) nthreads = 1;
    int64_t *envs = malloc(sizeof(int64_t) * (size_t)E);
    if (!envs) return OR_ENOMEM;
    int64_t ne = scope_list(mask, E, envs);
    if (ne == 0) { free(envs); return OR_EEMPTY; }
    exh_job *jobs = calloc((size_t)nthreads, sizeof(exh_job));
    pthread_t *th = calloc((size_t)nthreads, sizeof(pthread_t));
    if (!jobs || !th) { free(envs); free(jobs); free(th); return OR_ENOMEM; }
    for (int t = 0; t < nthreads; t++) {
        jobs[t] = (exh_job){logeff, C, envs, ne, k, lo, hi, t, nthreads, {0}};
        if (nthreads == 1) exh_worker(&jobs[t]);
        else pthread_create(&th[t], NULL, exh_worker, &jobs[t]);
    }
    top2 all;
    memset(&all, 0, sizeof all);
    for (int t = 0; t < nthreads; t++) {
        if (nthreads > 1) pthread_join(th[t], NULL);
        if (jobs[t].res.have >= 1) top2_offer(&all, jobs[t].res.L1, jobs[t].res.s1, k);
        if (jobs[t].res.have >= 2) top2_offer(&all, jobs[t].res.L2, jobs[t].res.s2, k);
    }
    if (n_found) *n_found = all.have;
    if (all.have >= 1) {
        memcpy(best_set, all.s1, sizeof(int32_t) * (size_t)k);
        *G_best = exp(all.L1 / (double)ne);
    }
    if (all.have >= 2) {
        memcpy(runner_set, all.s2, sizeof(int32_t) * (size_t)k);
        *G_runner = exp(all.L2 / (double)ne);
    }
    free(envs); free(jobs); free(th);
    return OR_OK;
}

/*
 * or_greedy -- greedy forward selection (north_star; reading c12):
 * S = init;  for t = 1..k:  score G(S u {c}) for every c not in S
 * (ascending c), take the maximum, ties to the lowest c; record G and the
 * top-two gap G_best - G_second of that step (reading c7).
 * m[e] = max_{c in S} logeff[e][c] is kept between steps; it IS the
 * per-environment maximum of the definition, not a reformulation.
 * init may be NULL with n_init = 0.  Writes k indices (the picks after
 * init), their G trace and gap trace (gap = +inf when only one candidate).
 */
int or_greedy(const double *logeff, int64_t E, int64_t C, const uint8_t *mask,
              int k, const int32_t *init, int n_init,
              int32_t *out_idx, double *G_trace, double *gap_trace)
{
    if (k <= 0 || k + n_init > C) return OR_EINVAL;
    int64_t *envs = malloc(sizeof(int64_t) * (size_t)E);
    double *m = malloc(sizeof(double) * (size_t)E);
    uint8_t *in = calloc((size_t)C, 1);
    if (!envs || !m || !in) { free(envs); free(m); free(in); return OR_ENOMEM; }
    int64_t ne = scope_list(mask, E, envs);
    if (ne == 0) { free(envs); free(m); free(in); return OR_EEMPTY; }
    for (int64_t q = 0; q < ne; q++) m[q] = -INFINITY;   /* empty set */
    for (int u = 0; u < n_init; u++) {
        int32_t c = init[u];
        if (c < 0 || c >= C || in[c]) { free(envs); free(m); free(in); return OR_EINVAL; }
        in[c] = 1;
        for (int64_t q = 0; q < ne; q++) {
            double v = logeff[envs[q] * C + c];
            if (v > m[q]) m[q] = v;
        }
    }
    for (int t = 0; t < k; t++) {
        double L1 = -INFINITY, L2 = -INFINITY;
        int32_t c1 = -1;
        for (int64_t c = 0; c < C; c++) {
            if (in[c]) continue;
            double L = 0.0;
            for (int64_t q = 0; q < ne; q++) {
                double v = logeff[envs[q] * C + c];
                L += (v > m[q]) ? v : m[q];
            }
            if (c1 < 0 || L > L1) { L2 = L1; L1 = L; c1 = (int32_t)c; }
            else if (L > L2 || L2 == -INFINITY) { L2 = L; }
        }
        if (c1 < 0) { free(envs); free(m); free(in); return OR_EINVAL; }
        out_idx[t] = c1;
        in[c1] = 1;
        for (int64_t q = 0; q < ne; q++) {
            double v = logeff[envs[q] * C + c1];
            if (v > m[q]) m[q] = v;
        }
        G_trace[t] = exp(L1 / (double)ne);
        gap_trace[t] = (L2 == -INFINITY) ? INFINITY
                       : exp(L1 / (double)ne) - exp(L2 / (double)ne);
    }
    free(envs); free(m); free(in);
    return OR_OK;
}

/*
 * or_holdout -- leave-one-device-out generalization, the analogue of the
 * unseen-device experiment (Sec. 5.8; reading c13):
 *   train scope = envs with device != d; test scope = envs with device == d
 *   S_unseen = select(train, k)  (method 0 greedy, 1 exhaustive)
 *   G_train  = G(S_unseen, train);  G_unseen = G(S_unseen, test)
 *   S_known  = select(test, k);     G_known  = G(S_known, test)
 * best[e] is each env's own Oracle over all configs (S:L400 reading).
 */
int or_holdout(const double *logeff, int64_t E, int64_t C, const int32_t *env_device,
               int32_t d, int k, int method, int nthreads,
               int32_t *out_idx, double *G_train, double *G_unseen, double *G_known,
               int32_t *known_idx)
{
    uint8_t *tr = malloc((size_t)E), *te = malloc((size_t)E);
    int32_t *tmp = malloc(sizeof(int32_t) * 32);
    double *gt = malloc(sizeof(double) * (size_t)k), *gp = malloc(sizeof(double) * (size_t)k);
    if (!tr || !te || !tmp || !gt || !gp) { free(tr); free(te); free(tmp); free(gt); free(gp); return OR_ENOMEM; }
    int64_t ntr = 0, nte = 0;
    for (int64_t e = 0; e < E; e++) {
        tr[e] = env_device[e] != d; te[e] = env_device[e] == d;
        ntr += tr[e]; nte += te[e];
    }
    int rc = OR_OK;
    if (ntr == 0 || nte == 0) { rc = OR_EEMPTY; goto out; }
    double g2; int nf;
    for (int pass = 0; pass < 2; pass++) {
        const uint8_t *sel_mask = pass == 0 ? tr : te;
        int32_t *dst = pass == 0 ? out_idx : known_idx;
        if (method == 0) rc = or_greedy(logeff, E, C, sel_mask, k, NULL, 0, dst, gt, gp);
        else rc = or_exhaustive(logeff, E, C, sel_mask, k, 0, C, nthreads, dst, gt, tmp, &g2, &nf);
        if (rc) goto out;
    }
    if ((rc = or_score(logeff, E, C, tr, out_idx, k, G_train, NULL))) goto out;
    if ((rc = or_score(logeff, E, C, te, out_idx, k, G_unseen, NULL))) goto out;
    rc = or_score(logeff, E, C, te, known_idx, k, G_known, NULL);
out:
    free(tr); free(te); free(tmp); free(gt); free(gp);
    return rc;
}

/* ---- fleet objective, Eq. 2 (Sec. 4.4.2) -------------------- */

/*
 * or_fleet_rate -- the rate at which the fleet completes tasks:
 *
 *   R(S) = sum_{d} quantity(d) / sum_{i} y'_{d,i}(S) * quantity(i)
 *
 * y'_{d,i}(S) = min_{c in S} T[(d,i)][c], the runtime of the best member of S
 * on that environment (best-member reading, as for Eq. 1); a missing
 * cell costs penalty * best[e] (reading c4).  The inner sum runs over the
 * environments of device d in scope (a device's task = its available inputs,
 * P:L487); devices with no environment in scope do not contribute.
 *   T         env-major runtimes (ld = C), NaN/inf = missing
 *   best, penalty   from or_normalize
 *   env_device int32[E]; q_dev double[n_dev] indexed by device id;
 *   q_env     double[E] = quantity(i) of each environment's input
 * Units: tasks per millisecond.
 */
static double rt_cell(const float *T, int64_t C, const double *best, double penalty,
                      int64_t e, int32_t c)
{
    float t = T[e * C + c];
    return isfinite(t) ? (double)t : penalty * best[e];
}

int or_fleet_rate(const float *T, int64_t E, int64_t C, const double *best, double penalty,
                  const int32_t *env_device, int32_t n_dev, const double *q_dev,
                  const double *q_env, const uint8_t *mask, const int32_t *set, int k,
                  double *R_out)
{
    if (k <= 0) return OR_EEMPTY;
    for (int u = 0; u < k; u++)
        if (set[u] < 0 || set[u] >= C) return OR_EINVAL;
    double *den = calloc((size_t)n_dev, sizeof(double));
    int *present = calloc((size_t)n_dev, sizeof(int));
    if (!den || !present) { free(den); free(present); return OR_ENOMEM; }
    int any = 0;
    for (int64_t e = 0; e < E; e++) {
        if (mask && !mask[e]) continue;
        int32_t d = env_device[e];
        if (d < 0 || d >= n_dev) { free(den); free(present); return OR_EINVAL; }
        double y = rt_cell(T, C, best, penalty, e, set[0]);
        for (int u = 1; u < k; u++) {
            double v = rt_cell(T, C, best, penalty, e, set[u]);
            if (v < y) y = v;
        }
        den[d] += y * q_env[e];
        present[d] = 1;
        any = 1;
    }
    if (!any) { free(den); free(present); return OR_EEMPTY; }
    double R = 0.0;
    for (int32_t d = 0; d < n_dev; d++)
        if (present[d]) R += q_dev[d] / den[d];
    free(den); free(present);
    *R_out = R;
    return OR_OK;
}

/*
 * or_fleet_exhaustive -- exhaustive search maximising R (the tuner minimises
 * its reciprocal): every k-subset in lexicographic order, strict '>'
 * (first in lex order wins ties).  Writes best and runner-up and their R.
 * Single-threaded (test sizes only).
 */
int or_fleet_exhaustive(const float *T, int64_t E, int64_t C, const double *best, double penalty,
                        const int32_t *env_device, int32_t n_dev, const double *q_dev,
                        const double *q_env, const uint8_t *mask, int k,
                        int32_t *best_set, double *R_best, int32_t *runner_set, double *R_runner,
                        int *n_found)
{
    if (k <= 0 || k > 32 || k > C) return OR_EINVAL;
    int32_t s[32];
    top2 res;
    memset(&res, 0, sizeof res);
    for (int u = 0; u < k; u++) s[u] = u;
    for (;;) {
        double R;
        int rc = or_fleet_rate(T, E, C, best, penalty, env_device, n_dev, q_dev, q_env, mask, s, k, &R);
        if (rc) return rc;
        top2_offer(&res, R, s, k);          /* top2 orders by higher value first */
        int u = k - 1;
        while (u >= 0 && s[u] == (int32_t)(C - k + u)) u--;
        if (u < 0) break;
        s[u]++;
        for (int v = u + 1; v < k; v++) s[v] = s[v - 1] + 1;
    }
    *n_found = res.have;
    if (res.have >= 1) { memcpy(best_set, res.s1, sizeof(int32_t) * (size_t)k); *R_best = res.L1; }
    if (res.have >= 2) { memcpy(runner_set, res.s2, sizeof(int32_t) * (size_t)k); *R_runner = res.L2; }
    return OR_OK;
}

/*
 * or_fleet_exhaustive_par -- or_fleet_exhaustive with the first index dealt to
 * nthreads threads round-robin (each thread enumerates its tuples in the same
 * lexicographic order with the same or_fleet_rate, strict '>' keeps the first of
 * equal rates); the per-thread best two are merged in (R desc, tuple asc) order,
 * which is the order the sequential loop produces.  For full-size golden values.
 */
typedef struct {
    const float *T; int64_t E, C; const double *best; double penalty;
    const int32_t *env_device; int32_t n_dev; const double *q_dev, *q_env;
    const uint8_t *mask; int k, tid, nth, rc;
    top2 res;
} fleet_job;

static void *fleet_worker(void *arg)
{
    fleet_job *j = (fleet_job *)arg;
    int k = j->k;
    int32_t s[32];
    memset(&j->res, 0, sizeof j->res);
    for (int64_t a0 = j->tid; a0 + k <= j->C; a0 += j->nth) {
        s[0] = (int32_t)a0;
        for (int u = 1; u < k; u++) s[u] = s[u - 1] + 1;
        for (;;) {
            double R;
            int rc = or_fleet_rate(j->T, j->E, j->C, j->best, j->penalty, j->env_device, j->n_dev,
                                   j->q_dev, j->q_env, j->mask, s, k, &R);
            if (rc) { j->rc = rc; return NULL; }
            top2_offer(&j->res, R, s, k);
            int u = k - 1;
            while (u >= 1 && s[u] == (int32_t)(j->C - k + u)) u--;
            if (u < 1) break;
            s[u]++;
            for (int v = u + 1; v < k; v++) s[v] = s[v - 1] + 1;
        }
    }
    return NULL;
}

int or_fleet_exhaustive_par(const float *T, int64_t E, int64_t C, const double *best, double penalty,
                            const int32_t *env_device, int32_t n_dev, const double *q_dev,
                            const double *q_env, const uint8_t *mask, int k, int nthreads,
                            int32_t *best_set, double *R_best, int32_t *runner_set, double *R_runner,
                            int *n_found)
{
    if (k <= 0 || k > 32 || k > C) return OR_EINVAL;
    if (nthreads < 1) nthreads = 1;
    fleet_job *jobs = calloc((size_t)nthreads, sizeof(fleet_job));
    pthread_t *th = calloc((size_t)nthreads, sizeof(pthread_t));
    if (!jobs || !th) { free(jobs); free(th); return OR_ENOMEM; }
    for (int t = 0; t < nthreads; t++) {
        jobs[t] = (fleet_job){T, E, C, best, penalty, env_device, n_dev, q_dev, q_env, mask, k, t, nthreads, 0, {0}};
        pthread_create(&th[t], NULL, fleet_worker, &jobs[t]);
    }
    top2 all;
    memset(&all, 0, sizeof all);
    int rc = OR_OK;
    for (int t = 0; t < nthreads; t++) {
        pthread_join(th[t], NULL);
        if (jobs[t].rc) rc = jobs[t].rc;
        if (jobs[t].res.have >= 1) top2_offer(&all, jobs[t].res.L1, jobs[t].res.s1, k);
        if (jobs[t].res.have >= 2) top2_offer(&all, jobs[t].res.L2, jobs[t].res.s2, k);
    }
    if (rc == OR_OK) {
        *n_found = all.have;
        if (all.have >= 1) { memcpy(best_set, all.s1, sizeof(int32_t) * (size_t)k); *R_best = all.L1; }
        if (all.have >= 2) { memcpy(runner_set, all.s2, sizeof(int32_t) * (size_t)k); *R_runner = all.L2; }
    }
    free(jobs); free(th);
    return rc;
}

/*
 * or_fleet_greedy -- greedy forward selection maximising R: at each step
 * evaluate R(S u {c}) for every c not in S (ascending), take the maximum,
 * ties to the lowest c.  Writes picks, R trace and the top-two gap per step.
 */
int or_fleet_greedy(const float *T, int64_t E, int64_t C, const double *best, double penalty,
                    const int32_t *env_device, int32_t n_dev, const double *q_dev,
                    const double *q_env, const uint8_t *mask, int k,
                    int32_t *out_idx, double *R_trace, double *gap_trace)
{
    if (k <= 0 || k > C || k > 64) return OR_EINVAL;
    int32_t S[65];
    uint8_t *in = calloc((size_t)C, 1);
    if (!in) return OR_ENOMEM;
    for (int t = 0; t < k; t++) {
        double R1 = -INFINITY, R2 = -INFINITY;
        int32_t c1 = -1;
        for (int64_t c = 0; c < C; c++) {
            if (in[c]) continue;
            S[t] = (int32_t)c;
            double R;
            int rc = or_fleet_rate(T, E, C, best, penalty, env_device, n_dev, q_dev, q_env, mask, S, t + 1, &R);
            if (rc) { free(in); return rc; }
            if (c1 < 0 || R > R1) { R2 = R1; R1 = R; c1 = (int32_t)c; }
            else if (R > R2) R2 = R;
        }
        S[t] = c1;
        in[c1] = 1;
        out_idx[t] = c1;
        R_trace[t] = R1;
        gap_trace[t] = (R2 == -INFINITY) ? INFINITY : R1 - R2;
    }
    free(in);
    return OR_OK;
}

/* ---- swap local search ------------------- */

/*
 * or_swap_search -- deterministic best-improvement swap local search, the
 * stand-in for the paper's heuristic/stochastic search over sets (P:L280,
 * Sec. 4.3.1; "PortabilityTune"): start from the greedy k-set (or
 * `init` if given); repeatedly evaluate every swap (a in S out, b not in S in)
 * with the full Eq. 1 score, take the best (highest L; ties -> the
 * lexicographically smallest resulting sorted tuple); apply it if it strictly
 * improves L, else stop.  At most max_moves moves.
 * Writes the final sorted set, its G and the number of moves applied.
 */
static int cmp_i32(const void *a, const void *b)
{
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

int or_swap_search(const double *logeff, int64_t E, int64_t C, const uint8_t *mask, int k,
                   const int32_t *init, int max_moves, int32_t *out_set, double *G_out,
                   int *moves_out)
{
    if (k <= 0 || k > 32 || k >= C) return OR_EINVAL;
    int64_t *envs = malloc(sizeof(int64_t) * (size_t)E);
    uint8_t *in = calloc((size_t)C, 1);
    if (!envs || !in) { free(envs); free(in); return OR_ENOMEM; }
    int64_t ne = scope_list(mask, E, envs);
    if (ne == 0) { free(envs); free(in); return OR_EEMPTY; }
    int32_t S[32], T[32], Tb[32];
    if (init) {
        memcpy(S, init, sizeof(int32_t) * (size_t)k);
    } else {
        double *gt = malloc(sizeof(double) * (size_t)k), *gp = malloc(sizeof(double) * (size_t)k);
        int rc = or_greedy(logeff, E, C, mask, k, NULL, 0, S, gt, gp);
        free(gt); free(gp);
        if (rc) { free(envs); free(in); return rc; }
    }
    qsort(S, (size_t)k, sizeof(int32_t), cmp_i32);
    for (int u = 0; u < k; u++) in[S[u]] = 1;
    double L = logsum(logeff, C, envs, ne, S, k);
    int moves = 0;
    while (moves < max_moves) {
        double Lb = -INFINITY;
        int have = 0;
        for (int a = 0; a < k; a++)
            for (int64_t b = 0; b < C; b++) {
                if (in[b]) continue;
                memcpy(T, S, sizeof(int32_t) * (size_t)k);
                T[a] = (int32_t)b;
                qsort(T, (size_t)k, sizeof(int32_t), cmp_i32);
                double Lt = logsum(logeff, C, envs, ne, T, k);
                if (!have || precedes(Lt, T, Lb, Tb, k)) {
                    Lb = Lt;
                    memcpy(Tb, T, sizeof(int32_t) * (size_t)k);
                    have = 1;
                }
            }
        if (!have || !(Lb > L)) break;
        for (int u = 0; u < k; u++) in[S[u]] = 0;
        memcpy(S, Tb, sizeof(int32_t) * (size_t)k);
        for (int u = 0; u < k; u++) in[S[u]] = 1;
        L = Lb;
        moves++;
    }
    memcpy(out_set, S, sizeof(int32_t) * (size_t)k);
    *G_out = exp(L / (double)ne);
    *moves_out = moves;
    free(envs); free(in);
    return OR_OK;
}

/* ---- k-means selector (Sec. 4.3.2) --------- */

/*
 * or_kmeans -- "perform unsupervised clustering ... k = |kappa| centroids";
 * each environment is a point in N-dimensional space, N = number of variants,
 * of its performance results, here its slowdowns T/best (reading
 * k1); "from the performance results vector of the centroid, we select
 * the highest-performing variant": per cluster the config with the
 * smallest centroid slowdown (ties -> lowest index); duplicates collapse.
 *   init (reading k2, deterministic): centroid 0 = the point nearest the mean
 *   of all points; centroid j = the point farthest (max over points of the
 *   min squared distance to the chosen centroids), ties -> lowest env index.
 *   Lloyd: assign each point to its nearest centroid (ties -> lowest j),
 *   centroids = mean of their points; an emptied cluster is re-seeded with the
 *   point farthest from its own centroid; stop when no assignment
 *   changes or after max_iter iterations.
 * Squared distances sum (x - mu)^2 over configs ascending; means sum points in
 * ascending env order then divide.  Writes the sorted unique selection
 * (n_sel <= k), the iteration count and the within-cluster sum of squares
 * after each iteration (wcss[max_iter], may be NULL).
 */
static double sqdist(const double *x, const double *mu, int64_t C)
{
    double d = 0.0;
    for (int64_t c = 0; c < C; c++) {
        double t = x[c] - mu[c];
        d += t * t;
    }
    return d;
}

/* Lloyd iterations from the centroids in M (k x C) and the selection; shared by
 * or_kmeans (maximin start) and or_kmeans_from (given start).  dmin, asg, cnt are
 * scratch (ne, ne, k).  Same arithmetic and order as before the split. */
static void kmeans_lloyd(const double *X, int64_t ne, int64_t C, int k, int max_iter, double *M,
                         double *dmin, int *asg, int *cnt, int32_t *sel, int *n_sel, int *iters,
                         double *wcss)
{
    for (int64_t q = 0; q < ne; q++) asg[q] = -1;
    int it = 0;
    while (it < max_iter) {
        int changed = 0;
        double w = 0.0;
        for (int64_t q = 0; q < ne; q++) {
            int bj = 0;
            double bdist = INFINITY;
            for (int j = 0; j < k; j++) {
                double d = sqdist(X + q * C, M + (int64_t)j * C, C);
                if (d < bdist) { bdist = d; bj = j; }
            }
            if (asg[q] != bj) changed = 1;
            asg[q] = bj;
            dmin[q] = bdist;
            w += bdist;
        }
        it++;
        if (!changed && it > 1) { if (wcss) wcss[it - 1] = w; break; }
        /* update */
        for (int j = 0; j < k; j++) cnt[j] = 0;
        for (int64_t i = 0; i < (int64_t)k * C; i++) M[i] = 0.0;
        for (int64_t q = 0; q < ne; q++) {
            cnt[asg[q]]++;
            for (int64_t c = 0; c < C; c++) M[(int64_t)asg[q] * C + c] += X[q * C + c];
        }
        for (int j = 0; j < k; j++) {
            if (cnt[j] == 0) {
                /* re-seed: the point farthest from its own centroid */
                int64_t far = 0;
                double fd = -1.0;
                for (int64_t q = 0; q < ne; q++)
                    if (dmin[q] > fd) { fd = dmin[q]; far = q; }
                memcpy(M + (int64_t)j * C, X + far * C, sizeof(double) * (size_t)C);
                dmin[far] = 0.0;
            } else {
                for (int64_t c = 0; c < C; c++) M[(int64_t)j * C + c] /= (double)cnt[j];
            }
        }
        if (wcss) wcss[it - 1] = w;
    }
    *iters = it;
    /* selection: per centroid the best config, unique, sorted */
    int n = 0;
    for (int j = 0; j < k; j++) {
        int32_t bc = 0;
        double bv = INFINITY;
        for (int64_t c = 0; c < C; c++)
            if (M[(int64_t)j * C + c] < bv) { bv = M[(int64_t)j * C + c]; bc = (int32_t)c; }
        int dup = 0;
        for (int u = 0; u < n; u++) dup |= sel[u] == bc;
        if (!dup) sel[n++] = bc;
    }
    qsort(sel, (size_t)n, sizeof(int32_t), cmp_i32);
    *n_sel = n;
}

int or_kmeans(const float *T, int64_t E, int64_t C, const double *best, double penalty,
              const uint8_t *mask, int k, int max_iter, int32_t *sel, int *n_sel, int *iters,
              double *wcss)
{
    int64_t *envs = malloc(sizeof(int64_t) * (size_t)E);
    if (!envs) return OR_ENOMEM;
    int64_t ne = scope_list(mask, E, envs);
    if (ne == 0) { free(envs); return OR_EEMPTY; }
    if (k < 1 || k > ne) { free(envs); return OR_EINVAL; }
    double *X = malloc(sizeof(double) * (size_t)(ne * C));
    double *M = malloc(sizeof(double) * (size_t)(k * C));
    double *mean = calloc((size_t)C, sizeof(double));
    double *dmin = malloc(sizeof(double) * (size_t)ne);
    int *asg = malloc(sizeof(int) * (size_t)ne), *cnt = malloc(sizeof(int) * (size_t)k);
    if (!X || !M || !mean || !dmin || !asg || !cnt) {
        free(envs); free(X); free(M); free(mean); free(dmin); free(asg); free(cnt);
        return OR_ENOMEM;
    }
    for (int64_t q = 0; q < ne; q++)
        for (int64_t c = 0; c < C; c++) {
            float t = T[envs[q] * C + c];
            double tt = isfinite(t) ? (double)t : penalty * best[envs[q]];
            X[q * C + c] = tt / best[envs[q]];
        }
    /* init */
    for (int64_t q = 0; q < ne; q++)
        for (int64_t c = 0; c < C; c++) mean[c] += X[q * C + c];
    for (int64_t c = 0; c < C; c++) mean[c] /= (double)ne;
    int64_t first = 0;
    double bd = INFINITY;
    for (int64_t q = 0; q < ne; q++) {
        double d = sqdist(X + q * C, mean, C);
        if (d < bd) { bd = d; first = q; }
    }
    memcpy(M, X + first * C, sizeof(double) * (size_t)C);
    for (int64_t q = 0; q < ne; q++) dmin[q] = sqdist(X + q * C, M, C);
    for (int j = 1; j < k; j++) {
        int64_t far = 0;
        double fd = -1.0;
        for (int64_t q = 0; q < ne; q++)
            if (dmin[q] > fd) { fd = dmin[q]; far = q; }
        memcpy(M + (int64_t)j * C, X + far * C, sizeof(double) * (size_t)C);
        for (int64_t q = 0; q < ne; q++) {
            double d = sqdist(X + q * C, M + (int64_t)j * C, C);
            if (d < dmin[q]) dmin[q] = d;
        }
    }
    kmeans_lloyd(X, ne, C, k, max_iter, M, dmin, asg, cnt, sel, n_sel, iters, wcss);
    free(envs); free(X); free(M); free(mean); free(dmin); free(asg); free(cnt);
    return OR_OK;
}

/*
 * or_kmeans_from -- or_kmeans with the initial centroids given (init: k x C doubles,
 * row j = centroid j in the same slowdown space as the points) instead of the maximin
 * start; the Lloyd iterations, the empty-cluster re-seed and the selection are the
 * same code.  A start far from every point empties a cluster on the first pass, which
 * is how the re-seed rule is pinned (tests/test_oracle_kmeans.py).
 */
int or_kmeans_from(const float *T, int64_t E, int64_t C, const double *best, double penalty,
                   const uint8_t *mask, int k, int max_iter, const double *init, int32_t *sel,
                   int *n_sel, int *iters, double *wcss)
{
    int64_t *envs = malloc(sizeof(int64_t) * (size_t)E);
    if (!envs) return OR_ENOMEM;
    int64_t ne = scope_list(mask, E, envs);
    if (ne == 0) { free(envs); return OR_EEMPTY; }
    if (k < 1 || k > ne || !init) { free(envs); return OR_EINVAL; }
    double *X = malloc(sizeof(double) * (size_t)(ne * C));
    double *M = malloc(sizeof(double) * (size_t)(k * C));
    double *dmin = malloc(sizeof(double) * (size_t)ne);
    int *asg = malloc(sizeof(int) * (size_t)ne), *cnt = malloc(sizeof(int) * (size_t)k);
    if (!X || !M || !dmin || !asg || !cnt) {
        free(envs); free(X); free(M); free(dmin); free(asg); free(cnt);
        return OR_ENOMEM;
    }
    for (int64_t q = 0; q < ne; q++)
        for (int64_t c = 0; c < C; c++) {
            float t = T[envs[q] * C + c];
            double tt = isfinite(t) ? (double)t : penalty * best[envs[q]];
            X[q * C + c] = tt / best[envs[q]];
        }
    memcpy(M, init, sizeof(double) * (size_t)(k * C));
    kmeans_lloyd(X, ne, C, k, max_iter, M, dmin, asg, cnt, sel, n_sel, iters, wcss);
    free(envs); free(X); free(M); free(dmin); free(asg); free(cnt);
    return OR_OK;
}

