// swap.cu -- deterministic best-improvement swap local search (SURVEY §8(f)
// NEXT #2), the stand-in for the paper's heuristic/stochastic
// search over variant sets (Sec. 4.3.1; "PortabilityTune").
//
// From the greedy k-set (or a caller's set) S, every move scores all k*(C-k)
// swaps (a in S out, b not in S in) and applies the best one if it strictly
// lowers s(S) = sum_e min_{c in S} l[c][e] (= raises Eq. 1's G).  With the
// leave-one-out minima M_a[e] = min_{c in S\{a}} l[c][e] (prefix/suffix mins)
//     s(S - a + b) = sum_e min(M_a[e], l[b][e])
// -- the same (min,+) pattern as the exhaustive search, k rows x C columns.
// Exact fp64 (k x C x E per move is small); ties -> the lexicographically
// smallest resulting sorted tuple.
#include <algorithm>
#include <cmath>
#include <vector>

#include "pt_internal.cuh"

// M[a][e] = min over S without its a-th member (prefix/suffix mins), thread per env
__global__ void k_swap_loo(const double *__restrict__ l64, int64_t E_pad, const int32_t *__restrict__ S,
                           int k, double *__restrict__ M)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E_pad) return;
    double v[PT_SWAP_MAXK], suf[PT_SWAP_MAXK + 1];
    for (int u = 0; u < k; u++) v[u] = l64[(int64_t)S[u] * E_pad + e];
    suf[k] = INFINITY;
    for (int u = k - 1; u >= 0; u--) suf[u] = fmin(suf[u + 1], v[u]);
    double pre = INFINITY;
    for (int a = 0; a < k; a++) {
        M[(int64_t)a * E_pad + e] = fmin(pre, suf[a + 1]);
        pre = fmin(pre, v[a]);
    }
}

// warp per (a, b): score of S - S[a] + b (members of S: +inf)
__global__ void k_swap_score(const double *__restrict__ l64, int64_t E_pad, int64_t C,
                             const double *__restrict__ M, int k, const uint32_t *__restrict__ inS,
                             double *__restrict__ sc)
{
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= (int64_t)k * C) return;
    const int a = (int)(w / C);
    const int64_t b = w % C;
    if (inS[b >> 5] >> (b & 31) & 1u) {
        if (lane == 0) sc[w] = INFINITY;
        return;
    }
    const double *mrow = M + (int64_t)a * E_pad, *col = l64 + b * E_pad;
    double acc = 0.0;
    for (int64_t e = lane; e < E_pad; e += 32) acc += fmin(mrow[e], col[e]);
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) sc[w] = acc;
}

// sorted tuple of S - S[a] + b (S sorted ascending)
__device__ void swap_tuple(const int32_t *S, int k, int a, int32_t b, int32_t *out)
{
    int n = 0;
    bool placed = false;
    for (int u = 0; u < k; u++) {
        if (u == a) continue;
        if (!placed && b < S[u]) {
            out[n++] = b;
            placed = true;
        }
        out[n++] = S[u];
    }
    if (!placed) out[n++] = b;
}

// does move (sa, a, b) precede (sb, a2, b2)? (score, then resulting tuple)
__device__ bool move_less(double sa, int a, int32_t b, double sb, int a2, int32_t b2,
                          const int32_t *S, int k)
{
    if (sa < sb) return true;
    if (sa > sb || !(sa < INFINITY)) return false;
    int32_t t1[PT_SWAP_MAXK], t2[PT_SWAP_MAXK];
    swap_tuple(S, k, a, b, t1);
    swap_tuple(S, k, a2, b2, t2);
    for (int u = 0; u < k; u++) {
        if (t1[u] < t2[u]) return true;
        if (t1[u] > t2[u]) return false;
    }
    return false;
}

// one CTA: best move over the k x C score array
__global__ void __launch_bounds__(256) k_swap_best(const double *__restrict__ sc, int k, int64_t C,
                                                  const int32_t *__restrict__ S,
                                                  double *__restrict__ out_s, int2 *__restrict__ out_ab)
{
    __shared__ int32_t Ss[PT_SWAP_MAXK];
    __shared__ double bs[256];
    __shared__ int2 bab[256];
    if (threadIdx.x < k) Ss[threadIdx.x] = S[threadIdx.x];
    __syncthreads();
    double best = INFINITY;
    int2 ab = make_int2(0, 0x7fffffff);
    for (int64_t w = threadIdx.x; w < (int64_t)k * C; w += blockDim.x) {
        const double s = sc[w];
        const int a = (int)(w / C);
        const int32_t b = (int32_t)(w % C);
        if (move_less(s, a, b, best, ab.x, ab.y, Ss, k)) {
            best = s;
            ab = make_int2(a, b);
        }
    }
    bs[threadIdx.x] = best;
    bab[threadIdx.x] = ab;
    __syncthreads();
    for (int h = blockDim.x / 2; h > 0; h >>= 1) {
        if ((int)threadIdx.x < h) {
            const double so = bs[threadIdx.x + h];
            const int2 o = bab[threadIdx.x + h];
            if (move_less(so, o.x, o.y, bs[threadIdx.x], bab[threadIdx.x].x, bab[threadIdx.x].y, Ss, k)) {
                bs[threadIdx.x] = so;
                bab[threadIdx.x] = o;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *out_s = bs[0];
        *out_ab = bab[0];
    }
}

extern "C" pt_status pt_swap_search(pt_ctx *ctx, int32_t k, const uint8_t *env_mask, int32_t objective,
                                    int32_t max_moves, const int32_t *init, int32_t *out_idx,
                                    double *out_G, int32_t *out_moves)
{
    PT_NVTX();
    if (!ctx || !out_idx || !out_G) return pt_fail(PT_EINVAL, "NULL argument");
    if (objective != PT_OBJ_GEOMEAN)
        return pt_fail(PT_EINVAL, "swap search supports PT_OBJ_GEOMEAN only");
    PT_CK(cudaSetDevice(ctx->dev));
    const pt_view *v = nullptr;
    PT_TRY(pt_get_view(ctx, env_mask, &v));
    const int64_t C = v->C, E_pad = v->E_pad;
    if (k < 1 || k >= C || k > PT_SWAP_MAXK)
        return pt_fail(PT_EINVAL, "k=%d outside [1, min(C-1, %d)]", k, PT_SWAP_MAXK);
    std::vector<int32_t> S(k);
    if (init) {
        for (int u = 0; u < k; u++) {
            if (init[u] < 0 || init[u] >= C) return pt_fail(PT_EINVAL, "init index out of range");
            S[u] = init[u];
        }
        std::vector<int32_t> t(S);
        std::sort(t.begin(), t.end());
        if (std::adjacent_find(t.begin(), t.end()) != t.end())
            return pt_fail(PT_EINVAL, "init has a repeated index");
    } else {
        std::vector<double> s1(k), s2(k);
        PT_TRY(pt_greedy_view(ctx, v, k, S.data(), s1.data(), s2.data()));
    }
    std::sort(S.begin(), S.end());
    cudaStream_t st = ctx->stream;
    const int64_t nwords = (C + 31) / 32;
    int32_t *dS = nullptr;
    double *M = nullptr, *sc = nullptr, *ds = nullptr;
    uint32_t *inS = nullptr;
    int2 *dab = nullptr;
    PT_TRY(pt_dalloc(ctx, (void **)&dS, sizeof(int32_t) * k));
    PT_TRY(pt_dalloc(ctx, (void **)&M, sizeof(double) * k * E_pad));
    PT_TRY(pt_dalloc(ctx, (void **)&sc, sizeof(double) * k * C));
    PT_TRY(pt_dalloc(ctx, (void **)&ds, sizeof(double) * 2));
    PT_TRY(pt_dalloc(ctx, (void **)&inS, sizeof(uint32_t) * nwords));
    PT_TRY(pt_dalloc(ctx, (void **)&dab, sizeof(int2)));
    // current score (exact, same kernel family as pt_score_sets)
    PT_CK(cudaMemcpyAsync(dS, S.data(), sizeof(int32_t) * k, cudaMemcpyHostToDevice, st));
    PT_TRY(pt_score_view(ctx, v, dS, 1, k, ds));
    double cur = 0.0;
    PT_CK(cudaMemcpyAsync(&cur, ds, sizeof(double), cudaMemcpyDeviceToHost, st));
    PT_CK(cudaStreamSynchronize(st));
    int moves = 0;
    std::vector<uint32_t> hin(nwords);
    while (moves < max_moves) {
        std::fill(hin.begin(), hin.end(), 0u);
        for (int32_t c : S) hin[c >> 5] |= 1u << (c & 31);
        PT_CK(cudaMemcpyAsync(dS, S.data(), sizeof(int32_t) * k, cudaMemcpyHostToDevice, st));
        PT_CK(cudaMemcpyAsync(inS, hin.data(), sizeof(uint32_t) * nwords, cudaMemcpyHostToDevice, st));
        k_swap_loo<<<(unsigned)((E_pad + 127) / 128), 128, 0, st>>>(v->l64, E_pad, dS, k, M);
        const int64_t threads = (int64_t)k * C * 32;
        k_swap_score<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(v->l64, E_pad, C, M, k, inS, sc);
        k_swap_best<<<1, 256, 0, st>>>(sc, k, C, dS, ds, dab);
        ctx->stats.launches += 3;
        PT_CK(cudaGetLastError());
        double sb = 0.0;
        int2 ab;
        PT_CK(cudaMemcpyAsync(&sb, ds, sizeof(double), cudaMemcpyDeviceToHost, st));
        PT_CK(cudaMemcpyAsync(&ab, dab, sizeof(int2), cudaMemcpyDeviceToHost, st));
        PT_CK(cudaStreamSynchronize(st));
        if (!(sb < cur)) break;   // no strictly improving swap: local optimum
        S[ab.x] = ab.y;
        std::sort(S.begin(), S.end());
        cur = sb;
        moves++;
    }
    for (void *p : {(void *)dS, (void *)M, (void *)sc, (void *)ds, (void *)inS, (void *)dab}) pt_dfree(ctx, p);
    PT_CK(cudaStreamSynchronize(st));
    for (int u = 0; u < k; u++) out_idx[u] = S[u];
    *out_G = std::exp(-cur / (double)v->E);
    if (out_moves) *out_moves = moves;
    return PT_OK;
}
