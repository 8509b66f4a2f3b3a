// dist.cu -- the cross-GPU reduction of the sharded exhaustive search (SURVEY §8 row
// a8): every rank searches its shard of the k-subset space, the ranks exchange their
// exact (s, tuple) top-2 records over NCCL (a communicator the library builds from a
// caller-broadcast ncclUniqueId) or through a caller's stream-ordered all-gather, and
// every rank merges the records on the device and maps the winner's s to the
// objective (G = exp(-s/E), Eq. 1; R = 1/cost for Eq. 2).
// "Returns the variant combination with the highest ranking" across ranks.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2: in a PyTorch process this is
// the NCCL torch already loaded); nccl.h supplies only the types.
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstring>
#include <mutex>

#include "pt_internal.cuh"

// ---------------------------------------------------------------------------
// NCCL entry points
// ---------------------------------------------------------------------------
namespace {
struct nccl_api {
    ncclResult_t (*get_unique_id)(ncclUniqueId *);
    ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*all_gather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*comm_destroy)(ncclComm_t);
    const char *(*error_string)(ncclResult_t);
};

pt_status nccl_load(const nccl_api **out)
{
    static std::once_flag once;
    static nccl_api api;
    static bool ok = false;
    static std::string why;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            why = dlerror();
            return;
        }
        api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
        api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
        api.all_gather = (decltype(api.all_gather))dlsym(h, "ncclAllGather");
        api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
        api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
        ok = api.get_unique_id && api.comm_init_rank && api.all_gather && api.comm_destroy && api.error_string;
        if (!ok) why = "libnccl.so.2 lacks an entry point";
    });
    if (!ok) return pt_fail(PT_ENCCL, "NCCL unavailable: %s", why.c_str());
    *out = &api;
    return PT_OK;
}
}  // namespace

struct pt_comm {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1, dev = 0;
};

extern "C" pt_status pt_comm_unique_id(void *out_id)
{
    PT_NVTX();
    if (!out_id) return pt_fail(PT_EINVAL, "NULL argument");
    static_assert(sizeof(ncclUniqueId) == PT_COMM_ID_BYTES, "ncclUniqueId size");
    const nccl_api *n = nullptr;
    PT_TRY(nccl_load(&n));
    ncclUniqueId id;
    const ncclResult_t r = n->get_unique_id(&id);
    if (r != ncclSuccess) return pt_fail(PT_ENCCL, "ncclGetUniqueId: %s", n->error_string(r));
    memcpy(out_id, &id, sizeof id);
    return PT_OK;
}

extern "C" pt_status pt_comm_init(pt_comm **out, const void *id, int32_t rank, int32_t world, int cuda_device)
{
    PT_NVTX();
    if (!out || !id || world < 1 || rank < 0 || rank >= world)
        return pt_fail(PT_EINVAL, "bad argument (rank %d of %d)", rank, world);
    *out = nullptr;
    const nccl_api *n = nullptr;
    PT_TRY(nccl_load(&n));
    PT_CK(cudaSetDevice(cuda_device));
    pt_comm *c = new pt_comm();
    c->rank = rank;
    c->world = world;
    c->dev = cuda_device;
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof uid);
    const ncclResult_t r = n->comm_init_rank(&c->comm, world, uid, rank);
    if (r != ncclSuccess) {
        delete c;
        return pt_fail(PT_ENCCL, "ncclCommInitRank(rank %d of %d): %s", rank, world, n->error_string(r));
    }
    *out = c;
    return PT_OK;
}

extern "C" void pt_comm_free(pt_comm *c)
{
    PT_NVTX();
    if (!c) return;
    const nccl_api *n = nullptr;
    if (c->comm && nccl_load(&n) == PT_OK) {
        cudaSetDevice(c->dev);
        n->comm_destroy(c->comm);
    }
    delete c;
}

// ---------------------------------------------------------------------------
// records and their merge
// ---------------------------------------------------------------------------
// One rank's record, REC(k) doubles: [fingerprint, s1, s2, t1[k], t2[k]] -- the exact
// fp64 s of its best and second set in (s asc, tuple asc) order (s = +inf: absent) and
// their sorted tuples (exact in fp64).  The fingerprint identifies the shard plan
// (k, C, scope size, shard count, weights): ranks that dealt the task list differently
// would skip or repeat subsets, so a mismatch is an error, not a wrong answer.
__host__ __device__ static inline int rec_len(int k) { return 3 + 2 * k; }

// Merge n_rank records into the global top-2; out = [s1, s2, v1, v2, t1[k], t2[k]],
// v = G = exp(-s / n_env) (geomean) or R = 1/s (fleet: s is the cost 1/R).
// Returns 0, 1 (fingerprints differ) or 2 (no record present).
__host__ __device__ static int merge_records(const double *all, int n_rank, int k, double n_env, int objective,
                                             double *out)
{
    int32_t t1[PT_MAXK], t2[PT_MAXK], t[PT_MAXK];
    double s1 = INFINITY, s2 = INFINITY;
    bool have1 = false, have2 = false;
    const int L = rec_len(k);
    for (int r = 0; r < n_rank; r++) {
        const double *rec = all + (int64_t)r * L;
        if (rec[0] != all[0]) return 1;
        for (int q = 0; q < 2; q++) {
            const double s = rec[1 + q];
            if (!(s < INFINITY)) continue;
            for (int u = 0; u < k; u++) t[u] = (int32_t)rec[3 + q * k + u];
            if (!have1 || pt_key_less(s, t, s1, t1, k)) {
                if (have1) {
                    s2 = s1;
                    for (int u = 0; u < k; u++) t2[u] = t1[u];
                    have2 = true;
                }
                s1 = s;
                for (int u = 0; u < k; u++) t1[u] = t[u];
                have1 = true;
            } else if (!have2 || pt_key_less(s, t, s2, t2, k)) {
                bool same = s == s1;
                for (int u = 0; u < k && same; u++) same = t[u] == t1[u];
                if (!same) {
                    s2 = s;
                    for (int u = 0; u < k; u++) t2[u] = t[u];
                    have2 = true;
                }
            }
        }
    }
    if (!have1) return 2;
    auto value = [&](double s) { return objective == PT_OBJ_FLEET ? 1.0 / s : exp(-s / n_env); };
    out[0] = s1;
    out[1] = have2 ? s2 : INFINITY;
    out[2] = value(s1);
    out[3] = have2 ? value(s2) : NAN;
    for (int u = 0; u < k; u++) {
        out[4 + u] = t1[u];
        out[4 + k + u] = have2 ? t2[u] : -1.0;
    }
    return 0;
}

__global__ void k_merge_records(const double *__restrict__ all, int n_rank, int k, double n_env, int objective,
                                double *__restrict__ out, int *__restrict__ status)
{
    if (threadIdx.x == 0 && blockIdx.x == 0) *status = merge_records(all, n_rank, k, n_env, objective, out);
}

// the local shard's top-2 (device os/ot of the exhaustive search) -> this rank's record
__global__ void k_pack_record(const double *__restrict__ os, const int32_t *__restrict__ ot, int k, double fp,
                              double *__restrict__ rec)
{
    const int i = threadIdx.x;
    if (i == 0) rec[0] = fp;
    if (i < 2) rec[1 + i] = os[i];
    if (i < 2 * k) rec[3 + i] = (double)ot[i];
}

void pt_pack_record(pt_ctx *ctx, const double *d_os, const int32_t *d_ot, int k)
{
    if (!ctx->rec_out) return;
    k_pack_record<<<1, 32, 0, ctx->stream>>>(d_os, d_ot, k, ctx->rec_fp, ctx->rec_out);
    ctx->stats.launches++;
    ctx->rec_written = true;
}

// 52-bit FNV-1a of the plan parameters, as an exactly representable double
static double plan_fingerprint(int k, int64_t C, int64_t E, int world, const std::vector<double> &w, int objective)
{
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](const void *p, size_t n) {
        const unsigned char *b = (const unsigned char *)p;
        for (size_t i = 0; i < n; i++) h = (h ^ b[i]) * 1099511628211ull;
    };
    mix(&k, sizeof k);
    mix(&C, sizeof C);
    mix(&E, sizeof E);
    mix(&world, sizeof world);
    mix(&objective, sizeof objective);
    if ((int)w.size() == world)
        for (double x : w) mix(&x, sizeof x);
    return (double)(h >> 12);
}

extern "C" pt_status pt_merge_records(const double *records, int32_t n_rank, int32_t k, int64_t n_env,
                                      int32_t objective, int32_t *out_idx, double *out_G,
                                      int32_t *out_runner_idx, double *out_G_runner, double *out_s)
{
    PT_NVTX();
    if (!records || !out_idx || !out_G || n_rank < 1 || k < 1 || k > PT_MAXK || n_env < 1)
        return pt_fail(PT_EINVAL, "bad argument");
    std::vector<double> out(4 + 2 * k);
    const int rc = merge_records(records, n_rank, k, (double)n_env, objective, out.data());
    if (rc == 1) return pt_fail(PT_EINVAL, "shard plans differ across ranks (record fingerprints disagree)");
    if (rc == 2) return pt_fail(PT_EEMPTY, "no record present");
    for (int u = 0; u < k; u++) {
        out_idx[u] = (int32_t)out[4 + u];
        if (out_runner_idx) out_runner_idx[u] = (int32_t)out[4 + k + u];
    }
    *out_G = out[2];
    if (out_G_runner) *out_G_runner = out[3];
    if (out_s) {
        out_s[0] = out[0];
        out_s[1] = out[1];
    }
    return PT_OK;
}

extern "C" int32_t pt_record_len(int32_t k) { return k >= 1 && k <= PT_MAXK ? rec_len(k) : -1; }

// ---------------------------------------------------------------------------
// the sharded search
// ---------------------------------------------------------------------------
extern "C" pt_status pt_exhaustive_best_sharded(pt_ctx *ctx, int32_t k, const uint8_t *env_mask, int32_t objective,
                                                int32_t shard_rank, int32_t shard_count, pt_comm *comm,
                                                pt_dev_allgather_fn allgather, void *user, int32_t *out_idx,
                                                double *out_G, int32_t *out_runner_idx, double *out_G_runner,
                                                double *out_s)
{
    PT_NVTX();
    if (!ctx || !out_idx || !out_G) return pt_fail(PT_EINVAL, "NULL argument");
    if ((comm != nullptr) == (allgather != nullptr))
        return pt_fail(PT_EINVAL, "give exactly one of comm and allgather");
    if (comm && (comm->rank != shard_rank || comm->world != shard_count))
        return pt_fail(PT_EINVAL, "shard %d of %d does not match the communicator's rank %d of %d", shard_rank,
                       shard_count, comm->rank, comm->world);
    if (comm && comm->dev != ctx->dev)
        return pt_fail(PT_EINVAL, "communicator on device %d, context on device %d", comm->dev, ctx->dev);
    if (objective != PT_OBJ_GEOMEAN && objective != PT_OBJ_FLEET)
        return pt_fail(PT_EINVAL, "unknown objective %d", objective);
    if (k < 1 || k > PT_MAXK) return pt_fail(PT_EINVAL, "k=%d outside [1, %d]", k, PT_MAXK);
    if (shard_count < 1 || shard_rank < 0 || shard_rank >= shard_count)
        return pt_fail(PT_EINVAL, "bad shard %d of %d", shard_rank, shard_count);
    PT_CK(cudaSetDevice(ctx->dev));
    cudaStream_t s = ctx->stream;
    const pt_view *v = nullptr;
    PT_TRY(pt_get_view(ctx, env_mask, &v));
    const int L = rec_len(k);
    // device buffers: my record, everyone's, the merged result + status
    size_t off = 0;
    auto take = [&](size_t b) { size_t o = off; off += pt_round_up(b, 256); return o; };
    const size_t o_mine = take(sizeof(double) * L), o_all = take(sizeof(double) * L * shard_count),
                 o_out = take(sizeof(double) * (4 + 2 * k)), o_st = take(sizeof(int));
    char *b = nullptr;
    PT_TRY(pt_dalloc(ctx, (void **)&b, off));
    double *mine = (double *)(b + o_mine), *all = (double *)(b + o_all), *dout = (double *)(b + o_out);
    int *dst = (int *)(b + o_st);
    const double fp = plan_fingerprint(k, v->C, v->E, shard_count, ctx->shard_w, objective);

    // 1. this rank's shard, its exact top-2 packed on the device (geomean tiled/generic
    //    paths); the other paths return host values, packed here
    std::vector<int32_t> best(k), runner(k);
    double sv[2] = {INFINITY, INFINITY};
    int nf = 0;
    ctx->rec_out = mine;
    ctx->rec_fp = fp;
    ctx->rec_written = false;
    pt_status st;
    if (objective == PT_OBJ_FLEET) {
        double R[2];
        st = pt_fleet_exhaustive(ctx, k, env_mask, shard_rank, shard_count, best.data(), runner.data(), R, sv, &nf);
    } else {
        st = pt_exhaustive_view(ctx, v, k, shard_rank, shard_count, best.data(), runner.data(), sv, &nf);
    }
    const bool packed = ctx->rec_written;
    ctx->rec_out = nullptr;
    ctx->rec_written = false;
    if (st != PT_OK) {
        pt_dfree(ctx, b);
        return st;
    }
    if (!packed) {
        std::vector<double> rec(L);
        rec[0] = fp;
        rec[1] = nf >= 1 ? sv[0] : INFINITY;
        rec[2] = nf >= 2 ? sv[1] : INFINITY;
        for (int u = 0; u < k; u++) {
            rec[3 + u] = best[u];
            rec[3 + k + u] = runner[u];
        }
        PT_CK(cudaMemcpyAsync(mine, rec.data(), sizeof(double) * L, cudaMemcpyHostToDevice, s));
        PT_CK(cudaStreamSynchronize(s));   // rec is a host temporary
    }
    // 2. the exchange, stream-ordered on the context's stream
    if (comm) {
        const nccl_api *n = nullptr;
        if (const pt_status ls = nccl_load(&n); ls != PT_OK) {
            pt_dfree(ctx, b);
            return ls;
        }
        const ncclResult_t r = n->all_gather(mine, all, (size_t)L, ncclFloat64, comm->comm, s);
        if (r != ncclSuccess) {
            pt_dfree(ctx, b);
            return pt_fail(PT_ENCCL, "ncclAllGather: %s", n->error_string(r));
        }
    } else if (allgather(user, mine, L, all, (void *)s) != 0) {
        pt_dfree(ctx, b);
        return pt_fail(PT_ENCCL, "the all-gather callback failed");
    }
    // 3. merge + objective transform on the device; one copy back
    k_merge_records<<<1, 32, 0, s>>>(all, shard_count, k, (double)v->E, objective, dout, dst);
    ctx->stats.launches++;
    PT_CK(cudaGetLastError());
    std::vector<double> out(4 + 2 * k);
    int hst = 0;
    pt_hostio io(ctx);
    pt_status ios = io.d2h(out.data(), dout, sizeof(double) * out.size());
    if (ios == PT_OK) ios = io.d2h(&hst, dst, sizeof(int));
    if (ios == PT_OK) ios = io.finish();
    pt_dfree(ctx, b);
    if (ios != PT_OK) return ios;
    if (hst == 1) return pt_fail(PT_EINVAL, "shard plans differ across ranks (record fingerprints disagree)");
    if (hst == 2) return pt_fail(PT_EEMPTY, "no k-subset in any shard");
    for (int u = 0; u < k; u++) {
        out_idx[u] = (int32_t)out[4 + u];
        if (out_runner_idx) out_runner_idx[u] = (int32_t)out[4 + k + u];
    }
    *out_G = out[2];
    if (out_G_runner) *out_G_runner = out[3];
    if (out_s) {
        out_s[0] = out[0];
        out_s[1] = out[1];
    }
    return PT_OK;
}
