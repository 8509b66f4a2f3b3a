// holdout.cu -- pt_eval_holdout: leave-one-device-out generalization, the
// analogue of the paper's unseen-device experiment (Sec. 5.8):
// select on the environments of the other devices (train scope), evaluate the
// chosen set on the held-out device's environments, each normalised by its own
// Oracle best[e], and compare with a selection made directly on the
// held-out environments (the "known" baseline).
#include <cmath>
#include <vector>

#include "pt_internal.cuh"

static pt_status select_on(pt_ctx *ctx, const uint8_t *mask, int32_t k, int32_t method,
                           int32_t *idx, double *G)
{
    if (method == 0) {
        std::vector<double> gt(k), gp(k);
        PT_TRY(pt_greedy_select(ctx, k, mask, PT_OBJ_GEOMEAN, idx, gt.data(), gp.data()));
        *G = gt[k - 1];
    } else {
        PT_TRY(pt_exhaustive_best(ctx, k, mask, PT_OBJ_GEOMEAN, 0, 1, idx, G, nullptr, nullptr,
                                  nullptr));
    }
    return PT_OK;
}

extern "C" pt_status pt_eval_holdout(pt_ctx *ctx, int32_t heldout_device, int32_t k, int32_t method,
                                     int32_t *out_idx, double *out_G_train, double *out_G_unseen,
                                     double *out_G_known, int32_t *out_known_idx)
{
    if (!ctx || !out_idx || !out_G_train || !out_G_unseen || !out_G_known)
        return pt_fail(PT_EINVAL, "NULL argument");
    if (!ctx->have_device) return pt_fail(PT_EINVAL, "pt_load_perf was given no env_device");
    if (method != 0 && method != 1) return pt_fail(PT_EINVAL, "method must be 0 or 1");
    if (k < 1) return pt_fail(PT_EINVAL, "k < 1");
    std::vector<uint8_t> train(ctx->E), test(ctx->E);
    int64_t ntr = 0, nte = 0;
    for (int64_t e = 0; e < ctx->E; e++) {
        train[e] = ctx->env_device[e] != heldout_device;
        test[e] = !train[e];
        ntr += train[e];
        nte += test[e];
    }
    if (ntr == 0 || nte == 0)
        return pt_fail(PT_EEMPTY, "device %d leaves an empty train or test scope", heldout_device);
    PT_TRY(select_on(ctx, train.data(), k, method, out_idx, out_G_train));
    PT_TRY(pt_score_sets(ctx, out_idx, 1, k, test.data(), PT_OBJ_GEOMEAN, out_G_unseen));
    std::vector<int32_t> kidx(k);
    PT_TRY(select_on(ctx, test.data(), k, method, kidx.data(), out_G_known));
    if (out_known_idx)
        for (int u = 0; u < k; u++) out_known_idx[u] = kidx[u];
    return PT_OK;
}
