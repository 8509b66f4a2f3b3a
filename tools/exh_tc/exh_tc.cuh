// exh_tc.cuh -- the tcgen05 exhaustive kernel's parameters and entry points, shared by
// exhaustive.cu (host driver) and exh_tc.cu (kernel).
#pragma once

#include "pt_internal.cuh"

// first column of a row tile whose first row's largest member is j0: j0 + 1 rounded
// down to 8 configs (16-byte aligned tiles); the extra columns are <= every row's
// largest member and masked.  The task builder AND the kernels use this one function.
// (tile_lo: pt_internal.cuh)

#define TC_R 128   // rows per task = threads per CTA = TMEM lanes
#define TC_C 64    // columns per tile
#define TC_K 64    // environments per B stage (32 env pairs)
#define TC_S 3     // B ring stages
#define TC_NB 3    // TMEM staging buffers (64 columns each)

struct TcParams {
    int64_t C, E_pad, n_rows;
    int m;                     // members per row (k - 1)
    const int4 *tasks;         // (row tile, first column tile, end column tile, 0)
    int task_hi;               // end of this shard's task range
    int *task_ctr;             // dynamic scheduler (starts at the shard's first task)
    float tau_seed;            // host seed of the window (+inf when U is seeded on the device)
    float c1, c2, c3, c4;      // LB = RD(s*c1 - c2), UB = RU(s*c3 + c4) on the fp32 sum s
    unsigned *U;               // float bits: min over warps of their 2nd-smallest UB
    unsigned long long *cand_key;
    float *cand_s;
    unsigned *cand_n;
    unsigned cap;
    const uint32_t *hTileP;    // [8 shifts][n_ct][E_pad/2][64] f16x2 env pairs, natural column order
    int64_t n_ct;
    const uint16_t *hC;        // [C_pad][E_pad] fp16 config-major (A staging)
};

// builds the view's hC and hTileP (once per view)
pt_status pt_exh_tc_prepare(pt_ctx *ctx, const pt_view *v);
// dynamic shared memory of k_exh_tc for a scope
size_t pt_exh_tc_smem(int64_t E_pad);
// the kernel entry (for attributes / occupancy) and its launch
const void *pt_exh_tc_kernel();
pt_status pt_exh_tc_launch(const TcParams &p, int grid, size_t smem, cudaStream_t s);
