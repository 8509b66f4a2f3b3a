"""bench.py -- candidate variant-sets scored per second for the portability-tuning
hot path (arXiv 2507.15277) on B200, one JSON line on rank 0.

Workload (BASELINE.json configs[1..3] on the paper-shaped matrix, 1,775 configs x
320 envs = 5 devices x 64 GEMM inputs, synthetic, seed 1).  One STEP = one pass
of the whole hot path over that matrix:
    pt_load_perf (normalise; T already resident in HBM)
  + pt_greedy_select k=24                     (42,324 sets)
  + pt_exhaustive_best k=2                    (1,574,425 sets)
  + pt_exhaustive_best k=3                    (930,485,175 sets)
  + pt_eval_holdout_all, 5 folds, greedy k=5  (88,655 sets)
With N GPUs the k=3 search is sharded across ranks and the library exchanges and
merges the (score, tuple) records over its own NCCL communicator (strong scaling:
the job is fixed); every rank loads the matrix, greedy k=24 runs on rank 0, the
(batched, one-launch) holdout on rank 1 and the latency-bound k=2 search on rank 2
(all on rank 0 at N=1), and those ranks take a smaller share of the k=3 tasks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {pt,reference}]
"""
import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

E_PAPER, C_PAPER = 320, 1775
K_GREEDY, K_HOLDOUT = 24, 5
SETS = {
    "greedy24": sum(C_PAPER - t for t in range(K_GREEDY)),
    "exh2": math.comb(C_PAPER, 2),
    "exh3": math.comb(C_PAPER, 3),
    # per fold: greedy on train + greedy on the held-out device + 1 scored set
    "holdout": 5 * (2 * sum(C_PAPER - t for t in range(K_HOLDOUT)) + 1),
}
SETS_PER_STEP = sum(SETS.values())
WORKLOAD = ("paper-shaped 1775 configs x 320 envs (5 devices x 64 GEMM inputs): load + greedy k=24 "
            "+ exhaustive k=2 + exhaustive k=3 + 5-fold holdout (greedy k=5)")


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# BENCH_SAME_GPU=1 (debug only): every rank on cuda:0 with the gloo backend, to smoke-test
# the multi-process path on a one-GPU box; never used for a reported number
SAME_GPU = os.environ.get("BENCH_SAME_GPU") == "1"


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            0 if SAME_GPU else int(os.environ.get("LOCAL_RANK", 0)))


class ClockSampler:
    """SM clock + throttle reasons sampled (NVML, in-process) during the timed region."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, gpu, period=0.05):
        self.gpu, self.period, self.rows, self.stop = gpu, period, [], threading.Event()
        self.max_mhz = None

    def _init(self):
        # NVML initialised before the timed region starts (in __enter__, ahead of
        # the first event record), not concurrently with it
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.h = None

    def _run(self):
        if self.h is None:
            return
        pynvml, h = self.nv, self.h
        while not self.stop.is_set():
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((sm, rs))
            except Exception:
                pass
            self.stop.wait(self.period)

    def __enter__(self):
        self._init()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        reasons = sorted({n for _, rs in self.rows for n, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": float(np.median([r[0] for r in self.rows])), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.rows), "source": "NVML"}


# --------------------------------------------------------------------------- oracle
def oracle_sample_rate(T, dev, target_s=12.0, threads=None):
    """The CPU oracle (as it stands) on a bounded sample of the k=3 search: all
    triples whose first index is in [0, n0).  Returns (sets/s, cores, sample)."""
    from oracle import Oracle, default_threads
    threads = threads or default_threads()
    o = Oracle(T, dev)
    C = T.shape[1]

    def n_sets(n0):
        return sum(math.comb(C - 1 - a, 2) for a in range(n0))

    # the oracle deals first indices to its threads round-robin, so the sample
    # always spans a multiple of `threads` first indices (every thread busy)
    n1 = threads
    for _ in range(5):
        t0 = time.perf_counter()
        o.exhaustive(3, lo=0, hi=n1, threads=threads)
        dt = time.perf_counter() - t0
        rate = n_sets(n1) / dt
        if dt >= 0.6 * target_s or n1 + threads > C - 3:
            break
        n2 = n1
        while n2 + threads <= C - 3 and n_sets(n2 + threads) / rate < target_s:
            n2 += threads
        n1 = max(n2, n1 + threads)
    return rate, threads, (f"exhaustive k=3 over the paper-shaped matrix restricted to first index "
                           f"in [0,{n1}): {n_sets(n1)} triples x 320 envs, {dt:.1f} s, {threads} threads")


def run_reference(args):
    """--impl reference: the CPU oracle timed on bounded samples of the workload."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2507_15277_b200 import synth
    from oracle import Oracle, default_threads
    T, dev = synth.paper_matrix(1)
    threads = default_threads()
    o = Oracle(T, dev)
    C = T.shape[1]
    per_step_target = max(1.0, 150.0 / max(1, args.steps + args.warmup))
    # calibrate a first-index range so one step takes ~per_step_target seconds; the
    # oracle deals first indices to its threads round-robin, so the range is a multiple
    # of `threads` (every thread busy -- calibrating on one index left all but one idle)
    def n_sets(n):
        return sum(math.comb(C - 1 - a, 2) for a in range(n))
    t0 = time.perf_counter()
    o.exhaustive(3, lo=0, hi=threads, threads=threads)
    r = n_sets(threads) / (time.perf_counter() - t0)
    n0 = threads
    while n0 + threads <= C - 3 and n_sets(n0 + threads) / r < per_step_target:
        n0 += threads
    nsets = n_sets(n0)
    for _ in range(args.warmup):
        o.exhaustive(3, lo=0, hi=n0, threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        o.exhaustive(3, lo=0, hi=n0, threads=threads)
    dt = time.perf_counter() - t0
    value = nsets * args.steps / dt
    sample = (f"exhaustive k=3, first index in [0,{n0}) ({nsets} triples x 320 envs) per step, "
              f"{threads} threads")
    print(json.dumps({
        "impl": "reference", "metric": "candidate variant-sets scored/sec", "value": value,
        "unit": "sets/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, paper shape)",
        "config": {"workload": WORKLOAD + " -- oracle on a bounded k=3 sample per step"},
        "cpu_baseline": {"value": value, "unit": "sets/s", "cores": threads, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": "sets/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# --------------------------------------------------------------------------- GPU arm
def measure_scaled(pt, synth, local, pk, steps=3, world=1):
    """Secondary line, BASELINE config 5: greedy k=32 on the scaled 65,536 x 4,096
    matrix (HBM-bound: every step streams the whole fp32 matrix, 1 GiB).  With
    world > 1 the configurations are sharded (pt_greedy_sharded: each rank
    streams 1/world of the matrix per step, 2 records all-gathered over the
    process group); the time is the max over ranks."""
    import torch
    T, dev = synth.scaled(1)
    dT = torch.from_numpy(T).cuda()
    del T
    ctx = pt.pt_load_perf(dT, dev, device=local)

    def run():
        if world > 1:
            return pt.greedy_select_distributed(ctx, 32)
        return pt.pt_greedy_select(ctx, 32)

    run()                                             # warm-up
    ms = []
    for _ in range(steps):
        run()
        ms.append(pt.pt_get_stats(ctx)["greedy_ms"])
    st = pt.pt_get_stats(ctx)
    km = None
    if world == 1:
        # k-means selector at the same shape: 4,096 points x 65,536 dims, k = 32,
        # bit-identical to the oracle's order of operations; fp64 CUDA cores
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        pt.pt_kmeans_select(ctx, 32)
        e0.record()
        sel, _, iters = pt.pt_kmeans_select(ctx, 32)
        e1.record()
        torch.cuda.synchronize()
        kms = e0.elapsed_time(e1)
        nsm = torch.cuda.get_device_properties(local).multi_processor_count
        dp_peak = nsm * 58.3 * pk.get("sm_max_mhz", 1965.0) * 1e6          # DP instructions / s (ubench_fp64)
        dp_ops = 3.0 * 4096 * 65536 * (32 * iters + 32 + 1)                 # sub, mul, add per (point, centroid, dim)
        km = {"workload": "k-means selector, 4,096 envs x 65,536 configs, k=32", "ms": kms, "iterations": iters,
              "selected": len(sel),
              "roofline": {"bound": "fp64", "achieved": dp_ops / (kms * 1e-3) / 1e12, "peak": dp_peak / 1e12,
                           "unit": "T DP-instr/s", "frac": dp_ops / (kms * 1e-3) / dp_peak,
                           "basis": "distance passes only (init + Lloyd), each (point, centroid, config) a "
                                    "DSUB + DMUL + DADD in the oracle's order; peak 58.3 DP/clk/SM"}}
    pt.pt_free(ctx)
    del dT
    torch.cuda.empty_cache()
    t = float(np.median(ms))
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([t], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    C, E = 65536, 4096
    sets = sum(C - i for i in range(32))
    bytes_ = 32.0 * C * E * 4                          # algorithmic: one fp32 read per (config, env) per step
    gbs = bytes_ / (t * 1e-3) / 1e9
    peak = pk.get("hbm_gbs", 6650.0) * world
    return {"workload": "scaled synthetic 65,536 configs x 4,096 envs (64 devices x 64 inputs), greedy k=32"
                        + (f", configs sharded x{world} (pt_greedy_sharded)" if world > 1 else ""),
            "value": sets / (t * 1e-3), "unit": "sets/s", "ms": t,
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                         "basis": "4 B per (candidate, env) per step over the whole selection "
                                  "(scan + window pick), MEASURED_PEAKS hbm_gbs (x world for sharded runs)"},
            "fp64_refined_candidates": st["greedy_candidates"], "kmeans_scaled": km}



def measure_per_config(pt, dT, dev, local, pk, reps=5):
    """One sub-line per BASELINE config on the paper-shaped matrix (each
    config has its own bounding roofline): the call alone, inputs resident, CUDA
    events on the library's stream around it (median of `reps` after a warm-up), and
    for the exhaustive searches the main kernel's own CUDA-event time."""
    import torch
    nsm = torch.cuda.get_device_properties(local).multi_processor_count
    alu_peak = nsm * 128 * pk.get("sm_max_mhz", 1965.0) * 1e6
    ctx = pt.pt_load_perf(dT, dev, device=local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def dev_ms(fn, stat=None):
        fn()
        ms, kms = [], []
        for _ in range(reps):
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
            if stat:
                kms.append(pt.pt_get_stats(ctx)[stat])
        return float(np.median(ms)), (float(np.median(kms)) if kms else None)

    out = {}
    ms, _ = dev_ms(lambda: pt.pt_greedy_select(ctx, K_GREEDY))
    out["paper_greedy_k24"] = {
        "config": "BASELINE configs[1]: greedy k=1..24 over 1,775 x 320", "ms": ms,
        "us_per_step": ms * 1e3 / K_GREEDY, "sets_per_s": SETS["greedy24"] / (ms * 1e-3),
        "roofline": {"bound": "latency", "basis": "24 dependent steps, each a grid barrier + a merge of "
                     "per-CTA records (DESIGN.md 6.4); ALU work per step ~0.03 us at the ALU ceiling",
                     "alu_frac": SETS["greedy24"] * E_PAPER / (ms * 1e-3) / alu_peak}}
    for k, name in ((2, "paper_exhaustive_k2"), (3, "paper_exhaustive_k3")):
        ms, kms = dev_ms(lambda: pt.pt_exhaustive_best(ctx, k), "exh_main_ms")
        sets = SETS[f"exh{k}"]
        stk = pt.pt_get_stats(ctx)
        q8 = stk["exh_kernel"] == 4
        pk_k = alu_peak * (2 if q8 else 1)   # u8 tier: 4 (set,env) per VABSDIFF4
        roof = {"bound": "alu", "kernel": "k_exh_q8" if q8 else "k_exh_tiled", "unit": "T(set,env)/s",
                "achieved": sets * E_PAPER / (kms * 1e-3) / 1e12, "peak": pk_k / 1e12,
                "frac": sets * E_PAPER / (kms * 1e-3) / pk_k}
        if stk["exh_kernel"] == 5:   # tc tier: tensor-bound
            fp8 = 2.0 * float(peaks().get("bf16_tflops", 1590.0))
            tf = 2.0 * stk["exh_tc_nt"] * stk["exh_env_pad"] * sets / (kms * 1e-3) / 1e12
            roof = {"bound": "tensor", "kernel": "k_exh_tc", "unit": "TFLOP/s", "achieved": tf, "peak": fp8,
                    "frac": tf / fp8, "survivors": stk["exh_tc_survivors"], "nt": stk["exh_tc_nt"]}
        out[name] = {"config": f"BASELINE configs[2]: exhaustive k={k} over 1,775 x 320", "ms": ms,
                     "kernel_ms": kms, "sets_per_s": sets / (ms * 1e-3), "roofline": roof}
    ms, _ = dev_ms(lambda: pt.pt_eval_holdout_all(ctx, K_HOLDOUT, 5))
    out["holdout_5fold_greedy_k5"] = {
        "config": "BASELINE configs[3]: leave-one-device-out, 5 folds, greedy k=5 (one batched launch)",
        "ms": ms, "sets_per_s": SETS["holdout"] / (ms * 1e-3),
        "roofline": {"bound": "latency", "basis": "5 dependent greedy steps over 10 problems at once",
                     "alu_frac": SETS["holdout"] * E_PAPER / (ms * 1e-3) / alu_peak}}
    pt.pt_free(ctx)
    return out


FP64_PEAK_TFLOPS = 2 * 16.96   # tools/ubench_fp64.cu on this pool's B200: 58.3 DFMA/clk/SM (2 flops each)


def measure_next_rows(pt, T, dev, local, cpu=True):
    """The §8(f) NEXT rows at the paper shape, each timed on the device (CUDA events
    around the call on the library's stream, median of 3 after a warm-up) beside the
    CPU oracle on the same workload: fleet objective (Eq. 2) greedy k=24 and
    exhaustive k=2 / k=3 (tiled), swap local search k=24, k-means k=24.  Work = (set, env)
    evaluations of one min + one multiply-add (k-means: (point, centroid, dim) of
    one subtract + one multiply-add), counted as 2 fp64 flops; roofline = the
    measured DFMA rate."""
    import torch
    from oracle import Oracle
    C, E = T.shape[1], T.shape[0]
    qd = np.array([5.0, 2.0, 1.0, 3.0, 4.0])      # fleet mix (invented; tests/test_gpu_fleet.py)
    qe = np.ones(len(dev))
    ctx = pt.pt_load_perf(torch.from_numpy(T).cuda(), dev, device=local)
    pt.pt_set_fleet(ctx, qd, qe)
    o = Oracle(T, dev) if cpu else None
    if o is not None:
        o.set_fleet(qd, qe)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def dev_ms(fn):
        fn()
        ms = []
        for _ in range(3):
            e0.record()
            r = fn()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        return float(np.median(ms)), r

    def cpu_s(fn):
        if o is None:
            return None
        t0 = time.perf_counter()
        fn()
        return time.perf_counter() - t0

    rows = {}
    ms, _ = dev_ms(lambda: pt.pt_greedy_select(ctx, 24, objective=pt.PT_OBJ_FLEET))
    ev = sum(C - t for t in range(24)) * E
    rows["fleet_greedy_k24"] = (ms, ev, sum(C - t for t in range(24)), cpu_s(lambda: o.fleet_greedy(24)))
    # fleet exhaustive: the tiled (min,+) kernel with the per-device fold (k_exh_tiled<true>),
    # roofline = the f16x2 ALU ceiling of the geomean kernel (same inner loop)
    fleet_exh = {}
    for kk in (2, 3):
        ms, _ = dev_ms(lambda: pt.pt_exhaustive_best(ctx, kk, objective=pt.PT_OBJ_FLEET))
        st = pt.pt_get_stats(ctx)
        fleet_exh[kk] = (ms, st["exh_main_ms"], st["exh_kernel"], st["exh_candidates"])
    rows_alu = {}
    for kk, (ms, kms, path, cand) in fleet_exh.items():
        sets = math.comb(C, kk)
        nsm = torch.cuda.get_device_properties(local).multi_processor_count
        alu_peak = nsm * 128 * 1965.0e6
        rows_alu[f"fleet_exhaustive_k{kk}"] = {
            "ms": ms, "kernel_ms": kms, "path": {3: "tiled fp16 + per-device fold"}.get(path, str(path)),
            "candidates_refined": cand, "sets_per_s": sets / (ms * 1e-3),
            "roofline": {"bound": "alu", "unit": "T(set,env)/s", "achieved": sets * E / (kms * 1e-3) / 1e12,
                         "peak": alu_peak / 1e12, "frac": sets * E / (kms * 1e-3) / alu_peak}}
    if o is not None:
        t0 = time.perf_counter()
        o.fleet_exhaustive_par(2)
        rows_alu["fleet_exhaustive_k2"]["oracle_s"] = time.perf_counter() - t0
        rows_alu["fleet_exhaustive_k2"]["oracle_sets_per_s"] = math.comb(C, 2) / rows_alu["fleet_exhaustive_k2"]["oracle_s"]
    ms, (_, _, moves) = dev_ms(lambda: pt.pt_swap_search(ctx, 24))
    sets = (moves + 1) * 24 * (C - 24)
    rows["swap_k24"] = (ms, sets * E, sets, cpu_s(lambda: o.swap_search(24)))
    ms, (_, _, iters) = dev_ms(lambda: pt.pt_kmeans_select(ctx, 24))
    rows["kmeans_k24"] = (ms, iters * E * 24 * C, None, cpu_s(lambda: o.kmeans(24)))
    pt.pt_free(ctx)
    out = {}
    for name, (ms, evals, sets, cs) in rows.items():
        fl = 2.0 * evals
        r = {"ms": ms, "gflops": fl / (ms * 1e-3) / 1e9,
             "roofline": {"bound": "fp64", "achieved": fl / (ms * 1e-3) / 1e12, "peak": FP64_PEAK_TFLOPS,
                          "unit": "TFLOP/s", "frac": fl / (ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS}}
        if sets is not None:
            r["sets_per_s"] = sets / (ms * 1e-3)
        if cs is not None:
            r["oracle_s"] = cs
            r["oracle_sets_per_s"] = sets / cs if sets is not None else None
        out[name] = r
    out.update(rows_alu)
    if moves is not None:
        out["swap_k24"]["moves"] = moves
    out["kmeans_k24"]["iterations"] = iters
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="pt", choices=["pt", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-next", action="store_true", help="skip the NEXT-row measurements")
    ap.add_argument("--no-scaled", action="store_true",
                    help="skip the secondary config-5 measurement (scaled greedy, HBM-bound)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_2507_15277_b200 import pt, synth

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if SAME_GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()

    T, dev = synth.paper_matrix(args.seed)
    dT = torch.from_numpy(T).cuda()
    hT = torch.from_numpy(T).pin_memory()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2
    flush.fill_(0)                     # load the fill kernel's module before any timing
    torch.cuda.synchronize()

    # with N ranks the exhaustive searches are sharded; the two unsharded parts
    # (greedy k=24 and the batched holdout) run once per job, on ranks 0 and 1, and
    # those ranks take a correspondingly smaller share of the k=3 task list
    # (pt_set_shard_weights; extra work per_config-measured on one B200: greedy k=24
    # ~0.21 ms, the batched holdout ~0.16 ms, k=2 ~0.11 ms, against a k=3 search of
    # ~1.0 ms on one GPU on the tc tier)
    # exhaustive k=2 is latency-bound (1.6 M pairs = 13 us of ALU work on one GPU, one
    # 32 us wave of 128x64 tiles): sharding it would cost every rank a full call for
    # ~2 us of work each, so with N > 1 it runs unsharded on rank 2 (mod N); only the
    # k=3 search (930 M triples) is sharded
    do_greedy = rank == 0
    do_holdout = rank == 1 % world
    do_k2 = world == 1 or rank == 2 % world
    shard_w = None
    if world > 1:
        extra = [0.0] * world
        extra[0] += 0.21
        extra[1 % world] += 0.16
        extra[2 % world] += 0.11
        shard_w = [max(0.05, 1.0 - x * world / 1.0) for x in extra]

    def step(src):
        """One pass of the whole hot path; returns (results, d2h bytes)."""
        ctx = pt.pt_load_perf(src, dev, device=local)
        if shard_w is not None:
            pt.pt_set_shard_weights(ctx, shard_w)
        d2h = 0
        idx = None
        if do_greedy:
            idx, gt, gp = pt.pt_greedy_select(ctx, K_GREEDY)
            d2h += idx.__len__() * 4 + gt.nbytes + gp.nbytes
        r2 = pt.pt_exhaustive_best(ctx, 2) if do_k2 else None
        r3 = pt.exhaustive_best_distributed(ctx, 3) if world > 1 else pt.pt_exhaustive_best(ctx, 3)
        st3 = pt.pt_get_stats(ctx)
        d2h += (2 * 2 * 4 + 4 * 8 if do_k2 else 0) + 2 * 3 * 4 + 4 * 8
        if do_holdout:
            hold = pt.pt_eval_holdout_all(ctx, K_HOLDOUT, 5)      # all 5 folds, one batched launch
            d2h += len(hold) * (2 * K_HOLDOUT * 4 + 3 * 8)
        st_end = pt.pt_get_stats(ctx)
        pt.pt_free(ctx)
        return {"greedy": idx, "r2": r2, "r3": r3, "k3_ms": st3["exh_main_ms"],
                "k3_sets": st3["exh_sets"], "k3_slots": st3["exh_slots"], "k3_kernel": st3["exh_kernel"],
                "k3_cand": st3["exh_candidates"], "k3_nt": st3["exh_tc_nt"], "k3_env_pad": st3["exh_env_pad"],
                "launches": st_end["launches"]}, d2h

    def timed(src, steps, warmup):
        for _ in range(warmup):
            step(src)
        k3_ms, launches, res = [], 0, None
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        marks = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        with ClockSampler(local) as clk:
            ev0.record(stream)
            for i in range(steps):
                flush.fill_(1)                     # L2 flushed between steps
                marks[i].record(stream)
                res, d2h = step(src)
                k3_ms.append(res["k3_ms"])
                launches += res["launches"] + 1
            marks[steps].record(stream)
            ev1.record(stream)
            torch.cuda.synchronize()
        step_ms = [marks[i].elapsed_time(marks[i + 1]) for i in range(steps)]
        if world > 1:
            dist.barrier()
        ms = ev0.elapsed_time(ev1)
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, k3_ms, launches, res, d2h, dict(clk.summary(), step_ms=[round(x, 3) for x in step_ms])

    ms, k3_ms, launches, res, d2h, clocks = timed(dT, args.steps, args.warmup)
    ms_e2e, _, _, _, d2h_e2e, clocks_e2e = timed(hT, args.steps, 1)
    h2d_e2e = int(T.nbytes) * world            # every rank loads the matrix
    if world > 1:
        # job totals: the copies and launches of every rank
        agg = torch.tensor([float(d2h_e2e), float(launches)], dtype=torch.float64,
                           device="cpu" if SAME_GPU else "cuda")
        dist.all_reduce(agg)
        d2h_e2e, launches = int(agg[0].item()), int(agg[1].item())
    # secondary config-5 line: every rank takes part (sharded greedy for world > 1)
    scaled = None if args.no_scaled else measure_scaled(pt, synth, local, peaks(), world=world)
    per_config = measure_per_config(pt, dT, dev, local, peaks()) if world == 1 else None
    next_rows = None
    if world == 1 and not args.no_next:
        next_rows = measure_next_rows(pt, T, dev, local, cpu=not args.no_cpu_baseline)
    # shard balance of the k=3 search (single-GPU runs only): the N shards of the
    # multi-GPU partition run one after another on this GPU; max over shards = the
    # kernel time an N-GPU run would see per GPU.  A model, not a multi-GPU measurement.
    shard_bal = None
    if world == 1:
        ctx = pt.pt_load_perf(dT, dev, device=local)
        pt.pt_exhaustive_best(ctx, 3)
        full_ms = pt.pt_get_stats(ctx)["exh_main_ms"]
        shard_bal = {"basis": "k=3 kernel (CUDA events) of each shard of the N-way partition, "
                              "run sequentially on this GPU", "full_ms": full_ms}
        for n in (2, 4, 8):
            t = []
            for r in range(n):
                pt.pt_exhaustive_best(ctx, 3, shard_rank=r, shard_count=n)
                t.append(pt.pt_get_stats(ctx)["exh_main_ms"])
            shard_bal[str(n)] = {"max_ms": max(t), "mean_ms": float(np.mean(t)),
                                 "efficiency": full_ms / n / max(t)}
        pt.pt_free(ctx)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    pk = peaks()
    sm_max = pk.get("sm_max_mhz", 1965.0)
    nsm = torch.cuda.get_device_properties(local).multi_processor_count
    # roofline of the dominant kernel (k=3).  Algorithmic work: one min + one add per
    # (set, env), E = 320 envs per set.  Default tier (exh_kernel 4, k_exh_q8): the
    # quantised set score is 4 (set, env) evaluations per VABSDIFF4.U8.ACC, which
    # issues at 16 lanes/clk/SMSP (tools/ubench.cu: 2.06 warp-instr/clk/SM) -> 16 x 4
    # SMSP x 4 = 256 (set,env)/clk/SM.  fp16 tier (exh_kernel 0, k_exh_tiled): the
    # ALU-pipe min ceiling, 16 lanes/clk/SMSP x 4 SMSP x 2 mins per HMNMX2 = 128.
    # The FP32 roofline of the north star (one FMNMX at 16 lanes/clk/SMSP + one FADD
    # per (set, env)) is 64 (set,env)/clk/SM.
    # Threshold-count tier (exh_kernel 5, k_exh_tc, the default): a tensor-core
    # contraction; algorithmic work = 2 x K flops per set, K = nt x E_pad (the 0/1
    # vectors' length), against the dense fp8 peak = the MEASURED bf16 peak x 2 (the
    # guide's nominal fp8/bf16 ratio; burst figure: the kernel runs ~1 ms inside the step).
    tier_tc = res.get("k3_kernel") == 5
    tier_q8 = res.get("k3_kernel") == 4
    per_clk = 256 if tier_q8 else 128
    evals = float(E_PAPER) * res["k3_sets"]
    k3_avg = float(np.mean(k3_ms))
    achieved = evals / (k3_avg * 1e-3) / 1e12
    peak = nsm * per_clk * sm_max * 1e6 / 1e12
    peak_q8 = nsm * 256 * sm_max * 1e6 / 1e12
    peak_f16 = nsm * 128 * sm_max * 1e6 / 1e12
    peak_fp32 = nsm * 64 * sm_max * 1e6 / 1e12
    tc_roof = None
    if tier_tc:
        K_tc = int(res["k3_nt"]) * int(res["k3_env_pad"])
        tflops = 2.0 * K_tc * res["k3_sets"] / (k3_avg * 1e-3) / 1e12
        fp8_peak = 2.0 * float(pk.get("bf16_tflops", 1590.0))   # fallback: B200_PROFILING.md's 1.59 PF bf16
        tc_roof = {"bound": "tensor", "kernel": "k_exh_tc (k=3)", "achieved": tflops, "peak": fp8_peak,
                   "unit": "TFLOP/s", "frac": tflops / fp8_peak,
                   "work_per_set": f"2 x K = {2 * K_tc} flops (K = nt {res['k3_nt']} x E_pad {res['k3_env_pad']}: "
                                   "the 0/1 threshold vectors' dot product, DESIGN.md 6.2c)",
                   "peak_basis": "dense fp8 (E4M3, kind::f8f6f4) = MEASURED_PEAKS bf16_tflops (burst) x 2, "
                                 "the guide's nominal fp8/bf16 ratio"}
    traffic, l2 = None, None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "k3_dram_bytes.json")))
        traffic = prof["bytes_per_launch"]
        if prof.get("l2_bytes_per_launch"):
            l2 = {"bytes_per_launch": prof["l2_bytes_per_launch"],
                  "GB_s": prof["l2_bytes_per_launch"] / (k3_avg * 1e-3) / 1e9,
                  "pct_of_peak": prof.get("l2_throughput_pct_of_peak"),
                  "source": "ncu lts__t_sectors.sum x 32 B and lts__throughput, one --set full capture"}
    except Exception:
        pass

    cpu = None
    if not args.no_cpu_baseline:
        rate, cores, sample = oracle_sample_rate(T, dev)
        cpu = {"value": rate, "unit": "sets/s", "cores": cores, "kind": "oracle", "sample": sample}


    import json as _j
    gold = None
    try:
        g = _j.load(open(os.path.join(ROOT, "tests", "golden", "paper_exhaustive.json")))[f"seed{args.seed}_k3"]
        gold = tuple(g["best"]) == tuple(res["r3"]["best"])
    except Exception:
        pass
    line = {
        "metric": "candidate variant-sets scored/sec",
        "value": SETS_PER_STEP * args.steps / (ms * 1e-3),
        "unit": "sets/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": ("e4m3 0/1 threshold-count filter on tcgen05 (exact integer counts, fp32 accumulate), "
                  "f64 exact refine" if tier_tc else
                  "u8 (exact integer |a-b| score of the quantised matrix) filter, f64 exact refine" if tier_q8
                  else "f16x2 min + f32 sum filter, f64 exact refine"),
        "data": "synthetic (seeded generator, paper shape; private dataset unavailable)",
        "config": {"workload": WORKLOAD, "sets_per_step": SETS_PER_STEP, "seed": args.seed,
                   "l2": "flushed between steps (256 MiB write, inside the timed region)",
                   "parallelism": (f"subset-space shards x{world}" + (" (DEBUG: all ranks on one GPU, gloo)" if SAME_GPU else "")) if world > 1 else "single GPU"},
        "e2e": {"value": SETS_PER_STEP * args.steps / (ms_e2e * 1e-3), "unit": "sets/s",
                "h2d_bytes_per_step": h2d_e2e, "d2h_bytes_per_step": int(d2h_e2e)},
        "gpu_launches": int(launches),
        "roofline": dict(tc_roof, traffic=traffic, kernel_ms=k3_avg, kernel_share_of_step=k3_avg / (ms / args.steps),
                         l2=l2, set_env_rate={"achieved": achieved, "unit": "T(set,env)/s",
                                              "vs_u8_alu_ceiling": achieved / peak_q8,
                                              "vs_fp32_alu_ceiling": achieved / peak_fp32}) if tier_tc else
                    {"bound": "alu", "kernel": ("k_exh_q8" if tier_q8 else "k_exh_tiled") + " (k=3)",
                     "achieved": achieved,
                     "peak": peak, "unit": "T(set,env)/s", "frac": achieved / peak, "traffic": traffic,
                     "work_per_set": f"{E_PAPER} (set,env) evaluations = {E_PAPER} min + {E_PAPER} add",
                     "peak_basis": (f"VABSDIFF4.U8.ACC ceiling: {nsm} SMs x 4 SMSP x 16 lanes/clk x 4 (set,env) "
                                    f"per instruction x {sm_max:.0f} MHz (MEASURED_PEAKS sm_max_mhz); issue rate "
                                    "measured by tools/ubench.cu, the inner loop alone reaches 245/clk/SM "
                                    "(tools/ubench_sad.cu, DESIGN.md 6.2b)") if tier_q8 else
                                   (f"ALU-pipe min ceiling: {nsm} SMs x 4 SMSP x 16 lanes/clk x 2 mins "
                                    f"(f16x2 HMNMX2) x {sm_max:.0f} MHz (MEASURED_PEAKS sm_max_mhz); "
                                    "the packed adds (HADD2, half rate on the FMA pipe) and the issue "
                                    "port have the same ceiling (DESIGN.md 6.1)"),
                     "f16x2_roofline": {"peak": peak_f16, "frac": achieved / peak_f16,
                                        "basis": "the fp16 tier's HMNMX2 ceiling (128 (set,env)/clk/SM)"},
                     "fp32_roofline": {"peak": peak_fp32, "frac": achieved / peak_fp32,
                                       "basis": "one FMNMX (16 lanes/clk/SMSP) + one FADD per (set, env)"},
                     "kernel_ms": k3_avg, "kernel_share_of_step": k3_avg / (ms / args.steps),
                     "l2": l2},
        "cpu_baseline": cpu,
        "clocks": clocks,
        "clocks_e2e": clocks_e2e,
        "parity": {"k3_best": list(res["r3"]["best"]), "k3_matches_oracle_golden": gold,
                   "k3_candidates_refined": res["k3_cand"]},
        "per_config": per_config,
        "scaled_greedy": scaled,
        "k3_shard_balance": shard_bal,
        "next_rows": next_rows,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
