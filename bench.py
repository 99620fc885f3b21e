#!/usr/bin/env python
"""bench.py — the driver's benchmark contract for the extreme-precision Hankel path.

Metric (BASELINE.json): time to lambda_min and MP-FMA/s of the Hankel LDLT.
One *step* = one pass of the hot path over one input: moments mu -> LDLT ->
first k columns of L^{-1} -> k x k block of H^{-1} -> eigensolve -> lambda_min.
Reported throughput = N(N^2-1)/6 LDLT MP-FMAs (the reference's update_count,
ldlt.cpp:128) per step time, i.e. MP-FMA/s over time-to-lambda.

Workload (default): BASELINE configs[3] = C4, beta = 1/2, N = 1024,
p = 49152 bits, k = 16 — the configuration the metric is quoted on "at
1/2/4/8 B200" and the largest that fits one GPU (C5 is the 8-GPU run).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c1..c5]

N > 1: one rank per GPU (torchrun; `--gpus N` without WORLD_SIZE re-launches
itself under torch.distributed.run).  The LDLT is column-sharded across the
ranks (boustrophedon ownership, ncclBroadcast of the pivot column each step,
gather to rank 0 for L^{-1}/block/eigen) — the same job split over N GPUs
(strong scaling); timing is the max over ranks.

`value` times the path with the moments resident on the device; `e2e` times the
public call a user makes (hk_moments on the host into pinned buffers, then
hk_compute: H2D of the moments, the whole path, D2H of the block and lambdas)
— the same span as the reference's RunRecord::wall_s, which includes its
build_hankel (pipeline.cpp:39-41).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# keep stdout to the one JSON line: NCCL's debug text (the version banner already at WARN; INFO if
# the caller asks for it) goes to stderr
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")

# BASELINE.json configs.  K_ref = the reference's K of the golden runs
# (1024 ceil(N/500) + 1024); K_equiv = (p - bits(mu_{2N-2})) / 2, the fixed-point
# K whose 2K fraction bits equal the float's absolute precision on the largest
# entry — the like-for-like precision for timing the reference.
CONFIGS = {
    "c1": dict(beta=(1, 2), n=64, p=3072, k=8, K_ref=2048, K_equiv=705),
    "c2": dict(beta=(1, 1), n=256, p=6144, k=8, K_ref=2048, K_equiv=1143),
    "c3": dict(beta=(1, 3), n=512, p=36864, k=12, K_ref=3072, K_equiv=2872),
    "c4": dict(beta=(1, 2), n=1024, p=49152, k=16, K_ref=4096, K_equiv=2968),
    "c5": dict(beta=(1, 2), n=2048, p=114688, k=16, K_ref=6144, K_equiv=10020),
}
METRIC = "MP-FMA/s of Hankel LDLT over time to lambda_min (N(N^2-1)/6 FMAs per step)"
UNIT = "MP-FMA/s"
# CPU-baseline leg of our own line: a bounded sample (~10-30 s of host work) of
# the same workload — the reference on the leading N_s x N_s block of H_N (the
# LDLT of H_N begins with exactly that factorisation), at K_equiv
CPU_SAMPLE_N = {"c1": 64, "c2": 256, "c3": 256, "c4": 512, "c5": 512}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def ref_driver_path():
    return os.path.join(ROOT, "oracle", "_ref", "ref_driver")


def run_reference_once(cfg, workers, K, n=None):
    """hankel::compute() of the unmodified reference (oracle/_ref/ref_driver) -> its RunRecord JSON."""
    b = cfg["beta"]
    out = subprocess.run([ref_driver_path(), "time", "--beta", f"{b[0]}/{b[1]}", "--n", str(n or cfg["n"]),
                          "--bits", str(K), "--k", str(cfg["k"]), "--workers", str(workers)],
                         capture_output=True, text=True, check=True)
    return json.loads(out.stdout)


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def hbm_peak_gbps():
    """Measured HBM copy bandwidth of this pool (MEASURED_PEAKS.json), else the recipe's fallback."""
    return float(measured_peaks().get("hbm_gbs", 6650.0))


def fmas(n):
    return n * (n * n - 1) // 6


def workload_config(args, cfg, world):
    b = cfg["beta"]
    return {"workload": f"{args.config.upper()}: beta={b[0]}/{b[1]} Hankel N={cfg['n']}, p={cfg['p']} bits, "
                        f"k={cfg['k']} -> lambda_min", "n": cfg["n"], "p_bits": cfg["p"], "k": cfg["k"],
            "beta": f"{b[0]}/{b[1]}",
            "parallelism": f"column-sharded LDLT x{world} GPUs (NCCL pivot-column broadcast)" if world > 1 else "1 GPU",
            "l2": "256 MB written between timed steps (L2 flush); the LDLT working set is "
                  f"{cfg['n'] * (cfg['n'] + 1) // 2 * (cfg['p'] // 8 + 8) / 1e6:.0f} MB"}


# ---------------------------------------------------------------- reference arm


def bench_reference(args, cfg):
    """The reference's own CPU implementation (oracle/_ref: the unmodified sources
    compiled against the GMP shim) through its public hankel::compute, with every
    host core as a worker, on the same config.  A full C4 run takes minutes on
    the box's cores, so the step count is bounded by --ref-budget-s: full runs
    only (never a smaller N), as many as fit, at least one."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    budget = args.ref_budget_s
    t_start = time.perf_counter()
    warm, times, recs = 0, [], []
    for i in range(args.warmup + args.steps):
        rec = run_reference_once(cfg, cores, cfg["K_equiv"])
        if i < args.warmup and rec["timing"]["wall_s"] < 0.05 * budget:
            warm += 1
            continue
        times.append(rec["timing"]["wall_s"])
        recs.append(rec)
        elapsed = time.perf_counter() - t_start
        if len(times) >= args.steps or elapsed + times[-1] > budget:
            break
    t = statistics.mean(times)
    v = fmas(cfg["n"]) / t
    # the golden runs' precision (K_ref) beside it, on request (one more full run)
    k_ref = None
    if args.ref_golden_precision and cfg["K_ref"] != cfg["K_equiv"]:
        r2 = run_reference_once(cfg, cores, cfg["K_ref"])
        k_ref = {"K": cfg["K_ref"], "wall_s": r2["timing"]["wall_s"], "ldlt_s": r2["timing"]["ldlt_s"],
                 "value": fmas(cfg["n"]) / r2["timing"]["wall_s"]}
    sample = (f"{len(times)} full run(s) of the reference's hankel::compute (oracle/_ref, fixed point "
              f"K={cfg['K_equiv']} = K_equiv, workers={cores}) on the whole {args.config} workload "
              f"(N={cfg['n']}); mean wall_s {t:.3f}, ldlt_s {statistics.mean(r['timing']['ldlt_s'] for r in recs):.3f}"
              + (f"; {warm} warm-up run(s)" if warm else "; no warm-up runs (a full run exceeds 5% of the budget)")
              + (f"; steps bounded by the {budget:.0f} s budget ({args.steps} requested)" if len(times) < args.steps
                 else ""))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": len(times),
        "steps_requested": args.steps, "warmup": warm, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": f"fixed-point mpz, K={cfg['K_equiv']} (2K={2 * cfg['K_equiv']} in LDLT)",
        "data": "exact-integer moments (deterministic, no dataset)",
        "config": workload_config(args, cfg, 1),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "time_to_lambda_s": t,
        "reference_timing": recs[-1]["timing"],
        "lambda_min": recs[-1]["lambda"][0] if recs[-1]["lambda"] else None,
        "at_golden_precision": k_ref,
    }
    emit(line)
    return 0


# ---------------------------------------------------------------- our arm


def lambda_parity(name, cfg, lam):
    """Digits of this run's lambda_min (hi + lo) against the reference's golden
    value for the config (tests/golden/<config>.json: the reference built from
    its own sources, lambda from its fixed-point block at 80 digits)."""
    path = os.path.join(ROOT, "tests", "golden", f"{name}.json")
    if not os.path.exists(path):
        return {"golden": None}
    from decimal import Decimal, getcontext

    getcontext().prec = 60
    g = json.load(open(path))
    if g.get("n") != cfg["n"] or g.get("p") != cfg["p"]:
        return {"golden": None}
    want = Decimal(g["lambda"][0])
    got = Decimal(lam[0][0]) + Decimal(lam[1][0])  # exact binary values of hi and lo
    rel = abs(got / want - 1)
    digits = float(-rel.log10()) if rel > 0 else 60.0
    return {"lambda1_digits_vs_reference": round(digits, 2), "required_digits": 20,
            "lambda1_hi_plus_lo": f"{got:.33e}",
            "golden": f"tests/golden/{name}.json (reference at K={g.get('K')}, lambda at 80 digits)"}


def max_over_ranks(x, world, local):
    if world == 1:
        return x
    import torch

    t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def bench_ours(args, cfg):
    import numpy as np
    import torch

    from paper_1810_01478_b200 import api

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    n, p, k = cfg["n"], cfg["p"], cfg["k"]
    L = p // 32
    kk = min(k, n)
    s = min(3, kk)
    if world > 1 or args.sharded:  # column-sharded LDLT over NCCL (hk_create_sharded), results on rank 0
        import torch.distributed as dist

        if "RANK" not in os.environ:  # `--sharded` outside torchrun: a world of one
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                port = sk.getsockname()[1]
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK=str(local), MASTER_ADDR="127.0.0.1",
                              MASTER_PORT=str(port))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [api.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = api.Context(L, device=local, rank=rank, world=world, nccl_id=obj[0])
    else:
        ctx = api.Context(L, device=local)
    # event-record nodes around every step's bulk kernels (graph-resident).  Inside
    # the timed region when a step's product launches are long (N >= 512: ms each,
    # the nodes cost nothing); for the short-step configs (C1/C2, latency-bound
    # chains of ~30 us launches, where the nodes would break the programmatic
    # launch edges) in one extra instrumented step after the timed region.
    kprof_timed = n >= 512
    ctx.set_kernel_timing(kprof_timed)
    ext = torch.cuda.ExternalStream(ctx.stream_ptr(), device=torch.device("cuda", local))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=f"cuda:{local}")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # ---- value: device-resident inputs (moments uploaded once, before timing)
    mu, exact = api.build_hankel(cfg["beta"], n, L)
    assert exact, "moments must be exact at this precision"
    ctx.load_moments(mu)

    def step():
        if world == 1 and not args.sharded:
            ctx.decompose_invert(kk)  # as compute() does: L^-1 steps ride in the LDLT graph when latency-bound
        else:
            # every call is collective on a sharded context: all ranks factor, and (unless
            # HK_DIST_INV=0 keeps them on rank 0) all ranks take part in L^-1 and the block;
            # rank 0 holds the block and runs the eigensolve (as compute_tail does)
            ctx.decompose()
            if rank != 0 and os.environ.get("HK_DIST_INV") == "0":
                return [float("nan")], [0.0], [0.0]
            ctx.invert_L_partial(kk)
        ctx.assemble_truncated_inverse(kk)
        if rank != 0:
            return [float("nan")], [0.0], [0.0]
        return ctx.smallest_eigs_of_H(s)

    for _ in range(args.warmup):
        step()
    barrier()
    sampler = ClockSampler(local)
    total_ms = 0.0
    launches0 = ctx.launch_count()
    kt_sum = {}
    with sampler:
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ext)
            lam = step()
            e1.record(ext)
            e1.synchronize()
            total_ms += e0.elapsed_time(e1)
            if kprof_timed:
                for kk_, v in ctx.kernel_times().items():  # this step's LDLT graph (event nodes)
                    kt_sum[kk_] = kt_sum.get(kk_, 0.0) + v
    barrier()
    launches = ctx.launch_count() - launches0
    ms = max_over_ranks(total_ms / args.steps, world, local)
    value = fmas(n) / (ms * 1e-3)  # one job split over `world` GPUs (strong scaling)
    kt = {kk_: v / args.steps for kk_, v in kt_sum.items()}
    if not kprof_timed:  # one instrumented step after the timed region
        ctx.set_kernel_timing(True)
        step()
        kt = ctx.kernel_times()
        ctx.set_kernel_timing(False)

    # ---- e2e: the public call with host buffers: moments generated on the host
    # into pinned arrays (hk_moments), then hk_compute (H2D, path, D2H of the
    # block + lambdas) — the span of the reference's wall_s incl. build_hankel
    def pinned(shape, dtype):
        t = torch.empty(shape, dtype=torch.int32, pin_memory=True)
        return t, t.numpy().view(dtype)

    keep = [pinned((2 * n - 1, L), np.uint32), pinned((2 * n - 1,), np.int32), pinned((2 * n - 1,), np.int32)]
    mu_pinned = api.MPArray(keep[0][1], keep[1][1], keep[2][1])

    def e2e_step():
        _, ex = api.build_hankel(cfg["beta"], n, L, out=mu_pinned)
        assert ex
        return ctx.compute(mu_pinned, k)

    e2e_step()  # graphs are cached per context: one warm-up suffices
    barrier()
    e2e_ms = 0.0
    for _ in range(args.steps):
        flush.zero_()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        rec = e2e_step()
        e1.record(ext)
        e1.synchronize()
        e2e_ms += e0.elapsed_time(e1)
    e2e_ms = max_over_ranks(e2e_ms / args.steps, world, local)
    h2d = mu.limbs.nbytes + mu.exps.nbytes + mu.signs.nbytes

    # ---- the same call with the moments generated on the device (hk_compute_generated,
    # SURVEY 8 f4): scalars in, lambdas out — reported beside e2e, not instead of it
    gen_ms = None
    if (2 * cfg["beta"][1] // cfg["beta"][0]) % 2 == 0:
        ctx.compute_generated(cfg["beta"], n, k)
        barrier()
        gen_ms, gsteps = 0.0, min(args.steps, 2)
        for _ in range(gsteps):
            flush.zero_()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ext)
            rec_g = ctx.compute_generated(cfg["beta"], n, k)
            e1.record(ext)
            e1.synchronize()
            gen_ms += e0.elapsed_time(e1)
        gen_ms = max_over_ranks(gen_ms / gsteps, world, local)
        gen_moments_ms = ctx.timings()[5] * 1e3
        assert rank != 0 or rec_g.lambda_hi == rec.lambda_hi, "device-generated moments changed lambda"
    d2h = kk * kk * (4 * L + 8) + 9 * 8 if rank == 0 else 11 * 8

    # ---- roofline of the dominant kernel: its graph-resident event times over the timed steps
    alg_macs = fmas(n) * L * L  # L^2 limb-MACs per MP-FMA
    tc_path = L >= 128 and L % 4 == 0
    steps_k = max(kt.get("steps", 0.0), 1.0)
    ms_k = kt.get("products_ms", 0.0)
    ldlt_ms = kt.get("ldlt_ms", 0.0)
    roofline = None
    if ms_k == 0 and not tc_path and ldlt_ms > 0:
        # small p: the whole LDLT is the one dataflow kernel k_ldlt_flow (no per-step launches)
        peak = api.peak_imad(local) / 1e12
        achieved = alg_macs / (ldlt_ms * 1e-3) / 1e12
        roofline = {"bound": "imad", "unit": "Tlimb-MAC/s",
                    "kernel": "k_ldlt_flow: the LDLT as one dataflow kernel (a CTA per entry applies all its "
                              "updates in order, ldlt.cpp:91-135); latency-bound: its critical path is N x "
                              "(fms -> reciprocal -> mul)",
                    "peak_how": "hk_peak_imad: register-only IMAD.WIDE carry-chain microkernel, best of 5 "
                                "(MEASURED_PEAKS.json has no integer peak)",
                    "achieved": achieved, "peak": peak, "frac": achieved / peak, "traffic": None,
                    "per_launch": f"1 launch per step, {ldlt_ms:.4f} ms, {alg_macs:.3e} algorithmic limb-MACs",
                    "algorithmic_units": "L^2 limb-MACs per MP-FMA (SURVEY 8d)",
                    "how_timed": "CUDA events around the kernel on the context's stream (hk_timings ldlt_s)",
                    "share_of_ldlt": 1.0, "kernel_ms_per_step": kt}
    if ms_k > 0:
        # the look-ahead column (ldlt.cpp:122-129 for j = i+1) runs on the chain, not in these launches
        bulk_macs = sum((n - i - 2) * (n - i - 1) // 2 for i in range(n)) * L * L
        achieved = bulk_macs / (ms_k * 1e-3) / 1e12
        if tc_path:
            peak = api.peak_i8mma(local) / 16.0 / 1e12  # u8 MAC/s -> limb-MAC/s (16 u8 MACs per limb-MAC)
            ncu_file = os.path.join(ROOT, "profiles", f"ncu_tc_bulk_{args.config}.json")
            roofline = {"bound": "tensor", "unit": "Tlimb-MAC/s",
                        "kernel": "k_tc_prep + k_tc_bulk: tcgen05.mma kind::i8 limb products of the trailing "
                                  "update (ldlt.cpp:122-129)" + (", certified rounding fused into the epilogue"
                                                                 if kt.get("round_ms", 1.0) < 0.02 * ms_k else ""),
                        "peak_how": "hk_peak_i8mma: back-to-back tcgen05.mma.kind::i8 M128 N256 K32 on every SM, "
                                    "best of 5, /16 u8 MACs per limb-MAC (MEASURED_PEAKS.json has no integer peak)",
                        "imad_peak": api.peak_imad(local) / 1e12}
        else:
            peak = api.peak_imad(local) / 1e12
            ncu_file = os.path.join(ROOT, "profiles", f"ncu_trailing_{args.config}.json")
            roofline = {"bound": "imad", "unit": "Tlimb-MAC/s",
                        "kernel": "trailing update k_items_hot<ItemTrailing2> (ldlt.cpp:122-129)",
                        "peak_how": "hk_peak_imad: register-only IMAD.WIDE carry-chain microkernel, best of 5 "
                                    "(MEASURED_PEAKS.json has no integer peak)"}
        roofline.update({
            "achieved": achieved, "peak": peak, "frac": achieved / peak, "traffic": None,
            "per_launch": f"{int(steps_k)} launches per step (one per LDLT step i with columns >= i+2), "
                          f"avg {ms_k / steps_k:.4f} ms, {bulk_macs / steps_k:.3e} algorithmic limb-MACs",
            "algorithmic_units": "L^2 limb-MACs per MP-FMA (SURVEY 8d); the tensor-core kernel forms the short "
                                 "product (byte columns >= limb L-8, ~half of L^2), so frac can exceed the MMA "
                                 "utilisation (up to ~2x)",
            "how_timed": ("event-record nodes in the captured LDLT graph around each step's product launches, "
                          "summed over the step and averaged over the timed steps") if kprof_timed else
                         ("event-record nodes around each step's product launches, in one instrumented step "
                          "after the timed region (short launches: the nodes would perturb the timed chain)"),
            "share_of_ldlt": ms_k / ldlt_ms if ldlt_ms > 0 else None,
            "kernel_ms_per_step": kt,
        })
        if 0 < kt.get("round_ms", 0.0) < 0.02 * ms_k:  # fused rounding: only the rare exact redos are left
            roofline["exact_redo"] = {"kernel": "k_tc_fix (items the fused certificate left to the exact FMA)",
                                      "ms": kt["round_ms"]}
        elif kt.get("round_ms", 0.0) > 0:
            round_bytes = sum((n - i - 2) * (n - i - 1) // 2 for i in range(n)) * (12 * L + 32)
            gbps = round_bytes / (kt["round_ms"] * 1e-3) / 1e9
            roofline["rounding_pass"] = {"kernel": "k_cols<ItemTcRound> + k_tc_fix", "ms": kt["round_ms"],
                                         "bound": "hbm", "achieved_GBps": gbps, "peak_GBps": hbm_peak_gbps(),
                                         "frac": gbps / hbm_peak_gbps(),
                                         "bytes": "12 L + 32 per MP-FMA (read c, read product, write c)"}
        if os.path.exists(ncu_file):
            roofline["traffic"] = json.load(open(ncu_file)).get("dram_bytes_per_launch")

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None,
        "dtype": f"mp{p} (p-bit binary float, 32-bit limbs, RNE; integer limb arithmetic)",
        "data": "exact-integer moments (deterministic, no dataset)",
        "config": workload_config(args, cfg, world),
        "time_to_lambda_ms": ms,
        "lambda_min": repr(lam[0][0] + lam[1][0]) if rank == 0 else None,
        "parity": lambda_parity(args.config, cfg, lam) if rank == 0 else None,
        "e2e": {"value": fmas(n) / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                "includes": "host moment generation (hk_moments into pinned memory) + hk_compute"},
        "e2e_device_moments": None if gen_ms is None else {
            "value": fmas(n) / (gen_ms * 1e-3), "unit": UNIT, "ms_per_step": gen_ms, "h2d_bytes_per_step": 0,
            "moments_ms": gen_moments_ms,
            "includes": "hk_compute_generated: moments built on the device (k_moments_fact), path, D2H of the "
                        "block + lambdas; same lambdas as e2e"},
        "roofline": roofline,
        "gpu_launches": launches,
        "clocks": sampler.summary(),
    }
    if world > 1:
        line["comm"] = {"broadcast_ms_per_step_rank0": kt.get("comm_ms"), "broadcasts": kt.get("comm_steps"),
                        "what": "device time of this rank's pivot-column ncclBroadcasts incl. the wait for their "
                                "root (WorkerTimings::comm_s, ldlt.cpp:214-263)"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cores = os.cpu_count() or 1
            n_s = CPU_SAMPLE_N[args.config]
            rec = run_reference_once(cfg, cores, cfg["K_equiv"], n=n_s)
            line["cpu_baseline"] = {
                "value": fmas(n_s) / rec["timing"]["wall_s"], "unit": UNIT, "cores": cores, "kind": "reference",
                "sample": f"1 hankel::compute of the reference (oracle/_ref, K={cfg['K_equiv']} = K_equiv, "
                          f"workers={cores}) on the leading N={n_s} block of {args.config}'s H_N (bounded sample; "
                          f"`--impl reference` times the whole workload): wall_s {rec['timing']['wall_s']:.3f}, "
                          f"ldlt_s {rec['timing']['ldlt_s']:.3f}"}
        except Exception as e:  # the baseline is reported, not required
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0:
        emit(line)
    ctx.close()
    if torch.distributed.is_initialized():
        torch.distributed.destroy_process_group()
    return 0


def relaunch_distributed(n):
    """`bench.py --gpus N` outside torchrun: one rank per GPU via torch.distributed.run."""
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, stdout=_OUT)  # the children inherit the real stdout


_OUT = None  # the process's real stdout (main() points fd 1 at stderr for everything else)


def emit(line):
    out = _OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    # stdout carries exactly ONE line, the JSON: whatever a library prints there (NCCL's version
    # banner appears under torchrun even with NCCL_DEBUG unset) is sent to stderr
    global _OUT
    if _OUT is None:
        sys.stdout.flush()
        _OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c4")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="use the NCCL column-sharded path even on 1 GPU")
    ap.add_argument("--ref-budget-s", type=float, default=300.0,
                    help="reference arm: wall-clock budget for its full runs (at least one runs)")
    ap.add_argument("--ref-golden-precision", action="store_true",
                    help="reference arm: also time one full run at the golden runs' K (K_ref)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_distributed(args.gpus)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return bench_reference(args, cfg)
    return bench_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
