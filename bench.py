#!/usr/bin/env python
"""Benchmark of the B200 m-Cubes VEGAS iteration (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One "step" = one full adjusting m-Cubes iteration -- V-Sample (K1, with its
exact cross-block sum into the exchange words), [the all-reduce across
ranks], rounding, grid adaptation, weighted estimate and convergence gate --
of 8D Genz f4 (Gaussian) at maxcalls = 1e9: m = 12^8 = 429,981,696 sub-cubes,
p = 2, so 8.6e8 integrand evaluations per step (BASELINE config 2's largest
8D shape).  The grid starts uniform and adapts every step (warm-up steps
included), on both arms.  value = evals/s over the whole job, device-timed
with CUDA events, max over ranks; L2 is flushed (256 MiB write) between timed
steps.  Secondary GPU-only line: the same step at maxcalls 1e10 (m = 2^32).

Under torchrun (N > 1) there is one process per GPU; rank r samples its slice
of the linear work index and the exact exchange buffer is all-reduced over
NCCL before every rank finishes the iteration identically.

--impl reference runs the SAME workload through the reference CPU library
(oracle/_ref/libmcubes_ref.so: the unmodified /root/reference headers
compiled in place): v_sample + Grid::adjusted + weighted_estimate per step
(driver.hpp:231-252) on the evolving grid, all host threads, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "integrand evals/sec (m-Cubes adjusting iteration, 8D Genz f4)"
UNIT = "evals/s"
DIMS = 8
FAMILY = 4
MAXCALLS = 10 ** 9
MAXCALLS_LARGE = 10 ** 10  # secondary GPU-only line: m = 16^8 = 2^32 cubes
N_BINS = 50
ALPHA = 1.5
# Algorithmic FP64 ops per eval (SURVEY.md 8d convention: +-*/ = 1, exp = 20):
# map 10d + accumulate (9 + 1 + bin_axes) + integrand f4 (3d + 21).
OPS_PER_EVAL = 10 * DIMS + (9 + 1 + DIMS) + (3 * DIMS + 21)  # = 143 for d = 8
FP64_LANES_PER_SM = 64
RNG_DESC = {
    "philox": "philox (north-star Philox4x32-10 keyed by (seed, iteration), counter (cube, sample, axis block); "
              "FMA transform; statistically equivalent to the reference, bitwise equal to its C twin)",
    "compat": "compat (the reference's keyed SplitMix stream and arithmetic order; bitwise equal to the reference)",
    "reference": "the reference's keyed SplitMix stream (rng.hpp), its own code",
}
BINS_DESC = {
    "r24": "estimate/variance exact (superaccumulator); bins: (f J)^2 rounded to 24 significant bits, then "
           "summed exactly (deterministic, geometry- and GPU-count-independent)",
    "exact": "exact (superaccumulator): estimate, variance and bins, as the reference's ExactSum/ExactBins",
}
DATA = {
    "philox": "synthetic (counter-based Philox stream; no input data)",
    "compat": "synthetic (keyed SplitMix stream of the reference; no input data)",
    "reference": "synthetic (keyed SplitMix stream of the reference; no input data)",
}


def workload(maxcalls: int, m: int, p: int) -> dict:
    """The `config` both arms report -- the workload only (implementation
    details go to top-level keys), so the two lines describe the same job."""
    return {"workload": "8D Genz f4 (Gaussian): one adjusting m-Cubes iteration per step (V-Sample, exact "
                        "reductions, grid adaptation, weighted estimate); grid uniform at step 1, adapted every step",
            "integrand": "f4", "dims": DIMS, "n_bins": N_BINS, "alpha": ALPHA, "maxcalls": maxcalls, "m": m, "p": p,
            "evals_per_step": m * p, "seed": 0,
            "l2": "GPU arm: flushed (256 MiB write) between timed steps; CPU arm: per-step working set "
                  "(m * p evaluations) far beyond the host caches"}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = []
        reasons = set()
        smax = None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                smax = float(r[1])
            except (ValueError, IndexError):
                continue
            for name, val in zip(names, r[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ reference arm
def ref_adjusting_steps(maxcalls: int, steps: int, warmup: int, threads: int, seed: int = 0):
    """The reference's own adjusting iteration, timed per step on `threads`
    host cores: v_sample, Grid::adjusted and weighted_estimate
    (driver.hpp:231-252) through oracle/_ref, on the evolving grid (uniform at
    step 1).  Returns (per-step seconds of the timed steps, m, p, result)."""
    import oracle as O

    lower, upper = [0.0] * DIMS, [1.0] * DIMS
    sp = (O._U64 * 4)()
    lib = O.ref()
    rc = lib.ref_setup(DIMS, N_BINS, maxcalls, 15, 10, 1e-3, ALPHA, 1.5, O.darr(lower), O.darr(upper), threads, sp)
    assert rc == 0, lib.ref_last_error()
    m, s, p = sp[1], sp[3], sp[2]
    edges = O.uniform_edges(DIMS, N_BINS, lower, upper)
    he, hv, times = [], [], []
    est = (0.0, 0.0, 0.0)
    for it in range(1, warmup + steps + 1):
        t0 = time.perf_counter()
        r = O.v_sample("ref", FAMILY, None, DIMS, N_BINS, lower, upper, edges, m, s, p, seed, it, "all", threads)
        edges = O.grid_adjust("ref", DIMS, N_BINS, lower, upper, edges, r["contrib"], ALPHA)
        he.append(r["est"])
        hv.append(r["var"])
        est = O.weighted_estimate(he, hv)
        dt = time.perf_counter() - t0
        if it > warmup:
            times.append(dt)
    return times, m, p, {"estimate": est[0], "sigma": est[1], "chi2_dof": est[2]}


def run_reference(args, rank):
    if rank != 0:
        return 0
    import oracle as O

    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libmcubes_ref.so not built"}))
        return 0
    threads = os.cpu_count() or 1
    times, m, p, res = ref_adjusting_steps(args.maxcalls, args.steps, args.warmup, threads)
    total = sum(times)
    rate = m * p * len(times) / total
    sample = (f"the full workload every step: reference v_sample + Grid::adjusted + weighted_estimate "
              f"(oracle/_ref, compiled from /root/reference headers) at maxcalls={args.maxcalls:.0e} "
              f"(m={m}, p={p}: {m * p} evals/step), {threads} threads, {args.warmup} untimed + "
              f"{args.steps} timed steps, {total:.1f} s timed")
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": DATA["reference"], "config": workload(args.maxcalls, m, p),
        "rng": RNG_DESC["reference"], "bins": "exact", "parallelism": f"{threads} host threads",
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "result": res,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_2202_01753_b200 as M

    gpu = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    # a dedicated (non-default) stream: the library, the CUDA events, the L2
    # flush and NCCL all order on it
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    dist = None
    import torch.distributed as dist_mod
    if dist_mod.is_available() and dist_mod.is_initialized():  # N > 1, or MCB_FORCE_DIST=1 at N = 1
        dist = dist_mod

    ctx = M.Context(gpu)
    ctx.set_stream(stream.cuda_stream)
    f = M.make_suite_integrand(FAMILY, DIMS)
    # --transport peer (N > 1): K1 writes every rank's exchange buffer over
    # peer memory and no collective runs in the step (one PeerExchange per run)
    peer = dist is not None and args.transport == "peer"
    # --transport compact (N > 1): every rank rounds its slice, the ranks
    # all-gather d x n_bins + 6 doubles and sum them in rank order (dist.py)
    compact = dist is not None and args.transport == "compact"
    cbufs = {}
    exchanges = []
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def make_run(maxcalls, rng, bins, its, seed):
        cfg = M.RunConfig(dims=DIMS, n_bins=N_BINS, maxcalls=maxcalls, itmax=its, ita=its, tau_rel=1e-15,
                          alpha=ALPHA, seed=seed, lower=[0.0] * DIMS, upper=[1.0] * DIMS, rng=rng, bins=bins)
        run = M.Run(f, cfg, ctx)
        xbuf = torch.zeros(run.exchange_words(), dtype=torch.int64, device=dev)
        run.set_exchange(xbuf.data_ptr())
        if peer:
            from paper_2202_01753_b200.dist import PeerExchange
            torch.cuda.synchronize()
            px = PeerExchange(ctx, run.exchange_words())
            px.attach(run)
            exchanges.append(px)
        if compact:
            cl = run.compact_len()
            cbufs[id(run)] = (torch.zeros(cl, dtype=torch.float64, device=dev),
                              torch.zeros(world * cl, dtype=torch.float64, device=dev))
        m = run.work_items
        return run, xbuf, m, rank * m // world, (rank + 1) * m // world

    def exchange_finish(run, xbuf, it):
        """The step's exchange and finish: exact all-reduce (collective), none
        (peer: K1 already wrote every rank's buffer) or the compact all-gather."""
        if compact:
            from paper_2202_01753_b200.dist import all_gather_rank_major
            mine, every = cbufs[id(run)]
            run.round_local(it, mine.data_ptr())
            all_gather_rank_major(every, mine)
            run.combine(it, every.data_ptr(), world)
            run.finish_rounded(it)
            return
        if dist is not None and not peer:
            dist.all_reduce(xbuf)  # exact: integer digit sums (MCB_XWORDS words per accumulator)
        run.finish(it)

    def measure(maxcalls, rng, bins, steps, warmup, seed=0, clocks=None):
        """W warm-up + K timed adjusting steps of one run: the grid starts
        uniform and adapts every step.  Device-timed with CUDA events (whole
        step, and K1 alone for the roofline), max over ranks."""
        run, xbuf, m, n0, n1 = make_run(maxcalls, rng, bins, warmup + steps, seed)

        def step(it, k1_events=None):
            if k1_events:
                k1_events[0].record(stream)
            run.sample(it, n0, n1)
            if k1_events:
                k1_events[1].record(stream)
            run.reduce(it)
            exchange_finish(run, xbuf, it)

        for it in range(1, warmup + 1):
            step(it)
            flush.zero_()
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        if clocks:
            clocks.start()
            time.sleep(0.3)
        launches0 = ctx.launches
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        k1 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        for i in range(steps):
            ev[i][0].record(stream)
            step(warmup + 1 + i, k1[i])
            ev[i][1].record(stream)
            flush.zero_()  # L2 flush between timed steps (outside the events)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        launches = ctx.launches - launches0
        clk = clocks.stop() if clocks else None
        step_ms = [a.elapsed_time(b) for a, b in ev]
        k1_ms = [a.elapsed_time(b) for a, b in k1]
        total_ms = max_over_ranks(sum(step_ms))
        res = run.result()
        assert res.iterations_used == warmup + steps and np.isfinite(res.estimate), res
        run.close()
        p = res.params.p
        k1_s = 1e-3 * statistics.mean(k1_ms)
        return {"value": m * p * steps / (total_ms * 1e-3), "ms_per_step": total_ms / steps, "m": m, "p": p,
                "k1_s": k1_s, "k1_evals": (n1 - n0) * p, "share": 1e3 * k1_s * steps / sum(step_ms),
                "launches": launches, "clocks": clk, "result": res}

    # ---- the headline: device-timed steps with inputs resident in HBM
    clocks = ClockSampler(gpu) if rank == 0 else None
    bins = args.bins if args.rng == "philox" else ""  # compat always sums exact bins
    head = measure(args.maxcalls, args.rng, bins, args.steps, args.warmup, clocks=clocks)
    m, p = head["m"], head["p"]
    res = head["result"]

    # ---- end to end through the C ABI with host buffers (H2D grid in, D2H adapted grid out)
    run2, xbuf2, _, n0, n1 = make_run(args.maxcalls, args.rng, bins, args.warmup + args.steps, 1)
    host_edges = torch.empty(DIMS * N_BINS, dtype=torch.float64).pin_memory().numpy()
    host_edges[:] = np.asarray(M.Grid(DIMS, N_BINS, [0.0] * DIMS, [1.0] * DIMS).raw_edges)
    out_edges = torch.empty(DIMS * N_BINS, dtype=torch.float64).pin_memory().numpy()

    def e2e_step(it):
        run2.set_grid(host_edges)                # H2D: the step's input grid
        run2.sample(it, n0, n1)
        run2.reduce(it)
        exchange_finish(run2, xbuf2, it)
        run2.grid_into(out_edges)                # D2H: adapted grid (synchronises)
        host_edges[:] = out_edges                # the next step samples on it

    for it in range(1, args.warmup + 1):
        e2e_step(it)
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        e2e_step(args.warmup + 1 + i)
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    run2.result()
    run2.close()
    e2e_value = m * p * args.steps / e2e_s

    # ---- roofline of the dominant kernel (K1 vsample_kernel)
    achieved_tflops = OPS_PER_EVAL * head["k1_evals"] / head["k1_s"] / 1e12
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    sm_max = (head["clocks"] or {}).get("sm_max_mhz") or 1965.0
    peak_tflops = sms * FP64_LANES_PER_SM * sm_max * 1e6 / 1e12
    stream_key = args.rng if args.rng == "compat" else f"philox_{args.bins}"
    traffic, winst_per_eval, ncu_src = None, None, None
    tf_path = os.path.join(HERE, "profiles", "k1_traffic.json")
    if os.path.exists(tf_path):
        try:
            ent = json.load(open(tf_path)).get(stream_key) or {}
            traffic, winst_per_eval, ncu_src = (ent.get("bytes_per_launch"), ent.get("warp_instr_per_eval"),
                                                ent.get("source"))
        except (OSError, ValueError):
            pass
    issue = None
    if winst_per_eval:
        # the instruction-issue roofline: 4 warp schedulers per SM, one issue each per clock;
        # warp instructions per eval from the ncu capture (smsp__inst_executed.sum / evals)
        ach = head["k1_evals"] * winst_per_eval / head["k1_s"] / 1e9
        pk = sms * 4 * sm_max * 1e6 / 1e9
        issue = {"achieved": ach, "peak": pk, "unit": "G warp-instructions/s", "frac": ach / pk,
                 "warp_instr_per_eval": winst_per_eval, "source": ncu_src}

    line = {
        "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": DATA[args.rng],
        "config": workload(args.maxcalls, m, p),
        "rng": RNG_DESC[args.rng], "bins": args.bins if args.rng == "philox" else "exact",
        "reductions": BINS_DESC[args.bins if args.rng == "philox" else "exact"],
        "parallelism": ((f"cube-range partition x{world} + " +
                         ("exact exchange over peer memory inside K1" if peer
                          else f"compact all-gather of rounded partials ({dist.get_backend()})" if compact
                          else f"exact all-reduce ({dist.get_backend()})")) if world > 1 else "single GPU"),
        "clocks": head["clocks"],
        "gpu_launches": head["launches"],
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * DIMS * N_BINS,
                "d2h_bytes_per_step": 8 * DIMS * N_BINS,
                "path": "C ABI mcb_run_set_grid/sample/reduce/finish/grid (host grid in, adapted host grid out, "
                        "every step)"},
        "roofline": {"bound": "fp64", "achieved": achieved_tflops, "peak": peak_tflops, "unit": "TFLOP/s",
                     "frac": achieved_tflops / peak_tflops, "traffic": traffic, "issue": issue,
                     "kernel": f"vsample_kernel<F4,8,{stream_key}>", "kernel_ms": 1e3 * head["k1_s"],
                     "ops_per_eval": OPS_PER_EVAL,
                     "peak_source": f"FP64 issue: {sms} SMs x {FP64_LANES_PER_SM} lanes x {sm_max:.0f} MHz "
                                    "(MEASURED_PEAKS.json has no FP64 figure; profiles/microbench_r01.txt "
                                    "measures 1.75e13 DADD/s)",
                     "share_of_step": head["share"]},
        "result": {"estimate": res.estimate, "sigma": res.sigma, "chi2_dof": res.chi2_dof, "truth": f.reference,
                   "samples": res.total_samples, "bin_writes": res.bin_writes},
    }

    def secondary(maxcalls, rng, bins, steps, desc):
        r = measure(maxcalls, rng, bins, steps, args.warmup)
        ach = OPS_PER_EVAL * r["k1_evals"] / r["k1_s"] / 1e12
        return {"value": r["value"], "unit": UNIT, "maxcalls": maxcalls, "m": r["m"], "p": r["p"], "rng": rng,
                "bins": bins or "exact", "what": desc, "kernel_ms": 1e3 * r["k1_s"], "roofline_achieved": ach,
                "roofline_frac": ach / peak_tflops,
                "result": {"estimate": r["result"].estimate, "sigma": r["result"].sigma}}

    if not args.no_secondary:
        if args.rng == "philox" and args.bins == "r24":
            line["philox_exact_bins"] = secondary(args.maxcalls, "philox", "exact", args.steps,
                                                  "the same steps with exact bins (the reference's ExactBins "
                                                  "precision)")
        if args.rng == "philox":
            line["compat"] = secondary(args.maxcalls, "compat", "", args.steps,
                                       "the same steps on the reference's own stream and arithmetic order "
                                       "(bitwise the reference)")
        line["maxcalls_1e10"] = secondary(MAXCALLS_LARGE, args.rng, bins, min(args.steps, 5),
                                          "GPU-only: 8D f4 at maxcalls 1e10 (m = 16^8 = 2^32 sub-cubes)")

    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args.maxcalls)
        line["time_to_epsrel"] = time_to_epsrel(M, ctx)
    elif world > 1 and not args.no_cpu:
        tte = time_to_epsrel_dist(M, ctx, dist, dev, rank, args.transport)
        if rank == 0:
            line["time_to_epsrel"] = tte
    if not args.no_cpu:
        tte = time_to_epsrel_headline(M, ctx, dist if world > 1 else None, dev, rank, world, args,
                                      with_cpu=rank == 0 and world == 1)
        if rank == 0:
            line["time_to_epsrel_headline"] = tte
    if rank == 0:
        print(json.dumps(line), flush=True)
    torch.cuda.synchronize()
    for px in exchanges:  # collective: every rank unmaps, then frees
        px.close()
    return 0


def cpu_baseline(maxcalls):
    """The reference's own adjusting iteration at the bench workload, timed on
    all host cores: one untimed step, then two timed (~10-20 s of CPU work)."""
    import oracle as O

    if not O.ref_available():
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": "oracle/_ref not built"}
    threads = os.cpu_count() or 1
    times, m, p, _ = ref_adjusting_steps(maxcalls, 2, 1, threads, seed=7)
    total = sum(times)
    return {"value": m * p * len(times) / total, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"the same workload: 2 timed reference adjusting steps (v_sample + Grid::adjusted + "
                      f"weighted_estimate) of 8D f4 at maxcalls={maxcalls:.0e} (m={m}, p={p}) after 1 untimed, "
                      f"{threads} threads, {total:.2f} s"}


def time_to_epsrel(M, ctx, runs: int = 2, cpu_budget_s: float = 120.0):
    """Time-to-target-relative-error, BASELINE config 2: the 8D suite f1..f6,
    the reference tool's sweep schedule (tools/mcubes_bench.cpp:145-165:
    tau_rel from 1e-3, divided by 5 per level, `runs` seeds per level, stop
    tightening once fewer than half converge) with the acceptance protocol
    (maxcalls 1e7, itmax 30, ita 10, n_bins 50).  Per level: GPU integrate()
    on both streams and the reference integrate() on all host cores, same
    seeds; the compat stream reaches the reference's estimates bit for bit
    (+-*/ integrands) or to the libdevice ulp (the others).  The CPU legs stop
    once they have used cpu_budget_s."""
    import oracle as O
    import torch

    d, maxcalls, itmax, ita = 8, 10 ** 7, 30, 10
    threads = os.cpu_count() or 1
    have_cpu = O.ref_available()
    cpu_used = 0.0

    def cfg(seed, tau, rng):
        return M.RunConfig(dims=d, maxcalls=maxcalls, itmax=itmax, ita=ita, tau_rel=tau, seed=seed,
                           lower=[0.0] * d, upper=[1.0] * d, rng=rng)

    def gpu(f, seed, tau, rng):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = M.integrate(f, cfg(seed, tau, rng), ctx=ctx)
        return r, 1e3 * (time.perf_counter() - t0)

    rows = []
    for fam in range(1, 7):
        f = M.make_suite_integrand(fam, d)
        gpu(f, 1, 1e-3, "compat")  # warm (loads this integrand's kernels)
        gpu(f, 1, 1e-3, "philox")
        tau, level = 1e-3, 0
        live = {"compat": True, "philox": True, "cpu": have_cpu}
        while any(live.values()) and tau >= 1e-9:
            seeds = [1 + level * runs + i for i in range(runs)]
            row = {"integrand": f"f{fam}", "tau_rel": tau, "seeds": seeds}
            for rng in ("compat", "philox"):
                if not live[rng]:
                    continue
                rr = [gpu(f, sd, tau, rng) for sd in seeds]
                conv = sum(r.converged for r, _ in rr)
                row[f"gpu_{rng}"] = {"median_ms": statistics.median(ms for _, ms in rr), "converged": conv,
                                     "iterations": [r.iterations_used for r, _ in rr],
                                     "estimates": [r.estimate for r, _ in rr], "sigmas": [r.sigma for r, _ in rr]}
                live[rng] = conv * 2 >= runs
            if live["cpu"] and cpu_used < cpu_budget_s:
                cr = []
                for sd in seeds:
                    t0 = time.perf_counter()
                    o = O.integrate("ref", fam, None, d, 50, maxcalls, itmax, ita, tau, 1.5, 1.5, sd, 0,
                                    [0.0] * d, [1.0] * d, workers=threads)
                    cr.append((o, 1e3 * (time.perf_counter() - t0)))
                cpu_used += sum(ms for _, ms in cr) / 1e3
                conv = sum(o["converged"] for o, _ in cr)
                row["cpu_reference"] = {"median_ms": statistics.median(ms for _, ms in cr), "converged": conv,
                                        "iterations": [o["iterations_used"] for o, _ in cr],
                                        "estimates": [o["estimate"] for o, _ in cr],
                                        "sigmas": [o["sigma"] for o, _ in cr], "threads": threads}
                live["cpu"] = conv * 2 >= runs
                if "gpu_compat" in row:
                    g = row["gpu_compat"]
                    row["compat_same_iterations"] = g["iterations"] == row["cpu_reference"]["iterations"]
                    row["compat_estimates_bitwise"] = g["estimates"] == row["cpu_reference"]["estimates"]
                    row["speedup_compat"] = row["cpu_reference"]["median_ms"] / g["median_ms"]
                if "gpu_philox" in row:
                    g = row["gpu_philox"]
                    row["philox_within_3_combined_sigma"] = all(
                        abs(a - b) <= 3 * math.hypot(sa, sb) for a, b, sa, sb in
                        zip(g["estimates"], row["cpu_reference"]["estimates"], g["sigmas"],
                            row["cpu_reference"]["sigmas"]))
                    row["speedup_philox"] = row["cpu_reference"]["median_ms"] / g["median_ms"]
            elif live["cpu"]:
                row["cpu_reference"] = "skipped: CPU budget spent"
                live["cpu"] = False
            rows.append(row)
            tau /= 5.0
            level += 1
    return {"protocol": f"8D f1..f6, maxcalls 1e7, itmax 30, ita 10; tau 1e-3 / 5^k, {runs} seeds per level, "
                        "a stream stops tightening once < 50% converge (mcubes_bench.cpp:145-165)",
            "cpu_threads": threads, "cpu_seconds": cpu_used, "levels": rows}


def time_to_epsrel_headline(M, ctx, dist, dev, rank, world, args, with_cpu):
    """time_to_epsrel at the headline size, where GPUs matter: 8D f4 at the
    bench's maxcalls (1e9: 8.6e8 evals per iteration) to tau_rel 3e-5, on
    this launch's GPUs (dist.integrate over the ranks for N > 1, wall time
    max over ranks), both streams; at N = 1 also the reference CPU integrate
    on the host cores (same schedule and seed; its stream is compat's)."""
    import torch

    import oracle as O
    from paper_2202_01753_b200 import dist as mdist

    d, tau, itmax, ita, seed = DIMS, 3e-5, 8, 6, 1  # bounded: <= 8 reference iterations of ~4.6 s
    out = {"protocol": f"8D f4, maxcalls {args.maxcalls:.0e}, tau_rel {tau:g}, itmax {itmax}, ita {ita}, seed {seed}",
           "gpus": world}
    f = M.make_suite_integrand(FAMILY, d)
    for rng, bins in (("philox", "r24"), ("compat", "")):
        cfg = M.RunConfig(dims=d, maxcalls=args.maxcalls, itmax=itmax, ita=ita, tau_rel=tau, seed=seed,
                          lower=[0.0] * d, upper=[1.0] * d, rng=rng, bins=bins)
        run = (lambda: mdist.integrate(f, cfg, ctx=ctx, transport=args.transport)) if dist is not None else \
            (lambda: M.integrate(f, cfg, ctx=ctx))
        run()  # warm
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        r = run()
        ms = 1e3 * (time.perf_counter() - t0)
        if dist is not None:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        out[f"gpu_{rng}"] = {"ms": ms, "iterations": r.iterations_used, "converged": r.converged,
                             "estimate": r.estimate, "sigma": r.sigma, "chi2_dof": r.chi2_dof}
    if with_cpu and O.ref_available():
        threads = os.cpu_count() or 1
        t0 = time.perf_counter()
        o = O.integrate("ref", FAMILY, None, d, N_BINS, args.maxcalls, itmax, ita, tau, ALPHA, 1.5, seed, 0,
                        [0.0] * d, [1.0] * d, workers=threads)
        cms = 1e3 * (time.perf_counter() - t0)
        out["cpu_reference"] = {"ms": cms, "iterations": o["iterations_used"], "converged": o["converged"],
                                "estimate": o["estimate"], "sigma": o["sigma"], "threads": threads}
        out["speedup_compat"] = cms / out["gpu_compat"]["ms"]
        out["speedup_philox"] = cms / out["gpu_philox"]["ms"]
        out["compat_same_iterations"] = o["iterations_used"] == out["gpu_compat"]["iterations"]
    return out


def time_to_epsrel_dist(M, ctx, dist, dev, rank, transport="collective"):
    """time_to_epsrel at N GPUs: paper_2202_01753_b200.dist.integrate (cube
    ranges per rank, exact all-reduce per iteration), wall time max over ranks;
    the reference CPU integrate is timed on rank 0's host cores."""
    import torch

    import oracle as O
    from paper_2202_01753_b200 import dist as mdist

    d, maxcalls, tau = 8, 10 ** 7, 1e-3
    cfg = M.RunConfig(dims=d, maxcalls=maxcalls, itmax=30, ita=10, tau_rel=tau, seed=1, lower=[0.0] * d,
                      upper=[1.0] * d)
    f = M.make_suite_integrand(5, d)
    mdist.integrate(f, cfg, ctx=ctx, transport=transport)  # warm
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    r = mdist.integrate(f, cfg, ctx=ctx, transport=transport)
    ms = 1e3 * (time.perf_counter() - t0)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out = {"integrand": "f5", "dims": d, "maxcalls": maxcalls, "tau_rel": tau, "itmax": 30, "ita": 10, "seed": 1,
           "gpu_ms": float(t.item()), "gpu_iterations": r.iterations_used, "gpu_converged": r.converged,
           "gpu_estimate": r.estimate, "gpu_sigma": r.sigma, "path": "dist.integrate over all ranks"}
    if rank == 0 and O.ref_available():
        threads = os.cpu_count() or 1
        t0 = time.perf_counter()
        o = O.integrate("ref", 5, None, d, 50, maxcalls, 30, 10, tau, 1.5, 1.5, 1, 0, [0.0] * d, [1.0] * d,
                        workers=threads)
        out.update(cpu_ms=1e3 * (time.perf_counter() - t0), cpu_iterations=o["iterations_used"],
                   cpu_converged=o["converged"], cpu_estimate=o["estimate"], cpu_sigma=o["sigma"],
                   cpu_threads=threads)
    dist.barrier()
    return out


def run_suite(path: str):
    """BASELINE.json configs 1-5 beside the reference CPU library (oracle/_ref,
    all host threads), one JSON line per measurement, written to `path`.
    Bounded: CPU legs stop at 1e8-1e9 evals."""
    import numpy as np
    import torch

    import oracle as O
    import paper_2202_01753_b200 as M

    ctx = M.Context(0)
    threads = os.cpu_count() or 1
    out = open(path, "w")

    def emit(d):
        line = json.dumps(d, default=lambda x: x.item() if hasattr(x, "item") else str(x))
        out.write(line + "\n")
        out.flush()
        log(line[:300])

    def gpu_run(f, cfg, reps=3):
        M.integrate(f, cfg, ctx=ctx)
        if cfg.maxcalls >= 10 ** 10:
            reps = 1  # seconds per run already; the warm-up above loaded everything
        best, r = 1e30, None
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = M.integrate(f, cfg, ctx=ctx)
            best = min(best, time.perf_counter() - t0)
        return r, 1e3 * best

    def cpu_run(fid, params, d, mc, itmax, ita, tau, seed, lo, hi):
        t0 = time.perf_counter()
        o = O.integrate("ref", fid, params, d, 50, mc, itmax, ita, tau, 1.5, 1.5, seed, 0, lo, hi, workers=threads)
        return o, 1e3 * (time.perf_counter() - t0)

    def both(config, name, f, fid, params, d, mc, itmax, ita, tau, seed=1, lo=None, hi=None, cpu=True):
        lo = lo or [0.0] * d
        hi = hi or [1.0] * d
        cfg = M.RunConfig(dims=d, maxcalls=mc, itmax=itmax, ita=ita, tau_rel=tau, seed=seed, lower=lo, upper=hi)
        r, gms = gpu_run(f, cfg)
        cfgp = M.RunConfig(dims=d, maxcalls=mc, itmax=itmax, ita=ita, tau_rel=tau, seed=seed, lower=lo, upper=hi,
                           rng="philox")
        rp, pms = gpu_run(f, cfgp)
        row = dict(config=config, integrand=name, dims=d, maxcalls=mc, itmax=itmax, ita=ita, tau_rel=tau, seed=seed,
                   evals=r.total_samples, gpu_ms=gms, gpu_evals_per_s=r.total_samples / (gms * 1e-3),
                   gpu_iterations=r.iterations_used, gpu_converged=r.converged, gpu_estimate=r.estimate,
                   gpu_sigma=r.sigma, gpu_chi2_dof=r.chi2_dof, truth=f.reference,
                   philox_ms=pms, philox_evals=rp.total_samples, philox_evals_per_s=rp.total_samples / (pms * 1e-3),
                   philox_iterations=rp.iterations_used, philox_converged=rp.converged, philox_estimate=rp.estimate,
                   philox_sigma=rp.sigma, philox_chi2_dof=rp.chi2_dof)
        if f.reference is not None and rp.sigma > 0:
            row["philox_pull_vs_truth"] = (rp.estimate - f.reference) / rp.sigma
        if cpu:
            o, cms = cpu_run(fid, params, d, mc, itmax, ita, tau, seed, lo, hi)
            row.update(cpu_ms=cms, cpu_threads=threads, cpu_iterations=o["iterations_used"],
                       cpu_converged=o["converged"], cpu_estimate=o["estimate"], cpu_sigma=o["sigma"],
                       speedup=cms / gms, same_iterations=o["iterations_used"] == r.iterations_used,
                       same_convergence=o["converged"] == r.converged,
                       estimate_bitwise_equal=o["estimate"] == r.estimate,
                       within_3_combined_sigma=abs(o["estimate"] - r.estimate) <= 3 * math.hypot(o["sigma"], r.sigma),
                       philox_speedup=cms / pms,
                       philox_within_3_combined_sigma=abs(o["estimate"] - rp.estimate)
                       <= 3 * math.hypot(o["sigma"], rp.sigma))
        emit(row)

    # C1: 5D f4, ncall 1e6, 10 iterations (the reference's CPU-runnable case)
    both("C1", "f4", M.make_suite_integrand(4, 5), 4, None, 5, 10 ** 6, 10, 10, 1e-9, seed=0)
    # C2: the 8D suite, time-to-epsrel at tau 1e-3 and 2e-4 (itmax 30, ita 10)
    for fam in range(1, 7):
        for tau in (1e-3, 2e-4):
            both("C2", f"f{fam}", M.make_suite_integrand(fam, 8), fam, None, 8, 10 ** 7, 30, 10, tau)
    for fam in (3, 5):  # GPU-only deeper tolerances at 1e9 evals/iteration
        for tau in (4e-5, 8e-6, 1.6e-6):
            both("C2", f"f{fam}", M.make_suite_integrand(fam, 8), fam, None, 8, 10 ** 9, 30, 10, tau, cpu=False)
    # C3: 6D f4 at 1e9 evals/iteration (3 iterations on both sides)
    both("C3", "f4", M.make_suite_integrand(4, 6), 4, None, 6, 10 ** 9, 3, 3, 1e-12)
    # C4: 6D table integrand (device-resident interpolation tables, CPU twin on the host)
    d, n = 6, 4096
    t = np.linspace(0, 1, n)
    rng = np.random.default_rng(0)
    tabs = np.array([0.2 + np.exp(-0.5 * ((t - rng.uniform(0.3, 0.7)) / rng.uniform(0.05, 0.2)) ** 2)
                     for _ in range(d)])
    ft = M.make_table_integrand(tabs, [0.0] * d, [1.0] * d)
    both("C4", "table6d", ft, 9, ft.params, d, 10 ** 8, 10, 10, 1e-12)
    both("C4", "table6d", ft, 9, ft.params, d, 10 ** 10, 3, 3, 1e-12, cpu=False)
    # C5: dims x ncall scaling (itmax 5, ita 3); CPU legs up to 1e8
    for dd in (2, 4, 6, 8, 10):
        for mc in (10 ** 6, 10 ** 8, 10 ** 10):
            both("C5", "f4", M.make_suite_integrand(4, dd), 4, None, dd, mc, 5, 3, 1e-15, cpu=mc <= 10 ** 8)
    for dd in (2, 6, 8):  # the top of the ncall range, GPU only
        both("C5", "f4", M.make_suite_integrand(4, dd), 4, None, dd, 10 ** 11, 3, 2, 1e-15, cpu=False)
    out.close()


def run_scale(args):
    """bench_cli scale (GPU columns, at this launch's GPU count) with the
    reference CPU adjusting iteration -- v_sample + Grid::adjusted through
    oracle/_ref on all host threads -- timed beside each cell (rank 0)."""
    import types

    import oracle as O
    from paper_2202_01753_b200 import bench_cli

    threads = os.cpu_count() or 1

    def cpu_timer(integrand, d, maxcalls):
        if not O.ref_available() or integrand not in {f"f{i}" for i in range(1, 7)}:
            return None
        fam = int(integrand[1])
        lo, hi = [0.0] * d, [1.0] * d
        sp = (O._U64 * 4)()
        assert O.ref().ref_setup(d, N_BINS, maxcalls, 3, 3, 1e-3, ALPHA, 1.5, O.darr(lo), O.darr(hi), threads, sp) == 0
        edges = O.uniform_edges(d, N_BINS, lo, hi)
        t0 = time.perf_counter()
        r = O.v_sample("ref", fam, None, d, N_BINS, lo, hi, edges, sp[1], sp[3], sp[2], 0, 1, "all", threads)
        O.grid_adjust("ref", d, N_BINS, lo, hi, edges, r["contrib"], ALPHA)
        return threads, 1e3 * (time.perf_counter() - t0)

    o = types.SimpleNamespace(integrand=args.scale_integrand, dims=args.scale_dims, ncalls=args.scale_ncalls,
                              rng=args.rng, cpu_max_evals=args.scale_cpu_max_evals, out=args.scale)
    return bench_cli.cmd_scale(o, cpu_timer)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--maxcalls", type=int, default=MAXCALLS)
    ap.add_argument("--rng", choices=["philox", "compat"], default="philox",
                    help="philox = the north-star stream (headline); compat = the reference's stream, bit-exact")
    ap.add_argument("--bins", choices=["r24", "exact"], default="r24",
                    help="philox: contribution addends rounded to 24 significant bits (headline) or exact")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the secondary lines (exact bins, compat stream, maxcalls 1e10)")
    ap.add_argument("--transport", choices=["collective", "peer", "compact"], default="collective",
                    help="N > 1: exchange through an exact NCCL all-reduce (216 KB at 8D, results independent of "
                         "N), K1 writing every rank's buffer over peer memory (CUDA IPC over NVLink), or the compact "
                         "all-gather of each rank's rounded d*n_bins+6 doubles (3.2 KB per rank, N-dependent last "
                         "bits)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline / time_to_epsrel legs")
    ap.add_argument("--suite", default=None, help="run BASELINE configs 1-5 (GPU + reference CPU) into this JSONL")
    ap.add_argument("--scale", default=None,
                    help="BASELINE config 5: bench_cli's scale sweep at this launch's GPU count (torchrun for N > 1) "
                         "with the reference CPU iteration timed on the host cores beside each cell, CSV here")
    ap.add_argument("--scale-dims", default="2,4,6,8,10")
    ap.add_argument("--scale-ncalls", default="1e6,1e8,1e10")
    ap.add_argument("--scale-integrand", default="f4")
    ap.add_argument("--scale-cpu-max-evals", type=float, default=1e9)
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup < 3 is not allowed by the timing rules; using 3")
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank)
    if args.suite:
        return run_suite(args.suite)
    if args.scale:
        return run_scale(args)
    # MCB_FORCE_DIST=1 runs the multi-rank code path (process group, exchange
    # all-reduce, barriers, max over ranks) even at N = 1: on a one-GPU box
    # that is the only way to exercise NCCL itself (tests/test_gpu_bench_dist.py)
    use_dist = world > 1 or os.environ.get("MCB_FORCE_DIST") == "1"
    if use_dist:
        import torch
        import torch.distributed as dist

        gpu = local_rank % torch.cuda.device_count()
        torch.cuda.set_device(gpu)
        # NCCL over NVLink in production; MCB_DIST_BACKEND=gloo lets several
        # ranks share one GPU for testing the multi-rank path
        backend = os.environ.get("MCB_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
        else:
            dist.init_process_group(backend)
    try:
        return run_ours(args, rank, world, local_rank)
    finally:
        if use_dist:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
