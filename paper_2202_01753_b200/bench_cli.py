"""GPU-backed equivalent of the reference's benchmark CLI
(proj/tools/mcubes_bench.cpp): same subcommands, flags, CSV schema, exit codes.

    python -m paper_2202_01753_b200.bench_cli run --integrand f4 --dim 8 --maxcalls 100000000
    python -m paper_2202_01753_b200.bench_cli sweep --integrand f5 --dim 8 --runs 20 --out s.csv
    python -m paper_2202_01753_b200.bench_cli summarize s.csv
    python -m paper_2202_01753_b200.bench_cli scale --integrand f4 --dims 2,4,6,8,10 --ncalls 1e6,1e8,1e10

run:       one seeded integration, one CSV row; exit 0 converged, 2 not (mcubes_bench.cpp:135-143)
sweep:     --runs seeded runs per tolerance level; tau starts at --tau-rel and is
           divided by 5 while at least half converge, down to 1e-9; seeds
           seed + level*runs + i (mcubes_bench.cpp:145-165)
summarize: per-(integrand, dims, tau) run counts, convergence rate and R-7
           quartiles of rel_error over converged runs (mcubes_bench.cpp:192-244)
scale:     (B200 addition, BASELINE config 5) per (d, ncall) cell at the launch's
           GPU count (torchrun for N > 1): one adjusting iteration's device
           throughput, a whole-run wall time, and the reference CPU iteration
           on the host cores beside it (gpus, cpu_* columns).
Usage and I/O errors exit 1.
"""
from __future__ import annotations

import argparse
import csv
import io
import math
import sys
import time
from typing import Optional

from . import mcubes as M

CSV_HEADER = ("integrand,dims,tau_rel,run,seed,estimate,sigma,chi2_dof,converged,"
              "true_value,rel_error,iterations,total_samples,wall_ms")
SUMMARY_HEADER = ("integrand,dims,tau_rel,runs,converged,convergence_rate,"
                  "min_rel_error,q1_rel_error,median_rel_error,q3_rel_error,max_rel_error")


def fmt17(v: float) -> str:
    return "%.17g" % v


def _config(o, spec: M.IntegrandSpec, tau: float, seed: int) -> M.RunConfig:
    return M.RunConfig(dims=spec.dims, n_bins=o.n_bins, maxcalls=o.maxcalls, itmax=o.itmax, ita=o.ita,
                       tau_rel=tau, alpha=o.alpha, seed=seed, variant=M.parse_variant(o.variant),
                       lower=spec.lower, upper=spec.upper, workers=o.workers, rng=o.rng)


def _timed(spec, cfg, ctx):
    ctx.synchronize()
    t0 = time.perf_counter()
    r = M.integrate(spec, cfg, ctx=ctx)
    return r, 1e3 * (time.perf_counter() - t0)


def _row(spec, tau, run, seed, r, wall_ms) -> str:
    fields = [spec.name, str(spec.dims), fmt17(tau), str(run), str(seed), fmt17(r.estimate), fmt17(r.sigma),
              fmt17(r.chi2_dof), "1" if r.converged else "0"]
    if spec.reference is not None:
        truth = spec.reference
        fields += [fmt17(truth), fmt17(abs(r.estimate - truth) / abs(truth))]
    else:
        fields += ["", ""]
    fields += [str(r.iterations_used), str(r.total_samples), fmt17(wall_ms)]
    return ",".join(fields)


class _Out:
    def __init__(self, path: Optional[str]):
        self.fh = open(path, "w") if path else sys.stdout

    def write(self, line: str):
        self.fh.write(line + "\n")
        self.fh.flush()  # interrupted sweeps keep completed rows

    def close(self):
        if self.fh is not sys.stdout:
            self.fh.close()


def cmd_run(o) -> int:
    spec = M.make_integrand(o.integrand, o.dim)
    ctx = M.default_context()
    r, ms = _timed(spec, _config(o, spec, o.tau_rel, o.seed), ctx)
    out = _Out(o.out)
    out.write(CSV_HEADER)
    out.write(_row(spec, o.tau_rel, 0, o.seed, r, ms))
    out.close()
    return 0 if r.converged else 2


def cmd_sweep(o) -> int:
    spec = M.make_integrand(o.integrand, o.dim)
    ctx = M.default_context()
    out = _Out(o.out)
    out.write(CSV_HEADER)
    tau = o.tau_rel
    level = 0
    while True:
        converged = 0
        for i in range(o.runs):
            seed = o.seed + level * o.runs + i
            r, ms = _timed(spec, _config(o, spec, tau, seed), ctx)
            converged += 1 if r.converged else 0
            out.write(_row(spec, tau, i, seed, r, ms))
        if converged * 2 < o.runs:
            break
        tau /= 5.0
        if tau < 1e-9:
            break
        level += 1
    out.close()
    return 0


def quantile(sorted_vals, q):
    """R-7 quantile (mcubes_bench.cpp:192-200)."""
    if not sorted_vals:
        return math.nan
    h = q * (len(sorted_vals) - 1)
    lo = int(h)
    if lo + 1 >= len(sorted_vals):
        return sorted_vals[-1]
    return sorted_vals[lo] + (h - lo) * (sorted_vals[lo + 1] - sorted_vals[lo])


def cmd_summarize(path: str, out_path: Optional[str]) -> int:
    try:
        fh = open(path)
    except OSError:
        print(f'cannot open input file "{path}"', file=sys.stderr)
        return 1
    lines = fh.read().splitlines()
    if not lines or len(lines[0].split(",")) != 14:
        print("input is not a result CSV (bad header)", file=sys.stderr)
        return 1
    groups = {}
    for n, line in enumerate(lines[1:], start=2):
        if not line:
            continue
        f = line.split(",")
        if len(f) != 14:
            print(f"malformed row at line {n}", file=sys.stderr)
            return 1
        key = (f[0], int(f[1]), float(f[2]))
        g = groups.setdefault(key, [0, 0, []])
        g[0] += 1
        if f[8] == "1":
            g[1] += 1
            if f[10]:
                g[2].append(float(f[10]))
    out = _Out(out_path)
    out.write(SUMMARY_HEADER)
    for key in sorted(groups):
        runs, conv, errs = groups[key]
        errs.sort()
        q = ["" if not errs else fmt17(quantile(errs, x)) for x in (0.0, 0.25, 0.5, 0.75, 1.0)]
        out.write(",".join([key[0], str(key[1]), fmt17(key[2]), str(runs), str(conv), fmt17(conv / runs)] + q))
    out.close()
    return 0


def _scale_dist():
    """(world, rank, dist module or None): torchrun sets WORLD_SIZE/RANK; one
    process per GPU, NCCL (MCB_DIST_BACKEND=gloo lets ranks share a GPU)."""
    import os

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world == 1:
        return 1, 0, None
    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % torch.cuda.device_count())
    if not dist.is_initialized():
        backend = os.environ.get("MCB_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
        else:
            dist.init_process_group(backend)
    return world, dist.get_rank(), dist


def cmd_scale(o, cpu_timer=None) -> int:
    """BASELINE config 5: throughput over d x ncall at the launch's GPU count.

    Per cell: one adjusting iteration device-timed through the stepped run
    (each rank samples its slice of the cube walk, the exact exchange is
    all-reduced, max over ranks) and the wall time of a whole itmax=5/ita=3
    integrate (dist.integrate when gpus > 1).  Launch with torchrun for
    gpus > 1; rank 0 writes the CSV.  The cpu_* columns are filled when a
    caller passes `cpu_timer(integrand, dims, maxcalls) -> (threads, ms)`
    timing the reference CPU iteration on the host cores in the same run
    (bench.py --scale does, with the compiled reference); the library itself
    never runs a CPU path."""
    import torch

    world, rank, dist = _scale_dist()
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.Stream(dev)
    ctx = M.Context(dev.index)
    ctx.set_stream(stream.cuda_stream)
    if rank != 0:
        cpu_timer = None
    out = _Out(o.out) if rank == 0 else None
    if out:
        out.write("integrand,dims,maxcalls,g,m,p,gpus,evals_per_iteration,iteration_ms,evals_per_s,run5_wall_ms,"
                  "cpu_threads,cpu_iteration_ms,cpu_evals_per_s,speedup")

    def max_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for d in [int(x) for x in o.dims.split(",")]:
        for nc in [int(float(x)) for x in o.ncalls.split(",")]:
            spec = M.make_integrand(o.integrand, d) if o.integrand not in ("fA", "fB") else M.make_integrand(
                o.integrand, 0)
            d_eff = spec.dims
            if nc < (2 << d_eff):
                continue
            cfg = M.RunConfig(dims=d_eff, maxcalls=nc, itmax=3, ita=3, tau_rel=1e-15, lower=spec.lower,
                              upper=spec.upper, rng=o.rng)
            sp = M.setup(cfg)
            with torch.cuda.stream(stream):
                run = M.Run(spec, cfg, ctx)
                m = run.work_items
                n0, n1 = rank * m // world, (rank + 1) * m // world
                x = torch.zeros(run.exchange_words(), dtype=torch.int64, device=dev)
                run.set_exchange(x.data_ptr())

                def step(it):
                    run.sample(it, n0, n1)
                    run.reduce(it)
                    if dist is not None:
                        dist.all_reduce(x[:run.exchange_words(it)])
                    run.finish(it)

                step(1)  # warm
                torch.cuda.synchronize()
                if dist is not None:
                    dist.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                step(2)
                e1.record(stream)
                torch.cuda.synchronize()
                it_ms = max_ranks(e0.elapsed_time(e1))
                run.close()
            cfg5 = M.RunConfig(dims=d_eff, maxcalls=nc, itmax=5, ita=3, tau_rel=1e-15, lower=spec.lower,
                               upper=spec.upper, rng=o.rng)
            with torch.cuda.stream(stream):
                if dist is None:
                    _, run_ms = _timed(spec, cfg5, ctx)
                else:
                    from . import dist as mdist
                    torch.cuda.synchronize()
                    dist.barrier()
                    t0 = time.perf_counter()
                    mdist.integrate(spec, cfg5, ctx=ctx)
                    run_ms = max_ranks(1e3 * (time.perf_counter() - t0))
            ev = sp.m * sp.p
            cpu_cols = ["", "", "", ""]
            if cpu_timer is not None and ev <= o.cpu_max_evals:
                timed = cpu_timer(o.integrand, d_eff, nc)
                if timed:
                    threads, cms = timed
                    cpu_cols = [str(threads), fmt17(cms), fmt17(ev / (cms * 1e-3)), fmt17(cms / it_ms)]
            if out:
                out.write(",".join(str(v) for v in [spec.name, d_eff, nc, sp.g, sp.m, sp.p, world, ev, fmt17(it_ms),
                                                    fmt17(ev / (it_ms * 1e-3)), fmt17(run_ms)] + cpu_cols))
    if out:
        out.close()
    return 0


def _common(p):
    p.add_argument("--integrand", required=True, help="integrand id: f1..f6, fA, fB")
    p.add_argument("--dim", type=int, default=0, help="dimension for f1..f6 (fA, fB are fixed)")
    p.add_argument("--tau-rel", type=float, default=1e-3)
    p.add_argument("--maxcalls", type=int, default=1_000_000)
    p.add_argument("--itmax", type=int, default=15)
    p.add_argument("--ita", type=int, default=10)
    p.add_argument("--n-bins", type=int, default=50)
    p.add_argument("--alpha", type=float, default=1.5)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--variant", choices=["mcubes", "mcubes1d"], default="mcubes")
    p.add_argument("--workers", type=int, default=0, help="accepted for compatibility (results are worker-invariant)")
    p.add_argument("--rng", choices=["compat", "philox"], default="compat")
    p.add_argument("--out", default=None, help="write CSV here instead of standard output")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="mcubes_bench", description="adaptive Monte Carlo integration benchmark (B200)")
    sub = ap.add_subparsers(dest="cmd")
    run = sub.add_parser("run", help="single seeded integration")
    _common(run)
    sweep = sub.add_parser("sweep", help="tolerance-schedule sweep")
    _common(sweep)
    sweep.add_argument("--runs", type=int, default=20)
    summ = sub.add_parser("summarize", help="quartile summary of a sweep CSV")
    summ.add_argument("input")
    summ.add_argument("--out", default=None)
    scale = sub.add_parser("scale", help="throughput sweep over dims x ncall (BASELINE config 5)")
    scale.add_argument("--integrand", default="f4")
    scale.add_argument("--dims", default="2,4,6,8,10")
    scale.add_argument("--ncalls", default="1e6,1e8,1e10")
    scale.add_argument("--rng", choices=["compat", "philox"], default="compat")
    scale.add_argument("--cpu-max-evals", type=float, default=1e9,
                       help="with a CPU timer (bench.py --scale): time the reference CPU iteration for cells "
                            "with m*p up to this")
    scale.add_argument("--out", default=None)
    try:
        o = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 1
    if o.cmd is None:
        ap.print_usage(sys.stderr)
        return 1
    if o.cmd == "sweep" and o.runs < 1:
        print("--runs must be positive", file=sys.stderr)
        return 1
    try:
        if o.cmd == "run":
            return cmd_run(o)
        if o.cmd == "sweep":
            return cmd_sweep(o)
        if o.cmd == "scale":
            return cmd_scale(o)
        return cmd_summarize(o.input, o.out)
    except (ValueError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
