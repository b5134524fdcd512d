"""Summarise ncu captures into profiles/ (tracked evidence).

    python tools/summarize_ncu.py gpurun_out/prof_k1.ncu-rep gpurun_out/launches.csv r01

Writes profiles/ncu_k1_<tag>.md (key metrics of the full-set capture of the
sampling kernel, the per-source-line instruction mix), profiles/launches_<tag>.md
(per-kernel share of the launch list) and profiles/k1_traffic.json
(DRAM bytes per launch, read by bench.py's roofline.traffic).
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))

KEYS = [
    ("gpu__time_duration.sum", "duration (ms, ncu replay)"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe cycles active %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe (IMAD) %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("smsp__inst_executed_op_shared_atom.sum", "shared atomics (warp-level)"),
    ("l1tex__t_set_accesses_pipe_lsu_mem_global_op_atom.sum", "GLOBAL atomics"),
    ("l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum", "GLOBAL reductions"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum", "GLOBAL atomic requests (none on the histogram path)"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_red.sum",
     "GLOBAL reduction requests (only the per-block flush of nonzero exchange words; per-sample deposits stay in shared memory)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum", "smem atomic bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
     "shared-memory data pipe busy % (one wavefront per clock per SM)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum.pct_of_peak_sustained_elapsed",
     "  of which shared loads (grid table, reciprocals) %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum.pct_of_peak_sustained_elapsed",
     "  of which shared atomics (exact deposits) %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "shared-load wavefronts"),
    ("smsp__sass_inst_executed_op_shared_ld.sum", "shared-load warp instructions"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "shared-atomic wavefronts"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
]


def ncu_csv(rep, page, *extra):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True,
                         check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep, launches, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    evals = float(sys.argv[4]) if len(sys.argv) > 4 else None
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    raw = ncu_csv(rep, "raw")
    hdr, units, val = raw[0], raw[1], raw[2]
    m = dict(zip(hdr, val))
    u = dict(zip(hdr, units))
    name = m.get("Kernel Name", "?")
    lines = [f"# ncu --set full: sampling kernel K1 ({tag})", "", f"kernel: `{name}`", "",
             "| metric | value | unit |", "|---|---|---|"]
    for k, label in KEYS:
        if k in m:
            lines.append(f"| {label} (`{k}`) | {m[k]} | {u.get(k, '')} |")
    stalls = sorted(((k, float(v)) for k, v in m.items()
                     if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                     and v not in ("", "n/a")), key=lambda x: -x[1])
    lines += ["", "Top stall reasons (warps per issue-active cycle):", ""]
    for k, v in stalls[:8]:
        lines.append(f"- {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}: {v:.3f}")

    # per-source-file instruction mix
    src = ncu_csv(rep, "source", "--print-source", "cuda,sass")
    agg = defaultdict(float)
    cur, ie = None, None
    for r in src:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            ie = r.index("Instructions Executed")
            continue
        if ie is not None and len(r) > ie and r[0].isdigit():  # cuda rows carry their line's total
            try:
                agg[cur] += float(r[ie])
            except ValueError:
                pass
    tot = sum(agg.values())
    if evals:
        lines += ["", f"Thread instructions per integrand evaluation ({evals:.0f} evals in the captured launch): "
                      f"{32 * tot / evals:.0f}", "", "| source | instr/eval | share |", "|---|---|---|"]
        for f, n in sorted(agg.items(), key=lambda x: -x[1]):
            lines.append(f"| {f} | {32 * n / evals:.1f} | {100 * n / tot:.1f}% |")
    dram = float(m.get("dram__bytes_read.sum", 0) or 0) + float(m.get("dram__bytes_write.sum", 0) or 0)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u.get("dram__bytes_read.sum", "byte"), 1)
    with open(os.path.join(ROOT, "profiles", f"ncu_k1_{tag}.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    # per-stream entry (vsample_kernel<F, D, Rng, NB>), read by bench.py
    tf = os.path.join(ROOT, "profiles", "k1_traffic.json")
    try:
        table = json.load(open(tf))
        if "bytes_per_launch" in table:  # the older flat format
            table = {}
    except (OSError, ValueError):
        table = {}
    targs = [a.strip() for a in name.split("<", 1)[1].split(">", 1)[0].split(",")] if "<" in name else []
    kind = targs[2] if len(targs) > 2 else "0"  # RngKind: 0 compat, 1 philox (r24 bins), 2 philox_exact
    kind = kind.replace("(mcubes::gpu::RngKind)", "")
    rng = {"1": "philox_r24", "2": "philox_exact"}.get(kind, "compat")
    winst = float(m.get("smsp__inst_executed.sum", 0) or 0)
    table[rng] = {"bytes_per_launch": dram * scale, "source": f"profiles/ncu_k1_{tag}.md", "kernel": name,
                  "warp_instr_per_eval": (winst / evals) if (evals and winst) else None}
    with open(tf, "w") as fh:
        json.dump(table, fh, indent=1)

    # launch list
    rows = list(csv.reader(open(launches)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    per = defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) > iv and r[im] == "gpu__time_duration.sum":
            k = r[ik].split("(")[0]
            per[k][0] += 1
            per[k][1] += float(r[iv].replace(",", ""))
    tot = sum(v[1] for v in per.values())
    out = [f"# ncu launch list ({tag}): gpu__time_duration.sum, --clock-control none", "",
           "Cold-cache, serialised replays: compare shares, not absolute times.", "",
           "| kernel | launches | total | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(per.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {n} | {t:.1f} | {100 * t / tot:.2f}% |")
    with open(os.path.join(ROOT, "profiles", f"launches_{tag}.md"), "w") as fh:
        fh.write("\n".join(out) + "\n")
    print("\n".join(lines[:40]))
    print("\n".join(out))


if __name__ == "__main__":
    main()
