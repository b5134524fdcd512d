"""Per-source-line instruction counts from `ncu --page source --csv
--print-source cuda,sass` output (tools/gpu_evidence2.sh): the cuda rows
carry per-line totals, the sass rows below them the instructions.

    python tools/ncu_lines2.py gpurun_out/ncu/src_philoxbinsr24.csv.gz EVALS [top]
"""
import csv
import gzip
import io
import sys
from collections import defaultdict


def main():
    path, evals = sys.argv[1], float(sys.argv[2])
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    op = gzip.open if path.endswith(".gz") else open
    rows = list(csv.reader(io.TextIOWrapper(op(path, "rb"))))
    cur, hdr, ti = None, None, None
    per_line, per_file, per_op = {}, defaultdict(float), defaultdict(float)
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            ti = hdr.index("Thread Instructions Executed")
            continue
        if hdr is None or len(r) <= ti:
            continue
        try:
            v = float(r[ti])
        except ValueError:
            continue
        if r[0]:  # a cuda line (totals of the sass below it)
            per_line[(cur, int(r[0]), r[1][:90])] = v
            per_file[cur] += v
        else:  # a sass row
            toks = r[3].split()
            if toks and toks[0].startswith("@"):
                toks = toks[1:]
            per_op[(toks[0] if toks else "?").split(".")[0]] += v
    tot = sum(per_file.values())
    print(f"thread instructions per eval: {tot / evals:.1f}")
    for f, v in sorted(per_file.items(), key=lambda x: -x[1]):
        print(f"  {f:24s} {v / evals:7.1f}")
    print("by opcode:")
    for o, v in sorted(per_op.items(), key=lambda x: -x[1])[:25]:
        print(f"  {o:12s} {v / evals:7.1f}")
    print("top lines:")
    for (f, ln, src), v in sorted(per_line.items(), key=lambda x: -x[1])[:top]:
        print(f"  {v / evals:6.1f}  {f}:{ln}  {src}")


if __name__ == "__main__":
    main()
