"""Per-source-line thread instructions per eval from an ncu report.
    python tools/ncu_lines.py rep.ncu-rep EVALS [top]"""
import csv, io, subprocess, sys
rep, evals = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, ie, src = None, None, {}
agg = {}
for r in rows:
    if len(r) >= 2 and r[0] in ("File Path", "File Name"):
        cur = r[1].split("/")[-1]; continue
    if len(r) > 2 and r[0] == "Line No":
        ie = r.index("Instructions Executed"); continue
    if ie is not None and len(r) > ie and r[0].isdigit():
        try:
            v = float(r[ie])
        except ValueError:
            continue
        agg[(cur, int(r[0]))] = agg.get((cur, int(r[0])), 0) + v
        src[(cur, int(r[0]))] = r[1][:90]
tot = sum(agg.values())
print(f"total thread instr/eval: {32 * tot / evals:.1f}")
byf = {}
for (f, l), v in agg.items():
    byf[f] = byf.get(f, 0) + v
for f, v in sorted(byf.items(), key=lambda x: -x[1]):
    print(f"  {f:40s} {32 * v / evals:7.1f}")
for (f, l), v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{f}:{l:<5d} {32 * v / evals:7.1f}  {src[(f, l)]}")
