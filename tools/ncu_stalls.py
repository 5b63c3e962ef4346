"""Aggregate ncu source-page stall samples of one kernel by SASS opcode and by
source line: python tools/ncu_stalls.py report.ncu-rep kernel_regex [top]."""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name-base", "demangled", "--kernel-name", f"regex:{kre}",
                      "--launch-count", "1"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
iS = h.index("Source")
iN = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
by_op = defaultdict(Counter)
tot = Counter()
per_ins = []
for r in rows[1:]:
    if len(r) < len(h) or not r[iN].isdigit():
        continue
    op = r[iS].strip().split()[0] if r[iS].strip() else "?"
    if op.startswith("@"):
        op = r[iS].strip().split()[1]
    op = op.split(".")[0]
    n = int(r[iN] or 0)
    for i, c in stall_cols:
        v = int(r[i] or 0)
        if v:
            by_op[op][c[6:]] += v
            tot[c[6:]] += v
    per_ins.append((n, r[0], r[iS].strip()))
T = sum(tot.values())
print("total samples", T)
print("by reason:", ", ".join(f"{k} {100*v/T:.0f}%" for k, v in tot.most_common(10)))
print("\nby opcode (samples, top reasons):")
for op, c in sorted(by_op.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
    s = sum(c.values())
    print(f"  {op:10s} {100*s/T:5.1f}%  " + ", ".join(f"{k} {100*v/T:.1f}" for k, v in c.most_common(3)))
print("\ntop instructions:")
for n, a, s in sorted(per_ins, reverse=True)[:top]:
    print(f"  {100*n/T:5.2f}%  {a[-5:]}  {s[:70]}")
