"""Per-SASS-instruction warp-stall samples from an ncu report's source page.

    python tools/ncu_stalls.py report.ncu-rep [top_n]

Prints the top instructions by samples with their dominant stall reasons, and totals by
stall reason and by opcode (reads `ncu -i --page source --csv --print-source sass`)."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
stall_cols = [c for c in rows[0] if c.startswith("stall_") and "Not Issued" not in c]


def num(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return 0.0


tot = defaultdict(float)
by_op = defaultdict(float)
allsamp = 0.0
recs = []
for r in rows:
    s = num(r["Warp Stall Sampling (All Samples)"])
    allsamp += s
    op = r["Source"].split()[0] if r["Source"].split() else "?"
    if op.startswith("@"):
        op = r["Source"].split()[1]
    by_op[op.split(".")[0]] += s
    st = {c: num(r[c]) for c in stall_cols}
    for c, v in st.items():
        tot[c] += v
    recs.append((s, r["Address"], r["Source"][:70], st, num(r["Instructions Executed"])))
print(f"total samples {allsamp:.0f}")
print("by stall reason:", ", ".join(f"{k[6:]}={100 * v / allsamp:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v > 0.005 * allsamp))
print("by opcode:", ", ".join(f"{k}={100 * v / allsamp:.1f}%" for k, v in sorted(by_op.items(), key=lambda x: -x[1])[:20]))
recs.sort(key=lambda x: -x[0])
for s, a, src, st, ex in recs[:top]:
    reasons = ", ".join(f"{k[6:]}={v:.0f}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3] if v > 0)
    print(f"{100 * s / allsamp:5.2f}% {a} {src:70s} exec={ex:.0f} [{reasons}]")
