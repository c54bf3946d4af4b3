"""Per-source-line warp-stall samples of one kernel in an ncu report.

    python tools/ncu_lines.py report.ncu-rep kernel.dis [top_n]

kernel.dis = `nvdisasm -g -c <cubin>` output restricted to the kernel's .text section (line-info
comments `// ## File "...", line N`).  ncu's SASS page gives absolute addresses; offsets from the
first instruction are matched to the disassembly, then samples are summed per source line."""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep, dis = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
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


base = min(int(r["Address"], 16) for r in rows)
line_of = {}
cur = None
for l in open(dis):
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if m and '##' in l:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
    if m:
        line_of[int(m.group(1), 16)] = cur
samp = defaultdict(float)
why = defaultdict(lambda: defaultdict(float))
tot = 0.0
for r in rows:
    s = num(r.get("Warp Stall Sampling (All Samples)", "0"))
    off = int(r["Address"], 16) - base
    ln = line_of.get(off)
    samp[ln] += s
    tot += s
    for c in stall_cols:
        why[ln][c] += num(r[c])
for ln, s in sorted(samp.items(), key=lambda x: -x[1])[:top]:
    w = sorted(why[ln].items(), key=lambda x: -x[1])[:3]
    print(f"{100 * s / tot:5.1f}%  {ln}  " + ", ".join(f"{k[6:]}={v:.0f}" for k, v in w if v))
