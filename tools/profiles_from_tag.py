"""Summarise a tools/profile_all.sh run (gpurun_out/<TAG>_*) into profiles/:
<TAG>_<config>_ncu.json, <TAG>_longformer_launches.{csv,json}, <TAG>_bench_*.json, and
profiles/ncu_summary.json (the per-step DRAM traffic bench.py reports as roofline.traffic).

    python tools/profiles_from_tag.py r01c
"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
src = os.path.join(ROOT, "gpurun_out")
dst = os.path.join(ROOT, "profiles")
summ = os.path.join(ROOT, "tools", "ncu_summary.py")


def nbytes(s):
    v, u = s.split()
    return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]


out = {}
for c in ["longformer", "bigbird", "mistral", "sparse_transformer"]:
    rep = os.path.join(src, f"{tag}_prof_{c}.ncu-rep")
    if not os.path.exists(rep):
        continue
    js = subprocess.check_output([sys.executable, summ, rep, "--label", f"{c} {tag}"], text=True)
    open(os.path.join(dst, f"{tag}_{c}_ncu.json"), "w").write(js)
    ks = json.loads(js)["full"]
    out[c] = {
        "kernel": " + ".join(k["kernel"].split("(")[0].replace("void ", "").replace("unnamed>::", "") for k in ks),
        "launches_per_step": len(ks),
        "dram_bytes_per_launch": sum(nbytes(k["dram__bytes_read.sum"]) + nbytes(k["dram__bytes_write.sum"]) for k in ks),
        "dram_read": " + ".join(k["dram__bytes_read.sum"] for k in ks),
        "dram_write": " + ".join(k["dram__bytes_write.sum"] for k in ks),
        "duration_under_ncu": " + ".join(k["gpu__time_duration.sum"] for k in ks),
        "tensor_pipe_active": " / ".join(k["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"] for k in ks),
        "xu_pipe_active": " / ".join(k["sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"] for k in ks),
        "source": f"profiles/{tag}_{c}_ncu.json (ncu --set full, one capture per kernel, cold L2 per replay)",
    }
json.dump(out, open(os.path.join(dst, "ncu_summary.json"), "w"), indent=1)
lc = os.path.join(src, f"{tag}_launches.csv")
if os.path.exists(lc):
    shutil.copy(lc, os.path.join(dst, f"{tag}_longformer_launches.csv"))
    js = subprocess.check_output([sys.executable, summ, "--launches", lc], text=True)
    open(os.path.join(dst, f"{tag}_longformer_launches.json"), "w").write(js)
for f in os.listdir(src):
    if f.startswith(f"{tag}_bench_") and f.endswith(".json"):
        shutil.copy(os.path.join(src, f), os.path.join(dst, f))
print(json.dumps(out, indent=1))
