"""Copy the latest GPU measurements into profiles/ (round tag argv[1], default r01): bench line,
ncu launch list + kernel-share table, and the per-kernel ncu --set full summaries."""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG = sys.argv[1] if len(sys.argv) > 1 else "r01"
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
shutil.copy(os.path.join(G, "bench.json"), os.path.join(P, f"bench_{TAG}.json"))
shutil.copy(os.path.join(G, "launches.csv"), os.path.join(P, f"launches_{TAG}.csv"))
lines = open(os.path.join(G, "launches.csv")).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = [r for r in csv.reader(lines[start:]) if r]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
d = defaultdict(list)
for r in rows[1:]:
    d[r[ki].split("(")[0].replace("void ", "")[:44]].append(float(r[vi]))
tot = sum(sum(v) for v in d.values())
out = ["ncu launch list (gpu__time_duration.sum, --clock-control none) of `python bench.py --steps 2 --warmup 3 --no-cpu`",
       f"(profiles/launches_{TAG}.csv): cold-cache, serialised per-launch times over all launches of that run (warm-up,",
       "timed steps, the debug pass and the host-path chunks of the e2e runs); the shares are what must agree with bench.py.", "",
       "| kernel | launches | mean us | share |", "|---|---|---|---|"]
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    out.append(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {100 * sum(v) / tot:.1f}% |")
open(os.path.join(P, f"launches_{TAG}.md"), "w").write("\n".join(out) + "\n")
summ = []
for k in ("k1full", "k2full", "krays", "kfit"):
    rep = os.path.join(G, k + ".ncu-rep")
    if os.path.exists(rep):
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep, f"/tmp/sum_{k}", "64"],
                       capture_output=True)
        summ += json.load(open(f"/tmp/sum_{k}.json"))
json.dump(summ, open(os.path.join(P, f"ncu_summary_{TAG}.json"), "w"), indent=1)
cols = ["kernel", "duration", "dram_bytes", "warp_inst", "issue_active_pct", "warps_active_pct", "fp64_pipe_pct",
        "alu_pipe_pct", "lsu_pipe_pct", "smem_wavefront_pct", "regs", "dyn_smem"]
with open(os.path.join(P, f"ncu_summary_{TAG}.md"), "w") as f:
    f.write("ncu --set full, one launch each on 64 cfg3 frames (tools/prof_step.py 3 64 2; tools/prof_round.sh)\n\n")
    f.write("| " + " | ".join(cols) + " |\n|" + "---|" * len(cols) + "\n")
    for s in summ:
        f.write("| " + " | ".join(str(round(s[c], 2)) if isinstance(s.get(c), float) else str(s.get(c, ""))
                                  for c in cols) + " |\n")
for k, name in (("k1full", "k1"), ("k2full", "k2")):   # per-source-line stall / instruction summaries
    src = os.path.join(G, f"{k}_src.csv")
    if os.path.exists(src):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), src, "40"], capture_output=True,
                           text=True)
        open(os.path.join(P, f"ncu_lines_{name}_{TAG}.txt"), "w").write(
            f"tools/ncu_lines.py gpurun_out/{k}_src.csv 40 (ncu --set full --import-source, 64 cfg3 frames)\n" + r.stdout)
print(open(os.path.join(P, f"launches_{TAG}.md")).read())
print(open(os.path.join(P, f"ncu_summary_{TAG}.md")).read())
