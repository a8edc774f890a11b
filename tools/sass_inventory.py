"""Static SASS inventory of librd.so's main kernels (cuobjdump -sass): per kernel, how many
TMA tensor loads (UTMALDG), 1-D bulk copies (UBLKCP), mbarrier ops (SYNCS), shared atomics
(ATOMS), dp4a (IDP), fp64 and memory instructions the code holds.  Writes
profiles/sass_inventory_<tag>.md.  usage: sass_inventory.py [tag]"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG = sys.argv[1] if len(sys.argv) > 1 else "r02"
LIB = os.path.join(ROOT, "paper_1310_1371_b200", "librd.so")
txt = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", txt)
want = {"k_ridges2ItLi5ELi4ELb0ELb1E": "K1 k_ridges2<u16, K_s 5, RB 4, ridges, TMA>",
        "k_raysENS_6ParamsE": "K1.5 k_rays",
        "k_hough2ILb0ELi4ELi512ELi2ELi1ELb1E": "K2 k_hough2<G 4, 512 thr, 2/SM, byte counters, R16>",
        "k_hough2ILb0ELi4ELi512ELi1ELi2ELb1E": "K2 redo k_hough2<G 4, 512 thr, 1/SM, 16-bit, R16>",
        "k_fitENS_6ParamsE": "K3 k_fit"}
ops = ["UTMALDG", "UBLKCP", "SYNCS", "ATOMS", "ATOMG", "IDP", "DMUL", "DFMA", "DADD", "F2I", "MUFU", "BAR",
       "LDS", "STS", "LDG", "STG"]
out = [f"SASS inventory of librd.so (sm_100a; `python tools/sass_inventory.py {TAG}`): static instruction counts per",
       "kernel.  UTMALDG = TMA tensor load (K1's input rows), UBLKCP = 1-D bulk copy on the TMA engine (K2's ray",
       "intervals / rays, the level-buffer clear and the window weight words), SYNCS = mbarrier operations,",
       "ATOMS = shared-memory atomic (votes, list appends), IDP = dp4a (window sums).", "",
       "| kernel | " + " | ".join(ops) + " |", "|---|" + "---|" * len(ops)]
for f in funcs:
    name = f.split("\n", 1)[0].strip()
    for k, lab in want.items():
        if k in name:
            out.append(f"| {lab} | " + " | ".join(str(len(re.findall(r"\b" + o + r"[\.\s]", f))) for o in ops) + " |")
path = os.path.join(ROOT, "profiles", f"sass_inventory_{TAG}.md")
open(path, "w").write("\n".join(out) + "\n")
print("\n".join(out))
