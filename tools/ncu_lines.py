"""Aggregate an ncu source page (`ncu -i X --page source --csv --print-source cuda,sass`) per CUDA
source line: warp-stall samples with the top stall reasons, executed instructions, lane
utilisation and excessive shared-memory wavefronts (bank conflicts).

Usage: ncu_lines.py page.csv [topN] [first_line last_line]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, 10 ** 9)
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr_i]
col = {n: i for i, n in enumerate(h) if n not in col} if False else {}
for i, n in enumerate(h):
    col.setdefault(n, i)
si, ie, ti = col["Warp Stall Sampling (All Samples)"], col["Instructions Executed"], col["Thread Instructions Executed"]
xw = col.get("L1 Wavefronts Shared Excessive")
reasons = [n for n in h if n.startswith("stall_") and "(Not Issued)" not in n]
lines = []
for r in rows[hdr_i + 1:]:
    if len(r) <= ie or r[0] in ("", "Line No") or r[2] != "-":
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    if not (lo <= ln <= hi):
        continue
    rs = sorted(((int(r[col[n]] or 0), n[6:]) for n in reasons), reverse=True)[:3]
    lines.append((int(r[si] or 0), int(r[ie] or 0), int(r[ti] or 0), int(r[xw] or 0) if xw else 0, ln, r[1][:90], rs))
tot = sum(x[0] for x in lines) or 1
print(f"samples {tot}  instructions {sum(x[1] for x in lines)}")
for s, e, t, x, ln, src, rs in sorted(lines, reverse=True)[:top]:
    why = " ".join(f"{n}:{100 * v / max(s, 1):.0f}%" for v, n in rs if v)
    util = t / (32 * e) if e else 0
    print(f"{100 * s / tot:5.1f}% L{ln:<4d} inst={e:>10} util={util:.2f} xsw={x:>8} [{why}] {src}")
