"""Aggregate ncu source-page warp-stall samples per CUDA source line (reads `ncu --page source --csv
--print-source cuda,sass` output).  Usage: ncu_lines.py file.csv [topN]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr_i]
si = h.index("Warp Stall Sampling (All Samples)")
ni = h.index("Warp Stall Sampling (Not-issued Samples)")
ie = h.index("Instructions Executed")
lines = []
for r in rows[hdr_i + 1:]:
    if len(r) > ie and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            lines.append((int(r[si]), int(r[ni]), int(r[ie]), r[0], r[1][:110]))
        except ValueError:
            pass
tot = sum(x[0] for x in lines) or 1
for s, n, e, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% ns={100 * n / tot:5.1f}% inst={e:>10} L{ln}: {src}")
