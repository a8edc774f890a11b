"""Summarise an ncu report (--set full) into per-kernel key metrics (JSON + markdown table).

usage: ncu_summary.py report.ncu-rep out_prefix [frames_per_launch]
Writes out_prefix.json and out_prefix.md (commit these under profiles/)."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "smsp__inst_executed.sum": "warp_inst",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_wavefront_pct",
    "smsp__inst_executed_op_shared_atom.sum": "smem_atom_inst",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "launch__registers_per_thread": "regs",
    "launch__shared_mem_per_block_dynamic": "dyn_smem",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    frames = int(sys.argv[3]) if len(sys.argv) > 3 else None
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:60]}
        for k, name in KEYS.items():
            if k in hdr:
                v = r[hdr.index(k)].replace(",", "")
                try:
                    d[name] = float(v)
                except ValueError:
                    d[name] = v
                if name == "duration" and units[hdr.index(k)] == "ms":
                    d[name] *= 1e6
                if name == "duration" and units[hdr.index(k)] == "us":
                    d[name] *= 1e3
        if "dram_read" in d:
            # bytes units may be reported scaled (KB/MB); normalise via the unit row
            for nm, k in (("dram_read", "dram__bytes_read.sum"), ("dram_write", "dram__bytes_write.sum")):
                u = units[hdr.index(k)]
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                d[nm] *= scale
            d["dram_bytes"] = d["dram_read"] + d["dram_write"]
            if frames:
                d["frames_per_launch"] = frames
                d["dram_bytes_per_frame"] = d["dram_bytes"] / frames
        res.append(d)
    json.dump(res, open(out + ".json", "w"), indent=1)
    with open(out + ".md", "w") as f:
        cols = ["kernel", "duration", "dram_bytes", "warp_inst", "issue_active_pct", "warps_active_pct",
                "fp64_pipe_pct", "alu_pipe_pct", "lsu_pipe_pct", "smem_wavefront_pct", "regs", "dyn_smem"]
        f.write("| " + " | ".join(cols) + " |\n|" + "---|" * len(cols) + "\n")
        for d in res:
            f.write("| " + " | ".join(str(round(d[c], 2)) if isinstance(d.get(c), float) else str(d.get(c, ""))
                                      for c in cols) + " |\n")
    print(open(out + ".md").read())


if __name__ == "__main__":
    main()
