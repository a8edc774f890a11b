"""Mutation check of the oracle's pins (test infrastructure).

Each mutation is a plausible slip in oracle/oracle.c (a rounding mode, a units factor, a
sign, an off-by-one).  For each, a mutated copy of the oracle is built under /tmp and the
CPU pin suites run against it through ORACLE_LIB_PATH; a mutation is "killed" when at least
one pin fails.  Writes profiles/mutation_<round>.json.

  python tools/mutate_oracle.py [round_tag]
"""
from __future__ import annotations

import json
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITES = ["tests/test_oracle_pins.py", "tests/test_oracle_units.py", "tests/test_oracle_edges.py"]

# (name, function it lives in, exact source text, replacement)
MUTATIONS = [
    ("gauss_taps: llround -> floor", "orc_gauss_taps",
     "taps[i + K] = (int32_t)llround(1024.0 * exp(", "taps[i + K] = (int32_t)floor(1024.0 * exp("),
    ("level_weight: llround -> floor", "orc_level_weight",
     "return (int32_t)llround(4096.0 * exp(-num / den));", "return (int32_t)floor(4096.0 * exp(-num / den));"),
    ("curvature threshold units: 64 -> 128", "orc_curvature_threshold_int",
     "return p->curvature_threshold * (64.0 * (double)sq * (double)sq);",
     "return p->curvature_threshold * (128.0 * (double)sq * (double)sq);"),
    ("edge threshold units: 128 -> 64", "orc_edge_threshold_int2",
     "double t = p->edge_threshold * (128.0 * (double)sq * (double)sq);",
     "double t = p->edge_threshold * (64.0 * (double)sq * (double)sq);"),
    ("votes: Hough range starts at r_min", "orc_votes",
     "const int r_lo = p->r_min - 1, r_hi = p->r_max + 1;\n  int64_t votes = 0;",
     "const int r_lo = p->r_min, r_hi = p->r_max + 1;\n  int64_t votes = 0;"),
    ("votes: x offset rounded toward zero", "orc_votes",
     "long long ox = llround((double)r * ridges[k].dx);", "long long ox = (long long)((double)r * ridges[k].dx);"),
    ("votes: one sense only", "orc_votes", "for (int s = 1; s >= -1; s -= 2) {", "for (int s = 1; s >= 1; s -= 2) {"),
    ("eigen: branch on e > 0 instead of e >= 0", "orc_eigen", "  if (e >= 0.0) {\n    vx = -b;",
     "  if (e > 0.0) {\n    vx = -b;"),
    ("eigen: kappa = larger eigenvalue", "orc_eigen", "*kappa = 0.5 * (T - s);", "*kappa = 0.5 * (T + s);"),
    ("window sum: K_r - 1", "orc_window_sum", "const int K = orc_level_halfwidth(p, r);\n  const int32_t* lvl",
     "const int K = orc_level_halfwidth(p, r) - 1;\n  const int32_t* lvl"),
    ("hotspot: raw >= T_raw", "hot_and_peaks", "if (v > p->vote_threshold_raw) {", "if (v >= p->vote_threshold_raw) {"),
    ("NMS: ties to the larger key", "hot_and_peaks", "cmp_key(v->r, v->y, v->x, ur, uy, ux) < 0);",
     "cmp_key(v->r, v->y, v->x, ur, uy, ux) > 0);"),
    ("NMS: 3x3 in-level only", "hot_and_peaks", "for (int dr = -1; dr <= 1 && is_peak; ++dr)",
     "for (int dr = 0; dr <= 0 && is_peak; ++dr)"),
    ("annulus: exclusive outer edge", "classify_fit", "    if (z < lo2 || z > hi2) continue;\n    ++n;",
     "    if (z < lo2 || z >= hi2) continue;\n    ++n;"),
    ("fit: centre sign", "fit_moments", "*uc = -D / 2.0;", "*uc = D / 2.0;"),
]


def build(src_dir, out):
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-o", out,
           os.path.join(src_dir, "oracle.c"), os.path.join(src_dir, "streamed.c"), "-lm", "-lpthread"]
    subprocess.run(cmd, check=True, capture_output=True)


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    src = open(os.path.join(ROOT, "oracle", "oracle.c")).read()
    results = []
    for name, fn, old, new in MUTATIONS:
        n = src.count(old)
        if n != 1:
            results.append({"mutation": name, "function": fn, "error": f"pattern found {n} times"})
            continue
        with tempfile.TemporaryDirectory() as d:
            for f in ("oracle.h", "streamed.c"):
                shutil.copy(os.path.join(ROOT, "oracle", f), d)
            open(os.path.join(d, "oracle.c"), "w").write(src.replace(old, new))
            lib = os.path.join(d, "liboracle_mut.so")
            build(d, lib)
            env = dict(os.environ, ORACLE_LIB_PATH=lib)
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider"] + SUITES,
                               cwd=ROOT, env=env, capture_output=True, text=True)
            failed = [ln.split(" ")[1] for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
            results.append({"mutation": name, "function": fn, "killed": r.returncode != 0,
                            "first_failing_test": failed[0] if failed else None})
        print(json.dumps(results[-1]), flush=True)
    out = os.path.join(ROOT, "profiles", f"mutation_{tag}.json")
    json.dump({"suites": SUITES, "results": results,
               "killed": sum(1 for r in results if r.get("killed")), "total": len(results)}, open(out, "w"), indent=1)
    print(out)
    return 0 if all(r.get("killed") for r in results) else 1


if __name__ == "__main__":
    sys.exit(main())
