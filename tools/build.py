"""Build the three native libraries in-tree.

* synth/libsynth.so     — seeded input generator (gcc)
* oracle/liboracle.so   — CPU oracle, test infrastructure only (gcc, -ffp-contract=off)
* paper_1310_1371_b200/librd.so — the product: CUDA kernels for sm_100a + C ABI (nvcc)
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _run(cmd):
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {cmd[0]} ... -> {cmd[-1] if cmd else ''}")
    return r


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def build_synth(force=False):
    out = os.path.join(ROOT, "synth", "libsynth.so")
    srcs = [os.path.join(ROOT, "synth", f) for f in ("synth.c", "synth.h")]
    if force or _stale(out, srcs):
        _run(["gcc", "-O2", "-fPIC", "-shared", "-Wall", "-o", out, srcs[0], "-lm", "-lpthread"])
    return out


def build_oracle(force=False):
    out = os.path.join(ROOT, "oracle", "liboracle.so")
    srcs = [os.path.join(ROOT, "oracle", f) for f in ("oracle.c", "streamed.c", "oracle.h")]
    if force or _stale(out, srcs):
        _run(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-Wall", "-o", out, srcs[0],
              srcs[1], "-lm", "-lpthread"])
    return out


def build_rd(force=False, checked=False):
    """librd.so, or with checked=True librd_checked.so: the same sources with -DRD_CHECKED (bounds
    assertions in every kernel, tests/test_checked.py)."""
    pkg = os.path.join(ROOT, "paper_1310_1371_b200")
    out = os.environ.get("RD_BUILD_OUT") or os.path.join(pkg, "librd_checked.so" if checked else "librd.so")
    csrc = os.path.join(pkg, "csrc")
    srcs = sorted(glob.glob(os.path.join(csrc, "*.cu")) + glob.glob(os.path.join(csrc, "*.cpp")))
    deps = srcs + glob.glob(os.path.join(csrc, "*.cuh")) + glob.glob(os.path.join(csrc, "*.h")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    if not (force or _stale(out, deps)):
        return out
    prof = ["-DRD_K2_PROF"] if os.environ.get("RD_BUILD_PROF") else []   # K2 phase-cycle counters (tools/phase_probe.py)
    prof += os.environ.get("RD_BUILD_DEFS", "").split()   # variant builds for A/B runs (-DNAME=VALUE ...)
    if checked:
        prof += ["-DRD_CHECKED"]
    cmd = [NVCC, "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo"] + prof + [
           "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off", "-shared",
           "-Xptxas", "-v", "-I", os.path.join(ROOT, "include"), "-o", out] + srcs + ["-lcudart"]
    r = _run(cmd)
    with open(os.path.join(pkg, "build_ptxas_checked.log" if checked else "build_ptxas.log"), "w") as f:
        f.write(r.stdout + r.stderr)
    return out


def build_all(force=False):
    return [build_synth(force), build_oracle(force), build_rd(force), build_rd(force, checked=True)]


if __name__ == "__main__":
    for p in build_all(force="--force" in sys.argv):
        print(p)
