"""Checked build (the sanitizer tier T5 of SURVEY.md §4 by assertion; -m gpu).

compute-sanitizer is not available on this pool, so librd_checked.so (the same sources built
with -DRD_CHECKED) tests every shared-memory and global index the kernels form against its
array's bounds and reports the first failure through rd_sync / rd_detect_host.  The runner
(tests/helpers/checked_run.py) drives the whole path on cfg1/2/3, the forced 16-bit redo pass,
the host path, the edge variant and K_r >= 16, compared with the oracle; with RD_JITTER=1 the
Hough kernel's warps sleep pseudo-random times at each phase start, so a missing barrier
between the phases (PAPER.md:426-434's register-and-undo becomes shared-memory clears and list
rebuilds here) would show as a result difference or a failed check.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1310_1371_b200", "librd_checked.so")


@pytest.mark.parametrize("mode", ["plain", "jitter", "redo_jitter"])
def test_checked_build_clean(mode):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(LIB):
        from tools.build import build_rd
        build_rd(checked=True)
    env = dict(os.environ, RD_LIB_PATH=LIB)
    if "jitter" in mode:
        env["RD_JITTER"] = "1"
    if "redo" in mode:
        env["RD_K2_FORCE_REDO"] = "1"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "helpers", "checked_run.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "checked ok" in r.stdout, out[-3000:]
