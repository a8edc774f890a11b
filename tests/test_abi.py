"""The C-ABI library loads and exports every symbol include/rd.h declares; host-side
validation works without a GPU (-m "not gpu")."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rdlib():
    from tools.build import build_rd
    build_rd()
    from paper_1310_1371_b200 import _rd
    return _rd


def _declared():
    src = open(os.path.join(ROOT, "include", "rd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rd_[a-z_]+)\s*\(", src)))


def test_exports_match_header(rdlib):
    names = _declared()
    assert len(names) >= 14
    assert sorted(rdlib.EXPORTS) == names
    L = C.CDLL(rdlib.LIB_PATH)
    for n in names:
        assert hasattr(L, n), n


def test_status_strings_and_version(rdlib):
    L = rdlib.lib()
    assert L.rd_abi_version() == 4
    for s in range(7):
        assert len(L.rd_status_string(s)) > 0


def test_config_init_defaults(rdlib):
    c = rdlib.make_config(1024, 688, 2)
    assert (c.width, c.height, c.pixel, c.max_value) == (1024, 688, rdlib.RD_U16, 65535)
    assert (c.r_min, c.r_max, c.vote_threshold_raw, c.sig_a, c.sig_b, c.sig_den) == (8, 70, 3, 1, 5, 20)
    assert c.smoothing_sigma == 1.5 and c.vote_threshold_norm == 0.5


@pytest.mark.parametrize("bad,status", [
    (dict(width=4), 2), (dict(smoothing_sigma=0.0), 1), (dict(smoothing_sigma=6.0), 1), (dict(smoothing_sigma=4.34), 1),
    (dict(curvature_threshold=0.5), 1), (dict(r_min=1), 1), (dict(r_max=5, r_min=9), 1),
    (dict(vote_threshold_raw=0), 1), (dict(vote_threshold_norm=0.0), 1), (dict(sig_den=0), 1),
    (dict(annulus_halfwidth=-1), 1), (dict(max_value=70000), 1)])
def test_create_rejects_invalid_config_without_gpu(rdlib, bad, status):
    c = rdlib.make_config(640, 480, 2)
    for k, v in bad.items():
        setattr(c, k, v)
    h = C.c_void_p()
    assert rdlib.lib().rd_create(C.byref(c), 1, 0, C.byref(h)) == status
    assert not h.value


def test_null_arguments(rdlib):
    L = rdlib.lib()
    assert L.rd_create(None, 1, 0, None) == rdlib.RD_ERR_PARAM
    assert L.rd_detect(None, None, 0, 0, 1, None, 0, None, None, None) == rdlib.RD_ERR_PARAM
    assert L.rd_detect_host(None, None, 0, 0, 1, None, 0, None, None) == rdlib.RD_ERR_PARAM
    assert L.rd_submit_host(None, None, 0, 0, 1, None, 0, None, None) == rdlib.RD_ERR_PARAM
    assert L.rd_wait_host(None) == rdlib.RD_ERR_PARAM
    assert L.rd_sync(None) == rdlib.RD_ERR_PARAM
    assert L.rd_query_overflow(None, None) == rdlib.RD_ERR_PARAM
    assert L.rd_debug_dump(None, 0, 0, None, 0, None) == rdlib.RD_ERR_PARAM
    assert L.rd_destroy(None) == rdlib.RD_OK


def test_product_does_not_import_oracle():
    """The product package never references the oracle (test infrastructure only)."""
    pkg = os.path.join(ROOT, "paper_1310_1371_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "oracle.h" not in txt and "orc_" not in txt, f
