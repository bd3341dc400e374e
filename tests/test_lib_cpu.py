"""CPU-only checks of the native library: it builds for sm_100a, loads, and exports every
symbol include/cks.h declares; host-only arithmetic (tree shape) matches the oracle's
closed form; argument errors are reported without touching a GPU."""
import ctypes
import os
import re
import subprocess

import pytest

import oracle
from conftest import ROOT


@pytest.fixture(scope="module")
def lib():
    from paper_2009_11543_b200 import _build
    _build.build()
    return ctypes.CDLL(_build.SO)


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "cks.h")).read()
    return sorted(set(re.findall(r"^(?:int|uint64_t|const char\*)\s+(cks_\w+)\(", src, flags=re.M)))


def test_header_symbols_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 15
    from paper_2009_11543_b200 import _build
    out = subprocess.run(["nm", "-D", "--defined-only", _build.SO], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (cks_\w+)", out))
    for s in syms:
        assert s in exported, s
        assert hasattr(lib, s)


def test_binding_names_cover_header():
    from paper_2009_11543_b200 import cks
    assert set(declared_symbols()) == set(cks.EXPORTS)


def test_sm100a_cubin(lib):
    from paper_2009_11543_b200 import _build
    out = subprocess.run(["cuobjdump", "--list-elf", _build.SO], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("n,fanout,fill", [(0, 64, 1.0), (1, 64, 1.0), (64, 64, 1.0), (65, 64, 1.0),
                                           (50_000_000, 64, 1.0), (16_392_000, 14, 0.9), (12345, 9, 0.9),
                                           (1000, 10, 0.9), (5000, 50, 0.9), (5000, 100, 0.9), (777, 7, 0.3)])
def test_tree_shape_closed_form(n, fanout, fill):
    from paper_2009_11543_b200 import cks
    s = cks.bulkload_shape(n, fanout, fill)
    per = int(fanout * fill)
    lv = oracle.tree_levels(n, per)
    assert s.height == len(lv) and s.per_node == per
    assert [int(s.level_nodes[i]) for i in range(s.height)] == lv
    assert int(s.total_nodes) == sum(lv)


def test_fill_is_double():
    # fill crosses the ABI as a double, so the library's entries per node agree with any
    # caller computing floor(fanout * fill) in double precision (10 x 0.9 = 9, not 8)
    from paper_2009_11543_b200 import cks
    for fanout, fill, per in [(10, 0.9, 9), (50, 0.9, 45), (100, 0.9, 90), (14, 0.9, 12), (9, 0.9, 8)]:
        assert cks.bulkload_shape(100, fanout, fill).per_node == per


@pytest.mark.parametrize("fanout,fill", [(1, 1.0), (64, 0.0), (64, 1.5), (2, 0.9)])
def test_tree_shape_rejects(fanout, fill, lib):
    from paper_2009_11543_b200 import cks
    with pytest.raises(cks.CksError):
        cks.bulkload_shape(100, fanout, fill)


def test_strerror_and_null_ctx(lib):
    lib.cks_strerror.restype = ctypes.c_char_p
    assert lib.cks_strerror(0) == b"ok"
    assert lib.cks_strerror(4) == b"CUDA error"
    assert lib.cks_ctx_destroy(None) == 1
    assert lib.cks_build(None, None, 0, 16, None, None) == 1


def test_binding_has_no_cpu_fallback():
    # the product package must not import the oracle or the generators
    pkg = os.path.join(ROOT, "paper_2009_11543_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            src = open(os.path.join(pkg, f)).read()
            assert "import oracle" not in src and "from oracle" not in src, f
            assert "cksgen" not in src, f


def test_paper_tree_shape_host():
    # NEXT-3 tree shape: host arithmetic against the oracle's level counts (INDBTAB-sized)
    from paper_2009_11543_b200 import cks
    s = cks.paper_tree_shape(16_392_000, 0.9)
    lv = oracle.paper_tree_levels(16_392_000, 12, 8)
    assert s.height == len(lv) and [int(s.level_nodes[i]) for i in range(s.height)] == lv
    assert s.per_node == 12 and s.reserved == 8 and int(s.total_nodes) == sum(lv)


def test_product_build_reads_no_environment(lib):
    # the timing-experiment knobs (one of them makes results wrong) exist only in a build
    # with -DCKS_EXPERIMENTS=1; the product library must not contain their names
    from paper_2009_11543_b200 import _build
    if os.environ.get("CKS_EXPERIMENTS") == "1":
        pytest.skip("experiments build")
    blob = open(_build.SO, "rb").read()
    for name in (b"CKS_LSD_DEBUG", b"CKS_LSD_ITEMS", b"CKS_REF_CTA", b"CKS_NO_TILE_RUNS", b"CKS_REFINE",
                 b"CKS_ROUND0_BITS"):
        assert name not in blob, name
    out = subprocess.run(["nm", "-D", _build.SO], capture_output=True, text=True).stdout
    assert " getenv" not in out
