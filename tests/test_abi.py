"""CPU-side checks of the C ABI: the library loads, exports every symbol include/pipnn.h declares, and host
validation / workspace sizing work without a GPU (no compute calls)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pipnn.h")


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"PIPNN_API\s+[\w\s\*]+?\b(\w+)\s*\(", txt)))


def P():
    import paper_2602_21247_b200 as P

    return P


def test_header_declares_the_north_star_entry_points():
    syms = header_symbols()
    for s in ("pipnn_partition", "pipnn_leaf_pick", "hashprune_insert", "pipnn_build", "pipnn_sketch",
              "pipnn_final_prune", "pipnn_workspace_size", "pipnn_last_error"):
        assert s in syms, s


def test_library_exports_every_declared_symbol():
    so = P().LIB_PATH
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing
    for s in header_symbols():
        assert hasattr(P().lib(), s)


def test_library_is_built_for_sm100a():
    so = P().LIB_PATH
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "UTCIMMA" in sass and "UTCHMMA" in sass  # tcgen05.mma kind::i8 and kind::f16
    assert "LDTM" in sass and "UBLKCP" in sass      # tcgen05.ld and bulk async copies


def fake_points(n=1_000_000, d=128, dtype=0, metric=0):
    return P().Points(0x1000, n, d, d, dtype, metric)


def test_workspace_size_and_validation_on_host():
    import synth

    L = P().lib()
    pts = fake_points()
    bp = P().build_params_from(synth.C2.params())
    nbytes = C.c_size_t(0)
    assert L.pipnn_workspace_size(C.byref(pts), C.byref(bp), C.byref(nbytes)) == 0
    assert 1 << 28 < nbytes.value < 40 << 30
    bad = P().build_params_from(synth.C2.params())
    bad.hp.m = 17  # m must fit the 2-byte hash
    assert L.pipnn_workspace_size(C.byref(pts), C.byref(bad), C.byref(nbytes)) == P().PIPNN_EINVAL
    assert b"m must be" in L.pipnn_last_error()
    bad = P().build_params_from(synth.C2.params())
    bad.part.c_min = 400  # 3*c_min >= c_max breaks the merge bound
    assert L.pipnn_workspace_size(C.byref(pts), C.byref(bad), C.byref(nbytes)) == P().PIPNN_EINVAL
    mips_u8 = fake_points(metric=1)
    assert L.pipnn_workspace_size(C.byref(mips_u8), C.byref(bp), C.byref(nbytes)) == P().PIPNN_EINVAL
    big_d = fake_points(d=300, dtype=1)
    assert L.pipnn_workspace_size(C.byref(big_d), C.byref(bp), C.byref(nbytes)) == P().PIPNN_EUNSUPPORTED


def test_null_workspace_is_a_size_query():
    L = P().lib()
    pts = fake_points(n=5000)
    pp = P().PickParams(8)
    off = C.c_void_p(0x2000)
    rc = L.pipnn_leaf_pick(C.byref(pts), off, off, 10, 5000, C.byref(pp), off, off, None, 0, None)
    assert rc == P().PIPNN_EWORKSPACE
    assert L.pipnn_required_workspace() > 5000 * 128
