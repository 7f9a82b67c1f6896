"""The C-ABI library loads and exports every entry point include/sirius.h declares (CPU only:
no compute call is made)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sirius.h")
LIB = os.path.join(ROOT, "paper_2409_03856_b200", "libsirius.so")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:sirius_status|const char\s*\*)\s*(\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for n in ("sirius_init", "sirius_prefill", "sparse_decode_step", "correct_kernel", "kv_rewrite",
              "sirius_destroy", "sirius_last_error", "sirius_version"):
        assert n in names


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        from paper_2409_03856_b200 import build
        build.build_sirius()
    lib = ctypes.CDLL(LIB)
    for n in declared_functions():
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    for n in declared_functions():
        assert re.search(rf"\bT {n}$", out, flags=re.M), n
    lib.sirius_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.sirius_version()


def test_binding_names_match_header():
    from paper_2409_03856_b200 import sirius as S
    assert set(S.ABI_SYMBOLS) == set(declared_functions())
    for n in ("sirius_prefill", "sparse_decode_step", "correct_kernel", "kv_rewrite", "sirius_destroy"):
        assert hasattr(S.Sirius, n)


def test_sass_is_sm100a_with_tcgen05_and_bulk_copies():
    """Evidence the product path is Blackwell-native: tcgen05 MMA (UTCHMMA), TMEM loads (LDTM),
    TMA tensor loads (UTMALDG) and TMEM allocation (UTCATOMSWS) in the built library SASS."""
    if not os.path.exists(LIB):
        pytest.skip("library not built")
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", LIB], capture_output=True, text=True).stdout or \
        "arch = sm_100a" in sass
    for mnem in ("UTCHMMA", "LDTM", "UTMALDG", "UTCATOMSWS"):
        assert mnem in sass, mnem


def test_library_resolves_all_its_own_symbols():
    """Every sirius:: symbol the library references is defined in it (a kernel launcher moved or
    deleted without its callers shows up here, not at first load on the GPU box)."""
    if not os.path.exists(LIB):
        pytest.skip("library not built")
    und = subprocess.run(["nm", "-D", "--undefined-only", LIB], capture_output=True, text=True).stdout
    assert "sirius" not in und, [l for l in und.splitlines() if "sirius" in l]
