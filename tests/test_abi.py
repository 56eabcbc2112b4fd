"""The C-ABI library: it builds, loads without a GPU, and exports every symbol
include/*.h declares; host-only helpers agree with the closed forms.  Also the
separation rules: the product path never imports the oracle and vice versa."""
import ctypes
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        txt = open(h).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        for m in re.finditer(r"^[A-Za-z_][\w \*]*?\b(dm_\w+)\s*\(", txt, flags=re.M):
            syms.add(m.group(1))
    return syms


@pytest.fixture(scope="module")
def lib():
    from paper_1109_6885_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_boundary():
    s = declared_symbols()
    for need in ("dm_merge_column", "dm_merge_column_async", "dm_merge_table", "dm_recompress", "dm_width",
                 "dm_words", "dm_workspace_bytes", "dm_pack_codes", "dm_unpack_codes", "dm_merge_column_host"):
        assert need in s


def test_every_declared_symbol_is_exported(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_sm100a_only(lib):
    from paper_1109_6885_b200 import build
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_host_helpers_match_closed_forms(lib, oracle_lib):
    lib.dm_width.restype = ctypes.c_uint32
    lib.dm_width.argtypes = [ctypes.c_uint64]
    lib.dm_words.restype = ctypes.c_uint64
    lib.dm_words.argtypes = [ctypes.c_uint64, ctypes.c_uint32]
    for n in list(range(0, 3000)) + [2**k + d for k in range(12, 33) for d in (-1, 0, 1)]:
        w = lib.dm_width(n)
        assert w == (1 if n <= 1 else (n - 1).bit_length())
    for n in (0, 1, 63, 64, 65, 10**9):
        for b in (1, 13, 31, 32):
            assert lib.dm_words(n, b) == -(-n * b // 64)


def test_invalid_arguments_rejected_before_launch():
    import paper_1109_6885_b200 as dm
    L = dm._lib()
    assert L.dm_merge_column(None, None, None, 0, None) == dm.Status.E_INVALID
    cin = dm._In(7, None, 0, None, 0, 3, None, 0)  # bad key
    cout = dm._Out()
    assert L.dm_merge_column_async(ctypes.byref(cin), ctypes.byref(cout), None, 0, None, None) == dm.Status.E_INVALID
    cin = dm._In(0, 16, 10, 32, 100, 2, None, 0)  # main_bits < width(10)
    assert L.dm_merge_column_async(ctypes.byref(cin), ctypes.byref(cout), None, 0, None, None) == dm.Status.E_INVALID
    assert L.dm_pack_codes(None, 0, 33, None, None) == dm.Status.E_INVALID


def test_workspace_grows_with_delta():
    import paper_1109_6885_b200 as dm
    a = dm.workspace_bytes(dm._In(0, 16, 1000, 16, 5000, 10, 16, 100))
    b = dm.workspace_bytes(dm._In(0, 16, 1000, 16, 5000, 10, 16, 100000))
    c = dm.workspace_bytes(dm._In(1, 16, 1000, 16, 5000, 10, 16, 100000))
    assert 0 < a < b < c


def test_product_and_oracle_are_separate():
    prod = glob.glob(os.path.join(ROOT, "paper_1109_6885_b200", "**", "*.*"), recursive=True)
    for p in prod:
        if p.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
            txt = open(p).read()
            assert not re.search(r"\bimport oracle\b|from oracle\b|dm_oracle", txt), p
    for p in glob.glob(os.path.join(ROOT, "oracle", "*.*")):
        if p.endswith((".py", ".cpp", ".h")):
            txt = open(p).read()
            assert not re.search(r"import paper_1109_6885_b200|from paper_1109_6885_b200|#include.*dictmerge\.h", txt), p


def test_tuning_knobs_validated_on_the_host():
    """dm_set_tuning (include/dictmerge.h): knobs 0..7 with their value ranges;
    anything else is DM_E_INVALID.  Pure host logic (no GPU needed)."""
    import paper_1109_6885_b200 as dm
    L = dm._lib()
    hi = {0: 3, 1: 3, 2: 3, 3: 1, 5: 2, 6: 1, 7: 2}
    try:
        for k, h in hi.items():
            for v in range(h + 1):
                assert L.dm_set_tuning(k, v) == dm.Status.OK, (k, v)
            assert L.dm_set_tuning(k, h + 1) == dm.Status.E_INVALID, k
            assert L.dm_set_tuning(k, -1) == dm.Status.E_INVALID, k
        for v in (0, 7, 8):
            assert L.dm_set_tuning(4, v) == dm.Status.OK
        for v in (1, 6, 9):
            assert L.dm_set_tuning(4, v) == dm.Status.E_INVALID
        assert L.dm_set_tuning(8, 0) == dm.Status.E_INVALID
        assert L.dm_get_tuning(8) == dm.Status.E_INVALID
    finally:
        for k in range(8):
            L.dm_set_tuning(k, 0)


def test_bucket_path_workspace():
    """The Step 1(a) bucket path (knob 5) sizes its own workspace: ~N_D/4 bucket
    offsets; forcing the LSD passes (knob 5 = 1) drops them."""
    import paper_1109_6885_b200 as dm
    L = dm._lib()
    cin = dm._In(0, 16, 1000, 16, 5000, 10, 16, 1_000_000)
    try:
        L.dm_set_tuning(5, 0)
        auto = dm.workspace_bytes(cin)
        L.dm_set_tuning(5, 1)
        lsd = dm.workspace_bytes(cin)
        assert auto > lsd
        assert auto - lsd >= 4 * (1_000_000 // 8)  # bucket offsets (u32, >= N_D / 8 buckets)
    finally:
        L.dm_set_tuning(5, 0)


def test_recompress_rejects_inconsistent_dictionary_length():
    """dm_recompress / dm_recompress_xc (include/dictmerge.h): with N_M > 0 the
    dictionary length must satisfy 1 <= |U_M| < 2^32 and b >= width(|U_M|) --
    else DM_E_INVALID before any launch (|U_M| = 0 would defeat the kernels'
    code clamp).  Host-only checks, no GPU needed."""
    import paper_1109_6885_b200 as dm
    L = dm._lib()
    P = 16  # any aligned non-NULL pointer value: the call must fail before touching it
    assert L.dm_recompress(P, 100, 8, 0, P, None, None, 0, 8, P, 100, None) == dm.Status.E_INVALID
    assert L.dm_recompress(P, 100, 8, 1 << 32, P, None, None, 0, 8, P, 100, None) == dm.Status.E_INVALID
    assert L.dm_recompress(P, 100, 3, 9, P, None, None, 0, 8, P, 100, None) == dm.Status.E_INVALID  # b < width(9)
    xc = dm._Xc(P, 1, P, 32, 8, 1)
    assert L.dm_recompress_xc(P, 100, 8, 0, ctypes.byref(xc), P, None, None, 0, 8, P, 100, None) == \
        dm.Status.E_INVALID


def test_host_entry_rejects_bad_host_buffers_before_copying():
    """dm_merge_column_host checks the caller's host buffers first: NULL context
    or structs are DM_E_INVALID (the capacity rules need a context, i.e. a GPU:
    tests/test_gpu_host_api.py)."""
    import paper_1109_6885_b200 as dm
    L = dm._lib()
    assert L.dm_merge_column_host(None, None, None) == dm.Status.E_INVALID


def test_get_tuning_round_trips():
    import paper_1109_6885_b200 as dm
    assert dm.get_tuning(4) == 0
    with dm.tuning(4, 7):
        assert dm.get_tuning(4) == 7
    assert dm.get_tuning(4) == 0
    assert dm._lib().dm_get_tuning(8) == dm.Status.E_INVALID
