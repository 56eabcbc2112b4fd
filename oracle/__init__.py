"""Python access to the plain CPU oracle (``liboracle_dm.so``, built from dm_oracle.cpp).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_1109_6885_b200``) never imports it, and it
never imports the product path.

Functions follow the paper (arXiv 1109.6885): see dm_oracle.h for the
passage each one implements.  Parity of every function here is pinned by
tests/test_oracle_pins.py against values and laws fixed by the paper and by
mathematics (Appendix-A worked example, closed forms, brute force) -- no
function is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dm_oracle.cpp")
_LIB_PATH = os.path.join(_HERE, "liboracle_dm.so")
_lib = None

OK, E_INVALID, E_TOO_WIDE, E_UNSORTED, E_CODE_RANGE = 0, -1, -3, -4, -5


def build(force: bool = False) -> str:
    """Compile the oracle with g++ (plain -O2, single-threaded)."""
    hdr = os.path.join(_HERE, "dm_oracle.h")
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= max(os.path.getmtime(_SRC), os.path.getmtime(hdr))):
        return _LIB_PATH
    tmp = _LIB_PATH + f".tmp{os.getpid()}"
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-o", tmp, _SRC])
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class _In(ctypes.Structure):
    _fields_ = [("key_bytes", ctypes.c_uint32), ("main_dict", ctypes.c_void_p),
                ("dict_len", ctypes.c_uint64), ("main_words", ctypes.c_void_p),
                ("n_main", ctypes.c_uint64), ("main_bits", ctypes.c_uint32),
                ("delta", ctypes.c_void_p), ("n_delta", ctypes.c_uint64)]


class _Out(ctypes.Structure):
    _fields_ = [("merged_dict", ctypes.c_void_p), ("merged_len", ctypes.c_uint64),
                ("merged_bits", ctypes.c_uint32), ("merged_words", ctypes.c_void_p),
                ("x_main", ctypes.c_void_p), ("x_delta", ctypes.c_void_p),
                ("delta_dict", ctypes.c_void_p), ("delta_dict_len", ctypes.c_uint64),
                ("delta_rank", ctypes.c_void_p), ("seconds", ctypes.c_double * 4)]


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.dmo_width.restype = ctypes.c_uint32
        _lib.dmo_width.argtypes = [ctypes.c_uint64]
        _lib.dmo_words.restype = ctypes.c_uint64
        _lib.dmo_words.argtypes = [ctypes.c_uint64, ctypes.c_uint32]
        for f in ("dmo_pack", "dmo_unpack"):
            getattr(_lib, f).restype = ctypes.c_int
            getattr(_lib, f).argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p]
        for f in ("dmo_merge_linear", "dmo_merge_definitional"):
            getattr(_lib, f).restype = ctypes.c_int
            getattr(_lib, f).argtypes = [ctypes.POINTER(_In), ctypes.POINTER(_Out)]
    return _lib


def _ptr(a: Optional[np.ndarray]) -> Optional[int]:
    return None if a is None or a.size == 0 else a.ctypes.data


def width(n: int) -> int:
    return int(lib().dmo_width(n))


def words(n: int, bits: int) -> int:
    return int(lib().dmo_words(n, bits))


def pack(codes, bits: int) -> np.ndarray:
    codes = np.ascontiguousarray(codes, dtype=np.uint32)
    out = np.zeros(max(words(codes.size, bits), 1), dtype=np.uint64)
    st = lib().dmo_pack(_ptr(codes), codes.size, bits, out.ctypes.data)
    if st != OK:
        raise ValueError(f"dmo_pack failed: {st}")
    return out[: words(codes.size, bits)]


def unpack(w: np.ndarray, n: int, bits: int) -> np.ndarray:
    w = np.ascontiguousarray(w, dtype=np.uint64)
    assert w.size >= words(n, bits)
    out = np.zeros(max(n, 1), dtype=np.uint32)
    st = lib().dmo_unpack(_ptr(w), n, bits, out.ctypes.data)
    if st != OK:
        raise ValueError(f"dmo_unpack failed: {st}")
    return out[:n]


@dataclasses.dataclass
class MergeResult:
    status: int
    merged_dict: np.ndarray = None     # U'
    merged_bits: int = 0               # b'
    merged_words: np.ndarray = None    # M' (exactly words(N', b') u64)
    x_main: np.ndarray = None          # X_M
    x_delta: np.ndarray = None         # X_D (|U_D| entries)
    delta_dict: np.ndarray = None      # U_D
    delta_rank: np.ndarray = None      # r
    seconds: tuple = ()

    @property
    def merged_len(self) -> int:
        return int(self.merged_dict.shape[0])


def merge(col, mode: str = "linear", main_words: Optional[np.ndarray] = None) -> MergeResult:
    """Run the oracle on a ``datagen.Column`` (or any object with the same fields).

    ``main_words``: the packed main vector; defaults to ``pack(col.main_codes, col.main_bits)``.
    """
    E = col.key_bytes
    kdt = {4: np.uint32, 8: np.uint64}.get(E, np.uint8)
    UM = np.ascontiguousarray(col.main_dict, dtype=kdt)
    D = np.ascontiguousarray(col.delta, dtype=kdt)
    nUM = UM.shape[0]
    nD = D.shape[0]
    nM = int(col.main_codes.shape[0]) if main_words is None else int(col.n_main)
    W = pack(col.main_codes, col.main_bits) if main_words is None else np.ascontiguousarray(main_words, np.uint64)
    cap_bits = width(nUM + nD)
    shape = (lambda n: (n,)) if E in (4, 8) else (lambda n: (n, 16))
    Uo = np.zeros(shape(max(nUM + nD, 1)), dtype=kdt)
    Mo = np.zeros(max(words(nM + nD, max(cap_bits, 1)), 1), dtype=np.uint64)
    XM = np.zeros(max(nUM, 1), dtype=np.uint32)
    XD = np.zeros(max(nD, 1), dtype=np.uint32)
    UD = np.zeros(shape(max(nD, 1)), dtype=kdt)
    R = np.zeros(max(nD, 1), dtype=np.uint32)
    cin = _In(E, _ptr(UM), nUM, _ptr(W), nM, col.main_bits, _ptr(D), nD)
    cout = _Out(Uo.ctypes.data, 0, 0, Mo.ctypes.data, XM.ctypes.data, XD.ctypes.data,
                UD.ctypes.data, 0, R.ctypes.data)
    fn = lib().dmo_merge_linear if mode == "linear" else lib().dmo_merge_definitional
    st = fn(ctypes.byref(cin), ctypes.byref(cout))
    if st != OK:
        return MergeResult(st)
    n_u, n_ud, nb = int(cout.merged_len), int(cout.delta_dict_len), int(cout.merged_bits)
    return MergeResult(
        st, Uo[:n_u].copy(), nb, Mo[: words(nM + nD, nb)].copy(), XM[:nUM].copy(), XD[:n_ud].copy(),
        UD[:n_ud].copy(), R[:nD].copy(), tuple(cout.seconds))


def codes_at(main_dict: np.ndarray, delta: np.ndarray, values: np.ndarray, key_bytes: int = 8):
    """Definitional codes of `values` in U' = set_union(U_M, sorted distinct D).  Returns (codes, |U'|)."""
    L = lib()
    L.dmo_codes_at.restype = ctypes.c_int
    L.dmo_codes_at.argtypes = [ctypes.c_uint32, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64,
                               ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64)]
    kdt = {4: np.uint32, 8: np.uint64}.get(key_bytes, np.uint8)
    UM = np.ascontiguousarray(main_dict, dtype=kdt)
    D = np.ascontiguousarray(delta, dtype=kdt)
    V = np.ascontiguousarray(values, dtype=kdt)
    nv = V.shape[0]
    out = np.zeros(max(nv, 1), dtype=np.uint32)
    n = ctypes.c_uint64(0)
    st = L.dmo_codes_at(key_bytes, _ptr(UM), UM.shape[0], _ptr(D), D.shape[0], _ptr(V), nv, out.ctypes.data,
                        ctypes.byref(n))
    if st != OK:
        raise ValueError(f"dmo_codes_at failed: {st}")
    return out[:nv], int(n.value)
