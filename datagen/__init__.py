"""Seeded synthetic inputs for the dictionary merge (shared by the oracle tests and the CUDA path).

This module holds NONE of the merge's arithmetic: no dictionary merge, no
translation tables, no bit packing.  (``width_hint`` only labels the generated
main vector with the input code width the configs state; neither side uses it
to compute an output.)  It only draws the three
inputs a merge consumes -- the sorted main dictionary U_M, the per-row main
codes (as plain u32, unpacked) and the raw delta values D in insertion order --
with the shapes and distributions of BASELINE.json's five configs (recipe:
SURVEY.md Appendix B, restated in DESIGN.md "Input recipe").

Everything is counter-based (SplitMix64 finaliser over (seed, stream, index)),
so any element can be regenerated independently and both sides of a parity
test see byte-identical inputs.

Keys:
  * ``"u64"``  -- numpy ``uint64`` arrays, compared as unsigned integers.
  * ``"b16"``  -- numpy ``uint8`` arrays of shape (n, 16): fixed-width
    zero-padded byte strings, compared bytewise (memcmp order).

The main codes are returned unpacked; each side packs them with its own
packer (the oracle's scalar packer, the library's ``dm_pack_codes``).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

__all__ = [
    "mix64", "rnd", "uniform_below", "uniform01", "bernoulli", "perm_pow2", "perm_below",
    "Column", "BASE_SEED", "config_seed", "make_config", "make_random_case",
    "make_string_pool", "bytes_to_hilo", "hilo_to_bytes", "sort_b16", "ALPHABET",
    "width_hint",
]

BASE_SEED = 11096885  # SURVEY.md §8d "Seeds"
GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
ALPHABET = np.frombuffer(
    b"0123456789ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz", dtype=np.uint8)
assert ALPHABET.size == 62


def _u64(x) -> np.ndarray:
    return np.asarray(x, dtype=np.uint64)


def mix64(x) -> np.ndarray:
    """SplitMix64 finaliser (a bijection on u64)."""
    z = _u64(x).copy()
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= _M1
        z ^= z >> np.uint64(27)
        z *= _M2
        z ^= z >> np.uint64(31)
    return z


def rnd(seed: int, stream: int, idx) -> np.ndarray:
    """Counter-based u64 draw number ``idx`` of ``stream`` under ``seed``."""
    with np.errstate(over="ignore"):
        key = mix64(_u64(seed & 0xFFFFFFFFFFFFFFFF) * GOLDEN + _u64(stream & 0xFFFFFFFFFFFFFFFF))
        return mix64(key + _u64(idx) * GOLDEN)


def uniform_below(seed: int, stream: int, idx, n: int) -> np.ndarray:
    """Integer uniform on [0, n) for n < 2^32 (multiply-shift of the top 32 bits)."""
    assert 0 < n <= (1 << 32)
    hi = rnd(seed, stream, idx) >> np.uint64(32)
    with np.errstate(over="ignore"):
        return (hi * np.uint64(n)) >> np.uint64(32)


def uniform01(seed: int, stream: int, idx) -> np.ndarray:
    return (rnd(seed, stream, idx) >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))


def bernoulli(seed: int, stream: int, idx, p: float) -> np.ndarray:
    return uniform01(seed, stream, idx) < p


def perm_pow2(seed: int, j, k: int) -> np.ndarray:
    """A keyed bijection on [0, 2^k): odd-multiply / xorshift / add rounds mod 2^k."""
    assert 1 <= k <= 64
    mask = np.uint64((1 << k) - 1) if k < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)
    x = _u64(j).copy() & mask
    sh = np.uint64(max(1, (k + 1) // 2))
    with np.errstate(over="ignore"):
        for r in range(4):
            m = int(rnd(seed, 900 + r, 0)) | 1
            a = int(rnd(seed, 950 + r, 0))
            x = (x * np.uint64(m)) & mask
            x ^= x >> sh
            x = (x + np.uint64(a)) & mask
    return x


def perm_below(seed: int, j, n: int) -> np.ndarray:
    """A keyed bijection on [0, n) by cycle-walking perm_pow2 with k = ceil(log2 n)."""
    assert n >= 1
    if n == 1:
        return np.zeros_like(_u64(j))
    k = max(1, (n - 1).bit_length())
    x = perm_pow2(seed, j, k)
    bad = x >= np.uint64(n)
    while bad.any():
        x[bad] = perm_pow2(seed, x[bad], k)
        bad = x >= np.uint64(n)
    return x


# ----------------------------------------------------------------------------- byte keys

def bytes_to_hilo(b: np.ndarray):
    """(n,16) u8 -> (hi, lo) u64 pair whose numeric order equals memcmp order."""
    b = np.ascontiguousarray(b, dtype=np.uint8).reshape(-1, 16)
    hi = b[:, :8].copy().view(">u8").ravel().astype(np.uint64)
    lo = b[:, 8:].copy().view(">u8").ravel().astype(np.uint64)
    return hi, lo


def hilo_to_bytes(hi: np.ndarray, lo: np.ndarray) -> np.ndarray:
    out = np.empty((hi.size, 16), dtype=np.uint8)
    out[:, :8] = hi.astype(">u8").view(np.uint8).reshape(-1, 8)
    out[:, 8:] = lo.astype(">u8").view(np.uint8).reshape(-1, 8)
    return out


def _b16_struct(b: np.ndarray) -> np.ndarray:
    hi, lo = bytes_to_hilo(b)
    s = np.empty(hi.size, dtype=[("hi", "<u8"), ("lo", "<u8")])
    s["hi"] = hi
    s["lo"] = lo
    return s


def sort_b16(b: np.ndarray) -> np.ndarray:
    """Sort 16-byte keys bytewise (input construction only)."""
    s = _b16_struct(b)
    order = np.argsort(s, kind="stable")
    return np.ascontiguousarray(b[order])


def make_string_pool(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    """``count`` candidate strings (draws start..start+count-1): length U{8..16},
    chars uniform over 0-9A-Za-z, zero padded to 16 bytes (reading A14)."""
    idx = np.arange(start, start + count, dtype=np.uint64)
    length = 8 + (rnd(seed, stream, idx) % np.uint64(9)).astype(np.int64)
    out = np.zeros((count, 16), dtype=np.uint8)
    for p in range(16):
        ch = ALPHABET[(rnd(seed, stream + 1 + p, idx) % np.uint64(62)).astype(np.int64)]
        out[:, p] = np.where(p < length, ch, 0)
    return out


def _distinct_strings(seed: int, stream: int, count: int, exclude: Optional[np.ndarray] = None) -> np.ndarray:
    """First ``count`` distinct strings of a draw sequence (in draw order), skipping ``exclude``."""
    got = np.zeros((0, 16), dtype=np.uint8)
    start = 0
    excl = _b16_struct(exclude) if exclude is not None and len(exclude) else None
    while got.shape[0] < count:
        need = count - got.shape[0]
        batch = make_string_pool(seed, stream, start, need + need // 64 + 16)
        start += batch.shape[0]
        cand = np.concatenate([got, batch])
        s = _b16_struct(cand)
        _, first = np.unique(s, return_index=True)
        keep = np.sort(first)
        cand = cand[keep]
        if excl is not None:
            cand = cand[~np.isin(_b16_struct(cand), excl)]
        got = cand[:count]
    return got


# ----------------------------------------------------------------------------- columns

@dataclasses.dataclass
class Column:
    """One column's merge inputs (unpacked codes; each side packs them itself)."""
    key: str                    # "u64" | "u32" | "b16"
    main_dict: np.ndarray       # sorted, unique. u64 (n,) or u8 (n,16)
    main_codes: np.ndarray      # u32 (N_M,), each < len(main_dict)
    main_bits: int              # code width of the packed main vector
    delta: np.ndarray           # u64 (N_D,) or u8 (N_D,16), insertion order
    name: str = ""

    @property
    def key_bytes(self) -> int:
        return {"u64": 8, "u32": 4}.get(self.key, 16)

    @property
    def n_main(self) -> int:
        return int(self.main_codes.shape[0])

    @property
    def n_delta(self) -> int:
        return int(self.delta.shape[0])

    @property
    def dict_len(self) -> int:
        return int(self.main_dict.shape[0])


def width_hint(n: int) -> int:
    """Input code width used by the generator for a main dictionary of n entries
    (the configs state widths: cfg1 14, cfg2 24, cfg3 20, cfg5 30).  Integer only:
    smallest w >= 1 with 2^w >= n."""
    w = 1
    while (1 << w) < n:
        w += 1
    return w


def config_seed(cfg: int, seed: int = BASE_SEED) -> int:
    return seed + 1000 * cfg


def _u64_column(seed, n_main, dict_len, n_delta, p_new, value_bits, code_dist="uniform",
                main_bits=None, name=""):
    j = np.arange(dict_len, dtype=np.uint64)
    main_dict = np.sort(perm_pow2(seed, j, value_bits))
    if dict_len == 0:
        assert n_main == 0
        p_new = 1.0
        codes = np.zeros(0, dtype=np.uint32)
    elif code_dist == "uniform":
        codes = uniform_below(seed, 1, np.arange(n_main, dtype=np.uint64), dict_len).astype(np.uint32)
    elif code_dist == "perm":
        codes = perm_below(seed + 7, np.arange(n_main, dtype=np.uint64), dict_len).astype(np.uint32)
    else:
        raise ValueError(code_dist)
    kidx = np.arange(n_delta, dtype=np.uint64)
    is_new = bernoulli(seed, 2, kidx, p_new)
    t = np.maximum(np.cumsum(is_new) - 1, 0)  # running count of new values
    new_vals = perm_pow2(seed, np.uint64(dict_len) + t.astype(np.uint64), value_bits)
    if dict_len > 0:
        reuse = main_dict[uniform_below(seed, 3, kidx, dict_len).astype(np.int64)]
    else:
        reuse = new_vals
    delta = np.where(is_new, new_vals, reuse).astype(np.uint64)
    mb = main_bits if main_bits is not None else width_hint(max(dict_len, 1))
    return Column("u64", main_dict, codes, mb, delta, name)


def _zipf_cdf(n: int, s: float = 1.0) -> np.ndarray:
    w = 1.0 / np.power(np.arange(1, n + 1, dtype=np.float64), s)
    c = np.cumsum(w)
    return c / c[-1]


def _zipf_codes(seed, stream, count, dict_len, cdf):
    u = uniform01(seed, stream, np.arange(count, dtype=np.uint64))
    rank = np.searchsorted(cdf, u, side="right")
    rank = np.minimum(rank, dict_len - 1).astype(np.uint64)
    return perm_below(seed + 17, rank, dict_len).astype(np.uint32)


def _b16_column(seed, n_main, dict_len, n_delta, p_new, code_dist="uniform", main_bits=None, name=""):
    main_dict = sort_b16(_distinct_strings(seed, 100, dict_len))
    if code_dist == "zipf":
        cdf = _zipf_cdf(dict_len)
        codes = _zipf_codes(seed, 1, n_main, dict_len, cdf)
    else:
        cdf = None
        codes = uniform_below(seed, 1, np.arange(n_main, dtype=np.uint64), dict_len).astype(np.uint32)
    kidx = np.arange(n_delta, dtype=np.uint64)
    is_new = bernoulli(seed, 2, kidx, p_new)
    n_new = int(is_new.sum())
    fresh = _distinct_strings(seed, 200, n_new, exclude=main_dict)
    delta = np.empty((n_delta, 16), dtype=np.uint8)
    delta[is_new] = fresh
    n_re = n_delta - n_new
    if code_dist == "zipf":
        rc = _zipf_codes(seed, 3, n_re, dict_len, cdf)
    else:
        rc = uniform_below(seed, 3, np.arange(n_re, dtype=np.uint64), dict_len).astype(np.uint32)
    delta[~is_new] = main_dict[rc.astype(np.int64)]
    mb = main_bits if main_bits is not None else width_hint(max(dict_len, 1))
    return Column("b16", main_dict, codes, mb, delta, name)


def _scaled(n: int, scale: float, lo: int = 1) -> int:
    return max(lo, int(round(n * scale)))


def cfg4_column_params(j: int, seed: Optional[int] = None):
    """cfg4 column j: (column seed, cardinality log-uniform on [2, 1e7], key type, new-value
    fraction: 1% below 2^16 distinct values else 10%, reading A13)."""
    s = config_seed(4, BASE_SEED if seed is None else seed)
    sj = int(mix64(np.uint64(s + 4000 + j)))
    u = float(uniform01(sj, 5, 0))
    card = max(2, int(round(math.exp(math.log(2) + u * (math.log(10**7) - math.log(2))))))
    return sj, card, ("u64" if j < 240 else "b16"), (0.01 if card < (1 << 16) else 0.10)


def make_config(cfg: int, seed: Optional[int] = None, scale: float = 1.0, column: Optional[int] = None):
    """Inputs for BASELINE.json configs[cfg-1] (cfg in 1..5).

    ``scale`` < 1 shrinks row and dictionary counts proportionally (parity tests
    at oracle-friendly sizes); ``scale == 1`` is the config as stated.
    cfg4 returns a list of 300 Columns (or only ``column`` if given).
    """
    s = config_seed(cfg, BASE_SEED if seed is None else seed)
    if cfg == 1:
        return _u64_column(s, _scaled(10**6, scale), _scaled(10**4, scale, 2), _scaled(10**4, scale),
                           0.5, 40, main_bits=14 if scale == 1.0 else None, name="cfg1")
    if cfg == 2:
        return _u64_column(s, _scaled(10**8, scale), _scaled(10**7, scale, 2), _scaled(10**6, scale),
                           0.1, 48, main_bits=24 if scale == 1.0 else None, name="cfg2")
    if cfg == 3:
        return _b16_column(s, _scaled(10**8, scale), _scaled(10**6, scale, 2), _scaled(5 * 10**6, scale),
                           0.2, code_dist="zipf", main_bits=20 if scale == 1.0 else None, name="cfg3")
    if cfg == 4:
        cols = []
        rng_cols = range(300) if column is None else [column]
        for j in rng_cols:
            sj, card, key, p_new = cfg4_column_params(j, seed)
            card = _scaled(card, scale, 2) if scale != 1.0 else card
            n_m, n_d = _scaled(10**7, scale), _scaled(10**5, scale)
            if j < 240:
                c = _u64_column(sj, n_m, card, n_d, p_new, 64, name=f"cfg4.col{j}")
            else:
                c = _b16_column(sj, n_m, card, n_d, p_new, name=f"cfg4.col{j}")
            cols.append(c)
        return cols if column is None else cols[0]
    if cfg == 5:
        # Reading A12: N_M = |U_M| = 2^30, codes a permutation, 5e7 all-new delta values.
        n = _scaled(1 << 30, scale, 2)
        nd = _scaled(5 * 10**7, scale)
        return _u64_column(s, n, n, nd, 1.0, 64, code_dist="perm",
                           main_bits=30 if scale == 1.0 else None, name="cfg5")
    raise ValueError(cfg)


def u32_column(col: Column) -> Column:
    """A u64 column whose values are < 2^32, as 4-byte keys (the paper's E = 4)."""
    assert col.key == "u64" and (col.main_dict.size == 0 or int(col.main_dict.max()) < 2 ** 32)
    assert col.delta.size == 0 or int(col.delta.max()) < 2 ** 32
    return Column("u32", col.main_dict.astype(np.uint32), col.main_codes, col.main_bits,
                  col.delta.astype(np.uint32), col.name)


def make_config_e4(seed: Optional[int] = None, scale: float = 1.0) -> Column:
    """cfg2's shape with 4-byte values (the paper's E = 4 of its Fig 8 value-length
    sweep): U_M = 1e7 distinct values in [0, 2^32)."""
    s = config_seed(2, BASE_SEED if seed is None else seed) + 4
    return u32_column(_u64_column(s, _scaled(10**8, scale), _scaled(10**7, scale, 2), _scaled(10**6, scale), 0.1, 32,
                                  main_bits=24 if scale == 1.0 else None, name="cfg2e4"))


def make_random_case(seed: int, n_main: int, dict_len: int, n_delta: int, p_new: float,
                     key: str = "u64", value_bits: int = 64, main_bits: Optional[int] = None) -> Column:
    """A generic random column (parity sweeps and edge cases)."""
    if key == "u64":
        return _u64_column(seed, n_main, dict_len, n_delta, p_new, value_bits, main_bits=main_bits,
                           name=f"rand{seed}")
    if key == "u32":
        return u32_column(_u64_column(seed, n_main, dict_len, n_delta, p_new, min(value_bits, 32),
                                      main_bits=main_bits, name=f"rand{seed}"))
    return _b16_column(seed, n_main, dict_len, n_delta, p_new, main_bits=main_bits, name=f"rand{seed}")


def make_clustered_case(seed: int, n_main: int, dict_len: int, n_delta: int, key: str = "u64") -> Column:
    """A column whose new delta values cluster: U_M[i] = 1000 (i + 1), and about half
    of the new values land in a few gaps of U_M (dozens per gap), the rest spread
    uniformly; 30% of the tuples reuse main values.  Exercises dense insertion
    runs (many new values between two neighbouring main values)."""
    SP = 1000
    UM = (np.arange(dict_len, dtype=np.uint64) + np.uint64(1)) * np.uint64(SP)
    n_new = int(n_delta * 0.7)
    n_hot = max(1, n_new // 60)  # gaps receiving ~30 new values each
    hot = uniform_below(seed, 1, np.arange(n_hot, dtype=np.uint64), dict_len + 1)
    gap = np.concatenate([np.repeat(hot, 30), uniform_below(seed, 2, np.arange(max(n_new - 30 * n_hot, 0),
                                                                                dtype=np.uint64), dict_len + 1)])
    off = uniform_below(seed, 3, np.arange(gap.size, dtype=np.uint64), SP - 1) + np.uint64(1)
    new = np.unique(gap.astype(np.uint64) * np.uint64(SP) + off)
    reuse = UM[uniform_below(seed, 4, np.arange(n_delta - min(new.size, n_delta), dtype=np.uint64), dict_len)]
    D = np.concatenate([new[:n_delta], reuse])
    D = D[np.argsort(rnd(seed, 5, np.arange(D.size, dtype=np.uint64)), kind="stable")]
    codes = uniform_below(seed, 6, np.arange(n_main, dtype=np.uint64), dict_len).astype(np.uint32)
    col = Column("u64", UM, codes, width_hint(dict_len), D.astype(np.uint64), f"clustered{seed}")
    return u32_column(col) if key == "u32" else col
