"""Device-side twin of the counter-based generators (datagen/__init__.py), for
inputs too large to build on the host (cfg5: a 2^30-entry dictionary).

Same formulas, same seeds, bit-identical results (checked against the numpy
version in tests/test_datagen.py on the CPU).  u64 values live in torch.int64
tensors as raw bit patterns; right shifts are made logical by masking.
Holds none of the merge's arithmetic.
"""
from __future__ import annotations

import torch

import datagen as _np_gen

_SIGN = -(1 << 63)


def _u(x: int) -> int:
    """Python int -> the int64 with the same 64-bit pattern."""
    x &= (1 << 64) - 1
    return x - (1 << 64) if x >= (1 << 63) else x


def _shr(x: torch.Tensor, s: int) -> torch.Tensor:
    return (x >> s) & ((1 << (64 - s)) - 1)


def _mask(x: torch.Tensor, k: int) -> torch.Tensor:
    return x if k == 64 else x & ((1 << k) - 1)


def perm_pow2(seed: int, j: torch.Tensor, k: int) -> torch.Tensor:
    """Twin of datagen.perm_pow2 (keyed bijection on [0, 2^k))."""
    x = _mask(j.to(torch.int64), k)
    sh = max(1, (k + 1) // 2)
    for r in range(4):
        m = int(_np_gen.rnd(seed, 900 + r, 0)) | 1
        a = int(_np_gen.rnd(seed, 950 + r, 0))
        x = _mask(x * _u(m), k)
        x = x ^ _shr(x, sh)
        x = _mask(x + _u(a), k)
    return x


def sort_u64(x: torch.Tensor) -> torch.Tensor:
    """Sort raw u64 bit patterns in unsigned order."""
    return torch.sort(x ^ _SIGN).values ^ _SIGN


def make_cfg5(seed: int | None = None, scale: float = 1.0, device="cuda", chunk: int = 1 << 26):
    """cfg5 (reading A12): U_M = sort(perm_64(j), j < 2^30), codes = perm_30(i) (a
    permutation), D = perm_64(2^30 + t), t < 5e7 -- identical to
    datagen.make_config(5, seed, scale) but built on `device`."""
    s = _np_gen.config_seed(5, _np_gen.BASE_SEED if seed is None else seed)
    n = max(2, int(round((1 << 30) * scale)))
    nd = max(1, int(round(5 * 10**7 * scale)))
    vals = torch.empty(n, dtype=torch.int64, device=device)
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        vals[c0:c1] = perm_pow2(s, torch.arange(c0, c1, device=device, dtype=torch.int64), 64)
    main_dict = sort_u64(vals)
    del vals
    k = max(1, (n - 1).bit_length())
    if n != (1 << k):
        raise ValueError("device cfg5 twin needs a power-of-two dictionary (scale = 2^-m)")
    codes = torch.empty(n, dtype=torch.int32, device=device)
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        codes[c0:c1] = perm_pow2(s + 7, torch.arange(c0, c1, device=device, dtype=torch.int64), k).to(torch.int32)
    delta = perm_pow2(s, n + torch.arange(nd, device=device, dtype=torch.int64), 64)
    main_bits = 30 if scale == 1.0 else _np_gen.width_hint(n)
    return main_dict, codes, main_bits, delta
