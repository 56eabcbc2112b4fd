"""cfg5 at its full size (reading A12: |U_M| = N_M = 2^30, N_D = 5e7 all new -> b' = 31),
in the launch configuration bench/merge_column uses.

The oracle cannot merge 1.1e9 rows in seconds, so parity is established by
properties that pin the output uniquely at any size, checked on EVERY row, plus
the oracle on sampled rows:
  * U' strictly increasing (unsigned), |U'| = |U_M| + |D| (all new), and U'
    contains every U_M and D value  =>  U' = sorted(U_M u D) exactly (Eq 3);
  * decode(U', M')[i] = decode(U_M, M)[i] for every main row and = D[k] for every
    delta row; with U' strictly increasing this fixes each code;
  * b' = 31 (Eq 4), pad bits zero;
  * 2^20 sampled rows: codes from the oracle's definitional dmo_codes_at.
The unpacking used for the checks is plain torch arithmetic written here, not
the library's unpack kernel.
"""
import numpy as np
import pytest
import torch

import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SIGN = -(1 << 63)


def codes_at_rows(words: torch.Tensor, rows: torch.Tensor, bits: int) -> torch.Tensor:
    """Code of each row of an LSB-first u64-word stream (int64 math, logical shifts)."""
    s = rows * bits
    w = s >> 6
    o = s & 63
    lo = words[w]
    hi = words[torch.clamp(w + 1, max=words.numel() - 1)]
    oc = torch.clamp(o, min=1)
    lo_part = torch.where(o == 0, lo, (lo >> oc) & ((torch.ones_like(oc) << (64 - oc)) - 1))
    hi_part = torch.where(o + bits > 64, hi << (64 - oc), torch.zeros_like(hi))
    return (lo_part | hi_part) & ((1 << bits) - 1)


def torch_unpack(words: torch.Tensor, start: int, count: int, bits: int) -> torch.Tensor:
    rows = torch.arange(start, start + count, device=words.device, dtype=torch.int64)
    return codes_at_rows(words, rows, bits)


@pytest.fixture(scope="module")
def merged():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1109_6885_b200 as dm
    from datagen import torch_gen
    UM, codes, bits, D = torch_gen.make_cfg5(device="cuda")
    M = dm.pack_codes(codes, bits)
    r = dm.merge_column(UM, M, UM.numel(), bits, D)
    torch.cuda.synchronize()
    return UM, codes, D, r


def test_cfg5_width_and_size(merged):
    UM, codes, D, r = merged
    assert UM.numel() == 1 << 30 and D.numel() == 5 * 10**7
    assert r.merged_bits == 31
    assert r.merged_len == (1 << 30) + 5 * 10**7
    n = UM.numel() + D.numel()
    nbits = n * 31
    assert r.merged_codes.numel() == (nbits + 63) // 64
    if nbits % 64:
        last = int(r.merged_codes[-1].item()) & ((1 << 64) - 1)
        assert last >> (nbits % 64) == 0


def test_cfg5_dictionary_is_the_sorted_union(merged):
    UM, codes, D, r = merged
    U = r.merged_dict ^ SIGN  # unsigned order as signed order
    assert bool((U[1:] > U[:-1]).all())
    for vals in (UM, D):
        v = vals ^ SIGN
        idx = torch.searchsorted(U, v)
        assert bool((idx < U.numel()).all())
        assert bool((U[idx] == v).all())


def test_cfg5_decode_identity_every_row(merged):
    UM, codes, D, r = merged
    n_main = UM.numel()
    step = 1 << 26
    for c0 in range(0, n_main, step):
        c1 = min(n_main, c0 + step)
        got = torch_unpack(r.merged_codes, c0, c1 - c0, 31)
        assert bool((r.merged_dict[got] == UM[codes[c0:c1].long()]).all()), c0
    for c0 in range(0, D.numel(), step):
        c1 = min(D.numel(), c0 + step)
        got = torch_unpack(r.merged_codes, n_main + c0, c1 - c0, 31)
        assert bool((r.merged_dict[got] == D[c0:c1]).all()), c0


def test_cfg5_sampled_rows_vs_oracle(merged):
    UM, codes, D, r = merged
    n_main, n = UM.numel(), UM.numel() + D.numel()
    g = torch.Generator(device="cpu").manual_seed(11096885)
    rows = torch.cat([torch.randint(0, n_main, (1 << 20,), generator=g),
                      torch.randint(n_main, n, (1 << 16,), generator=g),
                      torch.tensor([0, n_main - 1, n_main, n - 1])]).cuda()
    main_rows = rows[rows < n_main]
    delta_rows = rows[rows >= n_main] - n_main
    vals = torch.cat([UM[codes[main_rows].long()], D[delta_rows]]).cpu().numpy().view(np.uint64)
    got = codes_at_rows(r.merged_codes, torch.cat([main_rows, delta_rows + n_main]), 31)
    want, m = oracle.codes_at(UM.cpu().numpy().view(np.uint64), D.cpu().numpy().view(np.uint64), vals)
    assert m == r.merged_len
    assert np.array_equal(got.cpu().numpy().astype(np.uint32), want)
