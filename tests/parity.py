"""Parity helpers: run one seeded column through the CUDA path (C ABI via the
binding) and through the CPU oracle, and compare every output bit-exactly.

Test infrastructure only.  The oracle never sees a CUDA output as an input:
both sides start from the same datagen.Column and each packs the main codes
with its own packer (the packed words are compared too)."""
from __future__ import annotations

import numpy as np
import torch

import oracle


def to_device(col, dev="cuda"):
    import paper_1109_6885_b200 as dm
    if col.key in ("u64", "u32"):
        it = np.int64 if col.key == "u64" else np.int32
        UM = torch.from_numpy(col.main_dict.view(it).copy()).to(dev)
        D = torch.from_numpy(col.delta.view(it).copy()).to(dev)
    else:
        UM = torch.from_numpy(np.ascontiguousarray(col.main_dict).reshape(-1, 16)).to(dev)
        D = torch.from_numpy(np.ascontiguousarray(col.delta).reshape(-1, 16)).to(dev)
    codes = torch.from_numpy(col.main_codes.view(np.int32).copy()).to(dev)
    M = dm.pack_codes(codes, col.main_bits)
    return UM, M, D


def keys_np(t: torch.Tensor, key: str) -> np.ndarray:
    a = t.cpu().numpy()
    if key in ("u64", "u32"):
        return a.view(np.uint64 if key == "u64" else np.uint32)
    return a.reshape(-1, 16)


def run_gpu(col, dev="cuda"):
    import paper_1109_6885_b200 as dm
    UM, M, D = to_device(col, dev)
    r = dm.merge_column(UM, M, col.n_main, col.main_bits, D, x_tables=True, delta_dict=True)
    torch.cuda.synchronize()
    return M, r


def compare(col, gpu_M, r, ref=None, check_tables=True):
    """Element-by-element comparison; returns the oracle result."""
    ref = ref if ref is not None else oracle.merge(col, "linear")
    assert ref.status == oracle.OK, ref.status
    # packer parity (each side packs the main codes itself)
    want_M = oracle.pack(col.main_codes, col.main_bits)
    got_M = gpu_M.cpu().numpy().view(np.uint64)
    assert np.array_equal(got_M, want_M), "dm_pack_codes != oracle pack"
    assert r.merged_bits == ref.merged_bits, (r.merged_bits, ref.merged_bits)
    assert r.merged_len == ref.merged_len, (r.merged_len, ref.merged_len)
    assert r.delta_dict_len == ref.delta_dict.shape[0]
    assert np.array_equal(keys_np(r.merged_dict, col.key), ref.merged_dict), "U' differs"
    got = r.merged_codes.cpu().numpy().view(np.uint64)
    want = ref.merged_words
    if not np.array_equal(got, want):
        bad = np.nonzero(got != want)[0]
        raise AssertionError(f"M' differs in {bad.size} of {want.size} words; first at {bad[:8]}")
    if check_tables:
        assert np.array_equal(r.x_main.cpu().numpy().view(np.uint32), ref.x_main), "X_M differs"
        assert np.array_equal(r.x_delta.cpu().numpy().view(np.uint32), ref.x_delta), "X_D differs"
        assert np.array_equal(keys_np(r.delta_dict, col.key), ref.delta_dict), "U_D differs"
        assert np.array_equal(r.delta_rank.cpu().numpy().view(np.uint32), ref.delta_rank), "r differs"
    return ref
