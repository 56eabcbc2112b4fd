"""CUDA path vs the CPU oracle, element by element (bit-exact), through the C ABI.

Sizes span several tiles of every kernel (sort tile 4096/2048, merge tile 2048,
recompress chunk 4096 rows) with ragged tails; edge cases cover empty and
degenerate inputs; the configs run at BASELINE.json's full sizes where the
oracle finishes in seconds (cfg1, cfg2, cfg3, cfg4 columns) and at reduced
scale plus invariants for cfg5.
"""
import numpy as np
import pytest
import torch

import datagen
import oracle
from tests.parity import compare, run_gpu, to_device, keys_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1109_6885_b200  # noqa: F401  (fails loudly if the library is missing)
    oracle.build()


def bigint_words(codes, bits):
    s = 0
    for i, c in enumerate(codes):
        s |= int(c) << (i * bits)
    nw = (len(codes) * bits + 63) // 64
    return [(s >> (64 * w)) & ((1 << 64) - 1) for w in range(nw)]


# ----------------------------------------------------------------------- codec
@pytest.mark.parametrize("bits", list(range(1, 33)))
def test_pack_unpack_every_width(bits):
    import paper_1109_6885_b200 as dm
    rng = np.random.default_rng(bits)
    for n in (0, 1, 31, 32, 33, 1000, 4096, 4097, 100003):
        codes = rng.integers(0, 2 ** bits, size=n, dtype=np.uint64).astype(np.uint32)
        t = torch.from_numpy(codes.view(np.int32)).cuda()
        w = dm.pack_codes(t, bits).cpu().numpy().view(np.uint64)
        assert np.array_equal(w, oracle.pack(codes, bits))
        if n <= 100:
            assert w.tolist() == bigint_words(codes, bits)
        back = dm.unpack_codes(torch.from_numpy(w.view(np.int64)).cuda(), n, bits).cpu().numpy().view(np.uint32)
        assert np.array_equal(back, codes)


# ------------------------------------------------------ Step 2(b) every width pair
def _recompress_case(b, nb, n_main, n_delta, seed):
    import paper_1109_6885_b200 as dm
    rng = np.random.default_rng(seed)
    dict_len = int(min(2 ** b, 5000))
    codes = rng.integers(0, dict_len, size=n_main, dtype=np.uint64).astype(np.uint32)
    xm = rng.integers(0, 2 ** nb, size=dict_len, dtype=np.uint64).astype(np.uint32)
    nud = max(1, n_delta // 3)
    xd = rng.integers(0, 2 ** nb, size=nud, dtype=np.uint64).astype(np.uint32)
    r = rng.integers(0, nud, size=n_delta, dtype=np.uint64).astype(np.uint32)
    want_codes = np.concatenate([xm[codes], xd[r]]).astype(np.uint32)
    want = oracle.pack(want_codes, nb)
    M = torch.from_numpy(oracle.pack(codes, b).view(np.int64).copy()).cuda() if n_main else \
        torch.zeros(2, dtype=torch.int64, device="cuda")
    cap = max(dm.words(n_main + n_delta, nb), 2)
    out = torch.full((cap,), -1, dtype=torch.int64, device="cuda")
    T = lambda a: torch.from_numpy(a.view(np.int32).copy()).cuda()
    txm, txd, tr = T(xm), T(xd), T(r)  # keep the tensors alive across the call
    st = dm._lib().dm_recompress(M.data_ptr(), n_main, b, dict_len, txm.data_ptr(), txd.data_ptr(),
                                 tr.data_ptr(), n_delta, nb, out.data_ptr(), cap, torch.cuda.current_stream().cuda_stream)
    assert st == 0
    got = out.cpu().numpy().view(np.uint64)[: want.size]
    assert np.array_equal(got, want), (b, nb)


@pytest.mark.parametrize("b", list(range(1, 33)))
def test_recompress_all_width_pairs(b):
    # every (b, b') in [1,32]^2, including b > b' (input wider than minimal, reading A15)
    for nb in range(1, 33):
        _recompress_case(b, nb, 4096 * 2 + 77, 1000 + 13 * nb, seed=b * 100 + nb)


def test_recompress_seam_and_tails():
    for n_main in (0, 1, 31, 32, 33, 4095, 4096, 4097, 8191, 70001):
        for n_delta in (0, 1, 63, 4097):
            if n_main + n_delta:
                _recompress_case(21, 22, n_main, n_delta, seed=n_main + n_delta)


# ------------------------------------------------------------ whole merge, random
CASES = [
    # n_main, dict_len, n_delta, p_new
    (1000, 100, 17, 0.5),
    (100003, 5000, 4097, 0.1),
    (70001, 70000, 50001, 1.0),
    (65536, 2, 12289, 0.0),
    (200000, 30000, 300000, 0.3),
    (4096, 1, 4096, 0.001),
    (0, 1, 10000, 0.5),
    (5000, 3000, 0, 0.0),
]


@pytest.mark.parametrize("key", ["u64", "b16"])
@pytest.mark.parametrize("case", CASES)
def test_merge_random_cases(key, case):
    n_main, dict_len, n_delta, p_new = case
    for seed in (1, 2):
        col = datagen.make_random_case(seed * 7919 + n_main, n_main, dict_len, n_delta, p_new, key=key)
        M, r = run_gpu(col)
        compare(col, M, r)


@pytest.mark.parametrize("key", ["u64", "b16"])
def test_merge_wider_input_width(key):
    col = datagen.make_random_case(5, 50000, 1000, 3000, 0.2, key=key, main_bits=27)
    M, r = run_gpu(col)
    compare(col, M, r)


def test_edge_empty_main_and_delta():
    col = datagen.Column("u64", np.zeros(0, np.uint64), np.zeros(0, np.uint32), 1, np.zeros(0, np.uint64))
    M, r = run_gpu(col)
    assert r.merged_len == 0 and r.merged_bits == 1 and r.merged_codes.numel() == 0


def test_edge_empty_main_nonempty_delta():
    D = np.array([9, 3, 9, 2**64 - 1, 0, 3], dtype=np.uint64)
    col = datagen.Column("u64", np.zeros(0, np.uint64), np.zeros(0, np.uint32), 1, D)
    M, r = run_gpu(col)
    compare(col, M, r)


def test_edge_delta_all_equal_skips_every_pass():
    D = np.full(10000, 0xDEADBEEF, dtype=np.uint64)
    col = datagen.make_random_case(3, 20000, 500, 0, 0.0)
    col.delta = D
    M, r = run_gpu(col)
    compare(col, M, r)


def test_edge_delta_differs_in_one_byte_only():
    rng = np.random.default_rng(0)
    D = (np.uint64(0x1122334455667788) ^ (rng.integers(0, 256, 50000).astype(np.uint64) << np.uint64(40)))
    col = datagen.make_random_case(4, 20000, 500, 0, 0.0)
    col.delta = D.astype(np.uint64)
    M, r = run_gpu(col)
    compare(col, M, r)


def test_edge_b16_order_edges():
    strs = [b"", b"a", b"a\x00b", b"\x7f", b"\x80", b"\xff" * 16, b"ab", b"b"] * 700
    D = np.frombuffer(b"".join(s + b"\x00" * (16 - len(s)) for s in strs), np.uint8).reshape(-1, 16).copy()
    main = datagen.sort_b16(np.frombuffer(b"".join(s + b"\x00" * (16 - len(s)) for s in [b"a", b"zz", b"\x7f\x7f"]),
                                          np.uint8).reshape(-1, 16).copy())
    col = datagen.Column("b16", main, np.array([0, 1, 2, 1] * 1000, np.uint32), 2, D)
    M, r = run_gpu(col)
    compare(col, M, r)


def test_errors_code_range_and_unsorted():
    import paper_1109_6885_b200 as dm
    col = datagen.make_random_case(8, 10000, 100, 100, 0.5)
    col.main_codes = col.main_codes.copy()
    col.main_codes[5000] = 120  # >= |U_M| but < 2^7
    UM, M, D = to_device(col)
    with pytest.raises(dm.DictMergeError) as e:
        dm.merge_column(UM, M, col.n_main, col.main_bits, D)
    assert e.value.status == dm.Status.E_CODE_RANGE
    col = datagen.make_random_case(9, 10000, 100, 100, 0.5)
    md = col.main_dict.copy()
    md[40], md[41] = md[41], md[40]
    col.main_dict = md
    UM, M, D = to_device(col)
    with pytest.raises(dm.DictMergeError) as e:
        dm.merge_column(UM, M, col.n_main, col.main_bits, D)
    assert e.value.status == dm.Status.E_UNSORTED


def test_determinism_and_async_reuse():
    import paper_1109_6885_b200 as dm
    col = datagen.make_random_case(11, 300000, 20000, 30000, 0.2)
    UM, M, D = to_device(col)
    m = dm.ColumnMerger(UM, M, col.n_main, col.main_bits, D)
    outs = []
    for _ in range(3):
        m.run_async()
        r = m.result()
        outs.append((r.merged_dict.clone(), r.merged_codes.clone()))
    for d, c in outs[1:]:
        assert torch.equal(d, outs[0][0]) and torch.equal(c, outs[0][1])


def test_host_entry_point():
    import paper_1109_6885_b200 as dm
    col = datagen.make_config(1)
    ref = oracle.merge(col)
    ctx = dm.HostContext(0)
    UM = torch.from_numpy(col.main_dict.view(np.int64).copy()).pin_memory()
    D = torch.from_numpy(col.delta.view(np.int64).copy()).pin_memory()
    Mw = torch.from_numpy(oracle.pack(col.main_codes, col.main_bits).view(np.int64).copy()).pin_memory()
    Uo = torch.empty(col.dict_len + col.n_delta, dtype=torch.int64).pin_memory()
    Mo = torch.empty(dm.words(col.n_main + col.n_delta, 32), dtype=torch.int64).pin_memory()
    n, bits, nud = ctx.merge(UM, Mw, col.n_main, col.main_bits, D, Uo, Mo)
    assert n == ref.merged_len and bits == ref.merged_bits and nud == ref.delta_dict.shape[0]
    assert np.array_equal(Uo[:n].numpy().view(np.uint64), ref.merged_dict)
    assert np.array_equal(Mo[: ref.merged_words.size].numpy().view(np.uint64), ref.merged_words)
    ctx.close()


def test_row_sharded_step2_on_one_device():
    """The row-sharded path with G logical shards on one GPU: root
    Steps 1(a)/1(b)/2(a) via dm_dictionary_merge_async, then dm_recompress on each
    4096-row-aligned shard; the shards concatenate to the unsharded M'."""
    import paper_1109_6885_b200 as dm
    from paper_1109_6885_b200 import sharding
    col = datagen.make_random_case(41, 1 << 20, 1 << 16, 50001, 0.7, main_bits=18)
    UM, M, D = to_device(col)
    ref = oracle.merge(col)
    dmg = dm.DictionaryMerger(UM, col.n_main, col.main_bits, D)
    dmg.run_async()
    h = dmg.header()
    assert h.status == 0 and h.merged_bits == ref.merged_bits and h.merged_dict_len == ref.merged_len
    assert np.array_equal(keys_np(dmg.U[: h.merged_dict_len], "u64"), ref.merged_dict)
    for g in (1, 2, 3, 8):
        parts = []
        for s in sharding.plan_row_shards(col.n_main, col.n_delta, g):
            mslice = M[s.in_word(col.main_bits):] if s.n_main else M
            parts.append(dm.recompress(mslice, s.n_main, col.main_bits, col.dict_len, dmg.XM, dmg.XD,
                                       dmg.R[s.delta_begin:], s.n_delta, h.merged_bits))
        got = torch.cat(parts).cpu().numpy().view(np.uint64)
        # each shard's last word is complete except the final shard's
        assert np.array_equal(got, ref.merged_words), g


def test_merge_table_matches_per_column():
    import paper_1109_6885_b200 as dm
    cols = [datagen.make_config(4, scale=0.002, column=j) for j in (0, 7, 100, 239, 240, 299)]
    dev = [to_device(c) for c in cols]
    res = dm.merge_table([(UM, M, c.n_main, c.main_bits, D) for c, (UM, M, D) in zip(cols, dev)])
    for c, r in zip(cols, res):
        ref = oracle.merge(c)
        assert r.merged_bits == ref.merged_bits
        assert np.array_equal(keys_np(r.merged_dict, c.key), ref.merged_dict)
        assert np.array_equal(r.merged_codes.cpu().numpy().view(np.uint64), ref.merged_words)


# ------------------------------------------------------------------- the configs
def test_cfg1_full():
    col = datagen.make_config(1)
    M, r = run_gpu(col)
    ref = compare(col, M, r)
    ref_def = oracle.merge(col, "definitional")
    assert np.array_equal(ref_def.merged_words, ref.merged_words)


@pytest.mark.slow
def test_cfg2_full():
    col = datagen.make_config(2)
    M, r = run_gpu(col)
    ref = compare(col, M, r)
    assert r.merged_bits == 24


@pytest.mark.slow
def test_cfg3_full():
    col = datagen.make_config(3)
    M, r = run_gpu(col)
    ref = compare(col, M, r)
    assert ref.merged_bits == 21


# Seed S + 1 (SURVEY §8d "Seeds": every parity run repeats at S + 1), full size
@pytest.mark.slow
@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_configs_full_seed_s_plus_1(cfg):
    col = datagen.make_config(cfg, seed=datagen.BASE_SEED + 1)
    M, r = run_gpu(col)
    compare(col, M, r)


@pytest.mark.slow
def test_cfg2e4_full():
    """cfg2's shape with 4-byte values (E = 4; NEXT4) at full size."""
    col = datagen.make_config_e4()
    M, r = run_gpu(col)
    ref = compare(col, M, r)
    assert ref.merged_bits == 24


@pytest.mark.slow
def test_cfg4_columns_full_size():
    for j in (0, 3, 120, 239, 240, 271, 299):
        col = datagen.make_config(4, column=j)
        M, r = run_gpu(col)
        compare(col, M, r, check_tables=False)


def test_cfg5_reduced_scale_width_growth():
    # cfg5 shape (all-unique permuted main, all-new delta) at 2^20 rows: b' grows
    col = datagen.make_config(5, scale=1 / 1024)
    M, r = run_gpu(col)
    ref = compare(col, M, r)
    assert r.merged_len == col.dict_len + col.n_delta


@pytest.mark.parametrize("key,n_main,dict_len,n_delta,p_new", [
    ("u64", 13_000_003, 300_000, 200_001, 0.2),    # 3 chunks, ragged
    ("b16", 4_000_000, 50_000, 9_000_001, 0.6),    # delta rows span chunks
    ("u32", 9_000_000, 2_000, 1, 1.0),
])
def test_host_entry_point_pipelined(key, n_main, dict_len, n_delta, p_new):
    """dm_merge_column_host over several row chunks (copy-in / compute / copy-out
    pipeline): U', M' and the requested tables bit-exact; pinned and pageable."""
    import paper_1109_6885_b200 as dm
    col = datagen.make_random_case(5 + n_delta, n_main, dict_len, n_delta, p_new, key=key)
    ref = oracle.merge(col)
    E = col.key_bytes
    host = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64 if E == 8 else np.int32 if E == 4
                                                                    else np.uint8).copy())
    UM, D = host(col.main_dict), host(col.delta)
    if E == 16:
        UM, D = UM.reshape(-1, 16), D.reshape(-1, 16)
    Mw = torch.from_numpy(oracle.pack(col.main_codes, col.main_bits).view(np.int64).copy())
    for pinned in (True, False):
        ctx = dm.HostContext(0)
        args = [t.pin_memory() if pinned else t for t in (UM, Mw, D)]
        Uo = torch.empty((col.dict_len + col.n_delta,) + tuple(UM.shape[1:]), dtype=UM.dtype)
        Mo = torch.empty(dm.words(col.n_main + col.n_delta, 32), dtype=torch.int64)
        if pinned:
            Uo, Mo = Uo.pin_memory(), Mo.pin_memory()
        n, bits, nud = ctx.merge(args[0], args[1], col.n_main, col.main_bits, args[2], Uo, Mo)
        assert n == ref.merged_len and bits == ref.merged_bits and nud == ref.delta_dict.shape[0]
        assert np.array_equal(keys_np(Uo[:n], col.key), ref.merged_dict)
        assert np.array_equal(Mo[: ref.merged_words.size].numpy().view(np.uint64), ref.merged_words)
        ctx.close()


def test_host_entry_rejects_undersized_host_outputs():
    """dm_merge_column_host (ADVICE): host outputs are checked before any copy --
    NULL U' / M' buffers are DM_E_INVALID, capacities below dict_len + n_delta
    keys / dm_merged_codes_cap_words(in) words are DM_E_CAPACITY."""
    import ctypes
    import paper_1109_6885_b200 as dm
    col = datagen.make_random_case(77, 50_000, 3000, 4000, 0.4)
    UM = torch.from_numpy(col.main_dict.view(np.int64).copy())
    D = torch.from_numpy(col.delta.view(np.int64).copy())
    Mw = torch.from_numpy(oracle.pack(col.main_codes, col.main_bits).view(np.int64).copy())
    cin = dm._make_in(UM, Mw, col.n_main, col.main_bits, D)
    need = dm.merged_codes_cap_words(cin)
    Uo = torch.empty(col.dict_len + col.n_delta, dtype=torch.int64)
    Mo = torch.empty(need, dtype=torch.int64)
    ctx = dm.HostContext(0)
    L = dm._lib()
    cases = [(dm._Out(None, Uo.numel(), Mo.data_ptr(), need), dm.Status.E_INVALID),
             (dm._Out(Uo.data_ptr(), Uo.numel(), None, need), dm.Status.E_INVALID),
             (dm._Out(Uo.data_ptr(), Uo.numel() - 1, Mo.data_ptr(), need), dm.Status.E_CAPACITY),
             (dm._Out(Uo.data_ptr(), Uo.numel(), Mo.data_ptr(), need - 1), dm.Status.E_CAPACITY),
             (dm._Out(Uo.data_ptr(), Uo.numel(), Mo.data_ptr(), need), dm.Status.OK)]
    for cout, want in cases:
        assert L.dm_merge_column_host(ctx.h, ctypes.byref(cin), ctypes.byref(cout)) == want
    ref = oracle.merge(col)
    assert np.array_equal(Mo[: ref.merged_words.size].numpy().view(np.uint64), ref.merged_words)
    ctx.close()


def test_recompress_rejects_empty_dictionary_on_device():
    """dm_recompress with N_M > 0 and |U_M| = 0 (ADVICE): DM_E_INVALID, no launch."""
    import paper_1109_6885_b200 as dm
    M = torch.zeros(16, dtype=torch.int64, device="cuda")
    xm = torch.zeros(4, dtype=torch.int32, device="cuda")
    with pytest.raises(dm.DictMergeError) as e:
        dm.recompress(M, 10, 4, 0, xm, xm, xm, 0, 4)
    assert e.value.status == dm.Status.E_INVALID
