"""Compact translation table XC vs the oracle, bit-exact.

Auto placement runs with both Step 2(b) forms (knob 6: thread-per-group and
warp-per-group kernels).

XC replaces the Step 2(b) gather X_M[c] by c + #{new dictionary values inserted
at or before main position c} (the closed form of X_M; DESIGN.md
§7).  It must never change a result, so every case runs under each placement
knob (auto / plain X_M / XC with shared-memory preference / XC from L2), with
and without the translation tables requested, and is compared element by
element with the oracle.  The cases aim at the format's
edges: insertions before the first and after the last main entry, at 256- and
1024-code boundaries, blocks with exactly kXcMaxBlock (32) and 33 insertions
(flagged), list lengths 0..12 against the two-word read window, dictionary
sizes that are and are not multiples of the block sizes, and a new-value count
too large for shared memory (L2 companion kernel).
"""
import numpy as np
import pytest
import torch

import datagen
import oracle
from tests.parity import compare, run_gpu

pytestmark = pytest.mark.gpu

KNOBS = ((0, 0), (0, 1), (1, 0), (2, 0), (3, 0))  # (knob 0 placement, knob 6 Step 2(b) form)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1109_6885_b200  # noqa: F401
    oracle.build()


@pytest.fixture(autouse=True)
def _reset_knob():
    yield
    import paper_1109_6885_b200 as dm
    dm.set_tuning(0, 0)
    dm.set_tuning(6, 0)


SPACING = 1000  # U_M[i] = SPACING * (i + 1): value SPACING*p + k (0 < k < SPACING) lands before U_M[p]


def _column(n_dict, n_main, insert_at, n_reuse, seed, key="u64"):
    """insert_at: list of (position p, count) -> `count` distinct new values before U_M[p]."""
    rng = np.random.default_rng(seed)
    UM = (np.arange(n_dict, dtype=np.uint64) + 1) * np.uint64(SPACING)
    new = []
    for p, cnt in insert_at:
        ks = rng.choice(np.arange(1, SPACING), size=cnt, replace=False).astype(np.uint64)
        new.append(np.uint64(SPACING) * np.uint64(p) + ks)
    new = np.concatenate(new) if new else np.zeros(0, np.uint64)
    reuse = UM[rng.integers(0, n_dict, size=n_reuse)] if n_dict else np.zeros(0, np.uint64)
    D = np.concatenate([new, new[: len(new) // 3], reuse])  # some new values repeat
    D = D[rng.permutation(D.size)]
    codes = rng.integers(0, n_dict, size=n_main, dtype=np.uint64).astype(np.uint32)
    bits = datagen.width_hint(n_dict)
    if key == "u64":
        return datagen.Column("u64", UM, codes, bits, D)
    to16 = lambda v: datagen.hilo_to_bytes(np.zeros_like(v), v)
    return datagen.Column("b16", to16(UM), codes, bits, to16(D))


def _run_all_knobs(col):
    """Every placement knob, with X_M / X_D returned (compared too) and without:
    then a merge that reads XC from L2 does not materialise X_M at all and fills
    only the flagged superblocks' entries (k_xm_flagged), so M' checks them."""
    import paper_1109_6885_b200 as dm
    from tests.parity import to_device
    ref = None
    for k, form in KNOBS:
        dm.set_tuning(0, k)
        dm.set_tuning(6, form)
        M, r = run_gpu(col)
        ref = compare(col, M, r, ref=ref)
        UM, M, D = to_device(col)
        r = dm.merge_column(UM, M, col.n_main, col.main_bits, D)
        torch.cuda.synchronize()
        compare(col, M, r, ref=ref, check_tables=False)


def _spread(n_dict, n_new, seed):
    rng = np.random.default_rng(seed)
    pos = rng.integers(0, n_dict + 1, size=n_new)
    p, c = np.unique(pos, return_counts=True)
    return list(zip(p.tolist(), c.tolist()))


@pytest.mark.parametrize("key", ["u64", "b16"])
def test_xc_uniform_insertions(key):
    # X_M = 1.2 MB (> 96 KB smem staging) with ~1% new values: XC in shared memory
    n = 300_001
    col = _column(n, 1_000_003, _spread(n, 3000, 1), 20_000, seed=1, key=key)
    _run_all_knobs(col)


def test_xc_boundaries_and_overflow():
    n = 1024 * 80 + 77  # ragged last superblock
    ins = [(0, 5), (1, 2), (255, 3), (256, 4), (257, 1), (1023, 2), (1024, 6), (1025, 1),  # block / superblock edges
           (1024 * 3 + 10, 32),                                 # exactly kXcMaxBlock in one block
           (1024 * 5 + 300, 33),                                # one over: superblock flagged
           (1024 * 6 + 700, 6), (1024 * 6 + 701, 3),            # 9 entries: past the two-word window
           ]
    # 128 insertions in one superblock, 32 per block: fits
    ins += [(1024 * 7 + 256 * t + 5, 32) for t in range(4)]
    # every list length 0..12 at every start alignment (window edge k = 8 - start % 4)
    base = 1024 * 20
    for L in range(13):
        ins.append((base + 256 * L + 128, L))
    ins += [(n - 1, 9), (n, 11)]                               # before the last entry, after it
    col = _column(n, 400_000, [x for x in ins if x[1] > 0], 5000, seed=2)
    _run_all_knobs(col)


def test_xc_dictionary_multiple_of_superblock_and_tail_inserts():
    n = 1024 * 128  # 131072: multiple of both block sizes; new values after the last entry
    col = _column(n, 300_000, [(n, 40), (n - 256, 3), (1, 1)] + _spread(n, 500, 3), 1000, seed=3)
    _run_all_knobs(col)


@pytest.mark.parametrize("dense", [False, True])
def test_xc_block_shift(dense):
    # N_D / |U_M| > 6/256 selects 128-code blocks (cfg5's density), else 256
    n = 1024 * 50 + 3
    n_new = 4000 if dense else 150
    col = _column(n, 300_000, _spread(n, n_new, 7), 6000 if dense else 40, seed=7)
    _run_all_knobs(col)


def test_xc_too_large_for_shared_memory():
    # 300k distinct new values: XC exceeds the smem budget -> the L2 companion runs
    n = 100_000
    col = _column(n, 500_000, _spread(n, 300_000, 4), 1000, seed=4)
    _run_all_knobs(col)


def test_xc_no_new_values_and_all_new():
    n = 50_000
    _run_all_knobs(_column(n, 200_000, [], 30_000, seed=5))          # X_M = identity
    _run_all_knobs(_column(n, 200_000, _spread(n, 20_000, 6), 0, seed=6))


@pytest.mark.parametrize("cfg", [2, 3])
def test_xc_configs_scaled(cfg):
    col = datagen.make_config(cfg, scale=0.1)
    _run_all_knobs(col)


@pytest.mark.parametrize("key", ["u64", "u32"])
def test_xc_row_shards_with_exceptions(key):
    """Row-sharded Step 2 through XC (SURVEY §8e with NEXT3): the root's tables are
    copied as a receiving rank would get them, and that rank's X_M holds only the
    exception slices (flagged superblocks) -- every other entry is poisoned, so
    any read outside the exceptions breaks parity."""
    import paper_1109_6885_b200 as dm
    from paper_1109_6885_b200 import sharding
    from tests.parity import to_device
    n = 1024 * 80 + 77
    ins = [(0, 5), (1024 * 3 + 10, 32), (1024 * 5 + 300, 33), (1024 * 11 + 7, 40), (n - 1, 9), (n, 11)]
    ins += _spread(n, 800, 12)
    col = _column(n, 400_000, ins, 5000, seed=2, key="u64")
    if key == "u32":
        col = datagen.u32_column(col)
    UM, M, D = to_device(col)
    ref = oracle.merge(col)
    dmg = dm.DictionaryMerger(UM, col.n_main, col.main_bits, D)
    dmg.run_async()
    h = dmg.header()
    assert h.status == 0 and h.merged_bits == ref.merged_bits
    xc = dmg.xc()
    assert xc is not None
    ids, sl, cnt = dm.xc_exceptions_gather(xc, col.dict_len, dmg.XM)
    assert cnt >= 2  # the 33- and 40-insertion blocks
    tabs = dm.XcTables(xc.records.clone(), xc.offsets.clone(), xc.shift, xc.n_records)
    xm = torch.full((col.dict_len,), -1, dtype=torch.int32, device="cuda")
    dm.xc_exceptions_scatter(tabs, col.dict_len, ids.clone(), sl.clone(), cnt, xm)
    for g in (1, 3, 8):
        parts = []
        for s in sharding.plan_row_shards(col.n_main, col.n_delta, g):
            mslice = M[s.in_word(col.main_bits):] if s.n_main else M
            parts.append(dm.recompress_xc(mslice, s.n_main, col.main_bits, col.dict_len, tabs, xm, dmg.XD,
                                          dmg.R[s.delta_begin:], s.n_delta, h.merged_bits))
        got = torch.cat(parts).cpu().numpy().view(np.uint64)
        assert np.array_equal(got, ref.merged_words), g
