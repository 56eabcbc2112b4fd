"""Step 1(b) variants vs the oracle, bit-exact: the single-pass merge (default)
and the three-phase count / prefix-sum / write form, on tiles where
U_D is the smaller side, where it is the larger side, duplicate-heavy and
duplicate-free dictionaries, ties across tile boundaries, and both key types."""
import numpy as np
import pytest
import torch

import datagen
import oracle
from tests.parity import compare, run_gpu, to_device

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1109_6885_b200  # noqa: F401
    oracle.build()


@pytest.fixture(autouse=True)
def _reset():
    yield
    import paper_1109_6885_b200 as dm
    dm.set_tuning(1, 0)
    dm.set_tuning(dm.KNOB_SP_GRID, 0)


CASES = [
    # n_main, dict_len, n_delta, p_new: sparse U_D, dense U_D, all-new, all-reuse, balanced
    (300_000, 200_000, 20_000, 0.1),
    (50_000, 3_000, 200_000, 0.9),
    (10_000, 10_000, 300_000, 1.0),
    (100_000, 40_000, 100_000, 0.0),
    (100_000, 60_000, 60_000, 0.5),
    (7_000, 1, 5_000, 0.3),
]


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
@pytest.mark.parametrize("key", ["u64", "b16", "u32"])
@pytest.mark.parametrize("case", CASES)
def test_merge_variant(variant, key, case):
    import paper_1109_6885_b200 as dm
    dm.set_tuning(1, variant)
    n_main, dict_len, n_delta, p_new = case
    col = datagen.make_random_case(911 + n_delta, n_main, dict_len, n_delta, p_new, key=key)
    M, r = run_gpu(col)
    compare(col, M, r)


@pytest.mark.parametrize("key", ["u64", "b16", "u32"])
@pytest.mark.parametrize("case", CASES[:2] + CASES[3:])
def test_sparse_three_ctas_walk_all_tiles(key, case):
    """Sparse-delta Step 1(b) with knob 7 = 2: three persistent CTAs walk every
    U_M tile (the next tile prefetched while one is written)."""
    import paper_1109_6885_b200 as dm
    dm.set_tuning(1, 3)
    dm.set_tuning(dm.KNOB_SP_GRID, 2)
    n_main, dict_len, n_delta, p_new = case
    col = datagen.make_random_case(913 + n_delta, n_main, dict_len, n_delta, p_new, key=key)
    M, r = run_gpu(col)
    compare(col, M, r)


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
def test_merge_ties_at_every_tile_boundary(variant):
    # U_D = every other U_M value plus values between: duplicates land on both
    # sides of many merge-path tile boundaries (tile = 2048 merged elements)
    import paper_1109_6885_b200 as dm
    dm.set_tuning(1, variant)
    UM = np.arange(0, 40_000, 2, dtype=np.uint64) * np.uint64(3)
    D = np.concatenate([UM[::2], UM[1::5] + np.uint64(1), UM[-1:] + np.uint64(7), np.zeros(1, np.uint64)])
    rng = np.random.default_rng(5)
    D = D[rng.permutation(D.size)]
    codes = rng.integers(0, UM.size, size=60_000, dtype=np.uint64).astype(np.uint32)
    col = datagen.Column("u64", UM, codes, datagen.width_hint(UM.size), D)
    M, r = run_gpu(col)
    compare(col, M, r)


@pytest.mark.parametrize("grid", [0, 1, 2])
@pytest.mark.parametrize("shape", ["cluster", "all_below", "all_above", "boundaries", "one_tile", "many_chunks"])
def test_sparse_tiles_edges(shape, grid):
    """Step 1(b) sparse-delta tiles (knob 1 = 3): slices larger than one 2048-value
    chunk (several passes), every new value below U_M[0] or above U_M[-1], values
    equal to tile-boundary U_M entries (U_M[2048 t]) and their neighbours, a
    single partial tile.  Each under the three grids of knob 7 (one resident wave,
    one CTA per tile, three CTAs walking ~8 tiles each)."""
    import paper_1109_6885_b200 as dm
    dm.set_tuning(1, 3)
    dm.set_tuning(dm.KNOB_SP_GRID, grid)
    rng = np.random.default_rng(17)
    n_dict = 1500 if shape == "one_tile" else 50_000
    UM = (np.arange(n_dict, dtype=np.uint64) + np.uint64(1)) * np.uint64(1000)
    if shape == "cluster":       # 9000 new values in one gap (5 chunks) + some spread
        D = np.concatenate([np.uint64(1000 * 777) + rng.choice(np.arange(1, 1000, dtype=np.uint64) * np.uint64(1),
                                                                999, replace=False),
                            UM[rng.integers(0, n_dict, 3000)]])
    elif shape == "many_chunks":  # a slice of ~7000 values inside one tile: new and reused mixed
        base = np.uint64(1000 * 4100)
        D = np.concatenate([base + rng.choice(2_000_000, 7000, replace=False).astype(np.uint64) // np.uint64(1000) *
                            np.uint64(1000) + np.uint64(500), UM[4096:6000]])
    elif shape == "all_below":
        D = rng.choice(999, 600, replace=False).astype(np.uint64) + np.uint64(1)
    elif shape == "all_above":
        D = UM[-1] + rng.choice(10**6, 5000, replace=False).astype(np.uint64) + np.uint64(1)
    elif shape == "boundaries":
        t = np.arange(0, n_dict, 2048)
        D = np.concatenate([UM[t], UM[t] - np.uint64(1), UM[t] + np.uint64(1), UM[np.minimum(t + 2047, n_dict - 1)]])
    else:
        D = np.concatenate([UM[::7], UM[3::11] + np.uint64(5), np.zeros(1, np.uint64)])
    D = np.unique(D)[: max(1, n_dict // 2)]
    D = np.concatenate([D, D[::3]])
    D = D[rng.permutation(D.size)]
    codes = rng.integers(0, n_dict, size=80_000, dtype=np.uint64).astype(np.uint32)
    col = datagen.Column("u64", UM, codes, datagen.width_hint(n_dict), D)
    M, r = run_gpu(col)
    compare(col, M, r)


# ------------------------------------------------- Step 1(a) dedup front end (NEXT1)
@pytest.fixture()
def _reset_dedup():
    yield
    import paper_1109_6885_b200 as dm
    dm.set_tuning(2, 0)


DEDUP_CASES = CASES + [
    (50_000, 1000, 120_000, 0.01),   # heavy repeats: ~1.2k distinct of 120k
    (1000, 5, 70_000, 0.0),          # 5 distinct values
    (0, 1, 9_000, 1.0),              # empty main
]


@pytest.mark.parametrize("key", ["u64", "b16"])
@pytest.mark.parametrize("case", DEDUP_CASES)
def test_dedup_front_end(key, case, _reset_dedup):
    import paper_1109_6885_b200 as dm
    dm.set_tuning(2, 2)  # always deduplicate
    n_main, dict_len, n_delta, p_new = case
    col = datagen.make_random_case(311 + n_delta, n_main, dict_len, n_delta, p_new, key=key)
    M, r = run_gpu(col)
    compare(col, M, r)


def test_dedup_all_equal_and_zipf_strings(_reset_dedup):
    import paper_1109_6885_b200 as dm
    dm.set_tuning(2, 0)  # auto: on for 16-byte keys with N_D >= 65536
    col = datagen.make_config(3, scale=0.02)  # Zipf reuse, 100k delta strings
    M, r = run_gpu(col)
    compare(col, M, r)
    col = datagen.make_random_case(3, 20000, 500, 0, 0.0, key="b16")
    col.delta = np.repeat(col.main_dict[7:8], 70_000, axis=0)  # one value, 70k times
    M, r = run_gpu(col)
    compare(col, M, r)


# ------------------------------------------- NEXT4: 4-byte keys and the naive Step 2
@pytest.mark.parametrize("case", CASES)
def test_u32_keys(case):
    n_main, dict_len, n_delta, p_new = case
    col = datagen.make_random_case(733 + n_delta, n_main, dict_len, n_delta, p_new, key="u32")
    M, r = run_gpu(col)
    compare(col, M, r)


def test_u32_order_edges():
    UM = np.array([0, 1, 2**31 - 1, 2**31, 2**32 - 2], dtype=np.uint32)
    D = np.array([2**32 - 1, 2**31 + 1, 0, 5, 2**32 - 1, 2**31 - 1], dtype=np.uint32)
    codes = np.arange(5, dtype=np.uint32).repeat(7)
    col = datagen.Column("u32", UM, codes, 3, D)
    M, r = run_gpu(col)
    compare(col, M, r)


@pytest.fixture()
def _naive():
    import paper_1109_6885_b200 as dm
    dm.set_tuning(3, 1)
    yield
    dm.set_tuning(3, 0)


@pytest.mark.parametrize("key", ["u64", "b16", "u32"])
@pytest.mark.parametrize("case", CASES[:4] + [(100_003, 5000, 4097, 0.1)])
def test_naive_step2(key, case, _naive):
    n_main, dict_len, n_delta, p_new = case
    col = datagen.make_random_case(97 + n_main, n_main, dict_len, n_delta, p_new, key=key)
    M, r = run_gpu(col)
    compare(col, M, r)


# ------------------------------------------------- probe-first Step 1(a) (NEXT1)
@pytest.fixture()
def _reset_probe():
    yield
    import paper_1109_6885_b200 as dm
    dm.set_tuning(2, 0)


PROBE_CASES = [
    # key, n_main, dict_len, n_delta, p_new
    ("b16", 300_000, 40_000, 200_000, 0.2),   # cfg3-like: skewed reuse, some new
    ("b16", 50_000, 3_000, 100_000, 0.0),     # every delta value already in U_M: nothing to sort
    ("b16", 50_000, 3_000, 70_000, 1.0),      # all new
    ("u64", 400_000, 100_000, 300_000, 0.3),
    ("u32", 100_000, 20_000, 90_000, 0.5),
    ("u64", 20_000, 1, 5_000, 0.5),           # one-entry dictionary
]


@pytest.mark.parametrize("case", PROBE_CASES)
@pytest.mark.parametrize("knob", [3, 0])
def test_probe_first_step1a(case, knob, _reset_probe):
    """NEXT1 (knob 2 = 3, and auto for 16-byte keys): each delta value is looked up
    in U_M first, only the values not found are sorted, U' = merge(U_M, U_new).
    Active only when no U_D / X_D / r output is requested, so the merge runs
    without tables; U', M', b', |U'| and |U_D| must match the oracle."""
    import paper_1109_6885_b200 as dm
    dm.set_tuning(2, knob)
    key, n_main, dict_len, n_delta, p_new = case
    col = datagen.make_random_case(4242 + n_delta, n_main, dict_len, n_delta, p_new, key=key)
    UM, M, D = to_device(col)
    r = dm.merge_column(UM, M, col.n_main, col.main_bits, D)
    compare(col, M, r, check_tables=False)


def test_probe_first_cfg3_scaled(_reset_probe):
    import paper_1109_6885_b200 as dm
    dm.set_tuning(2, 0)  # auto: cfg3 takes the probe-first front end
    col = datagen.make_config(3, scale=0.05)
    UM, M, D = to_device(col)
    r = dm.merge_column(UM, M, col.n_main, col.main_bits, D)
    compare(col, M, r, check_tables=False)
