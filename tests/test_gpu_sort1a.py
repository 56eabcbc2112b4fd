"""Step 1(a) sort variants vs the oracle, bit-exact (U_D, r and everything
downstream): the bucket path (knob 5 = 2; counting pass into buckets by the top
bits below the keys' common prefix, then a rank among bucket mates) and the LSD
radix passes (knob 5 = 1), for u64, u32 and 16-byte keys.

The cases aim at the bucket path's edges: sizes around the auto threshold
(2^11) and tiny deltas, keys that differ only in their low bits (the digit
window reaches bit 0), 16-byte keys that differ only in the low or only in the
high word (shift across the 64-bit boundary), duplicates inside buckets
(ties broken by the original index), and skewed sets that overflow a bucket
(all keys equal; a cluster plus one outlier; heavy repeats with the dedup front
end off) -- those must fall back to the LSD passes on the device and still give
the oracle's result."""
import numpy as np
import pytest
import torch

import datagen
import oracle
from tests.parity import compare, run_gpu

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
    dm.set_tuning(5, 0)
    dm.set_tuning(2, 0)


def _run(col, variant, dedup=0):
    import paper_1109_6885_b200 as dm
    dm.set_tuning(5, variant)
    dm.set_tuning(2, dedup)
    M, r = run_gpu(col)
    compare(col, M, r)


CASES = [
    # n_main, dict_len, n_delta, p_new
    (20_000, 5_000, 1, 1.0),
    (20_000, 5_000, 3, 0.5),
    (20_000, 5_000, 2047, 0.5),
    (20_000, 5_000, 2049, 0.5),
    (100_000, 50_000, 100_000, 0.1),
    (300_000, 200_000, 250_000, 0.9),
    (50_000, 3_000, 200_000, 0.0),     # repeats of 3k main values
]


@pytest.mark.parametrize("variant", [0, 1, 2])
@pytest.mark.parametrize("key", ["u64", "u32", "b16"])
@pytest.mark.parametrize("case", CASES)
def test_sort_variant_random(variant, key, case):
    n_main, dict_len, n_delta, p_new = case
    col = datagen.make_random_case(4242 + n_delta, n_main, dict_len, n_delta, p_new, key=key)
    _run(col, variant)


@pytest.mark.parametrize("variant", [1, 2])
@pytest.mark.parametrize("dedup", [1, 2])
def test_sort_variant_with_and_without_dedup(variant, dedup):
    col = datagen.make_random_case(77, 40_000, 20_000, 150_000, 0.2, key="u64")
    _run(col, variant, dedup)
    col = datagen.make_random_case(78, 40_000, 20_000, 150_000, 0.2, key="b16")
    _run(col, variant, dedup)


def _u64_col(UM, D, n_main=30_000, seed=1):
    UM = np.unique(np.asarray(UM, dtype=np.uint64))
    rng = np.random.default_rng(seed)
    D = np.asarray(D, dtype=np.uint64)
    D = D[rng.permutation(D.size)]
    codes = rng.integers(0, UM.size, size=n_main, dtype=np.uint64).astype(np.uint32)
    return datagen.Column("u64", UM, codes, datagen.width_hint(UM.size), D)


@pytest.mark.parametrize("variant", [0, 2])
def test_low_bits_only(variant):
    # all keys < 2^10: the digit window [0, log2 B) covers every differing bit
    UM = np.arange(0, 1024, 3)
    D = np.concatenate([np.arange(1, 1024, 5), np.arange(0, 1024, 7), np.arange(0, 1024, 7)])
    _run(_u64_col(UM, D), variant)


@pytest.mark.parametrize("variant", [0, 2])
def test_high_prefix_shared(variant):
    # a long common prefix: keys differ only below bit 20
    base = np.uint64(0xABCD_0000_0000_0000)
    UM = base + np.arange(0, 1 << 20, 37, dtype=np.uint64)
    rng = np.random.default_rng(3)
    D = base + rng.integers(0, 1 << 20, size=60_000, dtype=np.uint64)
    _run(_u64_col(UM, D), variant)


@pytest.mark.parametrize("variant", [0, 2])
@pytest.mark.parametrize("dedup", [1, 2])
def test_overflow_falls_back(variant, dedup):
    # one outlier and a dense cluster: every cluster key lands in one bucket
    UM = np.array([5, 2**63, 2**63 + 10_000], dtype=np.uint64)
    D = np.concatenate([np.zeros(1, np.uint64), np.uint64(2**63) + np.arange(20_000, dtype=np.uint64)])
    _run(_u64_col(UM, D), variant, dedup)
    # all keys equal
    D = np.full(50_000, 2**40 + 7, dtype=np.uint64)
    _run(_u64_col(UM, D), variant, dedup)
    # heavy repeats of a few values (more than 256 copies each)
    D = np.repeat(np.array([1, 2**62, 2**63 + 3], dtype=np.uint64), 9000)
    _run(_u64_col(UM, D), variant, dedup)


def _b16(hi, lo):
    return datagen.hilo_to_bytes(np.asarray(hi, dtype=np.uint64), np.asarray(lo, dtype=np.uint64))


@pytest.mark.parametrize("variant", [0, 2])
@pytest.mark.parametrize("part", ["lo", "hi", "both"])
def test_b16_word_boundary(variant, part):
    rng = np.random.default_rng({"lo": 1, "hi": 2, "both": 3}[part])
    n_dict, n_d = 5000, 30_000
    if part == "lo":    # same high word: the shift stays below 64
        hi_m, lo_m = np.full(n_dict, 0x4142, np.uint64), rng.integers(0, 2**63, n_dict, dtype=np.uint64)
        hi_d, lo_d = np.full(n_d, 0x4142, np.uint64), rng.integers(0, 2**63, n_d, dtype=np.uint64)
    elif part == "hi":  # same low word: the shift is >= 64
        hi_m, lo_m = rng.integers(0, 2**63, n_dict, dtype=np.uint64), np.full(n_dict, 9, np.uint64)
        hi_d, lo_d = rng.integers(0, 2**63, n_d, dtype=np.uint64), np.full(n_d, 9, np.uint64)
    else:               # differing bits just above and below the word boundary
        hi_m, lo_m = rng.integers(0, 4, n_dict, dtype=np.uint64), rng.integers(0, 2**64 - 1, n_dict, dtype=np.uint64)
        hi_d, lo_d = rng.integers(0, 4, n_d, dtype=np.uint64), rng.integers(0, 2**64 - 1, n_d, dtype=np.uint64)
    UM = np.unique(_b16(hi_m, lo_m), axis=0)
    D = np.concatenate([_b16(hi_d, lo_d), UM[rng.integers(0, UM.shape[0], 5000)]])
    codes = rng.integers(0, UM.shape[0], size=20_000, dtype=np.uint64).astype(np.uint32)
    col = datagen.Column("b16", UM, codes, datagen.width_hint(UM.shape[0]), D)
    _run(col, variant)


@pytest.mark.parametrize("variant", [1, 2])
def test_cfg_shapes(variant):
    # BASELINE configs 1 and (scaled) 3: uniform u64 and Zipf-reused strings
    _run(datagen.make_config(1), variant)
    _run(datagen.make_config(3, scale=0.02), variant)
