"""The seeded input generators: determinism, bijections and the config shapes."""
import numpy as np
import pytest

import datagen as g


def test_counter_based_determinism():
    a = g.rnd(1, 2, np.arange(1000))
    b = g.rnd(1, 2, np.arange(500, 1000))
    assert np.array_equal(a[500:], b)
    assert not np.array_equal(g.rnd(1, 3, np.arange(10)), g.rnd(1, 2, np.arange(10)))


@pytest.mark.parametrize("k", [1, 2, 5, 12])
def test_perm_pow2_is_bijection(k):
    x = g.perm_pow2(123, np.arange(1 << k), k)
    assert sorted(x.tolist()) == list(range(1 << k))


@pytest.mark.parametrize("n", [1, 2, 3, 1000, 4097])
def test_perm_below_is_bijection(n):
    x = g.perm_below(5, np.arange(n), n)
    assert sorted(x.tolist()) == list(range(n))


def test_cfg1_shape():
    c = g.make_config(1)
    assert c.n_main == 10**6 and c.dict_len == 10**4 and c.n_delta == 10**4 and c.main_bits == 14
    assert np.all(np.diff(c.main_dict.astype(np.float64)) > 0) and c.main_dict.max() < 2**40
    assert c.main_codes.max() < c.dict_len
    new = ~np.isin(c.delta, c.main_dict)
    assert 0.45 < new.mean() < 0.55
    assert np.unique(c.delta[new]).size == new.sum()      # new values are distinct


def test_cfg3_small_scale_strings():
    c = g.make_config(3, scale=0.001)
    assert c.main_dict.shape[1] == 16 and c.delta.shape[1] == 16
    hi, lo = g.bytes_to_hilo(c.main_dict)
    rows = [bytes(r) for r in c.main_dict]
    assert all(a < b for a, b in zip(rows, rows[1:]))     # strictly increasing bytewise
    lens = (c.main_dict != 0).sum(1)
    assert lens.min() >= 8 and lens.max() <= 16
    # zipf skew: the most frequent code is far above the mean frequency
    cnt = np.bincount(c.main_codes, minlength=c.dict_len)
    assert cnt.max() > 20 * cnt.mean()


def test_cfg4_column_properties():
    c0 = g.make_config(4, scale=0.001, column=0)
    c299 = g.make_config(4, scale=0.001, column=299)
    assert c0.key == "u64" and c299.key == "b16"


def test_cfg5_small_scale_all_new():
    c = g.make_config(5, scale=1e-4)
    assert c.dict_len == c.n_main
    assert np.array_equal(np.sort(c.main_codes), np.arange(c.dict_len, dtype=np.uint32))
    assert not np.isin(c.delta, c.main_dict).any()
    assert np.unique(c.delta).size == c.n_delta


def test_torch_twin_matches_numpy_cfg5():
    import torch
    from datagen import torch_gen
    scale = 2.0 ** -14
    c = g.make_config(5, scale=scale)
    md, codes, bits, delta = torch_gen.make_cfg5(scale=scale, device="cpu")
    assert np.array_equal(md.numpy().view(np.uint64), c.main_dict)
    assert np.array_equal(codes.numpy().view(np.uint32), c.main_codes)
    assert np.array_equal(delta.numpy().view(np.uint64), c.delta)
    assert bits == c.main_bits
