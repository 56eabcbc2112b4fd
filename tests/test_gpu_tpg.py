"""Thread-per-group Step 2(b) (knob 6 = 0, csrc/recompress.cu k_recompress_tpg)
vs the oracle, bit-exact: Eq 11 for the main rows and the delta append
through X_D, run through the same merge as every other path.

The kernel handles b' = b and b' = b + 1 with XC in shared memory; the cases
cover both, the fast tiles (1024 main rows), the tail tiles (delta rows, the
main/delta boundary, the ragged end), the rare lookups that read the plain X_M
(a block with more than 8 insertions, a flagged superblock), and every key type.
Each case also runs with knob 6 = 1 (the warp-per-group kernel) and the two
must agree with the oracle and with each other.
"""
import numpy as np
import pytest
import torch

import datagen
import oracle
from tests.parity import compare, run_gpu
from tests.test_gpu_xc import _column, _spread

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
    dm.set_tuning(6, 0)


def _both_forms(col):
    import paper_1109_6885_b200 as dm
    ref = None
    words = []
    for form in (0, 1):
        dm.set_tuning(6, form)
        M, r = run_gpu(col)
        ref = compare(col, M, r, ref=ref)
        words.append(r.merged_codes.cpu().numpy())
    assert np.array_equal(words[0], words[1])
    return ref


@pytest.mark.parametrize("key", ["u64", "u32", "b16"])
def test_tpg_same_width(key):
    n = 300_001  # 19 bits; ~1% new values: b' = b
    col = _column(n, 1_000_003, _spread(n, 2500, 21), 20_000, seed=21, key="b16" if key == "b16" else "u64")
    if key == "u32":
        col = datagen.u32_column(col)
    ref = _both_forms(col)
    assert ref.merged_bits == col.main_bits


def test_tpg_width_grows_by_one():
    n = (1 << 19) - 40  # 19 bits; 3000 new values cross 2^19: b' = 20
    col = _column(n, 700_001, _spread(n, 3000, 22), 5000, seed=22)
    ref = _both_forms(col)
    assert (col.main_bits, ref.merged_bits) == (19, 20)


def test_tpg_rare_lookups_read_plain_xm():
    n = 1024 * 200 + 5
    ins = [(1024 * 3 + 10, 12), (1024 * 9 + 700, 9), (1024 * 17 + 3, 33), (1024 * 40 + 256, 40)]
    ins += _spread(n, 1500, 23)
    col = _column(n, 2 * 1024 * 64 + 1000, ins, 3000, seed=23)
    _both_forms(col)


@pytest.mark.parametrize("n_main", [0, 1, 1023, 1024, 1025, 32 * 1024 + 31])
def test_tpg_tiles_and_tails(n_main):
    n = 40_000
    col = _column(n, n_main, _spread(n, 300, 24), 2500, seed=24)
    _both_forms(col)


def test_tpg_cfg2_scaled():
    _both_forms(datagen.make_config(2, scale=0.05))


@pytest.mark.parametrize("n_dict,n_main", [(60_001, 200_000), (8_500_000, 3_000_007)])
@pytest.mark.parametrize("offset_words", [0, 2])
def test_tpg_wide_accesses_and_16_byte_aligned_codes(n_dict, n_main, offset_words):
    """b = b' = 16 / 24 (multiples of 8): the slot-free kernel moves a lane's words by
    32-byte accesses when M and M' are 32-byte aligned and by 16-byte ones otherwise
    (the ABI promises 16: include/dictmerge.h).  M at a 16-byte offset takes the second path;
    both must give the oracle's M' (Eq 11)."""
    import paper_1109_6885_b200 as dm
    from tests.parity import to_device
    col = _column(n_dict, n_main, _spread(n_dict, max(n_dict // 100, 64), 25), 4000, seed=25)
    assert col.main_bits in (16, 24)
    UM, M, D = to_device(col)
    buf = torch.empty(M.numel() + 4, dtype=M.dtype, device=M.device)
    Mo = buf[offset_words:offset_words + M.numel()]
    Mo.copy_(M)
    assert Mo.data_ptr() % 32 == (16 if offset_words else 0)
    r = dm.merge_column(UM, Mo, col.n_main, col.main_bits, D, x_tables=True, delta_dict=True)
    torch.cuda.synchronize()
    ref = compare(col, M, r)
    assert ref.merged_bits == col.main_bits
