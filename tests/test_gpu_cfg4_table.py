"""cfg4 -- the 300-column wide table (BASELINE configs[3]) -- merged exactly as
bench.py times it: every column on the device, one ``TableMerger`` issuing
``dm_merge_table_async`` (the library's 16-stream pool, per-column workspaces),
captured in a CUDA graph and replayed; then every column compared with the CPU
oracle: U' and the M' words bit for bit (digests of the exact bytes; a mismatch
re-runs that column for an element-wise report).  A second pass requests the
translation tables and checks X_M and X_D too.  Each column is merged separately
(P:184); the columns are independent tasks.

The oracle runs in forked host workers while the GPU merges (test
infrastructure only: the workers never see a GPU output)."""
import hashlib
import multiprocessing as mp
import os

import numpy as np
import pytest
import torch

import datagen
import oracle
from tests.parity import keys_np

pytestmark = pytest.mark.gpu

_COLS = None


def _digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _oracle_digest(j):
    c = _COLS[j]
    r = oracle.merge(c, "linear")
    return (r.status, r.merged_bits, r.merged_len, _digest(r.merged_dict), _digest(r.merged_words),
            _digest(r.x_main), _digest(r.x_delta))


def _check(cols, res, refs, tables):
    bad = []
    for j, (c, r, ref) in enumerate(zip(cols, res, refs)):
        st, nb, nu, du, dw, dxm, dxd = ref
        ok = st == 0 and r.merged_bits == nb and r.merged_len == nu and \
            _digest(keys_np(r.merged_dict, c.key)) == du and \
            _digest(r.merged_codes.cpu().numpy().view(np.uint64)) == dw
        if tables:
            ok = ok and _digest(r.x_main.cpu().numpy().view(np.uint32)) == dxm and \
                _digest(r.x_delta.cpu().numpy().view(np.uint32)) == dxd
        if not ok:
            bad.append(j)
    if bad:  # element-wise report for the first failing column
        j = bad[0]
        full = oracle.merge(cols[j], "linear")
        got = res[j].merged_codes.cpu().numpy().view(np.uint64)
        n_diff = int(np.count_nonzero(got != full.merged_words)) if got.size == full.merged_words.size else -1
        raise AssertionError(f"{len(bad)} of {len(cols)} columns differ, first {j} "
                             f"(b' {res[j].merged_bits} vs {full.merged_bits}, M' words differing {n_diff})")


def test_cfg4_full_table_as_benchmarked():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    global _COLS
    import bench
    import paper_1109_6885_b200 as dm
    oracle.build()
    cols = bench.host_columns("cfg4", 0, 1)  # all 300 columns, as bench.py builds them at N = 1
    assert len(cols) == 300
    _COLS = cols
    # fork the oracle workers before this process touches CUDA
    with mp.get_context("fork").Pool(max(2, min(32, (os.cpu_count() or 2) - 1))) as pool:
        pending = pool.map_async(_oracle_digest, range(len(cols)), chunksize=1)
        dev = torch.device("cuda", 0)
        dev_cols = [bench.device_inputs(c, dev) for c in cols]
        for tables in (False, True):
            tm = dm.TableMerger(dev_cols, x_tables=tables)
            if not tables:  # the benchmarked path: graph capture + replay
                tm.capture_graph()
                tm.replay_graph()
            else:
                tm.run_async()
            torch.cuda.synchronize()
            res = tm.results()
            refs = pending.get(timeout=1800)
            _check(cols, res, refs, tables)
            del tm, res
            torch.cuda.empty_cache()
