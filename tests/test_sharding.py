"""Multi-device partitioning: plans and their host logic on the CPU,
including 2-process gloo runs of the row-sharded Step 2 with the translation
tables broadcast from the root (the data path each GPU rank follows, with the
per-shard recompress done by numpy + the oracle's packer instead of the kernel)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import datagen
import oracle
from paper_1109_6885_b200 import sharding


def test_lpt_partition_properties():
    rng = np.random.default_rng(3)
    costs = rng.lognormal(10, 2, size=300).tolist()
    for parts in (1, 2, 3, 4, 8):
        p = sharding.lpt_partition(costs, parts)
        flat = sorted(i for q in p for i in q)
        assert flat == list(range(300))
        loads = [sum(costs[i] for i in q) for q in p]
        assert max(loads) - min(loads) <= max(costs) + 1e-6   # LPT bound
        assert p == sharding.lpt_partition(costs, parts)         # deterministic


@pytest.mark.parametrize("n_main,n_delta,g", [(10**6, 10**4, 2), (100003, 4097, 4), (4096, 0, 8), (0, 50000, 3),
                                              (1 << 20, 5 * 10**4, 8), (5, 3, 2)])
def test_plan_row_shards(n_main, n_delta, g):
    shards = sharding.plan_row_shards(n_main, n_delta, g)
    assert len(shards) == g and shards[0].row_begin == 0 and shards[-1].row_end == n_main + n_delta
    for a, b in zip(shards, shards[1:]):
        assert a.row_end == b.row_begin and a.row_end % sharding.ROW_ALIGN == 0
    assert sum(s.n_main for s in shards) == n_main and sum(s.n_delta for s in shards) == n_delta
    for s in shards:
        assert s.n_main + s.n_delta == s.row_end - s.row_begin
        for b in range(1, 33):
            assert (s.row_begin * b) % 64 == 0
            if s.n_main:
                assert (s.main_begin * b) % 64 == 0


def _shard_words(col, ref, shard, nb):
    """Packed words of one shard's rows (main rows through X_M, delta rows through X_D)."""
    codes = np.concatenate([ref.x_main[col.main_codes[shard.main_begin:shard.main_end].astype(np.int64)],
                            ref.x_delta[ref.delta_rank[shard.delta_begin:shard.delta_end].astype(np.int64)]])
    return oracle.pack(codes.astype(np.uint32), nb)


def test_row_shards_reassemble_to_the_full_output():
    col = datagen.make_random_case(21, 300007, 20000, 40001, 0.3)
    ref = oracle.merge(col)
    for g in (2, 3, 8):
        parts = [_shard_words(col, ref, s, ref.merged_bits) for s in sharding.plan_row_shards(col.n_main, col.n_delta, g)]
        assert np.array_equal(np.concatenate(parts), ref.merged_words)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        col = datagen.make_random_case(33, 200003, 15000, 30011, 0.2)
        shards = sharding.plan_row_shards(col.n_main, col.n_delta, world)
        # root: Steps 1(a)/1(b)/2(a); broadcast header + tables (the NCCL path's shape)
        hdr = torch.zeros(3, dtype=torch.int64)
        if rank == 0:
            ref = oracle.merge(col)
            hdr[:] = torch.tensor([ref.merged_bits, ref.x_delta.shape[0], col.n_delta])
        dist.broadcast(hdr, 0)
        nb, n_ud, nd = (int(x) for x in hdr)
        xm = torch.from_numpy(ref.x_main.view(np.int32)) if rank == 0 else torch.empty(col.dict_len, dtype=torch.int32)
        xd = torch.from_numpy(ref.x_delta.view(np.int32)) if rank == 0 else torch.empty(n_ud, dtype=torch.int32)
        rk = torch.from_numpy(ref.delta_rank.view(np.int32)) if rank == 0 else torch.empty(nd, dtype=torch.int32)
        for t in (xm, xd, rk):
            dist.broadcast(t, 0)

        class R:  # the tables as this rank received them
            x_main = xm.numpy().view(np.uint32)
            x_delta = xd.numpy().view(np.uint32)
            delta_rank = rk.numpy().view(np.uint32)

        mine = _shard_words(col, R, shards[rank], nb)
        gathered = [None] * world
        dist.all_gather_object(gathered, mine.tolist())
        costs = [float(c) for c in np.random.default_rng(5).lognormal(8, 1, 50)]
        plans = [None] * world
        dist.all_gather_object(plans, sharding.lpt_partition(costs, world))
        if rank == 0:
            full = np.array([w for part in gathered for w in part], dtype=np.uint64)
            q.put((bool(np.array_equal(full, ref.merged_words)), all(p == plans[0] for p in plans)))
    finally:
        dist.destroy_process_group()


def test_gloo_two_rank_row_sharded_step2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok, same_plan = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert ok and same_plan


def _gpu_worker(rank, world, port, q, tables):
    """One rank of sharded_merge_column on the (single) GPU: gloo carries the
    broadcasts of CUDA tensors between the processes; no kernel waits on another
    rank (every wait is a host-side collective)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1109_6885_b200 as dm  # noqa: F401
        from tests.parity import to_device
        torch.cuda.set_device(0)
        col = datagen.make_random_case(34, 1 << 20, 1 << 16, 60001, 0.6, main_bits=18)
        UM, M, D = to_device(col)
        shard = sharding.plan_row_shards(col.n_main, col.n_delta, world)[rank]
        mslice = M[shard.in_word(col.main_bits):] if shard.n_main else M
        if rank != 0:
            UM, D = UM[:0], D[:0]
        out, nb, n_u, U = sharding.sharded_merge_column(UM, mslice, col.n_main, col.main_bits, D, shard,
                                                        tables=tables)
        gathered = [None] * world
        dist.all_gather_object(gathered, out.cpu().numpy().view(np.uint64).tolist())
        if rank == 0:
            ref = oracle.merge(col)
            full = np.array([w for part in gathered for w in part], dtype=np.uint64)
            q.put(bool(np.array_equal(full, ref.merged_words)) and nb == ref.merged_bits and n_u == ref.merged_len)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("tables", ["xc", "plain"])
def test_sharded_merge_column_two_ranks_on_one_gpu(tables):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q, tables)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    assert ok


def _next2_worker(rank, world, port, q, key):
    """NEXT2: Step 1(b) sharded by U_M value ranges over `world` ranks on the one
    GPU (gloo broadcasts), then Step 2 of each rank's row shard through the
    assembled global XC; everything compared with the oracle."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1109_6885_b200 as dm
        from tests.parity import to_device, keys_np
        torch.cuda.set_device(0)
        col = datagen.make_random_case(35, 600_000, 200_000, 90_001, 0.5, key=key)
        UM, M, D = to_device(col)
        a, b = sharding.plan_dict_ranges(col.dict_len, world)[rank]
        sd = sharding.sharded_dictionary_merge(UM[a:b], a, col.dict_len, col.main_bits,
                                               D if rank == 0 else D[:0], shift=7)
        shard = sharding.plan_row_shards(col.n_main, col.n_delta, world)[rank]
        mslice = M[shard.in_word(col.main_bits):] if shard.n_main else M
        out = dm.recompress_xc(mslice, shard.n_main, col.main_bits, col.dict_len, sd.xc, sd.x_main_exceptions,
                               sd.x_delta, sd.delta_rank[shard.delta_begin:], shard.n_delta, sd.merged_bits)
        pieces = [None] * world
        dist.all_gather_object(pieces, (keys_np_list(keys_np(sd.u_slice, key), key), sd.u_offset,
                                        sd.x_main_range.cpu().numpy().view(np.uint32).tolist(),
                                        out.cpu().numpy().view(np.uint64).tolist()))
        if rank == 0:
            ref = oracle.merge(col)
            U = [v for p in sorted(pieces, key=lambda p: p[1]) for v in p[0]]
            want_U = keys_np_list(ref.merged_dict, key)
            xm = [v for p in pieces for v in p[2]]
            words = np.array([w for p in pieces for w in p[3]], dtype=np.uint64)
            xd = sd.x_delta.cpu().numpy().view(np.uint32)[: ref.x_delta.shape[0]]
            q.put((U == want_U, xm == ref.x_main.tolist(), bool(np.array_equal(xd, ref.x_delta)),
                   sd.merged_len == ref.merged_len and sd.merged_bits == ref.merged_bits,
                   bool(np.array_equal(words, ref.merged_words))))
    finally:
        dist.destroy_process_group()


def keys_np_list(a, key):
    return a.tolist() if key != "b16" else [bytes(r) for r in a]


@pytest.mark.gpu
@pytest.mark.parametrize("world,key", [(2, "u64"), (3, "u64"), (3, "b16"), (2, "u32")])
def test_next2_sharded_dictionary_merge(world, key):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_next2_worker, args=(r, world, port, q, key)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    assert all(res), res
