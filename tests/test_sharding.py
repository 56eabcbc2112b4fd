"""Multi-device partitioning: plans and their host logic on the CPU
-- the library's row plan (dm_plan_row_shards) and its host-callback transport
over 2- and 3-process gloo groups (dm_comm_selftest_host) -- a gloo model of the
row-sharded data exchange (numpy + the oracle), and, on the GPU, several ranks
sharing the one device through dm_merge_column_sharded (C ABI) bit-exact
against the oracle."""
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


def _comm_worker(rank, world, port, q):
    """Host-only: the library's callback transport over gloo (broadcast from every
    root, all-gather in rank order, point to point) and the library's row plan,
    identical on every rank."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1109_6885_b200 as dm
        comm = dm.Comm.callbacks()
        ok = comm.selftest_host() == dm.Status.OK and comm.rank == rank and comm.size == world
        plans = [None] * world
        dist.all_gather_object(plans, dm.plan_row_shards(10**8 + 7, 10**6 + 3, world))
        comm.close()
        if rank == 0:
            q.put((ok, all(p == plans[0] for p in plans), plans[0]))
        else:
            q.put((ok, True, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_library_transport_and_plan(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_comm_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[0] for r in res) and all(r[1] for r in res)
    cuts = next(r[2] for r in res if r[2] is not None)
    assert cuts[0] == 0 and cuts[-1] == 10**8 + 7 + 10**6 + 3
    assert all(c % 4096 == 0 for c in cuts[:-1]) and cuts == sorted(cuts)


def _gpu_worker(rank, world, port, q, tables, key, case):
    """One rank of dm_merge_column_sharded on the (single) GPU: the library's
    callback transport carries the collectives over gloo between the processes;
    no kernel waits on another rank (every wait is a host-side collective)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1109_6885_b200 as dm
        from tests.parity import to_device, keys_np
        torch.cuda.set_device(0)
        if case == "flagged":  # clustered new values: flagged XC superblocks (their X_M slices travel too)
            col = datagen.make_clustered_case(36, 1 << 19, 200_000, 20_000, key=key)
        else:
            col = datagen.make_random_case(34, 1 << 20, 1 << 16, 60001, 0.6, main_bits=18, key=key)
        UM, M, D = to_device(col)
        shard = sharding.plan_row_shards(col.n_main, col.n_delta, world)[rank]
        mslice = M[shard.in_word(col.main_bits):] if shard.n_main else M
        if rank != 0:
            UM, D = UM[:0], D[:0]
        comm = dm.Comm.callbacks()
        out, nb, n_u, U = sharding.sharded_merge_column(UM, mslice, col.n_main, col.main_bits, D, comm=comm,
                                                        tables=tables, dict_len=col.dict_len, n_delta=col.n_delta,
                                                        key=key)
        comm.close()
        gathered = [None] * world
        dist.all_gather_object(gathered, out.cpu().numpy().view(np.uint64).tolist())
        if rank == 0:
            ref = oracle.merge(col)
            full = np.array([w for part in gathered for w in part], dtype=np.uint64)
            q.put((bool(np.array_equal(full, ref.merged_words)), nb == ref.merged_bits, n_u == ref.merged_len,
                   bool(np.array_equal(keys_np(U, key), ref.merged_dict))))
    finally:
        dist.destroy_process_group()


def _ranges_worker(rank, world, port, q, key, case):
    """NEXT2 inside the library: dm_merge_column_sharded with step1b = "ranges" --
    every rank merges its U_M value range with the U_D values that fall into it
    (gloo callback transport, ranks sharing the one GPU); U' slices and M' words
    concatenated in rank order must equal the oracle's."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1109_6885_b200 as dm
        from tests.parity import to_device, keys_np
        torch.cuda.set_device(0)
        if case == "flagged":
            col = datagen.make_clustered_case(37, 1 << 19, 200_000, 20_000, key=key)
        elif case == "small":  # X_M <= 96 KB: the plain X_M is gathered instead of XC
            col = datagen.make_random_case(39, 300_000, 9_000, 7_001, 0.5, key=key)
        else:
            col = datagen.make_random_case(35, 600_000, 200_000, 90_001, 0.5, key=key)
        UM, M, D = to_device(col)
        a, b = dm.plan_dict_ranges(col.dict_len, world)[rank:rank + 2]
        shard = sharding.plan_row_shards(col.n_main, col.n_delta, world)[rank]
        mslice = M[shard.in_word(col.main_bits):] if shard.n_main else M
        comm = dm.Comm.callbacks()
        r = dm.merge_column_sharded(comm, mslice, col.n_main, col.main_bits, col.dict_len, col.n_delta,
                                    main_dict=UM[a:b].clone(), delta=D if rank == 0 else D[:0], key=key,
                                    step1b="ranges", range_begin=a)
        comm.close()
        pieces = [None] * world
        dist.all_gather_object(pieces, (r.merged_dict_offset, keys_np_list(keys_np(r.merged_dict, key), key),
                                        r.merged_codes.cpu().numpy().view(np.uint64).tolist(), r.merged_bits,
                                        r.merged_len))
        if rank == 0:
            ref = oracle.merge(col)
            U = [v for p in sorted(pieces, key=lambda p: p[0]) for v in p[1]]
            words = np.array([w for p in pieces for w in p[2]], dtype=np.uint64)
            q.put((U == keys_np_list(ref.merged_dict, key), bool(np.array_equal(words, ref.merged_words)),
                   all(p[3] == ref.merged_bits and p[4] == ref.merged_len for p in pieces)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,key,case", [(2, "u64", "random"), (3, "b16", "random"), (2, "u32", "random"),
                                            (3, "u64", "flagged"), (2, "u64", "small")])
def test_sharded_merge_column_ranges_in_library(world, key, case):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ranges_worker, args=(r, world, port, q, key, case)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    assert all(res), res


def _run_gpu_ranks(world, *args):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    return res


@pytest.mark.gpu
@pytest.mark.parametrize("world,tables,key,case", [(2, "xc", "u64", "random"), (2, "plain", "u64", "random"),
                                                   (3, "xc", "b16", "random"), (2, "xc", "u32", "random"),
                                                   (3, "xc", "u64", "flagged"), (2, "plain", "u64", "flagged")])
def test_sharded_merge_column_ranks_on_one_gpu(world, tables, key, case):
    res = _run_gpu_ranks(world, tables, key, case)
    assert all(res), res


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


def _nccl1_worker(port, q):
    """World size 1 over NCCL: the library resolves NCCL from the process and runs
    its broadcasts / all-gathers through it (NCCL collectives run even at one
    rank), bit-exact against the oracle."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        import paper_1109_6885_b200 as dm
        from tests.parity import to_device, keys_np
        col = datagen.make_random_case(38, 1 << 20, 1 << 16, 60001, 0.6, main_bits=18)
        UM, M, D = to_device(col)
        comm = dm.Comm.nccl()
        r = dm.merge_column_sharded(comm, M, col.n_main, col.main_bits, col.dict_len, col.n_delta, main_dict=UM,
                                    delta=D)
        comm.close()
        ref = oracle.merge(col)
        q.put((bool(np.array_equal(r.merged_codes.cpu().numpy().view(np.uint64), ref.merged_words)),
               r.merged_bits == ref.merged_bits, bool(np.array_equal(keys_np(r.merged_dict, "u64"),
                                                                     ref.merged_dict))))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_merge_column_nccl_one_rank():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl1_worker, args=(_free_port(), q))
    p.start()
    res = q.get(timeout=300)
    p.join(timeout=60)
    assert all(res), res


@pytest.mark.parametrize("dict_len,g", [(10**7, 8), (1 << 30, 8), (5000, 3), (1024, 4), (7, 2), (200_000, 3)])
def test_library_plan_dict_ranges(dict_len, g):
    """dm_plan_dict_ranges (host, pure): U_M cut into g contiguous ranges at
    multiples of 1024 positions (whole XC superblocks of 128- and 256-code
    blocks), tiling [0, |U_M|)."""
    import paper_1109_6885_b200 as dm
    cuts = dm.plan_dict_ranges(dict_len, g)
    assert len(cuts) == g + 1 and cuts[0] == 0 and cuts[-1] == dict_len
    assert cuts == sorted(cuts) and all(c % 1024 == 0 for c in cuts[:-1])
    py = sharding.plan_dict_ranges(dict_len, g)  # the Python NEXT2 orchestration's plan agrees
    assert [b for (b, _) in py] == cuts[:-1] and [e for (_, e) in py] == cuts[1:]
