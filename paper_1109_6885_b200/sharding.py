"""Multi-GPU partitioning of the merge.

* Whole columns are independent (each column is merged separately; the
  paper's first parallelisation scheme is a task queue over columns):
  ``lpt_partition`` assigns a wide table's columns to devices/ranks by longest
  processing time first on an estimated byte cost -- no collective on the data
  path.
* A very long single column is split by rows for Step 2 (the paper splits the
  N' tuples evenly over threads): ``plan_row_shards`` cuts [0, N') at
  multiples of 4096 rows so every shard starts on a u64-word boundary at both
  the input width b and the output width b' (4096·b and 4096·b' are multiples of
  64, and of 128 bits, so TMA bulk copies stay 16-byte aligned).
  ``sharded_merge_column`` is a thin wrapper of the C ABI's
  ``dm_merge_column_sharded``: the library runs Steps 1(a)/1(b)/2(a) on the root,
  broadcasts the header and the translation tables over its transport (NCCL, or
  host callbacks over a torch.distributed group) -- by default the compact table
  XC (~67 MB for cfg5) instead of the literal X_M (4.3 GB) -- and every rank
  recompresses its own row range.

The column partition (LPT) is plain Python; the row plan is the library's
(host-only, tested with gloo on the CPU); the merge itself needs CUDA devices.
"""
from __future__ import annotations

import dataclasses
from typing import List, Sequence

ROW_ALIGN = 4096  # rows per recompress chunk; multiple of 64 -> word-aligned at any width


def column_cost(n_main: int, n_delta: int, dict_len: int, main_bits: int, key_bytes: int) -> float:
    """Estimated bytes one column's merge moves (inputs read, outputs written, sort)."""
    b_hi = max(1, (dict_len + n_delta - 1).bit_length())
    passes = 8 if key_bytes == 8 else 16
    return (n_main * main_bits / 8 + (n_main + n_delta) * b_hi / 8 + 2 * dict_len * key_bytes
            + 4 * dict_len + passes * 2 * n_delta * (key_bytes + 4))


def lpt_partition(costs: Sequence[float], n_parts: int) -> List[List[int]]:
    """Longest-processing-time-first assignment of items to n_parts bins.
    Deterministic (ties broken by index), so every rank computes the same plan."""
    if n_parts < 1:
        raise ValueError("n_parts must be >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    load = [0.0] * n_parts
    parts: List[List[int]] = [[] for _ in range(n_parts)]
    for i in order:
        p = min(range(n_parts), key=lambda q: (load[q], q))
        parts[p].append(i)
        load[p] += costs[i]
    for p in parts:
        p.sort()
    return parts


@dataclasses.dataclass(frozen=True)
class RowShard:
    row_begin: int      # first output row (of N' = N_M + N_D)
    row_end: int        # one past the last
    main_begin: int     # main rows [main_begin, main_end)
    main_end: int
    delta_begin: int    # delta rows [delta_begin, delta_end) (0-based within D)
    delta_end: int

    @property
    def n_main(self) -> int:
        return self.main_end - self.main_begin

    @property
    def n_delta(self) -> int:
        return self.delta_end - self.delta_begin

    def in_word(self, b: int) -> int:
        """First u64 word of this shard's main codes in the packed input M (width b)."""
        assert (self.main_begin * b) % 64 == 0
        return self.main_begin * b // 64

    def out_word(self, nb: int) -> int:
        """First u64 word of this shard's rows in the packed output M' (width b')."""
        assert (self.row_begin * nb) % 64 == 0
        return self.row_begin * nb // 64

    def out_words(self, nb: int) -> int:
        """u64 words this shard writes: its rows at b' bits (the last shard may end mid-word)."""
        return (self.row_end * nb + 63) // 64 - self.out_word(nb)


def plan_row_shards(n_main: int, n_delta: int, n_shards: int, align: int = ROW_ALIGN) -> List[RowShard]:
    """The library's row plan (``dm_plan_row_shards``, a pure host function of the
    C ABI): the N' output rows cut into n_shards contiguous ranges at multiples of
    4096 (the delta rows follow the main rows)."""
    if align != ROW_ALIGN:
        raise ValueError("the library plans at 4096-row multiples")
    import paper_1109_6885_b200 as dm
    cuts = dm.plan_row_shards(n_main, n_delta, n_shards)
    shards = []
    for g in range(n_shards):
        r0, r1 = cuts[g], cuts[g + 1]
        m0, m1 = min(r0, n_main), min(r1, n_main)
        d0, d1 = max(r0, n_main) - n_main, max(r1, n_main) - n_main
        shards.append(RowShard(r0, r1, m0, m1, d0, d1))
    return shards


def sharded_merge_column(main_dict, main_codes_shard, n_main: int, main_bits: int, delta, comm=None,
                         tables: str = "xc", root: int = 0, dict_len=None, n_delta=None, key=None):
    """Row-sharded merge of one column across the ranks of `comm` (one GPU each),
    through the C ABI's ``dm_merge_column_sharded``: the root runs Steps
    1(a)/1(b)/2(a), the library broadcasts the header and XC (or X_M), sends the
    delta rows' codes to their owner and every rank recompresses its row range.

    Every rank passes its own packed main-code slice (`main_codes_shard`, the
    words of rows [shard.main_begin, shard.main_end) of ``plan_row_shards``); the
    root also passes U_M and D.  `comm`: a ``dm.Comm`` (default: callbacks over
    the torch.distributed default group).  Returns (this rank's M' words, b',
    |U'|, U' on the root else None)."""
    import paper_1109_6885_b200 as dm
    own = comm is None
    comm = comm if comm is not None else dm.Comm.callbacks()
    try:
        if key is None:
            key = {0: "u64", 1: "b16", 2: "u32"}[dm._key_of(main_dict)]
        r = dm.merge_column_sharded(comm, main_codes_shard, n_main, main_bits,
                                    main_dict.shape[0] if dict_len is None else dict_len,
                                    delta.shape[0] if n_delta is None else n_delta, main_dict=main_dict, delta=delta,
                                    key=key, tables=tables, root=root)
    finally:
        if own:
            comm.close()
    return r.merged_codes, r.merged_bits, r.merged_len, r.merged_dict


# ----------------------------------------------------------- NEXT2: sharded Step 1(b)
XC_SUPER = 1024  # U_M ranges start at multiples of every XC superblock size (4 << 7, 4 << 8)


def plan_dict_ranges(dict_len: int, n_ranges: int, align: int = XC_SUPER) -> List[tuple]:
    """Cut U_M's positions [0, |U_M|) into n_ranges contiguous ranges starting at
    multiples of `align` (so every range's XC superblocks are global ones)."""
    cuts = [0]
    for g in range(1, n_ranges):
        cuts.append(max(cuts[-1], (dict_len * g // n_ranges) // align * align))
    cuts.append(dict_len)
    return [(cuts[g], cuts[g + 1]) for g in range(n_ranges)]


@dataclasses.dataclass
class ShardedDictionary:
    """Result of sharded_dictionary_merge on one rank."""
    u_slice: object          # this rank's part of U' (its value range), keys
    u_offset: int            # global U' index of u_slice[0]
    merged_len: int          # |U'|
    merged_bits: int         # b'
    x_main_range: object     # X_M for this rank's U_M range (global codes), int32
    xc: object               # the global XC (dm.XcTables), identical on every rank
    x_main_exceptions: object  # a |U_M|-entry int32 X_M holding the flagged superblocks' slices
    x_delta: object          # the global X_D (over U_D), int32
    delta_rank: object       # r (N_D), int32
    delta_dict_len: int      # |U_D|


def sharded_dictionary_merge(main_dict_range, range_begin: int, dict_len: int, main_bits: int, delta, group=None,
                             root: int = 0, shift: int = 7) -> ShardedDictionary:
    """Step 1(b) sharded by value ranges across the ranks of `group` (SURVEY §8f
    NEXT2; the paper's parallel merge splits both inputs at matching quantiles,
    P:302-314).  Rank g holds U_M[range_begin : range_begin + len] (a
    plan_dict_ranges range, non-empty); the root also holds D.

    1. root: Step 1(a) (U_D, r);
    2. the first U_M value of every range -> the root -> U_D cut points (lower bound);
    3. root -> rank g: the U_D values in [U_M[a_g], U_M[a_{g+1}));
    4. every rank merges its two ranges (dm_dictionary_merge_sorted_async) ->
       local U', X_M, X_D, XC;
    5. all-gather of (|U'_g|, new values_g) -> rebase X_M, X_D (by the |U'| of
       earlier ranges) and the XC records (by their new values);
    6. all-gather of the XC pieces, X_D pieces and flagged-superblock slices (rank
       order = value order), broadcast of r: every rank can run Step 2 on any rows.
    """
    import torch
    import torch.distributed as dist
    import paper_1109_6885_b200 as dm

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    with dm.tuning(dm.KNOB_XC_SHIFT, shift):  # process-wide knob: restored on exit
        return _sharded_dictionary_merge(main_dict_range, range_begin, dict_len, main_bits, delta, group, root,
                                         shift)


def _sharded_dictionary_merge(main_dict_range, range_begin, dict_len, main_bits, delta, group, root, shift):
    import torch
    import torch.distributed as dist
    import paper_1109_6885_b200 as dm

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device())
    SB = 4 << shift
    L = int(main_dict_range.shape[0])
    assert L > 0 and range_begin % XC_SUPER == 0

    def bcast(t, src):
        dist.broadcast(t, src=src, group=group)
        return t

    def allgather(t):  # equal-shape all-gather from broadcasts (gloo moves CUDA tensors only by broadcast)
        return [bcast(t.contiguous() if g == rank else torch.empty_like(t), g) for g in range(world)]

    # 1. Step 1(a) on the root
    meta = torch.zeros(2, dtype=torch.int64, device=dev)  # |U_D|, N_D
    if rank == root:
        dd = dm.DictionaryMerger(main_dict_range, 0, main_bits, delta, mode="delta")
        dd.run_async()
        h = dd.header()
        if h.status != 0:
            raise dm.DictMergeError(h.status, "dm_delta_dictionary_async")
        meta.copy_(torch.tensor([h.delta_dict_len, delta.shape[0]], dtype=torch.int64))
    bcast(meta, root)
    n_ud, n_delta = (int(x) for x in meta.tolist())
    # 2. cut points of U_D at every range's first U_M value
    firsts = allgather(main_dict_range[:1])
    cuts = torch.zeros(world + 1, dtype=torch.int64, device=dev)
    if rank == root:
        pos = dm.lower_bound(dd.UD[:n_ud], torch.cat(firsts[1:])) if world > 1 else cuts[:0]
        cuts[1:world] = pos
        cuts[world] = n_ud
    bcast(cuts, root)
    c = cuts.tolist()
    # 3. U_D to every rank (one broadcast), each keeps its value range
    ud = dd.UD[:n_ud].contiguous() if rank == root else \
        torch.empty((n_ud,) + tuple(main_dict_range.shape[1:]), dtype=main_dict_range.dtype, device=dev)
    if n_ud:
        bcast(ud, root)
    mine = ud[c[rank]:c[rank + 1]].clone()  # own allocation: the ABI wants 16-byte aligned buffers
    # 4. local merge of the two ranges
    lm = dm.DictionaryMerger(main_dict_range, 0, main_bits, mine, mode="sorted")
    lm.run_async()
    h = lm.header()
    if h.status != 0:
        raise dm.DictMergeError(h.status, "dm_dictionary_merge_sorted_async")
    # 5. counts -> offsets, rebase
    cnt = torch.tensor([h.merged_dict_len, h.merged_dict_len - L], dtype=torch.int64, device=dev)
    allc = allgather(cnt)
    n_u = [int(t[0]) for t in allc]
    n_new = [int(t[1]) for t in allc]
    off, new_off = sum(n_u[:rank]), sum(n_new[:rank])
    dm.rebase(lm.XM[:L], off)
    if mine.shape[0]:
        dm.rebase(lm.XD[:mine.shape[0]], off)
    xc_l = lm.xc()
    xc_l.rebase(new_off)
    # 6. the global tables, in rank (= value) order
    all_len = torch.tensor([L, int(mine.shape[0])], dtype=torch.int64, device=dev)
    all_l = allgather(all_len)
    Ls = [int(t[0]) for t in all_l]
    nds = [int(t[1]) for t in all_l]
    recs, offs, xds = [], [], []
    for g in range(world):
        nrec_g = (Ls[g] + SB - 1) // SB
        r_t = xc_l.records if g == rank else torch.empty(nrec_g * 8, dtype=torch.uint8, device=dev)
        recs.append(bcast(r_t.contiguous(), g))
        o_t = xc_l.offsets[:n_new[g]] if g == rank else torch.empty(n_new[g], dtype=torch.uint8, device=dev)
        if n_new[g]:
            offs.append(bcast(o_t.contiguous(), g))
        x_t = lm.XD[:nds[g]] if g == rank else torch.empty(nds[g], dtype=torch.int32, device=dev)
        if nds[g]:
            xds.append(bcast(x_t.contiguous(), g))
    n_off = sum(n_new)
    offsets = torch.zeros(((n_off + 31) // 16) * 16, dtype=torch.uint8, device=dev)
    if offs:
        offsets[:n_off] = torch.cat(offs)
    records = torch.cat(recs)
    xc = dm.XcTables(records, offsets, shift, records.numel() // 8)
    x_delta = torch.cat(xds) if xds else torch.empty(1, dtype=torch.int32, device=dev)
    # flagged superblocks: every rank ships its X_M slices, every rank scatters all
    ids, sl, nexc = dm.xc_exceptions_gather(xc_l, L, lm.XM)
    if nexc:
        dm.rebase(ids[:nexc], range_begin // SB)  # local -> global superblock ids
    ex = torch.tensor([nexc], dtype=torch.int64, device=dev)
    exs = allgather(ex)
    x_exc = torch.empty(max(dict_len, 1), dtype=torch.int32, device=dev)
    for g in range(world):
        k = int(exs[g].item())
        if not k:
            continue
        i_t = bcast((ids[:k] if g == rank else torch.empty(k, dtype=torch.int32, device=dev)).contiguous(), g)
        s_t = bcast((sl[:k * SB] if g == rank else torch.empty(k * SB, dtype=torch.int32, device=dev)).contiguous(), g)
        dm.xc_exceptions_scatter(xc, dict_len, i_t, s_t, k, x_exc)
    rk = bcast(dd.R[:max(n_delta, 1)].contiguous() if rank == root
               else torch.empty(max(n_delta, 1), dtype=torch.int32, device=dev), root)
    total = sum(n_u)
    return ShardedDictionary(lm.U[: h.merged_dict_len], off, total, dm.width(total), lm.XM[:L], xc, x_exc, x_delta,
                             rk, n_ud)
