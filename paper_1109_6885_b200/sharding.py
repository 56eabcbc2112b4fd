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
  ``sharded_merge_column`` runs Steps 1(a)/1(b)/2(a) on the root device,
  broadcasts the header and the translation tables over NCCL (torch.distributed)
  -- by default the compact table XC (~67 MB for cfg5) instead of the literal X_M
  (4.3 GB) -- and every rank recompresses its own row range with
  ``dm_recompress_xc`` (or ``dm_recompress``).

The planning functions are plain Python (tested with gloo on the CPU); the
merge itself needs CUDA devices.
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
    """Cut the N' output rows into n_shards contiguous ranges at multiples of `align`
    (the delta rows follow the main rows)."""
    total = n_main + n_delta
    cuts = [0]
    for g in range(1, n_shards):
        c = (total * g // n_shards) // align * align
        cuts.append(max(c, cuts[-1]))
    cuts.append(total)
    shards = []
    for g in range(n_shards):
        r0, r1 = cuts[g], cuts[g + 1]
        m0, m1 = min(r0, n_main), min(r1, n_main)
        d0, d1 = max(r0, n_main) - n_main, max(r1, n_main) - n_main
        shards.append(RowShard(r0, r1, m0, m1, d0, d1))
    return shards


def sharded_merge_column(main_dict, main_codes_shard, n_main: int, main_bits: int, delta, shard: RowShard,
                         group=None, root: int = 0, tables: str = "xc"):
    """Row-sharded merge of one column across the ranks of `group` (one GPU each).

    Every rank passes its own packed main-code slice (`main_codes_shard`, the words
    of rows [shard.main_begin, shard.main_end)).  The root also passes U_M and D
    (other ranks may pass empty tensors with the right dtype).  Returns this rank's
    packed output slice (rows [shard.row_begin, shard.row_end) at b'), b', |U'|, and
    on the root U' as well.

    tables="xc" (default): the root broadcasts the compact table XC (8-byte records
    + one byte per new value; ~67 MB for cfg5) and the X_M slices of the rare
    flagged superblocks, instead of the literal X_M (4.3 GB for cfg5, SURVEY §8e's
    control design, tables="plain").  X_D and r follow as before.
    """
    import torch
    import torch.distributed as dist
    import paper_1109_6885_b200 as dm

    rank = dist.get_rank(group)
    dev = torch.device("cuda", torch.cuda.current_device())
    # |U'|, |U_D|, b', |U_M|, N_D, use_xc, shift, n_records, offset bytes, exception count
    hdr = torch.zeros(10, dtype=torch.int64, device=dev)
    U = merger = xc = None
    if rank == root:
        merger = dm.DictionaryMerger(main_dict, n_main, main_bits, delta)
        merger.run_async()
        h = merger.header()
        if h.status != 0:
            raise dm.DictMergeError(h.status, "dm_dictionary_merge_async")
        U = merger.U[: h.merged_dict_len]
        xc = merger.xc() if tables == "xc" else None
        exc = dm.xc_exceptions_gather(xc, main_dict.shape[0], merger.XM) if xc is not None else None
        hdr.copy_(torch.tensor([h.merged_dict_len, h.delta_dict_len, h.merged_bits, main_dict.shape[0],
                                delta.shape[0], int(xc is not None), xc.shift if xc else 0,
                                xc.n_records if xc else 0, xc.offsets.numel() if xc else 0,
                                exc[2] if exc else 0], dtype=torch.int64))
    dist.broadcast(hdr, src=root, group=group)
    n_u, n_ud, nb, dict_len, n_delta, use_xc, shift, n_rec, n_off, n_exc = (int(x) for x in hdr.tolist())

    def bcast(t_root, shape, dtype):
        t = t_root if rank == root else torch.empty(shape, dtype=dtype, device=dev)
        dist.broadcast(t, src=root, group=group)
        return t

    if use_xc:
        rec = bcast(xc.records if xc else None, (n_rec * 8,), torch.uint8)
        offs = bcast(xc.offsets if xc else None, (n_off,), torch.uint8)
        tabs = dm.XcTables(rec, offs, shift, n_rec)
        if rank == root:
            xm = merger.XM[:dict_len]
        else:
            xm = torch.empty(max(dict_len, 1), dtype=torch.int32, device=dev)  # only exception slices are read
        if n_exc:
            sb = 4 << shift
            ids = bcast(exc[0] if rank == root else None, (n_exc,), torch.int32)
            sl = bcast(exc[1] if rank == root else None, (n_exc * sb,), torch.int32)
            if rank != root:
                dm.xc_exceptions_scatter(tabs, dict_len, ids, sl, n_exc, xm)
    else:
        xm = bcast(merger.XM[:dict_len] if rank == root else None, (max(dict_len, 1),), torch.int32)
    xd = bcast(merger.XD[: max(n_ud, 1)] if rank == root else None, (max(n_ud, 1),), torch.int32) if n_delta \
        else torch.empty(1, dtype=torch.int32, device=dev)
    rk = bcast(merger.R[: max(n_delta, 1)] if rank == root else None, (max(n_delta, 1),), torch.int32) if n_delta \
        else torch.empty(1, dtype=torch.int32, device=dev)
    if use_xc:
        out = dm.recompress_xc(main_codes_shard, shard.n_main, main_bits, dict_len, tabs, xm, xd,
                               rk[shard.delta_begin:], shard.n_delta, nb)
    else:
        out = dm.recompress(main_codes_shard, shard.n_main, main_bits, dict_len, xm, xd, rk[shard.delta_begin:],
                            shard.n_delta, nb)
    return out, nb, n_u, U
