"""paper_1109_6885_b200 -- B200-native online merge for dictionary-encoded column stores.

Thin Python binding over ``libdictmerge.so`` (C ABI: ``include/dictmerge.h``).
This module only marshals arguments: PyTorch allocates device memory and
supplies the CUDA stream; every step of the merge (Krueger et al., arXiv
1109.6885, Sec 5: Step 1(a) delta dictionary, Step 1(b) dictionary merge with
translation tables X_M / X_D, Step 2(a) width, Step 2(b) recompression) runs in
the library's sm_100a kernels.  There is no CPU fallback: importing this
package without the built library raises.

Key tensors: ``"u64"`` keys are 1-D ``torch.int64`` tensors holding the u64 bit
patterns (compared unsigned); ``"u32"`` keys (the paper's E = 4) are 1-D
``torch.int32`` tensors holding u32 bit patterns; ``"b16"`` keys are ``torch.uint8`` tensors of
shape (n, 16) (compared bytewise).  Packed code vectors are 1-D ``torch.int64``
tensors of little-endian u64 words (LSB-first bitstream).
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
from typing import Optional, Sequence

import torch

from . import build as _build

__all__ = [
    "KEY_U64", "KEY_B16", "Status", "DictMergeError", "width", "words", "merged_codes_cap_words",
    "workspace_bytes", "merge_column", "merge_column_async", "merge_table", "pack_codes", "unpack_codes",
    "ColumnMerger", "HostContext", "launch_count", "lib_path", "set_tuning", "XcTables", "recompress_xc",
    "xc_exceptions_gather", "xc_exceptions_scatter", "lower_bound", "rebase", "DictionaryMerger", "get_tuning",
    "tuning", "Comm", "plan_row_shards", "merge_column_sharded", "ShardedResult", "sharded_codes_cap_words",
    "plan_dict_ranges",
]

KEY_U64, KEY_B16, KEY_U32 = 0, 1, 2
_KEY = {"u64": KEY_U64, "b16": KEY_B16, "u32": KEY_U32}


class Status:
    OK, E_INVALID, E_CAPACITY, E_TOO_WIDE, E_UNSORTED, E_CODE_RANGE, E_CUDA, E_NCCL = 0, -1, -2, -3, -4, -5, -6, -7


class DictMergeError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = _lib().dm_status_str(status).decode()
        if status == Status.E_CUDA:
            msg += f" (cudaError {int(_lib().dm_last_cuda_error())})"
        super().__init__(f"{where}: {msg} [{status}]")
        self.status = status


class _In(ctypes.Structure):
    _fields_ = [("key", ctypes.c_int32), ("main_dict", ctypes.c_void_p), ("dict_len", ctypes.c_uint64),
                ("main_codes", ctypes.c_void_p), ("n_main", ctypes.c_uint64), ("main_bits", ctypes.c_uint32),
                ("delta", ctypes.c_void_p), ("n_delta", ctypes.c_uint64)]


class _Out(ctypes.Structure):
    _fields_ = [("merged_dict", ctypes.c_void_p), ("merged_dict_cap", ctypes.c_uint64),
                ("merged_codes", ctypes.c_void_p), ("merged_codes_cap_words", ctypes.c_uint64),
                ("x_main", ctypes.c_void_p), ("x_delta", ctypes.c_void_p), ("delta_dict", ctypes.c_void_p),
                ("delta_rank", ctypes.c_void_p), ("merged_dict_len", ctypes.c_uint64),
                ("delta_dict_len", ctypes.c_uint64), ("merged_bits", ctypes.c_uint32)]


class _Xc(ctypes.Structure):
    _fields_ = [("records", ctypes.c_void_p), ("n_records", ctypes.c_uint64), ("offsets", ctypes.c_void_p),
                ("offsets_cap", ctypes.c_uint64), ("shift", ctypes.c_uint32), ("built", ctypes.c_int32)]


class _ShIn(ctypes.Structure):
    _fields_ = [("key", ctypes.c_int32), ("tables", ctypes.c_int32), ("root", ctypes.c_int32),
                ("step1b", ctypes.c_int32), ("main_dict", ctypes.c_void_p), ("dict_len", ctypes.c_uint64),
                ("range_begin", ctypes.c_uint64), ("range_len", ctypes.c_uint64), ("delta", ctypes.c_void_p),
                ("n_delta", ctypes.c_uint64), ("main_codes", ctypes.c_void_p), ("n_main", ctypes.c_uint64),
                ("main_bits", ctypes.c_uint32)]


class _ShOut(ctypes.Structure):
    _fields_ = [("merged_dict", ctypes.c_void_p), ("merged_dict_cap", ctypes.c_uint64),
                ("merged_codes", ctypes.c_void_p), ("merged_codes_cap_words", ctypes.c_uint64),
                ("merged_dict_len", ctypes.c_uint64), ("merged_bits", ctypes.c_uint32),
                ("merged_dict_offset", ctypes.c_uint64), ("merged_slice_len", ctypes.c_uint64)]


_CB_BCAST = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p)
_CB_AGATHER = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p)
_CB_SENDRECV = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                ctypes.c_void_p)


class _Cbs(ctypes.Structure):
    _fields_ = [("broadcast", _CB_BCAST), ("allgather", _CB_AGATHER), ("sendrecv", _CB_SENDRECV),
                ("user", ctypes.c_void_p)]


class _Hdr(ctypes.Structure):
    _fields_ = [("merged_dict_len", ctypes.c_uint64), ("delta_dict_len", ctypes.c_uint64),
                ("merged_bits", ctypes.c_uint32), ("status", ctypes.c_int32)]


_L = None


def lib_path() -> str:
    return _build.LIB


def _lib():
    global _L
    if _L is None:
        if not os.path.exists(_build.LIB):
            raise ImportError(f"libdictmerge.so is not built ({_build.LIB}); run "
                              "`python -m paper_1109_6885_b200.build` or __graft_entry__.build(). "
                              "There is no CPU fallback.")
        L = ctypes.CDLL(os.environ.get("DM_LIB_PATH", _build.LIB))
        u64, u32, vp, i32 = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_int
        P = ctypes.POINTER
        sig = {
            "dm_width": (u32, [u64]),
            "dm_words": (u64, [u64, u32]),
            "dm_merged_codes_cap_words": (u64, [P(_In)]),
            "dm_workspace_bytes": (ctypes.c_size_t, [P(_In)]),
            "dm_merge_column_async": (i32, [P(_In), P(_Out), vp, ctypes.c_size_t, vp, vp]),
            "dm_merge_column_async_ev": (i32, [P(_In), P(_Out), vp, ctypes.c_size_t, vp, vp, P(vp)]),
            "dm_merge_column": (i32, [P(_In), P(_Out), vp, ctypes.c_size_t, vp]),
            "dm_recompress": (i32, [vp, u64, u32, u64, vp, vp, vp, u64, u32, vp, u64, vp]),
            "dm_merge_table": (i32, [i32, P(_In), P(_Out), P(vp), P(ctypes.c_size_t), vp]),
            "dm_merge_table_async": (i32, [i32, P(_In), P(_Out), P(vp), P(ctypes.c_size_t), P(vp), vp]),
            "dm_dictionary_merge_async": (i32, [P(_In), P(_Out), vp, ctypes.c_size_t, vp, vp]),
            "dm_delta_dictionary_async": (i32, [P(_In), P(_Out), vp, ctypes.c_size_t, vp, vp]),
            "dm_dictionary_merge_sorted_async": (i32, [P(_In), P(_Out), vp, ctypes.c_size_t, vp, vp]),
            "dm_lower_bound_async": (i32, [i32, vp, u64, vp, u64, vp, vp]),
            "dm_rebase_async": (i32, [vp, u64, u32, vp]),
            "dm_xc_rebase_async": (i32, [vp, u64, u32, vp]),
            "dm_pack_codes": (i32, [vp, u64, u32, vp, vp]),
            "dm_unpack_codes": (i32, [vp, u64, u32, vp, vp]),
            "dm_ctx_create": (vp, [i32]),
            "dm_ctx_destroy": (None, [vp]),
            "dm_merge_column_host": (i32, [vp, P(_In), P(_Out)]),
            "dm_launch_count": (u64, []),
            "dm_set_tuning": (i32, [i32, i32]),
            "dm_get_tuning": (i32, [i32]),
            "dm_xc_export": (i32, [P(_In), vp, ctypes.c_size_t, P(_Xc)]),
            "dm_xc_exceptions_gather": (i32, [P(_Xc), u64, vp, vp, vp, vp, vp]),
            "dm_xc_exceptions_scatter": (i32, [P(_Xc), u64, vp, vp, u64, vp, vp]),
            "dm_recompress_xc": (i32, [vp, u64, u32, u64, P(_Xc), vp, vp, vp, u64, u32, vp, u64, vp]),
            "dm_last_cuda_error": (i32, []),
            "dm_comm_nccl_unique_id": (i32, [vp]),
            "dm_comm_init_nccl": (vp, [vp, i32, i32, i32]),
            "dm_comm_init_callbacks": (vp, [P(_Cbs), i32, i32]),
            "dm_comm_destroy": (None, [vp]),
            "dm_comm_rank": (i32, [vp]),
            "dm_comm_size": (i32, [vp]),
            "dm_comm_selftest_host": (i32, [vp]),
            "dm_plan_row_shards": (None, [u64, u64, i32, P(u64)]),
            "dm_plan_dict_ranges": (None, [u64, i32, P(u64)]),
            "dm_sharded_codes_cap_words": (u64, [u64, u64, u64, i32, i32]),
            "dm_merge_column_sharded": (i32, [vp, P(_ShIn), P(_ShOut), vp]),
            "dm_status_str": (ctypes.c_char_p, [i32]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _L = L
    return _L


# ------------------------------------------------------------------ pure helpers
def width(n: int) -> int:
    """max(1, ceil(log2 n)) -- Eq 4, reading A1."""
    return int(_lib().dm_width(n))


def words(n: int, bits: int) -> int:
    return int(_lib().dm_words(n, bits))


def launch_count() -> int:
    return int(_lib().dm_launch_count())


XM_AUTO, XM_PLAIN, XM_COMPACT, XM_COMPACT_L2 = 0, 1, 2, 3
KNOB_XMODE, KNOB_MERGE, KNOB_DEDUP, KNOB_STEP2, KNOB_XC_SHIFT, KNOB_SORT1A, KNOB_STEP2_FORM, KNOB_SP_GRID = \
    0, 1, 2, 3, 4, 5, 6, 7


def set_tuning(knob: int, value: int) -> None:
    """dm_set_tuning (include/dictmerge.h): knob 0 = Step 2(b) translation-table
    placement (XM_* above), 1 = Step 1(b) variant, 2 = Step 1(a) dedup front end,
    3 = Step 2 variant (1 = the paper's naive binary-search baseline), 4 = XC
    block shift, 5 = Step 1(a) sort (0 auto, 1 LSD passes, 2 bucket path), 6 =
    Step 2(b) form with XC in shared memory (0 thread-per-group, 1 warp-per-group), 7 =
    sparse Step 1(b) grid (0 one resident wave, 1 a CTA per tile, 2 three CTAs).  Never
    changes results; used by tests and experiments to select kernel variants."""
    st = _lib().dm_set_tuning(knob, value)
    if st != Status.OK:
        raise DictMergeError(st, "dm_set_tuning")


def get_tuning(knob: int) -> int:
    """dm_get_tuning: the knob's current value."""
    v = int(_lib().dm_get_tuning(knob))
    if v < 0:
        raise DictMergeError(v, "dm_get_tuning")
    return v


class tuning:
    """Context manager: set a knob, restore its previous value on exit (the knobs
    are process-wide)."""

    def __init__(self, knob: int, value: int):
        self.knob, self.value, self.old = knob, value, None

    def __enter__(self):
        self.old = get_tuning(self.knob)
        set_tuning(self.knob, self.value)
        return self

    def __exit__(self, *exc):
        set_tuning(self.knob, self.old)
        return False


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None or t.numel() == 0 else t.data_ptr()


def _key_of(t: torch.Tensor) -> int:
    if t.dtype == torch.uint8 and t.dim() == 2:
        return KEY_B16
    return KEY_U32 if t.dtype == torch.int32 else KEY_U64


def _make_in(main_dict, main_codes, n_main, main_bits, delta) -> _In:
    key = _key_of(main_dict) if main_dict.numel() else _key_of(delta)
    return _In(key, _ptr(main_dict), main_dict.shape[0], _ptr(main_codes), n_main, main_bits, _ptr(delta),
               delta.shape[0])


def merged_codes_cap_words(cin: _In) -> int:
    return int(_lib().dm_merged_codes_cap_words(ctypes.byref(cin)))


def workspace_bytes(cin: _In) -> int:
    return int(_lib().dm_workspace_bytes(ctypes.byref(cin)))


def _stream_handle(stream) -> Optional[int]:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _empty_keys(key: int, n: int, device) -> torch.Tensor:
    if key == KEY_U64:
        return torch.empty(max(n, 2), dtype=torch.int64, device=device)
    if key == KEY_U32:
        return torch.empty(max(n, 4), dtype=torch.int32, device=device)
    return torch.empty((max(n, 1), 16), dtype=torch.uint8, device=device)


@dataclasses.dataclass
class MergeResult:
    merged_dict: torch.Tensor            # U' (|U'| keys)
    merged_codes: torch.Tensor           # M' (exactly words(N', b') u64 words, as int64)
    merged_bits: int                     # b'
    delta_dict_len: int                  # |U_D|
    x_main: Optional[torch.Tensor] = None
    x_delta: Optional[torch.Tensor] = None
    delta_dict: Optional[torch.Tensor] = None
    delta_rank: Optional[torch.Tensor] = None

    @property
    def merged_len(self) -> int:
        return int(self.merged_dict.shape[0])


class ColumnMerger:
    """Pre-allocated merge of one column shape: outputs, workspace and a device
    result header live as long as the object, so ``run_async`` launches the
    whole path with no allocation and no host synchronisation (graph-capturable)."""

    def __init__(self, main_dict: torch.Tensor, main_codes: torch.Tensor, n_main: int, main_bits: int,
                 delta: torch.Tensor, *, x_tables: bool = False, delta_dict: bool = False):
        dev = main_dict.device if main_dict.numel() else delta.device
        if dev.type != "cuda":
            raise ValueError("merge_column needs CUDA tensors (there is no CPU path)")
        self.inputs = (main_dict, main_codes, delta)
        self.cin = _make_in(main_dict, main_codes, n_main, main_bits, delta)
        key = self.cin.key
        nU = main_dict.shape[0] + delta.shape[0]
        self.n_total = n_main + delta.shape[0]
        self.U = _empty_keys(key, nU, dev)
        cap = merged_codes_cap_words(self.cin)
        self.M = torch.empty(max(cap, 2), dtype=torch.int64, device=dev)
        self.XM = torch.empty(max(main_dict.shape[0], 1), dtype=torch.int32, device=dev) if x_tables else None
        self.XD = torch.empty(max(delta.shape[0], 1), dtype=torch.int32, device=dev) if x_tables else None
        self.UD = _empty_keys(key, delta.shape[0], dev) if delta_dict else None
        self.R = torch.empty(max(delta.shape[0], 1), dtype=torch.int32, device=dev) if delta_dict else None
        self.cout = _Out(_ptr(self.U), nU, _ptr(self.M), cap, _ptr(self.XM), _ptr(self.XD), _ptr(self.UD),
                         _ptr(self.R), 0, 0, 0)
        self.ws_bytes = workspace_bytes(self.cin)
        self.ws = torch.empty(max(self.ws_bytes, 256), dtype=torch.uint8, device=dev)
        self.hdr = torch.zeros(4, dtype=torch.int64, device=dev)  # dm_header (24 B, 16-B aligned)

    def run_async(self, stream=None) -> None:
        st = _lib().dm_merge_column_async(ctypes.byref(self.cin), ctypes.byref(self.cout), self.ws.data_ptr(),
                                          self.ws_bytes, self.hdr.data_ptr(), _stream_handle(stream))
        if st != Status.OK:
            raise DictMergeError(st, "dm_merge_column_async")

    def capture_graph(self) -> "torch.cuda.CUDAGraph":
        """Capture one whole merge (memset + all kernels, no host sync) into a CUDA
        graph; ``replay_graph`` then relaunches it with one driver call."""
        self.run_async()  # warm the library's per-device launch caches outside capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        with torch.cuda.graph(g, stream=side):
            self.run_async()
        torch.cuda.synchronize()
        self.graph = g
        return g

    def replay_graph(self) -> None:
        self.graph.replay()

    def run_async_timed(self, events, stream=None) -> None:
        """As run_async, recording 4 torch.cuda.Events at the step boundaries
        (before 1(a), before 1(b), before 2(b), after 2(b))."""
        evs = (ctypes.c_void_p * 4)(*[e.cuda_event for e in events])
        st = _lib().dm_merge_column_async_ev(ctypes.byref(self.cin), ctypes.byref(self.cout), self.ws.data_ptr(),
                                             self.ws_bytes, self.hdr.data_ptr(), _stream_handle(stream), evs)
        if st != Status.OK:
            raise DictMergeError(st, "dm_merge_column_async_ev")

    def header(self) -> _Hdr:
        raw = self.hdr.cpu().numpy().tobytes()
        return _Hdr.from_buffer_copy(raw[: ctypes.sizeof(_Hdr)])

    def result(self) -> MergeResult:
        h = self.header()
        if h.status != Status.OK:
            raise DictMergeError(h.status, "dm_merge_column")
        nw = words(self.n_total, h.merged_bits)
        return MergeResult(
            self.U[: h.merged_dict_len], self.M[:nw], int(h.merged_bits), int(h.delta_dict_len),
            None if self.XM is None else self.XM[: self.cin.dict_len],
            None if self.XD is None else self.XD[: h.delta_dict_len],
            None if self.UD is None else self.UD[: h.delta_dict_len],
            None if self.R is None else self.R[: self.cin.n_delta])


def merge_column(main_dict: torch.Tensor, main_codes: torch.Tensor, n_main: int, main_bits: int,
                 delta: torch.Tensor, *, x_tables: bool = False, delta_dict: bool = False,
                 stream=None) -> MergeResult:
    """Merge one column (synchronous): returns U', M', b' (+ X_M / X_D / U_D / r on request)."""
    m = ColumnMerger(main_dict, main_codes, n_main, main_bits, delta, x_tables=x_tables, delta_dict=delta_dict)
    m.run_async(stream)
    return m.result()


def merge_column_async(merger: ColumnMerger, stream=None) -> None:
    merger.run_async(stream)


def merge_table(columns: Sequence[tuple], *, stream=None) -> list:
    """Merge independent columns of a wide table through dm_merge_table.

    ``columns``: sequence of (main_dict, main_codes, n_main, main_bits, delta) on one device."""
    n = len(columns)
    ms = [ColumnMerger(*c) for c in columns]
    ins = (_In * n)(*[m.cin for m in ms])
    outs = (_Out * n)(*[m.cout for m in ms])
    wss = (ctypes.c_void_p * n)(*[m.ws.data_ptr() for m in ms])
    wsb = (ctypes.c_size_t * n)(*[m.ws_bytes for m in ms])
    st = _lib().dm_merge_table(n, ins, outs, wss, wsb, _stream_handle(stream))
    if st != Status.OK:
        raise DictMergeError(st, "dm_merge_table")
    res = []
    for m, o in zip(ms, outs):
        nw = words(m.n_total, o.merged_bits)
        res.append(MergeResult(m.U[: o.merged_dict_len], m.M[:nw], int(o.merged_bits), int(o.delta_dict_len)))
    return res


class TableMerger:
    """Pre-allocated merge of a wide table's independent columns
    through ``dm_merge_table_async``: one call launches every column on the
    library's stream pool; graph-capturable like ColumnMerger."""

    def __init__(self, columns: Sequence[tuple], *, x_tables: bool = False):
        self.ms = [ColumnMerger(*c, x_tables=x_tables) for c in columns]
        n = len(self.ms)
        self.n = n
        self.ins = (_In * n)(*[m.cin for m in self.ms])
        self.outs = (_Out * n)(*[m.cout for m in self.ms])
        self.wss = (ctypes.c_void_p * n)(*[m.ws.data_ptr() for m in self.ms])
        self.wsb = (ctypes.c_size_t * n)(*[m.ws_bytes for m in self.ms])
        self.hdrs = (ctypes.c_void_p * n)(*[m.hdr.data_ptr() for m in self.ms])
        self.graph = None

    def run_async(self, stream=None) -> None:
        st = _lib().dm_merge_table_async(self.n, self.ins, self.outs, self.wss, self.wsb, self.hdrs,
                                         _stream_handle(stream))
        if st != Status.OK:
            raise DictMergeError(st, "dm_merge_table_async")

    def capture_graph(self):
        self.run_async()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        with torch.cuda.graph(g, stream=side):
            self.run_async()
        torch.cuda.synchronize()
        self.graph = g
        return g

    def replay_graph(self) -> None:
        self.graph.replay()

    def results(self) -> list:
        return [m.result() for m in self.ms]

    @property
    def tuples(self) -> int:
        return sum(m.n_total for m in self.ms)


class DictionaryMerger:
    """Steps 1(a), 1(b), 2(a) only (``dm_dictionary_merge_async``): U', X_M, X_D,
    U_D, r and the header -- the root's part of the row-sharded merge.

    mode "delta": Step 1(a) alone (``dm_delta_dictionary_async``: U_D, r);
    mode "sorted": ``delta`` already is U_D (sorted, distinct), Steps 1(b)/2(a)
    only (``dm_dictionary_merge_sorted_async``) -- one value range of the
    sharded Step 1(b)."""

    _ENTRY = {"dict": "dm_dictionary_merge_async", "delta": "dm_delta_dictionary_async",
              "sorted": "dm_dictionary_merge_sorted_async"}

    def __init__(self, main_dict: torch.Tensor, n_main: int, main_bits: int, delta: torch.Tensor,
                 mode: str = "dict"):
        self.mode = mode
        dev = main_dict.device if main_dict.numel() else delta.device
        self.cin = _make_in(main_dict, None, n_main, main_bits, delta)
        self.cin.main_codes = None
        key = self.cin.key
        nU = main_dict.shape[0] + delta.shape[0]
        self.U = _empty_keys(key, nU, dev)
        self.XM = torch.empty(max(main_dict.shape[0], 1), dtype=torch.int32, device=dev)
        self.XD = torch.empty(max(delta.shape[0], 1), dtype=torch.int32, device=dev)
        self.UD = _empty_keys(key, delta.shape[0], dev)
        self.R = torch.empty(max(delta.shape[0], 1), dtype=torch.int32, device=dev)
        self.cout = _Out(_ptr(self.U), nU, None, 0, _ptr(self.XM), _ptr(self.XD), _ptr(self.UD), _ptr(self.R),
                         0, 0, 0)
        self.ws_bytes = workspace_bytes(self.cin)
        self.ws = torch.empty(max(self.ws_bytes, 256), dtype=torch.uint8, device=dev)
        self.hdr = torch.zeros(4, dtype=torch.int64, device=dev)
        self.inputs = (main_dict, delta)

    def run_async(self, stream=None) -> None:
        name = self._ENTRY[self.mode]
        st = getattr(_lib(), name)(ctypes.byref(self.cin), ctypes.byref(self.cout), self.ws.data_ptr(),
                                   self.ws_bytes, self.hdr.data_ptr(), _stream_handle(stream))
        if st != Status.OK:
            raise DictMergeError(st, name)

    def header(self) -> _Hdr:
        raw = self.hdr.cpu().numpy().tobytes()
        return _Hdr.from_buffer_copy(raw[: ctypes.sizeof(_Hdr)])

    def xc(self) -> Optional["XcTables"]:
        """The compact table XC built by the last run (None when |U_M| * 4 <= 96 KB,
        where the plain X_M is as small)."""
        x = _Xc()
        st = _lib().dm_xc_export(ctypes.byref(self.cin), self.ws.data_ptr(), self.ws_bytes, ctypes.byref(x))
        if st != Status.OK:
            raise DictMergeError(st, "dm_xc_export")
        if not x.built:
            return None
        h = self.header()
        n_new = int(h.merged_dict_len) - int(self.cin.dict_len)
        base = self.ws.data_ptr()
        r0 = x.records - base
        o0 = x.offsets - base
        return XcTables(self.ws[r0: r0 + x.n_records * 8], self.ws[o0: o0 + ((n_new + 31) // 16) * 16],
                        int(x.shift), int(x.n_records))


def lower_bound(sorted_keys: torch.Tensor, values: torch.Tensor, n: Optional[int] = None, stream=None) -> torch.Tensor:
    """pos[i] = #{sorted_keys[j] < values[i]} (``dm_lower_bound_async``), int64."""
    key = _key_of(sorted_keys if sorted_keys.numel() else values)
    nv = values.shape[0]
    pos = torch.empty(max(nv, 1), dtype=torch.int64, device=values.device)
    st = _lib().dm_lower_bound_async(key, _ptr(sorted_keys), sorted_keys.shape[0] if n is None else n,
                                     _ptr(values), nv, pos.data_ptr(), _stream_handle(stream))
    if st != Status.OK:
        raise DictMergeError(st, "dm_lower_bound_async")
    return pos[:nv]


def rebase(x: torch.Tensor, add: int, stream=None) -> None:
    """x += add in place for an int32 tensor of u32 values (``dm_rebase_async``)."""
    st = _lib().dm_rebase_async(_ptr(x), x.numel(), add, _stream_handle(stream))
    if st != Status.OK:
        raise DictMergeError(st, "dm_rebase_async")


@dataclasses.dataclass
class XcTables:
    """The compact translation table XC of one merge (``dm_xc``): 8-byte records
    and one offset byte per new value (include/dictmerge.h).  ``records`` and
    ``offsets`` are uint8 device tensors (views into a workspace on the root, or
    received copies on other ranks)."""
    records: torch.Tensor
    offsets: torch.Tensor
    shift: int
    n_records: int

    def struct(self) -> _Xc:
        return _Xc(_ptr(self.records), self.n_records, _ptr(self.offsets), self.offsets.numel(), self.shift, 1)

    def rebase(self, add: int, stream=None) -> None:
        """R += add in every record (``dm_xc_rebase_async``): new values of earlier ranges."""
        st = _lib().dm_xc_rebase_async(_ptr(self.records), self.n_records, add, _stream_handle(stream))
        if st != Status.OK:
            raise DictMergeError(st, "dm_xc_rebase_async")


def xc_exceptions_gather(xc: XcTables, dict_len: int, x_main: torch.Tensor, stream=None):
    """X_M slices of XC's flagged superblocks -> (ids int32, slices int32, count)."""
    dev = x_main.device
    sb = 4 << xc.shift
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    # count first (ids = slices = NULL), then size the buffers by the count: the
    # flagged superblocks are rare, a worst-case buffer would be X_M-sized
    st = _lib().dm_xc_exceptions_gather(ctypes.byref(xc.struct()), dict_len, _ptr(x_main), None, None,
                                        cnt.data_ptr(), _stream_handle(stream))
    if st != Status.OK:
        raise DictMergeError(st, "dm_xc_exceptions_gather")
    n = int(cnt[0].item())
    ids = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    slices = torch.empty(max(n * sb, 1), dtype=torch.int32, device=dev)
    if n:
        cnt.zero_()
        st = _lib().dm_xc_exceptions_gather(ctypes.byref(xc.struct()), dict_len, _ptr(x_main), ids.data_ptr(),
                                            slices.data_ptr(), cnt.data_ptr(), _stream_handle(stream))
        if st != Status.OK:
            raise DictMergeError(st, "dm_xc_exceptions_gather")
    return ids, slices, n


def xc_exceptions_scatter(xc: XcTables, dict_len: int, ids: torch.Tensor, slices: torch.Tensor, count: int,
                          x_main: torch.Tensor, stream=None) -> None:
    st = _lib().dm_xc_exceptions_scatter(ctypes.byref(xc.struct()), dict_len, _ptr(ids), _ptr(slices), count,
                                         _ptr(x_main), _stream_handle(stream))
    if st != Status.OK:
        raise DictMergeError(st, "dm_xc_exceptions_scatter")


def recompress_xc(main_codes: torch.Tensor, n_main: int, main_bits: int, dict_len: int, xc: XcTables,
                  x_main: torch.Tensor, x_delta: torch.Tensor, delta_rank: torch.Tensor, n_delta: int,
                  new_bits: int, stream=None) -> torch.Tensor:
    """Step 2(b) of a row shard through XC (``dm_recompress_xc``); x_main is read
    only for flagged superblocks."""
    dev = xc.records.device
    nw = words(n_main + n_delta, new_bits)
    out = torch.empty(max(nw, 2), dtype=torch.int64, device=dev)
    st = _lib().dm_recompress_xc(_ptr(main_codes) if n_main else None, n_main, main_bits, dict_len,
                                 ctypes.byref(xc.struct()), _ptr(x_main), _ptr(x_delta) if n_delta else None,
                                 _ptr(delta_rank) if n_delta else None, n_delta, new_bits, out.data_ptr(),
                                 out.numel(), _stream_handle(stream))
    if st != Status.OK:
        raise DictMergeError(st, "dm_recompress_xc")
    return out[:nw]


def recompress(main_codes: torch.Tensor, n_main: int, main_bits: int, dict_len: int, x_main: torch.Tensor,
               x_delta: torch.Tensor, delta_rank: torch.Tensor, n_delta: int, new_bits: int,
               stream=None) -> torch.Tensor:
    """Step 2(b) alone (``dm_recompress``): returns words(n_main + n_delta, new_bits) u64 words."""
    dev = x_main.device
    nw = words(n_main + n_delta, new_bits)
    out = torch.empty(max(nw, 2), dtype=torch.int64, device=dev)
    st = _lib().dm_recompress(_ptr(main_codes) if n_main else None, n_main, main_bits, dict_len,
                              _ptr(x_main), _ptr(x_delta) if n_delta else None,
                              _ptr(delta_rank) if n_delta else None, n_delta, new_bits, out.data_ptr(), out.numel(),
                              _stream_handle(stream))
    if st != Status.OK:
        raise DictMergeError(st, "dm_recompress")
    return out[:nw]


def pack_codes(codes: torch.Tensor, bits: int, stream=None) -> torch.Tensor:
    """Pack u32 codes (int32 tensor) at ``bits`` into words(n, bits) u64 words (library kernel)."""
    n = codes.numel()
    out = torch.empty(max(words(n, bits), 2), dtype=torch.int64, device=codes.device)
    st = _lib().dm_pack_codes(_ptr(codes), n, bits, out.data_ptr(), _stream_handle(stream))
    if st != Status.OK:
        raise DictMergeError(st, "dm_pack_codes")
    return out[: words(n, bits)]


def unpack_codes(w: torch.Tensor, n: int, bits: int, stream=None) -> torch.Tensor:
    out = torch.empty(max(n, 1), dtype=torch.int32, device=w.device)
    st = _lib().dm_unpack_codes(_ptr(w), n, bits, out.data_ptr(), _stream_handle(stream))
    if st != Status.OK:
        raise DictMergeError(st, "dm_unpack_codes")
    return out[:n]


class HostContext:
    """dm_ctx: merges columns held in HOST memory (inputs copied in, results copied
    back inside the call).  Buffers should be pinned for full PCIe bandwidth."""

    def __init__(self, device: int = 0):
        self.h = _lib().dm_ctx_create(device)
        if not self.h:
            raise DictMergeError(Status.E_CUDA, "dm_ctx_create")

    def close(self):
        if self.h:
            _lib().dm_ctx_destroy(self.h)
            self.h = None

    __del__ = close

    def merge(self, main_dict: torch.Tensor, main_codes: torch.Tensor, n_main: int, main_bits: int,
              delta: torch.Tensor, out_dict: torch.Tensor, out_codes: torch.Tensor) -> tuple:
        """All tensors on the CPU.  Returns (|U'|, b', |U_D|); U' and M' land in out_dict / out_codes."""
        cin = _make_in(main_dict, main_codes, n_main, main_bits, delta)
        cout = _Out(_ptr(out_dict), out_dict.shape[0], _ptr(out_codes), out_codes.numel(), None, None, None,
                    None, 0, 0, 0)
        st = _lib().dm_merge_column_host(self.h, ctypes.byref(cin), ctypes.byref(cout))
        if st != Status.OK:
            raise DictMergeError(st, "dm_merge_column_host")
        return int(cout.merged_dict_len), int(cout.merged_bits), int(cout.delta_dict_len)


# ------------------------------------------------------------------ sharded merge
def plan_row_shards(n_main: int, n_delta: int, nranks: int) -> list:
    """dm_plan_row_shards: output-row cuts [0, ..., N'] (every cut but the last a
    multiple of 4096) -- rank g owns rows [cuts[g], cuts[g+1])."""
    cuts = (ctypes.c_uint64 * (nranks + 1))()
    _lib().dm_plan_row_shards(n_main, n_delta, nranks, cuts)
    return [int(c) for c in cuts]


def plan_dict_ranges(dict_len: int, nranks: int) -> list:
    """dm_plan_dict_ranges: U_M position cuts for the value-range sharded Step 1(b)
    (every cut but the last a multiple of 1024)."""
    cuts = (ctypes.c_uint64 * (nranks + 1))()
    _lib().dm_plan_dict_ranges(dict_len, nranks, cuts)
    return [int(c) for c in cuts]


def sharded_codes_cap_words(dict_len: int, n_main: int, n_delta: int, nranks: int, rank: int) -> int:
    return int(_lib().dm_sharded_codes_cap_words(dict_len, n_main, n_delta, nranks, rank))


class Comm:
    """dm_comm: the transport of a sharded merge.  ``Comm.nccl()`` -- NCCL over
    NVLink (the library resolves NCCL from the process; the unique id travels over
    the torch.distributed default group); ``Comm.callbacks()`` -- host-buffer
    callbacks over a torch.distributed process group (gloo on the CPU: the
    multi-process tests; the library stages device data through pinned memory)."""

    def __init__(self, handle, keep=None):
        if not handle:
            raise DictMergeError(Status.E_NCCL, "dm_comm_init")
        self.h = handle
        self._keep = keep

    @property
    def rank(self) -> int:
        return int(_lib().dm_comm_rank(self.h))

    @property
    def size(self) -> int:
        return int(_lib().dm_comm_size(self.h))

    @classmethod
    def nccl(cls, group=None, device: Optional[int] = None) -> "Comm":
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            st = _lib().dm_comm_nccl_unique_id(uid.data_ptr())
            if st != Status.OK:
                raise DictMergeError(st, "dm_comm_nccl_unique_id")
        dev = torch.cuda.current_device() if device is None else device
        # the id over the process group (NCCL groups need a CUDA tensor)
        t = uid.cuda(dev) if dist.get_backend(group) == "nccl" else uid
        dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        uid = t.cpu()
        return cls(_lib().dm_comm_init_nccl(uid.data_ptr(), world, rank, dev))

    @classmethod
    def callbacks(cls, group=None) -> "Comm":
        import numpy as np
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        glob = (lambda r: dist.get_global_rank(group, r)) if group is not None else (lambda r: r)

        def view(ptr, n):
            return torch.from_numpy(np.ctypeslib.as_array((ctypes.c_uint8 * n).from_address(ptr)))

        def bcast(buf, n, root, _user):
            try:
                t = view(buf, n)
                dist.broadcast(t, src=glob(root), group=group)
                return 0
            except Exception:  # noqa: BLE001 -- reported to the library as a transport failure
                return 1

        def agather(send, recv, n, _user):
            try:
                out = [torch.empty(n, dtype=torch.uint8) for _ in range(world)]
                dist.all_gather(out, view(send, n).clone(), group=group)
                view(recv, n * world).copy_(torch.cat(out))
                return 0
            except Exception:  # noqa: BLE001
                return 1

        def sendrecv(buf, n, peer, is_send, _user):
            try:
                t = view(buf, n)
                if is_send:
                    dist.send(t.clone(), dst=glob(peer), group=group)
                else:
                    dist.recv(t, src=glob(peer), group=group)
                return 0
            except Exception:  # noqa: BLE001
                return 1

        cbs = _Cbs(_CB_BCAST(bcast), _CB_AGATHER(agather), _CB_SENDRECV(sendrecv), None)
        return cls(_lib().dm_comm_init_callbacks(ctypes.byref(cbs), world, rank), keep=cbs)

    def selftest_host(self) -> int:
        return int(_lib().dm_comm_selftest_host(self.h))

    def close(self):
        if self.h:
            _lib().dm_comm_destroy(self.h)
            self.h = None

    __del__ = close


@dataclasses.dataclass
class ShardedResult:
    merged_codes: torch.Tensor           # this rank's M' words (rows [cuts[g], cuts[g+1]) at b')
    merged_bits: int                     # b'
    merged_len: int                      # |U'|
    merged_dict: Optional[torch.Tensor]  # U' on the root (step1b "root"), this rank's U' slice ("ranges")
    row_begin: int
    row_end: int
    merged_dict_offset: int = 0          # "ranges": U' index of merged_dict[0]


def merge_column_sharded(comm: Comm, main_codes_shard: torch.Tensor, n_main: int, main_bits: int, dict_len: int,
                         n_delta: int, *, main_dict: Optional[torch.Tensor] = None,
                         delta: Optional[torch.Tensor] = None, key: str = "u64", tables: str = "xc",
                         root: int = 0, step1b: str = "root", range_begin: int = 0,
                         stream=None) -> ShardedResult:
    """dm_merge_column_sharded: this rank's part of one column's merge (collective).
    ``main_codes_shard``: the packed main codes of this rank's main rows
    (plan_row_shards); the root also passes D (``delta``).  step1b "root": the
    root passes the whole U_M (``main_dict``) and merges the dictionary;
    "ranges" (NEXT2): every rank passes its U_M range (``main_dict``, starting at
    ``range_begin``, a plan_dict_ranges cut) and gets its slice of U'."""
    nr, me = comm.size, comm.rank
    cuts = plan_row_shards(n_main, n_delta, nr)
    dev = main_codes_shard.device if main_codes_shard is not None else torch.device("cuda", torch.cuda.current_device())
    cap = sharded_codes_cap_words(dict_len, n_main, n_delta, nr, me)
    out_codes = torch.empty(max(cap, 2), dtype=torch.int64, device=dev)
    ranges = step1b == "ranges"
    rlen = int(main_dict.shape[0]) if ranges else 0
    ucap = rlen + n_delta if ranges else (dict_len + n_delta if me == root else 0)
    U = _empty_keys(_KEY[key], ucap, dev) if (ranges or me == root) else None
    md = _ptr(main_dict) if (ranges or me == root) else None
    cin = _ShIn(_KEY[key], 0 if tables == "xc" else 1, root, 1 if ranges else 0, md, dict_len, range_begin, rlen,
                _ptr(delta) if me == root else None, n_delta, _ptr(main_codes_shard), n_main, main_bits)
    cout = _ShOut(_ptr(U), ucap, out_codes.data_ptr(), out_codes.numel(), 0, 0, 0, 0)
    st = _lib().dm_merge_column_sharded(comm.h, ctypes.byref(cin), ctypes.byref(cout), _stream_handle(stream))
    if st != Status.OK:
        raise DictMergeError(st, "dm_merge_column_sharded")
    nb = int(cout.merged_bits)
    r0, r1 = cuts[me], cuts[me + 1]
    nw = (r1 * nb + 63) // 64 - r0 * nb // 64
    if ranges:
        Uo = U[: cout.merged_slice_len]
    else:
        Uo = U[: cout.merged_dict_len] if U is not None else None
    return ShardedResult(out_codes[:nw], nb, int(cout.merged_dict_len), Uo, r0, r1, int(cout.merged_dict_offset))
