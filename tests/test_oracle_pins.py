"""Pins for the CPU oracle (tests/../oracle) against what the paper and mathematics fix.

Each test names the pin it implements (DESIGN.md "Oracle pins" P1-P7).  None of
them re-types the oracle's own code: expected values come from the paper's
printed facts, closed forms, an independent big-integer formulation of the
bitstream, Python-set brute force on tiny domains, or agreement between the
oracle's two independently written modes.
"""
import itertools
import json
import os

import numpy as np
import pytest

import datagen
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def s16(s: str) -> bytes:
    b = s.encode()
    assert len(b) <= 16
    return b + b"\x00" * (16 - len(b))


def b16_array(strs):
    return np.frombuffer(b"".join(s16(s) for s in strs), dtype=np.uint8).reshape(-1, 16).copy()


class Col:
    def __init__(self, key, main_dict, main_codes, main_bits, delta):
        self.key = key
        self.main_dict = main_dict
        self.main_codes = np.asarray(main_codes, dtype=np.uint32)
        self.main_bits = main_bits
        self.delta = delta

    key_bytes = property(lambda s: {"u64": 8, "u32": 4}.get(s.key, 16))
    n_main = property(lambda s: int(s.main_codes.size))


def bigint_pack(codes, bits):
    """Independent formulation of the LSB-first stream: one big integer whose bit
    i*bits+t is bit t of code i; words are its little-endian 64-bit digits."""
    s = 0
    for i, c in enumerate(codes):
        s |= int(c) << (i * bits)
    nw = (len(codes) * bits + 63) // 64
    return np.array([(s >> (64 * w)) & ((1 << 64) - 1) for w in range(nw)], dtype=np.uint64)


def keys_as_tuples(a, key):
    return [int(x) for x in a] if key in ("u64", "u32") else [bytes(r) for r in a]


# ------------------------------------------------------------------------- P1
@pytest.mark.parametrize("mode", ["linear", "definitional"])
def test_p1_worked_example(mode):
    g = json.load(open(os.path.join(GOLDEN, "worked_example.json")))
    f = g["paper_facts"]
    col = Col("b16", b16_array(g["main_dict"]), g["main_codes"], f["main_bits"]["value"], b16_array(g["delta"]))
    # instance consistency with the paper's text
    assert len(g["main_dict"]) == f["main_dict_len"]["value"]
    assert oracle.width(len(g["main_dict"])) == f["main_bits"]["value"]
    assert len(g["delta"]) == f["n_delta"]["value"]
    assert [k for k, v in enumerate(g["delta"]) if v == "charlie"] == f["charlie_positions"]["value"]
    assert g["main_codes"][0] == f["first_main_code"]["value"]
    assert format(g["main_codes"][0], "03b") == f["first_main_code_bits_at_3"]["value"]
    assert g["main_dict"][f["hotel_code_before_after"]["value"][0]] == "hotel"

    r = oracle.merge(col, mode)
    assert r.status == oracle.OK
    assert r.delta_dict.shape[0] == f["delta_dict_len"]["value"]
    assert oracle.width(r.delta_dict.shape[0]) == f["delta_bits"]["value"]
    assert r.merged_len == f["merged_len"]["value"]
    assert r.merged_bits == f["merged_bits"]["value"]
    assert int(r.x_main[f["first_main_code"]["value"]]) == f["x_main_at_4"]["value"]
    hotel_new = [bytes(x) for x in r.merged_dict].index(s16("hotel"))
    assert hotel_new == f["hotel_code_before_after"]["value"][1]

    d = g["derived"]
    assert [bytes(x) for x in r.merged_dict] == [s16(s) for s in d["merged_dict"]]
    assert [bytes(x) for x in r.delta_dict] == [s16(s) for s in d["delta_dict"]]
    assert r.x_main.tolist() == d["x_main"]
    assert r.x_delta.tolist() == d["x_delta"]
    codes = oracle.unpack(r.merged_words, 12, r.merged_bits)
    assert codes.tolist() == d["merged_codes"]
    assert [hex(int(w)) for w in r.merged_words] == [hex(int(h, 16)) for h in d["merged_words_hex"]]
    assert [hex(int(w)) for w in oracle.pack(g["main_codes"], 3)] == [hex(int(h, 16)) for h in d["main_words_hex"]]
    if mode == "linear":
        assert r.delta_rank.tolist() == d["delta_rank"]
    # semantic identity (P5) on the example itself
    dec = [bytes(r.merged_dict[c]) for c in codes]
    want = [s16(g["main_dict"][c]) for c in g["main_codes"]] + [s16(s) for s in g["delta"]]
    assert dec == want


# ------------------------------------------------------------------------- P2
def test_p2_width_closed_form():
    # printed examples and the config widths BASELINE.json states
    assert oracle.width(6) == 3 and oracle.width(9) == 4
    assert oracle.width(10**4) == 14 and oracle.width(10**7) == 24 and oracle.width(10**6) == 20
    assert oracle.width(1 << 30) == 30
    assert oracle.width((1 << 30) + 5 * 10**7) == 31          # cfg5 under reading A12
    assert oracle.width(10**9 + 5 * 10**7) == 30              # the literal cfg5 (no growth)
    assert oracle.width(1) == 1 and oracle.width(0) == 1      # reading A1
    ns = list(range(2, 5000)) + [2**k + d for k in range(12, 33) for d in (-1, 0, 1)]
    for n in ns:
        w = oracle.width(n)
        assert 2 ** (w - 1) < n <= 2 ** w, n                   # the unique w of ceil(log2 n)


def test_p2_words():
    for n in range(0, 300):
        for b in (1, 3, 7, 14, 24, 31, 32):
            assert oracle.words(n, b) * 64 >= n * b > (oracle.words(n, b) - 1) * 64 or n * b == 0


# ------------------------------------------------------------------------- P6
def test_p6_layout_vectors():
    g = json.load(open(os.path.join(GOLDEN, "bit_layout.json")))
    for c in g["cases"]:
        codes = c["codes"] if "codes" in c else [i % 2 for i in range(70)]
        want = [int(h, 16) for h in c["words_hex"]]
        assert oracle.pack(codes, c["bits"]).tolist() == want
        assert bigint_pack(codes, c["bits"]).tolist() == want


@pytest.mark.parametrize("bits", list(range(1, 33)))
def test_p6_pack_matches_bigint_and_roundtrips(bits):
    rng = np.random.default_rng(bits)
    for n in (0, 1, 31, 32, 33, 63, 64, 65, 127, 200):
        codes = rng.integers(0, 2 ** bits, size=n, dtype=np.uint64).astype(np.uint32)
        w = oracle.pack(codes, bits)
        assert w.tolist() == bigint_pack(codes, bits).tolist()
        assert oracle.unpack(w, n, bits).tolist() == codes.tolist()


# ------------------------------------------------------------------------- P7
def brute(main_dict, main_codes, delta):
    """Definition by Python sets on tiny inputs: output column = main then delta,
    dictionary = sorted distinct union, code = position (Eq 3)."""
    U = sorted(set(main_dict) | set(delta))
    V = [main_dict[c] for c in main_codes] + list(delta)
    nb = 1
    while 2 ** nb < len(U):
        nb += 1
    codes = [U.index(v) for v in V]
    UD = sorted(set(delta))
    return U, nb, codes, [U.index(v) for v in main_dict], [U.index(v) for v in UD], UD


def _check_brute(mode, main_dict, main_codes, delta, bits, key="u64"):
    dt = np.uint64 if key == "u64" else np.uint32
    col = Col(key, np.array(main_dict, dtype=dt), main_codes, bits, np.array(delta, dtype=dt))
    r = oracle.merge(col, mode)
    assert r.status == oracle.OK
    U, nb, codes, xm, xd, UD = brute(main_dict, main_codes, delta)
    assert r.merged_dict.tolist() == U
    assert r.merged_bits == nb
    assert r.merged_words.tolist() == bigint_pack(codes, nb).tolist()
    assert r.x_main.tolist() == xm
    assert r.x_delta.tolist() == xd
    assert r.delta_dict.tolist() == UD


@pytest.mark.parametrize("mode", ["linear", "definitional"])
def test_p7_brute_force_exhaustive_tiny(mode):
    dom = [0, 3, 5, 9, 2**63, 2**64 - 1]  # includes unsigned-order edges (reading A5)
    n = 0
    for k in range(0, 4):
        for md in itertools.combinations(dom[:5], k):
            md = list(md)
            code_seqs = [[]] if not md else [list(s) for L in range(0, 3) for s in itertools.product(range(len(md)), repeat=L)]
            for cs in code_seqs:
                for L in range(0, 3):
                    for dl in itertools.product(dom, repeat=L):
                        bits = oracle.width(max(len(md), 1))
                        _check_brute(mode, md, cs, list(dl), bits)
                        n += 1
    assert n > 1000


@pytest.mark.parametrize("mode", ["linear", "definitional"])
def test_p7_brute_force_exhaustive_tiny_u32(mode):
    # 4-byte keys (NEXT4, E = 4): the same exhaustive sweep with u32 order edges
    dom = [0, 3, 9, 2**31, 2**32 - 1]
    n = 0
    for k in range(0, 4):
        for md in itertools.combinations(dom[:4], k):
            md = list(md)
            code_seqs = [[]] if not md else [list(s) for L in range(0, 3) for s in itertools.product(range(len(md)), repeat=L)]
            for cs in code_seqs:
                for L in range(0, 3):
                    for dl in itertools.product(dom, repeat=L):
                        _check_brute(mode, md, cs, list(dl), oracle.width(max(len(md), 1)), key="u32")
                        n += 1
    assert n > 500


# -------------------------------------------------------------- P3/P4/P5 random
def _invariants(col, r):
    key = col.key
    UM = keys_as_tuples(col.main_dict, key)
    D = keys_as_tuples(col.delta, key)
    U = keys_as_tuples(r.merged_dict, key)
    UD = keys_as_tuples(r.delta_dict, key)
    # P3: strictly increasing; the size law
    assert all(a < b for a, b in zip(U, U[1:]))
    assert set(U) == set(UM) | set(D)
    assert UD == sorted(set(D))
    assert len(U) == len(UM) + len(UD) - len(set(UM) & set(UD))
    # P2 on the output
    assert 2 ** (r.merged_bits - 1) < max(len(U), 2) <= 2 ** r.merged_bits
    # P4: closed forms X_M[i] = i + #{v in U_D \ U_M : v < U_M[i]}, symmetric for X_D
    new = np.array(sorted(set(UD) - set(UM)), dtype=object)
    old = np.array(sorted(set(UM) - set(UD)), dtype=object)
    xm = [i + int(np.searchsorted(new, v, side="left")) if len(new) else i for i, v in enumerate(UM)]
    xd = [j + int(np.searchsorted(old, v, side="left")) if len(old) else j for j, v in enumerate(UD)]
    assert r.x_main.tolist() == xm
    assert r.x_delta.tolist() == xd
    assert all(U[x] == v for x, v in zip(r.x_main.tolist(), UM))
    assert set(r.x_main.tolist()) | set(r.x_delta.tolist()) == set(range(len(U)))
    # P5: decode(U', M') == decode(U_M, M) ++ D
    codes = oracle.unpack(r.merged_words, col.n_main + len(D), r.merged_bits)
    assert [U[c] for c in codes.tolist()] == [UM[c] for c in col.main_codes.tolist()] + D
    # pad bits zero
    nbits = (col.n_main + len(D)) * r.merged_bits
    if nbits % 64:
        assert int(r.merged_words[-1]) >> (nbits % 64) == 0


@pytest.mark.parametrize("key", ["u64", "b16", "u32"])
@pytest.mark.parametrize("seed", range(6))
def test_p345_random_invariants_and_modes_agree(key, seed):
    rng = np.random.default_rng(seed)
    for t in range(8):
        n_main = int(rng.integers(0, 2000))
        dict_len = int(rng.integers(1, 600))
        n_delta = int(rng.integers(0, 500))
        p_new = [0.0, 0.001, 0.01, 0.1, 0.5, 1.0][t % 6]
        vb = int(rng.choice([10, 20, 64 if key != "u32" else 32]))
        col = datagen.make_random_case(1000 * seed + t, n_main, dict_len, n_delta, p_new, key=key,
                                       value_bits=vb, main_bits=oracle.width(dict_len) + int(rng.integers(0, 3)))
        a = oracle.merge(col, "linear")
        b = oracle.merge(col, "definitional")
        assert a.status == b.status == oracle.OK
        for f in ("merged_dict", "merged_words", "x_main", "x_delta", "delta_dict"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), f
        assert a.merged_bits == b.merged_bits
        _invariants(col, a)


# ------------------------------------------------------------------ edge cases
def test_edge_empty_delta_is_identity_when_width_minimal():
    col = datagen.make_random_case(7, 1000, 300, 0, 0.0)
    col.main_bits = oracle.width(300)
    r = oracle.merge(col)
    assert r.merged_words.tolist() == oracle.pack(col.main_codes, col.main_bits).tolist()
    assert r.x_main.tolist() == list(range(300))
    assert r.delta_dict.shape[0] == 0


def test_edge_empty_main():
    col = Col("u64", np.zeros(0, np.uint64), [], 1, np.array([5, 3, 5, 9], dtype=np.uint64))
    r = oracle.merge(col)
    assert r.merged_dict.tolist() == [3, 5, 9]
    assert oracle.unpack(r.merged_words, 4, r.merged_bits).tolist() == [1, 0, 1, 2]
    col = Col("u64", np.zeros(0, np.uint64), [], 1, np.zeros(0, np.uint64))
    r = oracle.merge(col)
    assert r.status == oracle.OK and r.merged_len == 0 and r.merged_bits == 1 and r.merged_words.size == 0


def test_edge_all_reuse_and_all_new():
    col = datagen.make_random_case(9, 500, 200, 300, 0.0)
    r = oracle.merge(col)
    assert r.x_main.tolist() == list(range(200))          # all-reuse -> identity
    col = datagen.make_random_case(10, 500, 200, 300, 1.0)
    r = oracle.merge(col)
    UD = r.delta_dict
    assert (r.x_main - np.arange(200)).tolist() == np.searchsorted(UD, col.main_dict, side="left").tolist()


def test_edge_single_entry_dictionary():
    col = Col("u64", np.array([42], np.uint64), [0] * 70, 1, np.array([42, 42], np.uint64))
    r = oracle.merge(col)
    assert r.merged_bits == 1 and r.merged_len == 1
    assert r.merged_words.tolist() == [0, 0]


def test_errors():
    col = Col("u64", np.array([5, 3], np.uint64), [0], 1, np.zeros(0, np.uint64))
    assert oracle.merge(col).status == oracle.E_UNSORTED
    col = Col("u64", np.array([3, 3], np.uint64), [0], 1, np.zeros(0, np.uint64))
    assert oracle.merge(col).status == oracle.E_UNSORTED
    col = Col("u64", np.array([3, 5, 7], np.uint64), [0, 3], 2, np.zeros(0, np.uint64))
    assert oracle.merge(col).status == oracle.E_CODE_RANGE
    col = Col("u64", np.array([3, 5, 7], np.uint64), [0, 1], 1, np.zeros(0, np.uint64))
    assert oracle.merge(col).status == oracle.E_INVALID


def test_b16_order_edges():
    # reading A5: unsigned bytewise order over all 16 bytes, zero padding included
    strs = [b"", b"a", b"a\x00b", b"\x7f", b"\x80", b"\xff" * 16, b"ab", b"b"]
    arr = np.frombuffer(b"".join(s + b"\x00" * (16 - len(s)) for s in strs), np.uint8).reshape(-1, 16)
    want = sorted(bytes(r) for r in arr)
    col = Col("b16", np.zeros((0, 16), np.uint8), [], 1, arr.copy())
    r = oracle.merge(col)
    assert [bytes(x) for x in r.merged_dict] == want
    assert want.index(b"\x7f" + b"\x00" * 15) < want.index(b"\x80" + b"\x00" * 15)


@pytest.mark.parametrize("key", ["u64", "b16", "u32"])
def test_codes_at_agrees_with_full_merge(key):
    col = datagen.make_random_case(77, 3000, 500, 700, 0.4, key=key)
    r = oracle.merge(col, "definitional")
    V = np.concatenate([col.main_dict[col.main_codes.astype(np.int64)], col.delta])
    codes, n = oracle.codes_at(col.main_dict, col.delta, V, key_bytes=col.key_bytes)
    assert n == r.merged_len
    assert codes.tolist() == oracle.unpack(r.merged_words, V.shape[0], r.merged_bits).tolist()
