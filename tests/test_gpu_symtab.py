"""Device SYMR ingest and dictionary build (symtab.cu; SURVEY.md §8(a) a3-a5,
§8(f) row 2): parse_symbols' checks (symfile.cpp:117-157) evaluated per entry on
the GPU with the reference's first-error semantics, and the byte-wise sorted
name dictionary (std::string order, folded.cpp:18) built by a device sort —
including names with NUL bytes, bytes >= 0x80, shared 8-byte prefixes and
prefix relations, and names shared between tables.
"""
import numpy as np
import pytest

import paper_2603_29235_b200 as stg
from oracle import ref
from tests.synth import build_id, pack_symr

pytestmark = pytest.mark.gpu

TRICKY = [b"a", b"a\x00", b"a\x00b", b"ab", b"b", b"\xff", b"\x80zz", b"\x7f",
          b"common_prefix_long_name_1", b"common_prefix_long_name_10", b"common_prefix_long_name_2",
          b"common_p", b"common_pr", b"common_prefix", b"x" * 300, b"x" * 299 + b"y", b"x" * 301,
          b"z\x00\x00\x00\x00\x00\x00\x00\x00", b"z\x00\x00\x00\x00\x00\x00\x00", b"z"]


def _table(label, names, seed):
    rng = np.random.default_rng(seed)
    starts = np.sort(rng.choice(np.arange(1, 1 << 20, dtype=np.uint64), size=len(names), replace=False)) * 16
    return build_id(label), starts, pack_symr(build_id(label), starts, np.full(len(names), 8, np.uint32), names)


def test_dictionary_order_and_sharing():
    c = stg.Context(0)
    try:
        n1 = TRICKY + [b"sym_%06d" % i for i in range(3000)]
        n2 = TRICKY[::-1][:12] + [b"sym_%06d" % i for i in range(2000, 5000)] + [b"only_in_2"]
        id1, s1, p1 = _table("dict-1", n1, 1)
        id2, s2, p2 = _table("dict-2", n2, 2)
        c.ingest(p1)
        c.ingest(p2)
        # entries are sorted by start inside pack_symr: map names to their starts
        q = np.concatenate([s1, s2])
        bins = np.concatenate([np.zeros(len(s1), np.uint16), np.ones(len(s2), np.uint16)])
        got_names, keys = c.resolve(q, bins, np.frombuffer(id1 + id2, np.uint8))
        names = list(n1) + list(n2)
        dict_sorted = sorted(set(names))
        exp = np.array([dict_sorted.index(n) for n in names], np.uint32)
        assert np.array_equal(keys, exp)
        assert got_names == [n.decode("utf-8", "surrogateescape") for n in names]
    finally:
        c.close()


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("case", ["unsorted_then_offset", "len_then_unsorted", "offset_only", "zero_len_last"])
def test_first_error_in_large_table(ctx, case):
    n = 100_000
    names = [b"f%d" % i for i in range(n)]
    bid, starts, good = _table("err-big", names, 9)
    b = bytearray(good)
    ent = lambda i: 36 + 16 * i
    strtab_len = len(good) - (36 + 16 * n)
    if case == "unsorted_then_offset":
        b[ent(70_000):ent(70_000) + 8] = (0).to_bytes(8, "little")                 # start regresses
        b[ent(90_000) + 12:ent(90_000) + 16] = (strtab_len + 5).to_bytes(4, "little")
    elif case == "len_then_unsorted":
        no = int.from_bytes(good[ent(50_000) + 12:ent(50_000) + 16], "little")
        s0 = 36 + 16 * n + no
        b[s0:s0 + 2] = (60_000).to_bytes(2, "little")                               # name runs past the end
        b[ent(60_000):ent(60_000) + 8] = (1).to_bytes(8, "little")
    elif case == "offset_only":
        b[ent(99_999) + 12:ent(99_999) + 16] = (strtab_len - 1).to_bytes(4, "little")
    else:
        no = int.from_bytes(good[ent(n - 1) + 12:ent(n - 1) + 16], "little")
        s0 = 36 + 16 * n + no
        b[s0:s0 + 2] = (0).to_bytes(2, "little")
    b = bytes(b)
    exp = ref.parse_error(b)
    assert exp is not None
    with pytest.raises(stg.StgError) as e:
        ctx.ingest(b)
    assert str(e.value) == exp
