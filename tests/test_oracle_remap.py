"""Pins for the C remap oracle (oracle/remap_oracle.c) -- SURVEY.md 8(c) c1.

Each test checks the oracle against something other than itself:
  (i)   numpy structured dtypes: a packed record of 'V<w>' fields *is* a
        cluster record (numpy computes the offsets), a field view of it *is*
        the field's slot (library routine);
  (ii)  special case: uniform-width AoS->SoA is the matrix transpose;
  (iii) invariants: round trip, composition, L->L, untouched gaps, record
        locality / shard equivalence, thread-split equality;
  (iv)  brute force over all 52^2 ordered layout pairs of 5 fields;
  (v)   tagged data names a misplaced slot; NaN payloads survive bit for bit.
"""

import numpy as np
import pytest

from adha_inputs import field_columns, tagged_columns, config_widths
from oracle import remap as O

SENT = 0xA5


def set_partitions(n):
    """All set partitions of range(n) as label lists (restricted growth strings)."""
    out = []

    def rec(i, labels, m):
        if i == n:
            out.append(list(labels))
            return
        for c in range(m + 1):
            labels.append(c)
            rec(i + 1, labels, max(m, c + 1))
            labels.pop()

    rec(0, [], 0)
    return out


def clusters_in_order(labels):
    """Clusters as lists of field indices: clusters by min decl index, fields by decl index.
    (The canonical order of SPEC.md:56, written here independently of the oracle.)"""
    order, members = [], {}
    for f, lab in enumerate(labels):
        if lab not in members:
            members[lab] = []
            order.append(lab)
        members[lab].append(f)
    return [members[lab] for lab in order]


def structured_regions(cols, widths, labels, n):
    """One numpy structured array per cluster, filled field by field from the columns."""
    out = []
    for cl in clusters_in_order(labels):
        dt = np.dtype([(f"f{f}", f"V{widths[f]}") for f in cl])     # numpy packs the record
        arr = np.zeros(n, dtype=dt)
        for f in cl:
            arr[f"f{f}"] = cols[f].reshape(n, widths[f]).view(f"V{widths[f]}").reshape(n)
        out.append((cl, arr))
    return out


def build_via_numpy(cols, widths, labels, n, fill=SENT):
    """Layout buffer built from numpy structured arrays, regions placed at the oracle's bases."""
    base, _, _, total = O.field_addresses(widths, labels, n)
    buf = np.full(total, fill, dtype=np.uint8)
    for cl, arr in structured_regions(cols, widths, labels, n):
        raw = arr.view(np.uint8)
        b = int(base[cl[0]])
        buf[b: b + raw.size] = raw
    return buf


def read_via_numpy(buf, widths, labels, n):
    base, _, _, _ = O.field_addresses(widths, labels, n)
    cols = [None] * len(widths)
    for cl in clusters_in_order(labels):
        dt = np.dtype([(f"f{f}", f"V{widths[f]}") for f in cl])
        b = int(base[cl[0]])
        arr = buf[b: b + n * dt.itemsize].view(dt)
        for f in cl:
            cols[f] = np.ascontiguousarray(arr[f"f{f}"]).view(np.uint8).reshape(n, widths[f])
    return cols


def test_structured_dtype_cross_oracle():
    rng = np.random.default_rng(1)
    for trial in range(60):
        F = int(rng.integers(1, 9))
        widths = [int(x) for x in rng.choice([1, 2, 3, 4, 8, 12], size=F)]
        ls = [int(x) for x in rng.integers(0, F, size=F)]
        ld = [int(x) for x in rng.integers(0, F, size=F)]
        n = int(rng.choice([0, 1, 7, 64, 1001]))
        cols = field_columns(100 + trial, n, widths)
        src = build_via_numpy(cols, widths, ls, n, fill=0x3C)
        assert np.array_equal(src, O.pack(cols, widths, ls, n, fill=0x3C))
        dst = np.full(O.layout_bytes(widths, ld, n), SENT, dtype=np.uint8)
        O.remap(src, ls, dst, ld, widths, n)
        back = read_via_numpy(dst, widths, ld, n)
        for f in range(F):
            assert np.array_equal(back[f], cols[f].reshape(n, widths[f])), (trial, f)
        # every byte that is not payload is still the sentinel
        mask = O.payload_mask(widths, ld, n)
        assert np.all(dst[~mask] == SENT)


def test_uniform_aos_to_soa_is_transpose():
    for F, n in [(3, 1024), (9, 333), (32, 100)]:
        widths = [4] * F
        src = np.frombuffer(np.random.default_rng(F).integers(0, 2 ** 32, size=n * F, dtype=np.uint32)
                            .tobytes(), dtype=np.uint8).copy()
        aos, soa = [0] * F, list(range(F))
        dst = np.zeros(O.layout_bytes(widths, soa, n), dtype=np.uint8)
        O.remap(src, aos, dst, soa, widths, n)
        T = src.view(np.uint32).reshape(n, F).T          # the transpose
        base, _, _, _ = O.field_addresses(widths, soa, n)
        for f in range(F):
            assert np.array_equal(dst[base[f]: base[f] + 4 * n].view(np.uint32), T[f])


def test_region_placement_reading_q3():
    widths = config_widths(16)
    for labels in ([0] * 16, list(range(16)), [0, 0, 1, 1, 2, 2, 2, 3, 4, 4, 5, 6, 7, 8, 8, 9]):
        for n in (0, 1, 3, 1000):
            base, stride, offset, total = O.field_addresses(widths, labels, n)
            first = {}
            for f in range(16):
                first.setdefault(labels[f], (int(base[f]), int(stride[f])))
            regs = list(first.values())                     # in canonical (first-sight) order
            assert regs[0][0] == 0
            for (b0, s0), (b1, s1) in zip(regs, regs[1:]):
                assert b1 % 256 == 0 and b1 >= b0 + n * s0 and b1 - (b0 + n * s0) < 256
                if n == 0:
                    assert b1 == 0
            assert total == regs[-1][0] + n * regs[-1][1]
            assert sum(s for _, s in regs) == sum(widths)


def test_round_trip_composition_and_identity():
    widths = config_widths(16)
    n = 777
    cols = field_columns(7, n, widths)
    aos, soa = [0] * 16, list(range(16))
    hyb = [0, 0, 0, 1, 2, 2, 3, 3, 3, 3, 4, 5, 6, 6, 6, 7]
    src = O.pack(cols, widths, aos, n)
    a2s = np.full(O.layout_bytes(widths, soa, n), SENT, np.uint8)
    O.remap(src, aos, a2s, soa, widths, n)
    back = np.full(src.size, SENT, np.uint8)
    O.remap(a2s, soa, back, aos, widths, n)
    assert np.array_equal(back, src)                       # AoS -> SoA -> AoS = identity
    a2h = np.full(O.layout_bytes(widths, hyb, n), SENT, np.uint8)
    O.remap(src, aos, a2h, hyb, widths, n)
    h2s = np.full(a2s.size, SENT, np.uint8)
    O.remap(a2h, hyb, h2s, soa, widths, n)
    assert np.array_equal(h2s, a2s)                        # AoS -> hybrid -> SoA = AoS -> SoA
    same = np.full(a2h.size, SENT, np.uint8)
    O.remap(a2h, hyb, same, hyb, widths, n)
    mask = O.payload_mask(widths, hyb, n)
    assert np.array_equal(same[mask], a2h[mask])           # L -> L copies the payload


def test_nan_payloads_survive():
    widths = [4, 8, 4, 8]
    n = 4096
    cols = field_columns(11, n, widths)
    f32 = cols[0].view(np.uint32).ravel()
    exp = (f32 >> 23) & 0xFF
    assert np.any((exp == 0xFF) & ((f32 & 0x400000) == 0) & ((f32 & 0x7FFFFF) != 0))   # sNaN present
    src = O.pack(cols, widths, [0, 0, 0, 0], n)
    dst = np.zeros(O.layout_bytes(widths, [0, 1, 2, 3], n), np.uint8)
    O.remap(src, [0, 0, 0, 0], dst, [0, 1, 2, 3], widths, n)
    out = O.unpack(dst, widths, [0, 1, 2, 3], n)
    for f in range(4):
        assert out[f].tobytes() == cols[f].tobytes()


def test_record_locality_and_shards():
    widths = config_widths(8)
    n = 1000
    cols = field_columns(3, n, widths)
    ls, ld = [0] * 8, [0, 1, 1, 2, 3, 3, 3, 4]
    src = O.pack(cols, widths, ls, n)
    full = np.full(O.layout_bytes(widths, ld, n), SENT, np.uint8)
    O.remap(src, ls, full, ld, widths, n)
    # range remap in two halves equals the full remap
    part = np.full(full.size, SENT, np.uint8)
    O.remap(src, ls, part, ld, widths, n, lo=0, hi=371)
    O.remap(src, ls, part, ld, widths, n, lo=371, hi=n)
    assert np.array_equal(part, full)
    # shards as their own layout instances: field-wise concatenation equals the full result
    G = 3
    full_cols = O.unpack(full, widths, ld, n)
    got = [[] for _ in widths]
    for g in range(G):
        lo, hi = g * n // G, (g + 1) * n // G
        sub = [c[lo:hi] for c in cols]
        s_src = O.pack(sub, widths, ls, hi - lo)
        s_dst = np.full(O.layout_bytes(widths, ld, hi - lo), SENT, np.uint8)
        O.remap(s_src, ls, s_dst, ld, widths, hi - lo)
        for f, c in enumerate(O.unpack(s_dst, widths, ld, hi - lo)):
            got[f].append(c)
    for f in range(len(widths)):
        assert np.array_equal(np.concatenate(got[f]), full_cols[f])


def test_thread_split_equals_single_thread():
    widths = config_widths(16)
    n = 50_000
    src = np.frombuffer(np.random.default_rng(5).bytes(n * 80), np.uint8).copy()
    ld = list(range(16))
    a = np.full(O.layout_bytes(widths, ld, n), SENT, np.uint8)
    b = a.copy()
    O.remap(src, [0] * 16, a, ld, widths, n)
    O.remap(src, [0] * 16, b, ld, widths, n, threads=4)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("n", [0, 1, 17, 33])
def test_brute_force_all_layout_pairs_5_fields(n):
    widths = [1, 2, 3, 4, 8]
    parts = set_partitions(5)
    assert len(parts) == 52
    cols = tagged_columns(n, widths)
    for ls in parts:
        src = build_via_numpy(cols, widths, ls, n, fill=0x11)
        for ld in parts:
            dst = np.full(O.layout_bytes(widths, ld, n), SENT, np.uint8)
            O.remap(src, ls, dst, ld, widths, n)
            exp = build_via_numpy(cols, widths, ld, n, fill=SENT)
            assert np.array_equal(dst, exp), (ls, ld)


def test_rejects_bad_arguments():
    with pytest.raises(ValueError):
        O.remap(np.zeros(4, np.uint8), [0, 0], np.zeros(100, np.uint8), [0, 1], [4, 4], 10)


# ----------------------------------------------------------------------------- generalised layouts (N4)

def _np_base(w):
    """numpy element type for a w-byte field: the largest power of two dividing w (<= 8) as an
    unsigned integer, repeated -- numpy's align=True then applies the C-struct rule."""
    a = 1
    while a < 8 and w % (a * 2) == 0:
        a *= 2
    t = {1: "u1", 2: "u2", 4: "u4", 8: "u8"}[a]
    return (t, (w // a,)) if w // a > 1 else t


def test_aligned_records_are_numpy_align_true_structs():
    """Natural alignment == numpy's align=True struct layout (offsets, itemsize) -- the C rule."""
    rng = np.random.default_rng(21)
    for trial in range(40):
        F = int(rng.integers(1, 8))
        widths = [int(x) for x in rng.choice([1, 2, 3, 4, 6, 8, 12, 16], size=F)]
        labels = [0] * F
        d = O.field_addresses_ex(widths, labels, 5, aligned=True)
        dt = np.dtype([(f"f{f}", _np_base(w)) for f, w in enumerate(widths)], align=True)
        assert int(d["stride"][0]) == dt.itemsize, (widths, dt)
        for f in range(F):
            assert int(d["offset"][f]) == dt.fields[f"f{f}"][1]
        # remap aligned AoS -> SoA -> aligned AoS: padding comes back as zeros, payload intact
        n = int(rng.integers(1, 300))
        cols = field_columns(trial, n, widths)
        src = np.zeros(n, dtype=dt)
        for f, w in enumerate(widths):
            src[f"f{f}"] = cols[f].reshape(n, w).view(dt.fields[f"f{f}"][0].base if dt.fields[f"f{f}"][0].shape
                                                     else dt.fields[f"f{f}"][0]).reshape(src[f"f{f}"].shape)
        src_b = src.view(np.uint8).copy()
        assert np.array_equal(src_b, O.pack_ex(cols, widths, labels, n, aligned=True))
        soa = np.full(O.layout_bytes_ex(widths, list(range(F)), n), SENT, np.uint8)
        O.remap_ex(src_b, labels, soa, list(range(F)), widths, n, src_aligned=True)
        back = np.full(src_b.size, SENT, np.uint8)
        O.remap_ex(soa, list(range(F)), back, labels, widths, n, dst_aligned=True)
        assert np.array_equal(back, src_b)


def test_aosoa_is_a_blocked_transpose():
    """AoSoA(B) of a uniform 4-byte record == reshape (N/B, B, F) -> transpose (0, 2, 1)."""
    for F, B, n in [(3, 8, 64), (5, 4, 37), (16, 32, 100), (2, 2, 9)]:
        widths = [4] * F
        x = np.random.default_rng(F * B).integers(0, 2 ** 32, size=(n, F), dtype=np.uint32)
        src = x.view(np.uint8).reshape(-1).copy()
        dst = np.full(O.layout_bytes_ex(widths, [0] * F, n, blocks=[B] * F), SENT, np.uint8)
        O.remap_ex(src, [0] * F, dst, [0] * F, widths, n, dst_blocks=[B] * F)
        nb = -(-n // B)
        pad = np.zeros((nb * B, F), np.uint32)
        pad[:n] = x
        exp = pad.reshape(nb, B, F).transpose(0, 2, 1).reshape(-1)
        assert np.array_equal(dst.view(np.uint32), exp)          # slots past N are zero


def test_generalised_round_trips_and_zero_fill():
    rng = np.random.default_rng(8)
    for trial in range(60):
        F = int(rng.integers(1, 7))
        widths = [int(x) for x in rng.choice([1, 2, 3, 4, 8], size=F)]
        ls = [int(x) for x in rng.integers(0, F, size=F)]
        ld = [int(x) for x in rng.integers(0, F, size=F)]
        cl_s = {lab: int(rng.choice([1, 2, 4, 8, 32])) for lab in set(ls)}
        cl_d = {lab: int(rng.choice([1, 2, 4, 8, 32])) for lab in set(ld)}
        bs, bd = [cl_s[l] for l in ls], [cl_d[l] for l in ld]
        als, ald = bool(rng.integers(2)), bool(rng.integers(2))
        n = int(rng.integers(0, 200))
        cols = field_columns(trial, n, widths)
        src = O.pack_ex(cols, widths, ls, n, bs, als)
        dst = np.full(O.layout_bytes_ex(widths, ld, n, bd, ald), SENT, np.uint8)
        O.remap_ex(src, ls, dst, ld, widths, n, bs, als, bd, ald)
        assert np.array_equal(dst, O.pack_ex(cols, widths, ld, n, bd, ald, fill=SENT))   # payload + zero padding
        back = np.full(src.size, 0x77, np.uint8)
        O.remap_ex(dst, ld, back, ls, widths, n, bd, ald, bs, als)
        assert np.array_equal(back, O.pack_ex(cols, widths, ls, n, bs, als, fill=0x77))
        for f, c in enumerate(O.unpack_ex(dst, widths, ld, n, bd, ald)):
            assert np.array_equal(c, cols[f])


def test_plain_layouts_unchanged_by_ex():
    """With blocks of 1 and no alignment the generalised oracle is the plain one."""
    widths = [1, 2, 3, 4, 8]
    for ls in set_partitions(5)[::7]:
        for ld in set_partitions(5)[::5]:
            n = 23
            cols = tagged_columns(n, widths)
            src = O.pack(cols, widths, ls, n)
            a = np.full(O.layout_bytes(widths, ld, n), SENT, np.uint8)
            b = a.copy()
            O.remap(src, ls, a, ld, widths, n)
            O.remap_ex(src, ls, b, ld, widths, n)
            assert np.array_equal(a, b)
