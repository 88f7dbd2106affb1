"""Property-based checks (hypothesis, CPU only) of the oracle and the C ABI's host logic, over
random widths, partitions, AoSoA blocks, alignment and record counts.  Each property is one the
paper's data model fixes: the remap is a bijection on payload bytes,
composes, round-trips, equals a structured-array view, and the C ABI's descriptor places every
field where the (independently written) oracle address model does."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from oracle import remap as O

A = pytest.importorskip("paper_1407_4859_b200")

SET = settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.too_slow])


@st.composite
def layouts(draw, max_fields=7):
    F = draw(st.integers(1, max_fields))
    widths = draw(st.lists(st.sampled_from([1, 2, 3, 4, 6, 8, 12, 16]), min_size=F, max_size=F))
    return widths


@st.composite
def partition(draw, F):
    labels = draw(st.lists(st.integers(0, F - 1), min_size=F, max_size=F))
    return labels


@st.composite
def layout_triple(draw):
    widths = draw(layouts())
    F = len(widths)
    parts = [draw(partition(F)) for _ in range(3)]
    n = draw(st.sampled_from([0, 1, 2, 31, 32, 33, 100, 257]))
    return widths, parts, n


def _random_src(widths, labels, n, seed):
    rng = np.random.default_rng(seed)
    cols = [rng.integers(0, 256, size=(n, w), dtype=np.uint8) for w in widths]
    return cols, O.pack(cols, widths, labels, n)


@SET
@given(layout_triple(), st.integers(0, 2 ** 31))
def test_oracle_round_trip_and_composition(t, seed):
    widths, (l1, l2, l3), n = t
    cols, src = _random_src(widths, l1, n, seed)
    b2 = np.zeros(O.layout_bytes(widths, l2, n), np.uint8)
    b3 = np.zeros(O.layout_bytes(widths, l3, n), np.uint8)
    O.remap(src, l1, b2, l2, widths, n)
    O.remap(b2, l2, b3, l3, widths, n)
    direct = np.zeros_like(b3)
    O.remap(src, l1, direct, l3, widths, n)
    assert np.array_equal(b3, direct)                       # L1 -> L2 -> L3 == L1 -> L3
    back = np.zeros(O.layout_bytes(widths, l1, n), np.uint8)
    O.remap(b2, l2, back, l1, widths, n)
    mask = O.payload_mask(widths, l1, n)
    assert np.array_equal(back[mask], src[mask])           # round trip restores every payload byte
    for f, c in enumerate(O.unpack(b3, widths, l3, n)):
        assert np.array_equal(c, cols[f])                   # fields land where the layout says


@SET
@given(layouts(), st.data())
def test_oracle_is_a_numpy_structured_view(widths, data):
    """A packed cluster record is a numpy structured dtype with V<w> fields at the packed offsets;
    its region is the contiguous array of those records (SURVEY 8(c) pin (i))."""
    F = len(widths)
    labels = data.draw(partition(F))
    n = data.draw(st.integers(0, 50))
    cols, buf = _random_src(widths, labels, n, data.draw(st.integers(0, 999)))
    base, stride, off, _ = O.field_addresses(widths, labels, n)
    for f in range(F):
        members = [g for g in range(F) if labels[g] == labels[f]]
        dt = np.dtype({"names": [f"f{g}" for g in members], "formats": [f"V{widths[g]}" for g in members],
                       "offsets": [int(off[g]) for g in members], "itemsize": int(stride[f])})
        region = buf[int(base[f]): int(base[f]) + n * int(stride[f])].view(dt) if n else np.zeros(0, dt)
        got = np.frombuffer(np.ascontiguousarray(region[f"f{f}"]).tobytes(), np.uint8).reshape(n, widths[f])
        assert np.array_equal(got, cols[f])


@SET
@given(layouts(max_fields=9), st.data())
def test_capi_descriptor_matches_oracle_address_model(widths, data):
    F = len(widths)
    labels = data.draw(partition(F))
    blocks = data.draw(st.one_of(st.none(), st.lists(st.sampled_from([1, 2, 4, 8, 16, 32]), min_size=F,
                                                     max_size=F)))
    aligned = data.draw(st.booleans())
    n = data.draw(st.integers(0, 5000))
    if blocks is not None:
        # one block size per cluster (the first field's)
        first = {}
        for f, c in enumerate(labels):
            first.setdefault(c, blocks[f])
        blocks = [first[c] for c in labels]
    L = A.Layout(widths, labels, blocks=blocks, aligned=aligned)
    d = O.field_addresses_ex(widths, labels, n, blocks, aligned)
    assert L.nbytes(n) == O.layout_bytes_ex(widths, labels, n, blocks, aligned)
    for f in range(F):
        r, s, o, b = L.field_address_ex(f, n)
        for i in sorted({0, 1, n // 2, max(0, n - 1)}):
            if i < n:
                assert r + (i // b) * (b * s) + o * b + (i % b) * widths[f] == O.addr_ex(d, f, i)


@SET
@given(layouts(max_fields=8), st.data())
def test_capi_layout_string_round_trip(widths, data):
    F = len(widths)
    labels = data.draw(partition(F))
    names = [f"x{i}" for i in range(F)]
    blocks = None
    if data.draw(st.booleans()):
        per = {c: data.draw(st.sampled_from([1, 2, 4, 8, 16, 32])) for c in sorted(set(labels))}
        blocks = [per[c] for c in labels]
    L = A.Layout(widths, labels, names=names, blocks=blocks, aligned=data.draw(st.booleans()))
    text = L.to_string()
    L2 = A.Layout.from_string(text, names, widths)
    assert L2.to_string() == text
    for f in range(F):
        assert L.field_address_ex(f, 77) == L2.field_address_ex(f, 77)
    assert L.nbytes(1001) == L2.nbytes(1001)


@SET
@given(st.integers(0, 10 ** 12), st.integers(1, 64))
def test_capi_shard_ranges_cover_and_balance(n, G):
    prev_hi = 0
    sizes = []
    for g in range(G):
        lo, hi = A.shard_range(n, G, g)
        assert lo == prev_hi and lo == g * n // G and hi == (g + 1) * n // G
        prev_hi = hi
        sizes.append(hi - lo)
    assert prev_hi == n and max(sizes) - min(sizes) <= 1


@settings(max_examples=300, deadline=None)
@given(st.text(max_size=80))
def test_capi_layout_parser_never_crashes(text):
    """Arbitrary text into adha_layout_from_string: a layout or ADHA_ERR_PARSE / INVALID_ARG,
    never a crash."""
    names, widths = ["a", "b", "c", "V1"], [4, 4, 8, 2]
    try:
        L = A.Layout.from_string(text, names, widths)
    except A.AdhaError as e:
        assert e.name in ("ADHA_ERR_PARSE", "ADHA_ERR_INVALID_ARG"), e
    else:
        assert sorted(f for c in L.to_string().strip("{}").split("}|{") for f in c.split(",")) == sorted(names)


def _mutations(doc: str):
    return st.one_of(
        st.just(doc),
        st.builds(lambda i, j: doc[:i] + doc[j:], st.integers(0, len(doc)), st.integers(0, len(doc))),
        st.builds(lambda i, c: doc[:i] + c + doc[i:], st.integers(0, len(doc)), st.sampled_from(list('{}[]",:0-1e'))),
        st.text(max_size=60))


_PROGRAM = None


def _medical():
    global _PROGRAM
    if _PROGRAM is None:
        import json
        from tests.conftest import golden
        _PROGRAM = (json.dumps(golden("medical_program.json")), json.dumps(golden("medical_arch.json")))
    return _PROGRAM


@settings(max_examples=200, deadline=None)
@given(st.data())
def test_capi_planner_rejects_malformed_json_cleanly(data):
    """Truncated, spliced or random planner documents: adha_plan_ods / adha_plan_pdl return a plan or
    a PARSE / PLANNER / CAPACITY / INVALID_ARG status, never a crash."""
    prog, arch = _medical()
    p = data.draw(_mutations(prog))
    a = data.draw(_mutations(arch))
    for call in (lambda: A.plan_pdl(p, a), lambda: A.plan_ods(p, a, "s1", "cpu")):
        try:
            call()
        except A.AdhaError as e:
            assert e.name in ("ADHA_ERR_PARSE", "ADHA_ERR_PLANNER", "ADHA_ERR_CAPACITY", "ADHA_ERR_INVALID_ARG"), e


@st.composite
def inplace_case(draw):
    F = draw(st.integers(1, 12))
    widths = draw(st.lists(st.sampled_from([1, 2, 3, 4, 4, 8, 8, 12, 16]), min_size=F, max_size=F))
    ls = draw(st.lists(st.integers(0, F - 1), min_size=F, max_size=F))
    ld = draw(st.lists(st.integers(0, F - 1), min_size=F, max_size=F))
    n = draw(st.one_of(st.sampled_from([0, 1, 63, 64, 65, 255, 256, 257, 4096]), st.integers(0, 300_000)))
    return widths, ls, ld, n


@SET
@given(inplace_case())
def test_inplace_plan_invariants(case):
    """Host plan of the in-place remap (slot-permutation mode) on random packed layout pairs:
    never crashes; the buffer is max(bytes(Ls), bytes(Ld)) by the oracle's address model; every
    src body slot is content; the permutation closes on src u dst slots; segments cover the moved
    slots in pieces of at most 64; the workspace holds a saved slot per segment; and (ADHA_IP_VERIFY)
    every moved slot sits in exactly one segment, in cycle order, each segment's predecessor ending
    on the slot whose content its first position receives."""
    import os
    widths, ls, ld, n = case
    os.environ["ADHA_INPLACE_STAGED_BYTES"] = "0"
    os.environ["ADHA_IP_VERIFY"] = "1"        # the library checks its segments against the permutation
    try:
        try:
            p = A.InplacePlan(A.Layout(widths, ls), A.Layout(widths, ld), n)
        except A.AdhaError as e:   # a record too wide for a tile in shared memory
            assert e.name == "ADHA_ERR_UNSUPPORTED"
            return
        d = p.describe()
    finally:
        os.environ.pop("ADHA_INPLACE_STAGED_BYTES", None)
        os.environ.pop("ADHA_IP_VERIFY", None)
    assert p.buffer_bytes == max(O.layout_bytes(widths, ls, n), O.layout_bytes(widths, ld, n))
    u, S, T = d["unit"], d["slot_bytes"], d["T"]
    assert S == T * u and all(w % u == 0 for w in widths)
    assert d["body_tiles"] == n // T and d["tail_records"] == n % T
    assert d["content_slots"] == (n // T) * sum(widths) // u
    assert d["moved_slots"] + d["fixed_slots"] == d["content_slots"] + d["junk_slots"]
    assert d["segments"] * 64 >= d["moved_slots"] and (d["moved_slots"] == 0) == (d["segments"] == 0)
    assert p.workspace_bytes >= d["segments"] * S
