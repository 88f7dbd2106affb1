"""GPU parity of the in-place remap (adha_remap_inplace, SURVEY.md 8(f) N1 "in-place").

The definition is the remap's with src and dst the same
buffer: after the call, every payload byte of the dst layout equals the oracle's out-of-place
remap of the buffer's old contents.  Bytes outside the dst payload are unspecified (adha.h), so
the comparison runs over oracle.remap.payload_mask(dst layout).  Bit-exact is the bar.
"""
import os

import numpy as np
import pytest

from adha_inputs import config_widths, field_columns, fill_random_device, SEED_BASE
from oracle import remap as O
from tests.test_oracle_remap import set_partitions

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1407_4859_b200 as A  # noqa: E402


@pytest.fixture(autouse=True)
def permute_mode(monkeypatch):
    """Every test here exercises the slot-permutation kernels (tile rewrite + cycles), also at
    the small sizes that would otherwise go through the staged mode (ADHA_INPLACE_STAGED_BYTES)."""
    monkeypatch.setenv("ADHA_INPLACE_STAGED_BYTES", "0")


def oracle_dst(src, ls, ld, widths, n):
    dst = np.zeros(O.layout_bytes(widths, ld, n), np.uint8)
    O.remap(src, ls, dst, ld, widths, n, threads=min(8, os.cpu_count() or 1))
    return dst


def run_inplace(widths, ls, ld, n, src_np):
    """Place src_np (layout ls) at the start of a buffer of plan.buffer_bytes, remap in place."""
    Ls, Ld = A.Layout(widths, ls), A.Layout(widths, ld)
    plan = A.InplacePlan(Ls, Ld, n)
    buf = torch.full((max(plan.buffer_bytes, 256),), 0x5A, dtype=torch.uint8, device="cuda")
    if src_np.size:
        buf[: src_np.size].copy_(torch.from_numpy(src_np))
    A.remap_inplace(buf, plan)
    torch.cuda.synchronize()
    return buf.cpu().numpy(), plan


def check_inplace(widths, ls, ld, n, seed=0):
    cols = field_columns(seed, n, widths)
    src = O.pack(cols, widths, ls, n, fill=0x3C)
    got, plan = run_inplace(widths, ls, ld, n, src)
    exp = oracle_dst(src, ls, ld, widths, n)
    mask = O.payload_mask(widths, ld, n)
    g = got[: exp.size]
    if not np.array_equal(g[mask], exp[mask]):
        bad = np.nonzero((g != exp) & mask)[0]
        raise AssertionError(f"in-place mismatch at {bad.size} payload bytes, first {bad[:8]} "
                             f"(widths={widths} ls={ls} ld={ld} n={n} plan={plan.describe()})")
    return plan


def _T(widths, ls, ld, n):
    return A.InplacePlan(A.Layout(widths, ls), A.Layout(widths, ld), n).describe()["T"]


# ----------------------------------------------------------------------------- small shapes

def test_c1_xyz_in_place_round_trip():
    """C1's record: AoS -> SoA in place, then back; payload equals the original AoS."""
    widths, n = [4, 4, 4], 1024
    cols = field_columns(SEED_BASE + 0, n, widths)
    aos, soa = [0, 0, 0], [0, 1, 2]
    src = O.pack(cols, widths, aos, n)
    mid, _ = run_inplace(widths, aos, soa, n, src)
    mask = O.payload_mask(widths, soa, n)
    exp = oracle_dst(src, aos, soa, widths, n)
    assert np.array_equal(mid[: exp.size][mask], exp[mask])
    back, _ = run_inplace(widths, soa, aos, n, mid[: O.layout_bytes(widths, soa, n)])
    assert np.array_equal(back[: src.size], src)


@pytest.mark.parametrize("widths", [[4, 4, 4, 8, 4], [1, 2, 3, 4, 8], [2, 2, 6, 4, 2]])
def test_all_layout_pairs_5_fields(widths):
    """All 52 x 52 ordered pairs of partitions of 5 fields (brute force, SURVEY.md 8(c) iv) at one
    N with a ragged tail and several tiles; a random quarter of the pairs at a second N."""
    parts = set_partitions(5)
    rng = np.random.default_rng(sum(widths) + 7)
    for k, ls in enumerate(parts):
        for ld in parts:
            T = _T(widths, ls, ld, 1 << 20)
            check_inplace(widths, ls, ld, 3 * T + 5, seed=k)
            if rng.random() < 0.25:
                check_inplace(widths, ls, ld, int(rng.integers(1, 9 * T)), seed=k + 1)


@pytest.mark.parametrize("n", [0, 1, 63, 64, 65, 255, 256, 257, 1000, 4097, 65536 + 3])
def test_edge_counts(n):
    """Empty, single record, below / at / above one tile, ragged tails (adha.h: N = 0 is a no-op)."""
    widths = config_widths(16)
    for ls, ld in [([0] * 16, list(range(16))), (list(range(16)), [0] * 16),
                   ([0, 0, 1, 1, 2, 2, 3, 3] * 2, [i % 5 for i in range(16)])]:
        check_inplace(widths, ls, ld, n, seed=n)


def test_narrow_units():
    """u = 1 and u = 2 (byte-atom transposes, T = 256 / 128 records per slot tile)."""
    for widths in ([1, 3, 4, 8, 2, 1], [2, 2, 6, 4, 2, 8]):
        F = len(widths)
        for ls, ld in [([0] * F, list(range(F))), (list(range(F)), [0] * F), ([0] * F, [0, 0, 1, 1, 2, 2])]:
            for n in (1000, 5003, 40_000):
                check_inplace(widths, ls, ld, n, seed=n + F)


def test_identical_layouts_move_nothing():
    widths, n = config_widths(16), 100_003
    lab = [0, 0, 1, 1, 2, 2, 3, 3] * 2
    plan = check_inplace(widths, lab, lab, n)
    d = plan.describe()
    assert d["moved_slots"] == 0 and d["pre_clusters"] == 0 and d["post_clusters"] == 0


def test_medical_aosv_to_soa_keeps_unchanged_regions():
    """Medical AoSV -> SoA (Table 2; the plan's remap edge): with N a
    multiple of 64 the six singleton regions have the same base in both layouts, so only the
    {V1,V2,V3} slots move (the moved-subset rule)."""
    widths, n = [4] * 9, 1 << 20
    aosv, soa = [0, 0, 0, 1, 2, 3, 4, 5, 6], list(range(9))
    plan = check_inplace(widths, aosv, soa, n, seed=21)
    d = plan.describe()
    S = d["slot_bytes"]
    assert 0 < d["moved_slots"] <= 3 * 4 * n // S          # V1..V3 (a few are fixed points)
    assert d["moved_slots"] + d["fixed_slots"] == 9 * 4 * n // S
    assert d["pre_clusters"] == 1 and d["post_clusters"] == 0


def test_random_pairs_config_widths():
    """Random partitions of C2's and C3's field sets (mixed 4/8-byte widths)."""
    rng = np.random.default_rng(14074859)
    for F in (16, 64):
        widths = config_widths(F)
        for k in range(12):
            ls = [int(x) for x in rng.integers(0, int(rng.integers(1, F + 1)), F)]
            ld = [int(x) for x in rng.integers(0, int(rng.integers(1, F + 1)), F)]
            check_inplace(widths, ls, ld, int(rng.integers(1, 200_000)), seed=k)


def test_nan_payloads_bit_exact():
    """sNaN/qNaN payloads, -0.0, denormals survive the in-place moves bit for bit (reading Q6)."""
    widths, n = [4, 8, 4, 4], 10_007
    cols = field_columns(5, n, widths)
    cols[0][::3] = np.frombuffer(np.array([0x7F800001], np.uint32).tobytes(), np.uint8)
    cols[1][::5] = np.frombuffer(np.array([0x7FF0000000000ABC], np.uint64).tobytes(), np.uint8)
    cols[2][::7] = np.frombuffer(np.array([0x80000000], np.uint32).tobytes(), np.uint8)
    src = O.pack(cols, widths, [0, 0, 0, 0], n)
    got, _ = run_inplace(widths, [0, 0, 0, 0], [0, 1, 2, 3], n, src)
    back = O.unpack(got, widths, [0, 1, 2, 3], n)
    for f in range(4):
        assert np.array_equal(back[f], cols[f])


def test_repeat_runs_and_errors():
    """A plan runs any number of times (each run remaps the current contents); argument errors."""
    widths, n = config_widths(16), 20_011
    aos, soa = [0] * 16, list(range(16))
    La, Ls = A.Layout(widths, aos), A.Layout(widths, soa)
    fwd, bwd = A.InplacePlan(La, Ls, n), A.InplacePlan(Ls, La, n)
    buf = torch.zeros(max(fwd.buffer_bytes, bwd.buffer_bytes), dtype=torch.uint8, device="cuda")
    fill_random_device(buf, 99)
    ref = buf[: La.nbytes(n)].clone()
    for _ in range(3):
        A.remap_inplace(buf, fwd)
        A.remap_inplace(buf, bwd)
    torch.cuda.synchronize()
    assert torch.equal(buf[: La.nbytes(n)], ref)
    # a buffer smaller than max(bytes) is rejected
    with pytest.raises(A.AdhaError) as e:
        A.remap_inplace(buf[: fwd.buffer_bytes - 256], fwd)
    assert e.value.name == "ADHA_ERR_INVALID_ARG"
    # misaligned buffer
    with pytest.raises(A.AdhaError) as e:
        A.remap_inplace(buf[16:], fwd)
    assert e.value.name in ("ADHA_ERR_ALIGNMENT", "ADHA_ERR_INVALID_ARG")
    # a plan must be uploaded to the workspace it runs with
    p3 = A.InplacePlan(La, Ls, n)
    ws = torch.empty(p3.workspace_bytes, dtype=torch.uint8, device="cuda")
    with pytest.raises(A.AdhaError) as e:
        A._check(A._lib.adha_remap_inplace(buf.data_ptr(), buf.numel(), p3._h, ws.data_ptr(), 0))
    assert e.value.name == "ADHA_ERR_INVALID_ARG"
    # a workspace inside the buffer is rejected
    p3.upload(buf[: p3.workspace_bytes])
    with pytest.raises(A.AdhaError) as e:
        A.remap_inplace(buf, p3)
    assert e.value.name == "ADHA_ERR_OVERLAP"


# ----------------------------------------------------------------------------- full BASELINE sizes

def test_c2_full_size_in_place_every_payload_byte():
    """C2 (16 mixed fields, 10M records) AoS -> SoA in place; every payload byte vs the oracle."""
    widths, n = config_widths(16), 10_000_000
    aos, soa = [0] * 16, list(range(16))
    La, Ls = A.Layout(widths, aos), A.Layout(widths, soa)
    plan = A.InplacePlan(La, Ls, n)
    buf = torch.empty(plan.buffer_bytes, dtype=torch.uint8, device="cuda")
    fill_random_device(buf, SEED_BASE + 1)
    h_src = buf[: La.nbytes(n)].cpu().numpy()
    A.remap_inplace(buf, plan)
    torch.cuda.synchronize()
    exp = oracle_dst(h_src, aos, soa, widths, n)
    mask = O.payload_mask(widths, soa, n)
    got = buf[: exp.size].cpu().numpy()
    assert np.array_equal(got[mask], exp[mask])


@pytest.mark.parametrize("variant", ["structured", "random"])
def test_c3_shape_in_place_exact(variant):
    """C3's remap (64 SoA fields -> the ODS hybrid of the structured program, or of the seeded
    random program variant) in place at 5M records: every dst payload byte against the oracle's
    out-of-place remap of a copy of the src (record-range chunks; the other bytes of the buffer are
    unspecified in place)."""
    from tests.test_gpu_parity import c3_labels, c3r_labels
    from tests.gpu_util import exact_chunked_check
    widths, n = config_widths(64), 5_000_003
    ls, ld = list(range(64)), (c3_labels() if variant == "structured" else c3r_labels())
    Ls, Ld = A.Layout(widths, ls), A.Layout(widths, ld)
    plan = A.InplacePlan(Ls, Ld, n)
    buf = torch.empty(plan.buffer_bytes, dtype=torch.uint8, device="cuda")
    fill_random_device(buf, SEED_BASE + 2)
    src = buf[: Ls.nbytes(n)].clone()
    A.remap_inplace(buf, plan)
    torch.cuda.synchronize()
    assert exact_chunked_check(O, src, ls, buf, ld, widths, n, check_gaps=False) == n * sum(widths)
    del buf, src
    torch.cuda.empty_cache()


def test_staged_mode_small_buffers(monkeypatch):
    """Buffers up to ADHA_INPLACE_STAGED_BYTES (16 MB by default) are remapped out of place into
    the workspace and copied back; same result on every dst payload byte."""
    monkeypatch.delenv("ADHA_INPLACE_STAGED_BYTES", raising=False)
    widths = config_widths(16)
    for ls, ld, n in [([0] * 16, list(range(16)), 1000), (list(range(16)), [0] * 16, 100_003),
                      ([0, 0, 1, 1, 2, 2, 3, 3] * 2, [i % 5 for i in range(16)], 65_537)]:
        plan = check_inplace(widths, ls, ld, n, seed=n)
        d = plan.describe()
        assert d["mode"] == "staged" and plan.workspace_bytes >= d["dst_bytes"]
    big = A.InplacePlan(A.Layout(widths, [0] * 16), A.Layout(widths, list(range(16))), 1_000_000)
    assert big.describe()["mode"] == "permute"
