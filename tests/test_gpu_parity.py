"""GPU parity: the CUDA remap (through the C ABI) against the CPU oracle.

Bit-exact is the bar (integer/byte work; SURVEY.md 8(c) c1 -- the result is
unique).  Small N: element by element over the whole dst buffer, including the
sentinel-filled gaps between regions.  Full BASELINE sizes (C2, C3, C3R, each
C4 hop, C5): every payload byte, C3/C4/C5 by record-range chunks against the
oracle (exact by record locality), in the launch configuration bench.py times.
"""
import os

import numpy as np
import pytest

from adha_inputs import config_widths, field_columns, tagged_columns, fill_random_device, SEED_BASE
from oracle import remap as O
from tests.gpu_util import SENT, run_remap, sentinel_dev, to_dev, exact_chunked_check
from tests.test_oracle_remap import set_partitions

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1407_4859_b200 as A  # noqa: E402


@pytest.fixture(params=["tiled", "tiled-components", "direct-small"])
def small_path(request, monkeypatch):
    """Run a test three times: with every remap on the tiled kernel (ADHA_SMALL_BYTES=0; remaps of
    up to merge_bytes take the merged one-component plan), on the tiled kernel with per-component
    tiles at every size (ADHA_MERGE_BYTES=0, the large-N plan), and with the default routing where
    small remaps (remap.cu direct_bytes) take the direct kernel."""
    monkeypatch.delenv("ADHA_MERGE_BYTES", raising=False)
    if request.param == "tiled":
        monkeypatch.setenv("ADHA_SMALL_BYTES", "0")
    elif request.param == "tiled-components":
        monkeypatch.setenv("ADHA_SMALL_BYTES", "0")
        monkeypatch.setenv("ADHA_MERGE_BYTES", "0")
    else:
        monkeypatch.delenv("ADHA_SMALL_BYTES", raising=False)
    return request.param


def oracle_dst(src, ls, ld, widths, n):
    dst = np.full(O.layout_bytes(widths, ld, n), SENT, np.uint8)
    O.remap(src, ls, dst, ld, widths, n, threads=min(8, os.cpu_count() or 1))
    return dst


def check_pair(widths, ls, ld, n, cols=None, seed=0):
    cols = cols if cols is not None else field_columns(seed, n, widths)
    src = O.pack(cols, widths, ls, n, fill=0x3C)
    got = run_remap(A, src, A.Layout(widths, ls), A.Layout(widths, ld), n)
    exp = oracle_dst(src, ls, ld, widths, n)
    assert got.shape == exp.shape
    if not np.array_equal(got, exp):
        bad = np.nonzero(got != exp)[0]
        raise AssertionError(f"mismatch at {bad.size} bytes, first {bad[:8]} (widths={widths} ls={ls} ld={ld} n={n})")


def plan_T(widths, ls, ld):
    return A.plan_describe(A.Layout(widths, ls), A.Layout(widths, ld))["T"]


# ----------------------------------------------------------------------------- C1

def test_c1_xyz_aos_soa_and_back(small_path):
    widths, n = [4, 4, 4], 1024
    cols = field_columns(SEED_BASE + 0, n, widths)
    aos, soa = [0, 0, 0], [0, 1, 2]
    src = O.pack(cols, widths, aos, n)
    La, Ls = A.Layout(widths, aos), A.Layout(widths, soa)
    mid = run_remap(A, src, La, Ls, n)
    assert np.array_equal(mid, oracle_dst(src, aos, soa, widths, n))
    back = run_remap(A, mid, Ls, La, n)
    assert np.array_equal(back, src)


# ----------------------------------------------------------------------------- brute force

@pytest.mark.parametrize("widths", [[1, 2, 3, 4, 8], [4, 4, 4, 8, 4], [2, 2, 6, 4, 2]])
def test_all_layout_pairs_5_fields(widths, small_path):
    parts = set_partitions(5)
    rng = np.random.default_rng(sum(widths))
    for ls in parts:
        for ld in parts:
            T = plan_T(widths, ls, ld)
            n = 3 * T + 5
            check_pair(widths, ls, ld, n, cols=tagged_columns(n, widths))
    for _ in range(60):                                   # edge record counts on random pairs
        ls, ld = parts[rng.integers(52)], parts[rng.integers(52)]
        T = plan_T(widths, ls, ld)
        for n in (0, 1, 15, 16, 17, 31, 32, 33, T - 1, T, T + 1):
            check_pair(widths, ls, ld, n, seed=n)


# ----------------------------------------------------------------------------- config shapes, small N

def c3_labels():
    from oracle import planner as P
    from tests.conftest import golden
    hyb = P.parse_layout(golden("expected.json")["c3_hybrid"]["value"], {f"f{i}": i for i in range(64)})
    lab = [0] * 64
    for c, cl in enumerate(hyb):
        for nm in cl:
            lab[int(nm[1:])] = c
    return lab


def c3r_labels():
    """The oracle's layout of the seeded random C3 program (tests/golden/c3_random_expected.json)."""
    from oracle import planner as P
    from tests.conftest import golden
    hyb = P.parse_layout(golden("c3_random_expected.json")["c3_random_hybrid"]["value"], {f"f{i}": i for i in range(64)})
    lab = [0] * 64
    for c, cl in enumerate(hyb):
        for nm in cl:
            lab[int(nm[1:])] = c
    return lab


AOSV = [0, 0, 0, 1, 2, 3, 4, 5, 6]


@pytest.mark.parametrize("name,widths,ls,ld", [
    ("C2", config_widths(16), [0] * 16, list(range(16))),
    ("C2-back", config_widths(16), list(range(16)), [0] * 16),
    ("C3", config_widths(64), list(range(64)), c3_labels()),
    ("C3-back", config_widths(64), c3_labels(), list(range(64))),
    ("C3R", config_widths(64), list(range(64)), c3r_labels()),
    ("C3R-back", config_widths(64), c3r_labels(), list(range(64))),
    ("C4-aos-aosv", [4] * 9, [0] * 9, AOSV),
    ("C4-aosv-soa", [4] * 9, AOSV, list(range(9))),
    ("C4-soa-aos", [4] * 9, list(range(9)), [0] * 9),
    ("P2-soa-4x8", [4] * 32, list(range(32)), [i // 8 for i in range(32)]),
    ("identity-hybrid", [4] * 9, AOSV, AOSV),
])
def test_config_shapes_small(name, widths, ls, ld, small_path):
    T = plan_T(widths, ls, ld)
    for n in (1, 33, T + 7, 5 * T + 31, 151 * T + 3):
        check_pair(widths, ls, ld, n, seed=n)


def test_nan_payloads_bit_exact():
    widths = [4, 8, 4, 8, 4, 4, 4, 8]
    n = 50_000
    cols = field_columns(7, n, widths)
    f32 = cols[0].view(np.uint32).ravel()
    assert np.any(((f32 >> 23) & 0xFF) == 0xFF)
    check_pair(widths, [0] * 8, list(range(8)), n, cols=cols)
    check_pair(widths, list(range(8)), [0, 0, 1, 1, 1, 2, 3, 3], n, cols=cols)


def test_naive_fallback_many_fields():
    widths = [4, 2, 1, 8] * 75                              # 300 fields > tiled limit
    d = A.plan_describe(A.Layout.aos(widths), A.Layout.soa(widths))
    assert not d["tiled"]
    check_pair(widths, [0] * 300, list(range(300)), 777)


# ----------------------------------------------------------------------------- errors on device pointers

def test_device_pointer_errors():
    a, s = A.Layout.aos([4, 4]), A.Layout.soa([4, 4])
    buf = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    with pytest.raises(A.AdhaError) as e:
        A.remap(buf[16:], a, buf[4096:], s, 10)
    assert e.value.name == "ADHA_ERR_ALIGNMENT"
    with pytest.raises(A.AdhaError) as e:
        A.remap(buf, a, buf[256:], s, 1000)
    assert e.value.name == "ADHA_ERR_OVERLAP"


def test_side_stream():
    widths = config_widths(16)
    n = 100_000
    cols = field_columns(1, n, widths)
    src = O.pack(cols, widths, [0] * 16, n)
    La, Ls = A.Layout.aos(widths), A.Layout.soa(widths)
    s = torch.cuda.Stream()
    d_src = to_dev(src)
    d_dst = sentinel_dev(Ls.nbytes(n))
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        A.remap(d_src, La, d_dst, Ls, n, stream=s)
    s.synchronize()
    assert np.array_equal(d_dst.cpu().numpy(), oracle_dst(src, [0] * 16, list(range(16)), widths, n))


@pytest.mark.parametrize("widths,ls,ld", [(config_widths(16), [0] * 16, list(range(16))),
                                           ([2, 4, 6, 4] * 4, [0] * 16, list(range(16))),
                                           (config_widths(64), list(range(64)), [i // 8 for i in range(64)])],
                         ids=["unit4", "byte-groups", "many-regions"])
def test_first_use_inside_cuda_graph_capture(widths, ls, ld, monkeypatch):
    """A layout pair's first tiled remap issued while the stream is being captured into a CUDA
    graph: its plan table is uploaded by a kernel inside the graph (remap.cu device_table), so
    every replay is correct; a later uncaptured call uploads it for good."""
    monkeypatch.setenv("ADHA_SMALL_BYTES", "0")
    n = 40_003
    cols = field_columns(7, n, widths)
    src = O.pack(cols, widths, ls, n, fill=0x3C)
    exp = oracle_dst(src, ls, ld, widths, n)
    Ls, Ld = A.Layout(widths, ls), A.Layout(widths, ld)          # fresh handles: a new plan
    d_src = to_dev(src)
    d_dst = sentinel_dev(Ld.nbytes(n))
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        A.remap(d_src, Ls, d_dst, Ld, n)
    for _ in range(2):
        d_dst.fill_(SENT)
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(d_dst.cpu().numpy(), exp)
    d_dst.fill_(SENT)
    A.remap(d_src, Ls, d_dst, Ld, n)
    torch.cuda.synchronize()
    assert np.array_equal(d_dst.cpu().numpy(), exp)


# ----------------------------------------------------------------------------- full BASELINE sizes

def test_c2_full_size_every_byte():
    widths, n = config_widths(16), 10_000_000
    aos, soa = [0] * 16, list(range(16))
    La, Ls = A.Layout(widths, aos), A.Layout(widths, soa)
    src = torch.empty(La.nbytes(n), dtype=torch.uint8, device="cuda")
    fill_random_device(src, SEED_BASE + 1)
    dst = sentinel_dev(Ls.nbytes(n))
    A.remap(src, La, dst, Ls, n)
    torch.cuda.synchronize()
    h_src = src.cpu().numpy()
    exp = oracle_dst(h_src, aos, soa, widths, n)
    assert np.array_equal(dst.cpu().numpy(), exp)


@pytest.mark.parametrize("cfg", ["C3", "C3R", "C5"])
def test_full_size_exact(cfg):
    """The bench workloads at full size, EVERY payload byte against the oracle by record-range
    chunks: C3 (50M x 320 B, SoA -> the 24-cluster hybrid), C3R (the seeded
    random-program hybrid) and C5 (8 GiB AoS -> SoA), in the launch configuration bench.py times."""
    if cfg in ("C3", "C3R"):
        widths, n, ls = config_widths(64), 50_000_000, list(range(64))
        ld = c3_labels() if cfg == "C3" else c3r_labels()
    else:
        widths, n, ls, ld = config_widths(16), 107_374_182, [0] * 16, list(range(16))
    Ls, Ld = A.Layout(widths, ls), A.Layout(widths, ld)
    src = torch.empty(Ls.nbytes(n), dtype=torch.uint8, device="cuda")
    fill_random_device(src, SEED_BASE + {"C3": 2, "C3R": 6, "C5": 4}[cfg])
    dst = sentinel_dev(Ld.nbytes(n))
    A.remap(src, Ls, dst, Ld, n)
    torch.cuda.synchronize()
    assert exact_chunked_check(O, src, ls, dst, ld, widths, n) == n * sum(widths)
    del src, dst
    torch.cuda.empty_cache()


@pytest.mark.parametrize("widths", [[4, 4], [1, 2, 1]], ids=["unit4", "byte-groups"])
def test_max_size_beyond_2_31_records(widths):
    """Maximum sizes: N > 2^31 records, so record indices need 64 bits and region offsets pass
    2^32 bytes (unit-4 permute path and byte-group path); every payload byte against the oracle,
    so every 2^k boundary a 32-bit index or byte offset would break at is covered."""
    n = 2 ** 31 + 4099
    F = len(widths)
    aos, soa = [0] * F, list(range(F))
    La, Ls = A.Layout(widths, aos), A.Layout(widths, soa)
    src = torch.empty(La.nbytes(n), dtype=torch.uint8, device="cuda")
    fill_random_device(src, SEED_BASE + 9)
    dst = sentinel_dev(Ls.nbytes(n))
    A.remap(src, La, dst, Ls, n)
    torch.cuda.synchronize()
    assert exact_chunked_check(O, src, aos, dst, soa, widths, n, chunk=1 << 24) == n * sum(widths)
    del src, dst
    torch.cuda.empty_cache()


@pytest.mark.parametrize("cfg", ["P1", "P2"])
def test_paper_shaped_chains_full_size_exact(cfg):
    """The extra paper-shaped bench configs at their bench sizes (P1 Medical 256^3 AoS->AoSV->SoA,
    P2 K-Means 2^23 SoA->4xAoS8->AoS), through adha_remap_chain; every payload byte of every hop
    against the oracle (record-range chunks)."""
    if cfg == "P1":
        widths, n, labs = [4] * 9, 256 ** 3, [[0] * 9, AOSV, list(range(9))]
    else:
        widths, n, labs = [4] * 32, 2 ** 23, [list(range(32)), [i // 8 for i in range(32)], [0] * 32]
    lays = [A.Layout(widths, l) for l in labs]
    bufs = [torch.empty(l.nbytes(n), dtype=torch.uint8, device="cuda") for l in lays]
    fill_random_device(bufs[0], SEED_BASE + 11)
    for b in bufs[1:]:
        b.fill_(SENT)
    A.remap_chain(bufs, lays, n)
    torch.cuda.synchronize()
    for k in range(len(labs) - 1):
        assert exact_chunked_check(O, bufs[k], labs[k], bufs[k + 1], labs[k + 1], widths, n) == n * sum(widths)
    del bufs
    torch.cuda.empty_cache()


@pytest.mark.parametrize("widths,kind", [([2, 4, 6, 4] * 4, "aos2soa"), ([2, 4, 6, 4] * 4, "soa2aos"),
                                         ([1] * 24 + [8], "aos2soa"), ([1, 3, 4, 8] * 4, "soa2aos")])
def test_byte_groups_large_n_exact(widths, kind):
    """The byte-group path (1/2-byte units) at the narrow-probe size N = 20M, in the tile
    configuration it runs there; every payload byte against the oracle (record-range chunks)."""
    n = 20_000_003
    F = len(widths)
    ls, ld = ([0] * F, list(range(F))) if kind == "aos2soa" else (list(range(F)), [0] * F)
    Ls, Ld = A.Layout(widths, ls), A.Layout(widths, ld)
    assert A.plan_describe(Ls, Ld)["byte_groups"]
    src = torch.empty(Ls.nbytes(n), dtype=torch.uint8, device="cuda")
    fill_random_device(src, SEED_BASE + 12)
    dst = sentinel_dev(Ld.nbytes(n))
    A.remap(src, Ls, dst, Ld, n)
    torch.cuda.synchronize()
    assert exact_chunked_check(O, src, ls, dst, ld, widths, n) == n * sum(widths)
    del src, dst
    torch.cuda.empty_cache()


@pytest.mark.parametrize("fuse", ["1", "0"])
def test_small_chain_fused_single_launch(fuse, monkeypatch):
    """adha_remap_chain over latency-bound hops runs as ONE launch (block-local record ranges,
    a barrier between hops) when every hop is <= ADHA_SMALL_BYTES and the layouts are packed;
    every intermediate is materialised and bit-exact vs the oracle, fused or not.  Includes C1
    (xyz AoS -> SoA -> AoS, 1024 records) and random 2-4 hop chains with ragged N."""
    monkeypatch.setenv("ADHA_CHAIN_FUSE", fuse)
    rng = np.random.default_rng(77)
    cases = [([4, 4, 4], [[0, 0, 0], [0, 1, 2], [0, 0, 0]], 1024)]
    for _ in range(12):
        F = int(rng.integers(1, 12))
        widths = [int(x) for x in rng.choice([1, 2, 4, 8, 3], size=F)]
        hops = int(rng.integers(2, 5))
        labs = [[int(x) for x in rng.integers(0, F, size=F)] for _ in range(hops + 1)]
        n = int(rng.integers(1, max(2, 60000 // sum(widths))))
        cases.append((widths, labs, n))
    for widths, labs, n in cases:
        cols = field_columns(n % 1000, n, widths)
        lays = [A.Layout(widths, l) for l in labs]
        bufs = [to_dev(O.pack(cols, widths, labs[0], n))] + [sentinel_dev(l.nbytes(n)) for l in lays[1:]]
        A.remap_chain(bufs, lays, n)
        torch.cuda.synchronize()
        exp = O.pack(cols, widths, labs[0], n)
        for k in range(1, len(labs)):
            e = np.full(O.layout_bytes(widths, labs[k], n), SENT, np.uint8)
            O.remap(exp, labs[k - 1], e, labs[k], widths, n)
            assert np.array_equal(bufs[k].cpu().numpy()[: e.size], e), (widths, labs, n, k)
            exp = e


@pytest.mark.parametrize("case", ["c4", "p2", "random"])
def test_chain_fused_tiled(case, monkeypatch):
    """adha_remap_chain as ONE tiled launch in chain mode (remap.cu chain_tiled; forced with
    ADHA_CHAIN_TILED_BYTES=1): every band runs through every hop in the same CTA, hop h reading hop
    h-1's output back; every intermediate is materialised and equals the oracle's chain, byte for
    byte, including the gaps between regions and ragged tails (a trailing single band per CTA)."""
    monkeypatch.setenv("ADHA_CHAIN_TILED_BYTES", "1")
    rng = np.random.default_rng({"c4": 1, "p2": 2, "random": 3}[case])
    if case == "c4":
        cases = [([4] * 9, [[0] * 9, AOSV, list(range(9)), [0] * 9], 1_234_567)]
    elif case == "p2":
        cases = [([4] * 32, [list(range(32)), [i // 8 for i in range(32)], [0] * 32], 700_001)]
    else:
        monkeypatch.setenv("ADHA_TILE_CAP", "512")     # short records: enough bands for two per SM
        cases = []
        for _ in range(6):
            F = int(rng.integers(2, 14))
            widths = [int(x) for x in rng.choice([4, 4, 8, 12], size=F)]
            hops = int(rng.integers(2, 5))
            labs = [[int(x) for x in rng.integers(0, F, size=F)] for _ in range(hops + 1)]
            cases.append((widths, labs, int(rng.integers(400_000, 900_000))))
    for widths, labs, n in cases:
        cols = field_columns(n % 977, n, widths)
        lays = [A.Layout(widths, l) for l in labs]
        bufs = [to_dev(O.pack(cols, widths, labs[0], n))] + [sentinel_dev(l.nbytes(n)) for l in lays[1:]]
        A.remap_chain(bufs, lays, n)
        torch.cuda.synchronize()
        exp = O.pack(cols, widths, labs[0], n)
        for k in range(1, len(labs)):
            e = np.full(O.layout_bytes(widths, labs[k], n), SENT, np.uint8)
            O.remap(exp, labs[k - 1], e, labs[k], widths, n, threads=min(8, os.cpu_count() or 1))
            got = bufs[k].cpu().numpy()[: e.size]
            if not np.array_equal(got, e):
                bad = np.nonzero(got != e)[0]
                raise AssertionError(f"hop {k}: {bad.size} bytes differ, first {bad[:6]} ({widths} {labs} n={n})")
            exp = e


def test_c4_pdl_chain_full_size():
    widths, n = [4] * 9, (2 ** 31) // 36
    labs = [[0] * 9, AOSV, list(range(9)), [0] * 9]
    lays = [A.Layout(widths, l) for l in labs]
    bufs = [torch.empty(l.nbytes(n), dtype=torch.uint8, device="cuda") for l in lays]
    fill_random_device(bufs[0], SEED_BASE + 3)
    for b in bufs[1:]:
        b.fill_(SENT)
    A.remap_chain(bufs, lays, n)
    torch.cuda.synchronize()
    for k in range(3):       # every hop, every payload byte, against the oracle (record-range chunks)
        assert exact_chunked_check(O, bufs[k], labs[k], bufs[k + 1], labs[k + 1], widths, n) == n * 36
    assert torch.equal(bufs[3], bufs[0])                    # AoS -> AoSV -> SoA -> AoS is the identity


def test_sharded_on_one_device():
    widths, n, G = config_widths(16), 3_000_001, 4
    aos, soa = [0] * 16, list(range(16))
    La, Ls = A.Layout(widths, aos), A.Layout(widths, soa)
    cols = field_columns(9, n, widths)
    srcs, dsts, exp_cols = [], [], []
    for g in range(G):
        lo, hi = A.shard_range(n, G, g)
        sub = [c[lo:hi] for c in cols]
        srcs.append(to_dev(O.pack(sub, widths, aos, hi - lo)))
        dsts.append(sentinel_dev(Ls.nbytes(hi - lo)))
    streams = [torch.cuda.Stream() for _ in range(G)]
    torch.cuda.synchronize()
    A.remap_sharded(srcs, La, dsts, Ls, n, [0] * G, streams)
    torch.cuda.synchronize()
    got = [[] for _ in widths]
    for g in range(G):
        lo, hi = A.shard_range(n, G, g)
        for f, c in enumerate(O.unpack(dsts[g].cpu().numpy(), widths, soa, hi - lo)):
            got[f].append(c)
    for f in range(16):                                      # shard union == the 1-GPU result
        assert np.array_equal(np.concatenate(got[f]), cols[f])


def test_remap_host_end_to_end():
    widths, n = config_widths(16), 2_000_003
    aos, soa = [0] * 16, list(range(16))
    La, Ls = A.Layout(widths, aos), A.Layout(widths, soa)
    h_src = torch.empty(La.nbytes(n), dtype=torch.uint8).pin_memory()
    h_src.copy_(torch.from_numpy(O.pack(field_columns(5, n, widths), widths, aos, n)))
    h_dst = torch.full((Ls.nbytes(n),), SENT, dtype=torch.uint8).pin_memory()
    scratch = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    A.remap_host(h_src, La, h_dst, Ls, n, scratch)
    torch.cuda.synchronize()
    assert np.array_equal(h_dst.numpy(), oracle_dst(h_src.numpy(), aos, soa, widths, n))


# ----------------------------------------------------------------------------- moved subset (NEXT N1)

def test_remap_regions_moves_only_changed_fields():
    """Medical AoSV -> SoA with the six unchanged singleton regions aliased between the two
    instances: only {V1,V2,V3} move, the aliased regions are untouched, and the
    result equals the full out-of-place remap."""
    widths, n = [4] * 9, 1_000_003
    aosv, soa = [0, 0, 0, 1, 2, 3, 4, 5, 6], list(range(9))
    Lv, Ls = A.Layout(widths, aosv), A.Layout(widths, soa)
    cols = field_columns(21, n, widths)
    src_full = O.pack(cols, widths, aosv, n)
    exp = oracle_dst(src_full, aosv, soa, widths, n)
    exp_cols = O.unpack(exp, widths, soa, n)
    # src instance as separate regions: the {V1,V2,V3} cluster and six singletons
    v_reg = to_dev(np.ascontiguousarray(np.concatenate([cols[0], cols[1], cols[2]], 1)).reshape(-1))
    singles = [to_dev(np.ascontiguousarray(cols[f]).reshape(-1)) for f in range(3, 9)]
    dst_v = [sentinel_dev(4 * n) for _ in range(3)]
    A.remap_regions([v_reg] + singles, Lv, dst_v + singles, Ls, n)
    torch.cuda.synchronize()
    for f in range(3):
        assert np.array_equal(dst_v[f].cpu().numpy().reshape(n, 4), exp_cols[f])
    for k, f in enumerate(range(3, 9)):
        assert np.array_equal(singles[k].cpu().numpy().reshape(n, 4), exp_cols[f])
    # a non-identical alias is rejected
    with pytest.raises(A.AdhaError) as e:
        A.remap_regions([v_reg] + singles, Lv, [v_reg] + dst_v[1:] + singles, Ls, n)
    assert e.value.name == "ADHA_ERR_OVERLAP"


@pytest.mark.parametrize("n", [50_003, 1_000_003])
def test_remap_regions_medical_edge_both_paths(n, small_path):
    """The Medical AoSV -> SoA edge through adha_remap_regions at a size the default routing
    sends to the direct kernel (1.8 MB) and one it sends to the tiled kernel (36 MB), both
    forced tiled too: the six aliased singleton regions keep their bytes, V1..V3 match the
    oracle."""
    widths = [4] * 9
    aosv, soa = [0, 0, 0, 1, 2, 3, 4, 5, 6], list(range(9))
    Lv, Ls = A.Layout(widths, aosv), A.Layout(widths, soa)
    cols = field_columns(22 + n, n, widths)
    exp_cols = O.unpack(oracle_dst(O.pack(cols, widths, aosv, n), aosv, soa, widths, n), widths, soa, n)
    v_reg = to_dev(np.ascontiguousarray(np.concatenate([cols[0], cols[1], cols[2]], 1)).reshape(-1))
    singles = [to_dev(np.ascontiguousarray(cols[f]).reshape(-1)) for f in range(3, 9)]
    dst_v = [sentinel_dev(4 * n) for _ in range(3)]
    A.remap_regions([v_reg] + singles, Lv, dst_v + singles, Ls, n)
    torch.cuda.synchronize()
    for f in range(3):
        assert np.array_equal(dst_v[f].cpu().numpy().reshape(n, 4), exp_cols[f])
    for k, f in enumerate(range(3, 9)):
        assert np.array_equal(singles[k].cpu().numpy().reshape(n, 4), exp_cols[f])


@pytest.mark.parametrize("n", [1003, 200_003])
def test_remap_regions_blocked_alias_untouched(n, small_path):
    """An aliased identity cluster with AoSoA blocks ({a,b}@8 on both sides) is left untouched
    by both kernel paths -- including the slots past N in its last block, which a zero pass
    would overwrite (adha.h adha_remap_regions: "left untouched") -- while {c},{d} -> {c,d}
    matches the oracle."""
    widths = [4, 4, 4, 4]
    ls, bs = [0, 0, 1, 2], [8, 8, 1, 1]
    ld, bd = [0, 0, 1, 1], [8, 8, 1, 1]
    Ls, Ld = A.Layout(widths, ls, blocks=bs), A.Layout(widths, ld, blocks=bd)
    cols = field_columns(77 + n, n, widths)
    ab = O.pack_ex(cols[:2], [4, 4], [0, 0], n, [8, 8], False)
    d = O.field_addresses_ex([4, 4], [0, 0], n, [8, 8], False)
    payload = np.zeros(ab.size, bool)
    i = np.arange(n, dtype=np.int64)
    for f in range(2):
        a = O.addr_ex(d, f, i)
        payload[(a[:, None] + np.arange(4)[None, :]).reshape(-1)] = True
    ab[~payload] = 0x77                        # slots past N in the last block: must survive
    x = to_dev(ab)
    c, dd = to_dev(np.ascontiguousarray(cols[2]).reshape(-1)), to_dev(np.ascontiguousarray(cols[3]).reshape(-1))
    cd = sentinel_dev(8 * n)
    A.remap_regions([x, c, dd], Ls, [x, cd], Ld, n)
    torch.cuda.synchronize()
    assert np.array_equal(x.cpu().numpy(), ab)
    assert np.array_equal(cd.cpu().numpy().reshape(n, 8), np.concatenate([cols[2], cols[3]], 1))


def test_remap_regions_rejects_non_identity_alias():
    """Aliasing needs an identity component, not only equal member sets: a padded (aligned)
    cluster, or one whose AoSoA block changes, is rejected with OVERLAP; overlap spans cover the
    whole blocked region (ceil(N/B)*B records), not N*stride."""
    n = 1000
    t = torch
    w = [1, 4, 4]
    # {a,b} aligned (stride 8, padding) -> {a,b} packed: same members, not an identity
    La = A.Layout(w, [0, 0, 1], aligned=True)
    Lp = A.Layout(w, [0, 0, 1])
    r0, r1 = t.zeros(8 * n, dtype=t.uint8, device="cuda"), t.zeros(4 * n, dtype=t.uint8, device="cuda")
    o1 = t.zeros(4 * n, dtype=t.uint8, device="cuda")
    with pytest.raises(A.AdhaError) as e:
        A.remap_regions([r0, r1], La, [r0, o1], Lp, n)
    assert e.value.name == "ADHA_ERR_OVERLAP"
    # {a,b}@4 -> {a,b}@8: the block changes
    w2 = [4, 4, 4]
    L4 = A.Layout(w2, [0, 0, 1], blocks=[4, 4, 1])
    L8 = A.Layout(w2, [0, 0, 1], blocks=[8, 8, 1])
    s0 = t.zeros(8 * (n + 8), dtype=t.uint8, device="cuda")
    with pytest.raises(A.AdhaError) as e:
        A.remap_regions([s0, r1], L4, [s0, o1], L8, n)
    assert e.value.name == "ADHA_ERR_OVERLAP"
    # a 16-byte field in 32-record blocks: 1 record occupies 512 region bytes, so a region 256
    # bytes further on overlaps it (N*stride = 16 would not see it)
    w3 = [16, 4]
    Lsrc = A.Layout(w3, [0, 1])
    Ldst = A.Layout(w3, [0, 1], blocks=[32, 1])
    big = t.zeros(4096, dtype=t.uint8, device="cuda")
    s_a, s_b = t.zeros(256, dtype=t.uint8, device="cuda"), t.zeros(256, dtype=t.uint8, device="cuda")
    with pytest.raises(A.AdhaError) as e:
        A.remap_regions([s_a, s_b], Lsrc, [big[:512], big[256:512]], Ldst, 1)
    assert e.value.name == "ADHA_ERR_OVERLAP"


def test_pdl_plan_drives_the_remap():
    """Planner -> remap: the Medical PDL plan (Table 4 row 1) has two runs, AoSV on
    the CPU side and SoA on the GPU side; materialising them runs the plan's one remap edge."""
    from tests.conftest import golden
    plan = A.plan_pdl(golden("medical_program.json"), golden("medical_arch.json"), golden("medical_profile.json"))
    names = [f["name"] for f in golden("medical_program.json")["fields"]]
    widths = [4] * 9
    n = 300_007
    lays = A.plan_layouts(plan, names, widths)
    assert [l.to_string() for l in lays] == [r["layout"] for r in plan["runs"]]
    labs = [l.cluster_of for l in lays]
    cols = field_columns(31, n, widths)
    src = O.pack(cols, widths, labs[0], n)
    bufs = [to_dev(src), sentinel_dev(lays[1].nbytes(n))]
    A.run_plan_remaps(plan, names, widths, bufs, n)
    torch.cuda.synchronize()
    assert np.array_equal(bufs[1].cpu().numpy(), oracle_dst(src, labs[0], labs[1], widths, n))


def test_random_layout_pairs_tiled(monkeypatch):
    """Random records (1..40 fields, widths 1..16 incl. odd), random partitions on both sides,
    random N around tile boundaries: tiled kernel forced (ADHA_SMALL_BYTES=0)."""
    monkeypatch.setenv("ADHA_SMALL_BYTES", "0")
    rng = np.random.default_rng(1407)
    for trial in range(120):
        F = int(rng.integers(1, 41))
        widths = [int(x) for x in rng.choice([1, 2, 3, 4, 4, 4, 8, 8, 12, 16], size=F)]
        k1, k2 = int(rng.integers(1, F + 1)), int(rng.integers(1, F + 1))
        ls = [int(x) for x in rng.integers(0, k1, size=F)]
        ld = [int(x) for x in rng.integers(0, k2, size=F)]
        T = plan_T(widths, ls, ld)
        n = int(rng.choice([T - 1, T, T + 1, 3 * T + int(rng.integers(0, T)), 160 * T + 7]))
        check_pair(widths, ls, ld, max(n, 1), seed=trial)


def test_section_run_matches_numpy():
    """Synthetic consumer section reads through the layout: streaming pass and
    irregular gather equal sum_f x_f^2 computed by numpy in fp32.  Tolerance: fp32 sums of <= 9
    squares of values in [1, 2): the kernel's FMA vs numpy's multiply-add differ by <= 9 ulps,
    so rel 4e-6."""
    names = ["V1", "V2", "V3", "U1", "U2", "U3", "S", "T", "interpT"]
    widths = [4] * 9
    n = 100_003
    rng = np.random.default_rng(3)
    x = rng.uniform(1, 2, size=(n, 9)).astype(np.float32)
    cols = [np.ascontiguousarray(x[:, f]).view(np.uint8).reshape(n, 4) for f in range(9)]
    for lay in ["{V1,V2,V3},U1,U2,U3,S,T,interpT", "V1,V2,V3,U1,U2,U3,S,T,interpT", "{V1,V2,V3,U1,U2,U3,S,T,interpT}"]:
        L = A.Layout.from_string(lay, names, widths)
        buf = to_dev(O.pack(cols, widths, L.cluster_of, n))
        for fields in ([0, 1, 2], [0, 1, 2, 6, 7, 8], [5]):
            out = torch.empty(n, dtype=torch.float32, device="cuda")
            A.section_run(buf, L, n, fields, out)
            exp = np.zeros(n, np.float32)
            for f in fields:
                exp = exp + x[:, f] * x[:, f]
            np.testing.assert_allclose(out.cpu().numpy(), exp, rtol=4e-6)
            idx = torch.from_numpy(rng.integers(0, n, size=5000)).cuda()
            out2 = torch.empty(5000, dtype=torch.float32, device="cuda")
            A.section_run(buf, L, n, fields, out2, idx=idx)
            np.testing.assert_allclose(out2.cpu().numpy(), exp[idx.cpu().numpy()], rtol=4e-6)
    with pytest.raises(A.AdhaError) as e:
        A.section_run(to_dev(np.zeros(1024, np.uint8)), A.Layout.aos([2, 2]), 10, [0], torch.empty(10, device="cuda"))
    assert e.value.name == "ADHA_ERR_UNSUPPORTED"


@pytest.mark.parametrize("mode,pinned", [("auto", True), ("hybrid", True), ("zero", True), ("staged", True),
                                         ("auto", False)])
def test_remap_host_modes(mode, pinned, monkeypatch):
    """adha_remap_host in every strategy (hybrid / zero-copy / staged; pageable memory falls back to
    staged) equals the oracle, C3-like multi-region layouts included; auto picks zero-copy for the
    64-region C3 src."""
    monkeypatch.setenv("ADHA_HOST_MODE", mode)
    monkeypatch.setenv("ADHA_HOST_CHUNK_BYTES", str(1 << 20))     # several chunks
    for widths, ls, ld, n in [(config_widths(16), [0] * 16, list(range(16)), 300_001),
                              (config_widths(64), list(range(64)), c3_labels(), 50_017),
                              ([1, 3, 4, 8] * 4, list(range(16)), [0] * 16, 120_000)]:
        La, Ld = A.Layout(widths, ls), A.Layout(widths, ld)
        src_np = O.pack(field_columns(n, n, widths), widths, ls, n)
        h_src = torch.from_numpy(src_np)
        h_dst = torch.full((Ld.nbytes(n),), SENT, dtype=torch.uint8)
        if pinned:
            h_src, h_dst = h_src.pin_memory(), h_dst.pin_memory()
        scratch = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
        A.remap_host(h_src, La, h_dst, Ld, n, scratch)
        torch.cuda.synchronize()
        assert np.array_equal(h_dst.numpy(), oracle_dst(src_np, ls, ld, widths, n)), (mode, pinned, widths[:4])


# ----------------------------------------------------------------------------- generalised layouts (N4)

def check_pair_ex(widths, ls, bs, als, ld, bd, ald, n, seed=0):
    cols = field_columns(seed, n, widths)
    src = O.pack_ex(cols, widths, ls, n, bs, als, fill=0x3C)
    Ls = A.Layout(widths, ls, blocks=bs, aligned=als)
    Ld = A.Layout(widths, ld, blocks=bd, aligned=ald)
    got = run_remap(A, src, Ls, Ld, n)
    exp = np.full(O.layout_bytes_ex(widths, ld, n, bd, ald), SENT, np.uint8)
    O.remap_ex(src, ls, exp, ld, widths, n, bs, als, bd, ald)
    if not np.array_equal(got, exp):
        bad = np.nonzero(got != exp)[0]
        raise AssertionError(f"mismatch at {bad.size} bytes, first {bad[:8]} (widths={widths} ls={ls} bs={bs} "
                             f"als={als} ld={ld} bd={bd} ald={ald} n={n})")


@pytest.mark.parametrize("case", [
    ("AoS->AoSoA8", [4] * 8, [0] * 8, [1] * 8, False, [0] * 8, [8] * 8, False),
    ("AoSoA32->SoA", config_widths(16), [0] * 16, [32] * 16, False, list(range(16)), [1] * 16, False),
    ("SoA->aligned AoS", [1, 4, 2, 8, 4, 2], list(range(6)), [1] * 6, False, [0] * 6, [1] * 6, True),
    ("aligned AoS->AoSoA4 hybrid", [1, 4, 2, 8, 4, 2], [0] * 6, [1] * 6, True, [0, 0, 1, 1, 2, 2], [4] * 6, True),
    ("Medical AoSV@8 -> SoA", [4] * 9, [0, 0, 0, 1, 2, 3, 4, 5, 6], [8, 8, 8, 1, 1, 1, 1, 1, 1], False,
     list(range(9)), [1] * 9, False),
])
def test_generalised_layouts(case, small_path):
    _, widths, ls, bs, als, ld, bd, ald = case
    T = A.plan_describe(A.Layout(widths, ls, blocks=bs, aligned=als), A.Layout(widths, ld, blocks=bd, aligned=ald))["T"]
    for n in (1, 31, 33, T + 7, 5 * T + 19, 150 * T + 3):
        check_pair_ex(widths, ls, bs, als, ld, bd, ald, n, seed=n)


def test_generalised_random_pairs(monkeypatch):
    import random as _r
    monkeypatch.setenv("ADHA_SMALL_BYTES", "0")
    rng = _r.Random(4859)
    for trial in range(80):
        F = rng.randint(1, 12)
        widths = [rng.choice([1, 2, 3, 4, 4, 4, 6, 8, 8, 12]) for _ in range(F)]
        ls = [rng.randrange(F) for _ in range(F)]
        ld = [rng.randrange(F) for _ in range(F)]
        cbs = {l: rng.choice([1, 1, 2, 4, 8, 32]) for l in set(ls)}
        cbd = {l: rng.choice([1, 1, 2, 4, 8, 32]) for l in set(ld)}
        bs, bd = [cbs[l] for l in ls], [cbd[l] for l in ld]
        als, ald = rng.random() < 0.5, rng.random() < 0.5
        T = A.plan_describe(A.Layout(widths, ls, blocks=bs, aligned=als), A.Layout(widths, ld, blocks=bd, aligned=ald))["T"]
        n = rng.choice([T - 1, T + 5, 3 * T + rng.randrange(T), 160 * T + 11])
        check_pair_ex(widths, ls, bs, als, ld, bd, ald, max(n, 1), seed=trial)


# ----------------------------------------------------------------------------- cross-device (NEXT N2)

def test_remap_peer_same_device_and_errors():
    """adha_remap_peer with src and dst on one device is adha_remap (bit-exact vs the oracle);
    bad device ids and non-device pointers are rejected before any launch."""
    widths = config_widths(16)
    n = 300_001
    aos, soa = [0] * 16, list(range(16))
    cols = field_columns(5, n, widths)
    src = O.pack(cols, widths, aos, n)
    La, Ls = A.Layout(widths, aos), A.Layout(widths, soa)
    d_src = to_dev(src)
    d_dst = sentinel_dev(Ls.nbytes(n))
    A.remap_peer(d_src, La, d_dst, Ls, n)
    torch.cuda.synchronize()
    assert np.array_equal(d_dst.cpu().numpy(), oracle_dst(src, aos, soa, widths, n))
    lib = A._lib
    nd = torch.cuda.device_count()
    rc = lib.adha_remap_peer(d_src.data_ptr(), La.handle, 0, d_dst.data_ptr(), Ls.handle, nd, n, None)
    assert A.STATUS[rc] == "ADHA_ERR_INVALID_ARG"
    h = torch.empty(Ls.nbytes(n), dtype=torch.uint8).pin_memory()
    rc = lib.adha_remap_peer(d_src.data_ptr(), La.handle, 0, h.data_ptr(), Ls.handle, 0, n, None)
    assert A.STATUS[rc] == "ADHA_ERR_INVALID_ARG" and b"not device memory" in lib.adha_last_error()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs (peer access)")
def test_remap_peer_two_devices():
    """One kernel on cuda:0 stores the remapped records into cuda:1's HBM; bit-exact vs the oracle."""
    widths = config_widths(16)
    n = 1_000_003
    aos, hyb = [0] * 16, [0, 0, 1, 1, 2, 2, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11]
    cols = field_columns(6, n, widths)
    src = O.pack(cols, widths, aos, n)
    La, Lh = A.Layout(widths, aos), A.Layout(widths, hyb)
    d_src = torch.from_numpy(src).to("cuda:0")
    d_dst = torch.full((Lh.nbytes(n),), SENT, dtype=torch.uint8, device="cuda:1")
    A.remap_peer(d_src, La, d_dst, Lh, n)
    torch.cuda.synchronize(0)
    assert np.array_equal(d_dst.cpu().numpy(), oracle_dst(src, aos, hyb, widths, n))


def test_concurrent_host_threads():
    """Several host threads call adha_remap at once (ctypes drops the GIL), each on its own stream
    with its own layout pair, so plan compilation and the plan cache run concurrently; every
    result is bit-exact vs the oracle."""
    import threading
    widths = config_widths(16)
    n = 50_001
    pairs = [([0] * 16, list(range(16))), (list(range(16)), [0] * 16),
             ([i // 4 for i in range(16)], [i % 4 for i in range(16)]),
             ([i % 2 for i in range(16)], [i // 8 for i in range(16)])]
    results, errors = {}, []

    def work(k):
        try:
            ls, ld = pairs[k % len(pairs)]
            cols = field_columns(100 + k, n, widths)
            src = O.pack(cols, widths, ls, n)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                d_src = to_dev(src)
                d_dst = sentinel_dev(A.Layout(widths, ld).nbytes(n))
                for _ in range(3):
                    A.remap(d_src, A.Layout(widths, ls), d_dst, A.Layout(widths, ld), n, stream=s)
            s.synchronize()
            results[k] = (src, ls, ld, d_dst.cpu().numpy())
        except Exception as e:  # surfaced below
            errors.append(e)

    threads = [threading.Thread(target=work, args=(k,)) for k in range(8)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for k, (src, ls, ld, got) in results.items():
        assert np.array_equal(got, oracle_dst(src, ls, ld, widths, n)), k


def test_concurrent_remap_host_threads(monkeypatch):
    """adha_remap_host from 4 host threads at once (own streams, own scratch, own pinned buffers):
    the per-device pipe is shared, so its enqueue is serialised; every result is bit-exact."""
    import threading
    monkeypatch.setenv("ADHA_HOST_MODE", "hybrid")
    monkeypatch.setenv("ADHA_HOST_CHUNK_BYTES", str(1 << 20))
    widths = config_widths(16)
    n = 120_001
    ls, ld = [0] * 16, list(range(16))
    La, Ld = A.Layout(widths, ls), A.Layout(widths, ld)
    out, errors = {}, []

    def work(k):
        try:
            src_np = O.pack(field_columns(200 + k, n, widths), widths, ls, n)
            h_src = torch.from_numpy(src_np).pin_memory()
            h_dst = torch.full((Ld.nbytes(n),), SENT, dtype=torch.uint8).pin_memory()
            scratch = torch.empty(16 << 20, dtype=torch.uint8, device="cuda")
            s = torch.cuda.Stream()
            for _ in range(3):
                A.remap_host(h_src, La, h_dst, Ld, n, scratch, stream=s)
            s.synchronize()
            out[k] = (src_np, h_dst.numpy().copy())
        except Exception as e:  # surfaced below
            errors.append(e)

    threads = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for k, (src_np, got) in out.items():
        assert np.array_equal(got, oracle_dst(src_np, ls, ld, widths, n)), k


@pytest.mark.parametrize("mode", ["tma", "stg", "auto"])
def test_write_back_modes(mode, monkeypatch):
    """Both write-back paths of the tiled kernel (consumer STG, or the TMA bulk-store warp chosen per
    launch for one large dst chunk per tile) are bit-exact, forced either way: K-Means chain edges,
    AoS->SoA (many small chunks), C-aligned and AoSoA dst (pre-zeroed padding), ragged N."""
    if mode != "auto":
        monkeypatch.setenv("ADHA_COPYOUT", mode)
    monkeypatch.setenv("ADHA_SMALL_BYTES", "0")
    w32 = [4] * 32
    cases = [
        (w32, list(range(32)), None, False, [i // 8 for i in range(32)], None, False, 200_003),
        (w32, [i // 8 for i in range(32)], None, False, [0] * 32, None, False, 100_001),
        (config_widths(16), [0] * 16, None, False, list(range(16)), None, False, 70_001),
        ([4, 8, 4, 4, 8], list(range(5)), None, False, [0] * 5, None, True, 50_017),
        ([4, 4, 8, 4], list(range(4)), None, False, [0] * 4, [8] * 4, False, 33_333),
    ]
    for w, ls, bs, als, ld, bd, ald, n in cases:
        check_pair_ex(w, ls, bs, als, ld, bd, ald, n, seed=n % 97)


@pytest.mark.parametrize("loader", ["tma", "cpa"])
@pytest.mark.parametrize("merge", ["merged", "components"])
def test_loaders(loader, merge, monkeypatch):
    """Both tile loaders of the tiled kernel are bit-exact: the producer warp's TMA bulk copies and
    the consumers' cp.async (remap.cu: auto for >= 32 src chunks per tile up to 24 MB), forced
    either way, on the merged one-component plan and on per-component plans (the cp.async
    look-ahead then crosses component boundaries), with padded / AoSoA dst and ragged N --
    including N below s_in tiles per CTA and CTAs without tiles."""
    monkeypatch.setenv("ADHA_LOADER", loader)
    monkeypatch.setenv("ADHA_SMALL_BYTES", "0")
    if merge == "components":
        monkeypatch.setenv("ADHA_MERGE_BYTES", "0")
    else:
        monkeypatch.delenv("ADHA_MERGE_BYTES", raising=False)
    w64 = config_widths(64)
    cases = [
        (w64, list(range(64)), None, False, c3_labels(), None, False, 100_003),
        (w64, list(range(64)), None, False, c3_labels(), None, False, 4_111),
        ([4] * 32, list(range(32)), None, False, [0] * 32, None, False, 200_003),
        (config_widths(16), [0] * 16, None, False, list(range(16)), None, False, 70_001),
        ([4] * 9, [0, 0, 0, 1, 2, 3, 4, 5, 6], None, False, list(range(9)), None, False, 300_007),
        ([4] * 9, [0, 0, 0, 1, 2, 3, 4, 5, 6], None, False, list(range(9)), None, False, 33),
        ([4, 8, 4, 4, 8], list(range(5)), None, False, [0] * 5, None, True, 50_017),
        ([4, 4, 8, 4], list(range(4)), None, False, [0] * 4, [8] * 4, False, 33_333),
    ]
    for w, ls, bs, als, ld, bd, ald, n in cases:
        check_pair_ex(w, ls, bs, als, ld, bd, ald, n, seed=n % 89)


@pytest.mark.parametrize("path", ["tiled", "direct"])
@pytest.mark.parametrize("pdl", ["1", "0"])
def test_back_to_back_hazards(pdl, path, monkeypatch):
    """Programmatic dependent launch (remap.cu launch_ex / launch_pdl, kernels.cuh grid_dep_wait), on the
    tiled and on the direct kernel: a remap may start
    while the previous one drains, but must not read what it writes (RAW) nor write what it still reads
    (WAR).  A ring of remaps on one stream -- A->B, B->C, C->A, then around again, every buffer both read
    and overwritten by neighbouring launches -- must end exactly where the oracle's ring ends."""
    monkeypatch.setenv("ADHA_PDL", pdl)
    monkeypatch.setenv("ADHA_SMALL_BYTES", "0" if path == "tiled" else str(1 << 40))
    widths = config_widths(16)
    n = 300_007
    labs = [[0] * 16, list(range(16)), [i // 4 for i in range(16)]]
    Ls = [A.Layout(widths, l) for l in labs]
    cols = field_columns(11, n, widths)
    src = O.pack(cols, widths, labs[0], n, fill=0x3C)
    bufs = [to_dev(src), sentinel_dev(Ls[1].nbytes(n)), sentinel_dev(Ls[2].nbytes(n))]
    torch.cuda.synchronize()
    for _ in range(4):
        for k in range(3):
            A.remap(bufs[k], Ls[k], bufs[(k + 1) % 3], Ls[(k + 1) % 3], n)
    torch.cuda.synchronize()
    # a full ring returns every payload byte to its AoS place: the oracle's ring, once, ends there too
    mid = oracle_dst(src, labs[0], labs[1], widths, n)
    last = oracle_dst(mid, labs[1], labs[2], widths, n)
    back = np.full(src.size, 0x3C, np.uint8)
    O.remap(last, labs[2], back, labs[0], widths, n)
    got = bufs[0].cpu().numpy()[: Ls[0].nbytes(n)]
    assert np.array_equal(got, back[: Ls[0].nbytes(n)])
    assert np.array_equal(bufs[1].cpu().numpy()[: Ls[1].nbytes(n)], mid)
    assert np.array_equal(bufs[2].cpu().numpy()[: Ls[2].nbytes(n)], last)
