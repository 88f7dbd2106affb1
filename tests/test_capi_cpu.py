"""CPU-side tests of the C ABI (no GPU): exported symbols, the layout descriptor
against the oracle's address model, shard ranges, error codes, the C++ planner
against the Python planner oracle and the paper pins, and the remap-plan
compiler's permutation table (coverage and bank-conflict freedom)."""
import json
import os
import random
import re
import ctypes

import numpy as np
import pytest

import paper_1407_4859_b200 as A
from oracle import planner as P
from oracle import remap as O
from tests.conftest import ROOT, golden


def header_symbols():
    text = open(os.path.join(ROOT, "include", "adha.h")).read()
    return sorted(set(re.findall(r"ADHA_API\s+[\w\s\*]*?\b(adha_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    syms = header_symbols()
    assert len(syms) >= 20
    lib = ctypes.CDLL(A.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert A.version() >= 100


def rand_layout(rng, F):
    widths = [rng.choice([1, 2, 3, 4, 8, 12]) for _ in range(F)]
    labels = [rng.randrange(F) for _ in range(F)]
    return widths, labels


def test_layout_descriptor_matches_oracle_addresses():
    rng = random.Random(3)
    for _ in range(300):
        F = rng.randint(1, 12)
        widths, labels = rand_layout(rng, F)
        L = A.Layout(widths, labels)
        for n in (0, 1, 5, 1000, 123457):
            base, stride, offset, total = O.field_addresses(widths, labels, n)
            assert L.nbytes(n) == total == O.layout_bytes(widths, labels, n)
            for f in range(F):
                assert L.field_address(f, n) == (base[f], stride[f], offset[f])
        assert L.record_bytes == sum(widths)


def test_layout_strings_and_paper_notation(expected):
    names = ["V1", "V2", "V3", "U1", "U2", "U3", "S", "T", "interpT"]
    w = [4] * 9
    l = A.Layout.from_string("V1,V2,V3,{U1,U2,U3},S,T,interpT", names, w)
    assert l.to_string() == expected["medical_aosu"]["value"]
    l2 = A.Layout.from_string(expected["medical_aosv"]["value"], names, w)
    assert l2.to_string() == expected["medical_aosv"]["value"]
    assert l2.n_clusters == 7 and l2.cluster_of == [0, 0, 0, 1, 2, 3, 4, 5, 6]
    decl = {n: i for i, n in enumerate(names)}
    rng = random.Random(8)
    for _ in range(100):
        labels = [rng.randrange(9) for _ in names]
        L = A.Layout(w, labels, names)
        groups = {}
        for n, lab in zip(names, labels):
            groups.setdefault(lab, []).append(n)
        assert L.to_string() == P.layout_string(P.canonical(list(groups.values()), decl))
        assert A.Layout.from_string(L.to_string(), names, w).to_string() == L.to_string()
    for bad in ["{V1,V2}", "V1,V1,V2,V3,U1,U2,U3,S,T,interpT", "{V1,{V2}},V3,U1,U2,U3,S,T,interpT", "X"]:
        with pytest.raises(A.AdhaError) as e:
            A.Layout.from_string(bad, names, w)
        assert e.value.name == "ADHA_ERR_PARSE"


def test_invalid_layouts_rejected():
    with pytest.raises(A.AdhaError):
        A.Layout([], [])
    with pytest.raises(A.AdhaError):
        A.Layout([0, 4], [0, 1])
    with pytest.raises(A.AdhaError):
        A.Layout.aos([4]).nbytes(-1)
    with pytest.raises(A.AdhaError) as e:
        A.Layout.aos([1 << 16]).nbytes(2 ** 62)
    assert e.value.name == "ADHA_ERR_TOO_LARGE"


def test_shard_range_floor_formula():
    for N in (0, 1, 7, 1000, 107374182, 2 ** 40 + 3):
        for G in (1, 2, 3, 4, 8):
            prev = 0
            for g in range(G):
                lo, hi = A.shard_range(N, G, g)
                assert lo == g * N // G and hi == (g + 1) * N // G and lo == prev
                prev = hi
            assert prev == N
    with pytest.raises(A.AdhaError):
        A.shard_range(10, 0, 0)
    with pytest.raises(A.AdhaError):
        A.shard_range(10, 2, 2)


def test_remap_validation_errors_without_gpu():
    # validation happens before any CUDA call
    a, s = A.Layout.aos([4, 4]), A.Layout.soa([4, 4])
    with pytest.raises(A.AdhaError) as e:
        A.remap(256, a, 1 << 20, A.Layout.aos([4, 8]), 10, stream=0)
    assert e.value.name == "ADHA_ERR_LAYOUT_MISMATCH"
    with pytest.raises(A.AdhaError) as e:
        A.remap(256 + 16, a, 1 << 20, s, 10, stream=0)
    assert e.value.name == "ADHA_ERR_ALIGNMENT"
    with pytest.raises(A.AdhaError) as e:
        A.remap(4096, a, 4096 + 256, s, 100, stream=0)
    assert e.value.name == "ADHA_ERR_OVERLAP"
    with pytest.raises(A.AdhaError) as e:
        A.remap(4096, a, 1 << 20, s, -1, stream=0)
    assert e.value.name == "ADHA_ERR_INVALID_ARG"
    A.remap(0, a, 0, s, 0, stream=0)          # N = 0 is a no-op


# ---------------------------------------------------------------- C++ planner vs Python oracle

def _prog_json(p: P.Program) -> str:
    return json.dumps({
        "schema_version": 1, "name": p.name, "record_count": p.record_count,
        "fields": [{"name": f.name, "elem_bytes": f.elem_bytes} for f in p.fields],
        "sections": [{"id": s.id, "trip_count": s.trip_count, "allowed_devices": list(s.allowed_devices),
                      "groups": [{"fields": list(g.fields), "freq": g.freq, "pattern": g.pattern, "ops": g.ops}
                                 for g in s.groups]} for s in p.sections],
        "order": p.order})


def _arch_json(a: P.Architecture) -> str:
    return json.dumps({
        "schema_version": 1,
        "devices": [{"name": d.name, "line_bytes": d.line_bytes, "line_time_ns": d.line_time_ns,
                     "throughput_ops_per_ns": d.throughput_ops_per_ns, "coalescing": d.coalescing,
                     "stream_cluster_penalty": d.stream_cluster_penalty,
                     "cluster_capacity_bytes": d.cluster_capacity_bytes} for d in a.devices],
        "links": [{"from": l.src, "to": l.dst, "bandwidth_bytes_per_ns": l.bandwidth_bytes_per_ns,
                   "latency_ns": l.latency_ns} for l in a.links],
        "same_device_remap_bandwidth_bytes_per_ns": a.same_device_remap_bandwidth_bytes_per_ns,
        "remap_fixed_overhead_ns": a.remap_fixed_overhead_ns})


def test_cpp_ods_fixtures(expected):
    prog, arch = golden("medical_aosu_program.json"), golden("medical_arch.json")
    assert A.plan_ods(prog, arch, "aosu", "cpu") == expected["medical_aosu"]["value"]
    km, t3 = golden("kmeans_program.json"), golden("kmeans_table3_arch.json")
    assert A.plan_ods(km, t3, "k1", "cpu") == expected["kmeans_cap32_noncoalescing"]["value"]
    assert A.plan_ods(km, t3, "k1", "gpu") == expected["kmeans_coalescing_soa"]["value"]
    assert A.plan_ods(golden("c3_program.json"), golden("b200_arch.json"), "c3", "b200") == \
        expected["c3_hybrid"]["value"]
    # SURVEY.md 8(d) random program variant: the C++ planner gives the oracle's layout
    assert A.plan_ods(golden("c3_random_program.json"), golden("b200_arch.json"), "c3r", "b200") == \
        golden("c3_random_expected.json")["c3_random_hybrid"]["value"]


def test_cpp_pdl_fixtures(expected):
    plan = A.plan_pdl(golden("medical_program.json"), golden("medical_arch.json"), golden("medical_profile.json"))
    assert [[r["sections"], r["device"], r["layout"]] for r in plan["runs"]] == expected["medical_plan"]["runs"]
    assert len(plan["remaps"]) == 1 and plan["remaps"][0]["moved"] == expected["medical_plan"]["remap_moved"]
    plan = A.plan_pdl(golden("kmeans_program.json"), golden("kmeans_arch.json"), golden("kmeans_profile.json"))
    assert [[r["sections"], r["device"], r["layout"]] for r in plan["runs"]] == expected["kmeans_plan"]["runs"]
    assert plan["remaps"] == []


def test_cpp_planner_errors():
    prog, arch = golden("medical_aosu_program.json"), golden("medical_arch.json")
    with pytest.raises(A.AdhaError) as e:
        A.plan_ods(prog, arch, "aosu", "gpu")                 # device not allowed for the section
    assert e.value.name == "ADHA_ERR_PLANNER"
    with pytest.raises(A.AdhaError) as e:
        A.plan_ods("{not json", arch, "aosu", "cpu")
    assert e.value.name == "ADHA_ERR_PARSE"
    bad = json.loads(json.dumps(prog))
    bad["sections"][0]["groups"][0]["fields"].append("X")
    with pytest.raises(A.AdhaError) as e:
        A.plan_ods(bad, arch, "aosu", "cpu")
    assert e.value.name == "ADHA_ERR_PLANNER"
    narrow = json.loads(json.dumps(arch))
    narrow["devices"][0]["cluster_capacity_bytes"] = 2
    with pytest.raises(A.AdhaError) as e:
        A.plan_ods(prog, narrow, "aosu", "cpu")
    assert e.value.name == "ADHA_ERR_CAPACITY"


def test_cpp_planner_equals_oracle_random():
    from tests.test_oracle_planner import random_program, random_arch
    rng = random.Random(2024)
    for _ in range(150):
        p, a = random_program(rng), random_arch(rng)
        pj, aj = _prog_json(p), _arch_json(a)
        for s in p.sections:
            for d in s.allowed_devices:
                try:
                    exp = P.layout_string(P.ods(s, a.device(d), p))
                except P.PlannerError:
                    with pytest.raises(A.AdhaError):
                        A.plan_ods(pj, aj, s.id, d)
                    continue
                assert A.plan_ods(pj, aj, s.id, d) == exp
        try:
            exp_plan = P.plan_to_json(P.shortest_plan(p, a), p)
        except P.PlannerError:
            with pytest.raises(A.AdhaError):
                A.plan_pdl(pj, aj)
            continue
        got = A.plan_pdl(pj, aj)
        assert got["total_ns"] == pytest.approx(exp_plan["total_ns"], rel=1e-12)
        assert [[r["sections"], r["device"], r["layout"]] for r in got["runs"]] == \
            [[r["sections"], r["device"], r["layout"]] for r in exp_plan["runs"]]
        assert [[m["boundary"], m["moved"]] for m in got["remaps"]] == \
            [[m["boundary"], m["moved"]] for m in exp_plan["remaps"]]


# ---------------------------------------------------------------- remap-plan compiler (host)

def _plan_checks(widths, ls, ld, merged=False):
    from tests.test_oracle_remap import clusters_in_order
    Ls, Ld = A.Layout(widths, ls), A.Layout(widths, ld)
    d = A.plan_describe(Ls, Ld, merged=merged)
    assert d["tiled"], d["why_naive"]
    if merged:
        assert len(d["components"]) == 1
    if d["byte_groups"]:
        if not merged:
            _check_byte_groups(widths, ls, ld)
        return d
    g = d["unit"]
    cs, cd = clusters_in_order(ls), clusters_in_order(ld)          # canonical clusters (field lists)
    csrc = {f: k for k, c in enumerate(cs) for f in c}
    cdst = {f: k for k, c in enumerate(cd) for f in c}
    comps = d["components"]
    # components partition the fields and are closed under "shares a src or dst cluster"
    allf = sorted(f for K in comps for f in K["fields"])
    assert allf == list(range(len(widths)))
    for K in comps:
        fs = set(K["fields"])
        assert sorted(K["src_clusters"]) == sorted({csrc[f] for f in fs})
        assert sorted(K["dst_clusters"]) == sorted({cdst[f] for f in fs})
        for c in K["src_clusters"]:
            assert set(cs[c]) <= fs
        for c in K["dst_clusters"]:
            assert set(cd[c]) <= fs
        assert K["R"] == sum(widths[f] for f in fs) and K["T"] % 32 == 0
        assert K["identity"] == (len(K["src_clusters"]) == 1 and len(K["dst_clusters"]) == 1
                                 and cs[K["src_clusters"][0]] == cd[K["dst_clusters"][0]])
    ent_in, ent_out = np.array(d["ent_in"]), np.array(d["ent_out"])
    ent_sc, ent_dc = np.array(d["ent_sc"]), np.array(d["ent_dc"])
    _, ss, os_, _ = O.field_addresses(widths, ls, 32)
    _, sd, od, _ = O.field_addresses(widths, ld, 32)
    total = 0
    for K in comps:
        if K["identity"]:
            assert K["n_instr"] == 0
            continue
        W = K["R"] // g
        assert K["n_instr"] == W
        lo, hi = 32 * K["instr_base"], 32 * (K["instr_base"] + W)
        total += hi - lo
        # every unit of the component's 32-record period moved exactly once, to the place the
        # oracle's record model gives (r*stride + offset + j, inside the unit's chunk)
        exp = set()
        for r in range(32):
            for f in K["fields"]:
                for j in range(0, widths[f], g):
                    exp.add((int(r * ss[f] + os_[f] + j) // g, int(r * sd[f] + od[f] + j) // g, csrc[f], cdst[f]))
        got = {(int(a), int(b), d["src_order"][c], d["dst_order"][e])
               for a, b, c, e in zip(ent_in[lo:hi], ent_out[lo:hi], ent_sc[lo:hi], ent_dc[lo:hi])}
        assert got == exp and len(got) == hi - lo
        if g == 4:
            assert d["matched"]
            for i in range(lo, hi, 32):           # conflict-free: 32 distinct banks on both sides
                assert len(set((ent_in[i: i + 32] % 32).tolist())) == 32
                assert len(set((ent_out[i: i + 32] % 32).tolist())) == 32
    assert total == ent_in.size
    return d


def test_plan_compiler_tables():
    w16 = [8 if i % 4 == 3 else 4 for i in range(16)]
    d = _plan_checks(w16, [0] * 16, list(range(16)))                    # C2 AoS -> SoA
    assert d["unit"] == 4
    w64 = [8 if i % 4 == 3 else 4 for i in range(64)]
    hyb = P.parse_layout(golden("expected.json")["c3_hybrid"]["value"], {f"f{i}": i for i in range(64)})
    lab = [0] * 64
    for c, cl in enumerate(hyb):
        for n in cl:
            lab[int(n[1:])] = c
    _plan_checks(w64, list(range(64)), lab)                             # C3 SoA -> hybrid
    med = [4] * 9
    _plan_checks(med, [0] * 9, [0, 0, 0, 1, 2, 3, 4, 5, 6])            # C4 AoS -> AoSV
    _plan_checks([4, 4, 4], [0, 0, 0], [0, 1, 2])                       # C1
    rng = random.Random(11)
    for _ in range(40):
        F = rng.randint(1, 10)
        widths = [rng.choice([1, 2, 3, 4, 8]) for _ in range(F)]
        _plan_checks(widths, [rng.randrange(F) for _ in range(F)], [rng.randrange(F) for _ in range(F)])


def test_merged_plan_tables():
    """The merged plan (one component over every cluster; remap.cu runs it for multi-component
    remaps up to ADHA_MERGE_BYTES) passes the same table checks: every unit of the 32-record period
    moved once to the oracle's address, 32 distinct banks per instruction on both sides."""
    w64 = [8 if i % 4 == 3 else 4 for i in range(64)]
    hyb = P.parse_layout(golden("expected.json")["c3_hybrid"]["value"], {f"f{i}": i for i in range(64)})
    lab = [0] * 64
    for c, cl in enumerate(hyb):
        for n in cl:
            lab[int(n[1:])] = c
    d = _plan_checks(w64, list(range(64)), lab, merged=True)             # C3 SoA -> hybrid
    assert d["matched"] and d["components"][0]["n_instr"] == 80
    _plan_checks(w64, lab, list(range(64)), merged=True)                 # C3 hybrid -> SoA
    med = [4] * 9
    _plan_checks(med, [0, 0, 0, 1, 2, 3, 4, 5, 6], list(range(9)), merged=True)   # Medical AoSV -> SoA
    rng = random.Random(12)
    for _ in range(40):
        F = rng.randint(2, 16)
        widths = [rng.choice([4, 4, 8, 12]) for _ in range(F)]
        _plan_checks(widths, [rng.randrange(F) for _ in range(F)], [rng.randrange(F) for _ in range(F)],
                     merged=True)


def test_plan_falls_back_beyond_limits():
    widths = [4] * 300
    d = A.plan_describe(A.Layout.aos(widths), A.Layout.soa(widths))
    assert not d["tiled"] and "fields" in d["why_naive"]


def test_plan_layouts_follow_the_plan(expected):
    plan = A.plan_pdl(golden("medical_program.json"), golden("medical_arch.json"), golden("medical_profile.json"))
    names = [f["name"] for f in golden("medical_program.json")["fields"]]
    lays = A.plan_layouts(plan, names, [4] * 9)
    assert [l.to_string() for l in lays] == [r[2] for r in expected["medical_plan"]["runs"]]
    # the remap edge moves exactly the fields whose cluster differs (same-device reading)
    a, b = lays
    moved = [names[f] for f in range(9)
             if {g for g in range(9) if a.cluster_of[g] == a.cluster_of[f]} !=
                {g for g in range(9) if b.cluster_of[g] == b.cluster_of[f]}]
    assert moved == expected["medical_plan"]["remap_moved"]


def test_plan_candidates_match_oracle_run_graph():
    """adha_plan_candidates = the oracle's build_run_graph nodes: same runs, devices,
    layouts, exec estimates."""
    from tests.test_oracle_planner import random_program, random_arch
    cases = [(golden("medical_program.json"), golden("medical_arch.json"), golden("medical_profile.json"))]
    rng = random.Random(77)
    for _ in range(40):
        p, a = random_program(rng), random_arch(rng)
        cases.append((json.loads(_prog_json(p)), json.loads(_arch_json(a)), None))
    for prog, arch, prof in cases:
        p, a = P.program_from_json(prog), P.arch_from_json(arch)
        pr = P.profile_from_json(prof) if prof else None
        try:
            exp = P.build_run_graph(p, a, pr)
        except P.PlannerError:
            with pytest.raises(A.AdhaError):
                A.plan_candidates(prog, arch, prof)
            continue
        got = A.plan_candidates(prog, arch, prof)["runs"]
        assert len(got) == len(exp)
        for g, e in zip(got, exp):
            assert (g["begin"], g["end"], g["device"], g["layout"]) == (e.begin, e.end, e.device, P.layout_string(e.layout))
            assert g["exec_ns"] == pytest.approx(e.exec_ns, rel=1e-12)
    assert len(A.plan_candidates(golden("medical_program.json"), golden("medical_arch.json"))["runs"]) == 56


def _prmt(a, b, sel):
    """__byte_perm semantics: bytes of {b:a} indexed 0..7, one selector nibble per result byte."""
    src = [(a >> (8 * i)) & 0xFF for i in range(4)] + [(b >> (8 * i)) & 0xFF for i in range(4)]
    return sum(src[(sel >> (4 * j)) & 7] << (8 * j) for j in range(4))


def _check_byte_groups(widths, ls, ld):
    """Simulate the byte-group plan of one 32-record period on the host: every dst byte must be
    produced exactly once, from the src byte the oracle's record model names."""
    from tests.test_oracle_remap import clusters_in_order
    Ls, Ld = A.Layout(widths, ls), A.Layout(widths, ld)
    d = A.plan_describe(Ls, Ld)
    assert d["tiled"] and d["unit"] < 4 and d["byte_groups"], d
    cs, cd = clusters_in_order(ls), clusters_in_order(ld)
    csrc = {f: k for k, c in enumerate(cs) for f in c}
    cdst = {f: k for k, c in enumerate(cd) for f in c}
    _, ss, os_, _ = O.field_addresses(widths, ls, 32)
    _, sd, od, _ = O.field_addresses(widths, ld, 32)
    # a distinct value per src byte: (src cluster, local byte) -> tag
    def tag(c, off):
        return (c * 7919 + off * 131) & 0xFF
    seen = {}
    for K in d["components"]:
        if K["identity"]:
            continue
        for gi in range(K["instr_base"], K["instr_base"] + K["n_instr"]):
            g = d["groups"][gi]
            n_out, n_src = g[0], g[1]
            out_off, out_dc, src_off, src_sc, sel = g[2:6], g[6:10], g[10:14], g[14:18], g[18:30]
            words = []
            for m in range(4):
                if m < n_src:
                    c = d["src_order"][src_sc[m]]
                    words.append(sum(tag(c, src_off[m] + j) << (8 * j) for j in range(4)))
                else:
                    words.append(0)
            for o in range(n_out):
                a = _prmt(words[0], words[1], sel[3 * o])
                b = _prmt(words[2], words[3], sel[3 * o + 1])
                v = _prmt(a, b, sel[3 * o + 2])
                c = d["dst_order"][out_dc[o]]
                for j in range(4):
                    key = (c, out_off[o] + j)
                    assert key not in seen
                    seen[key] = (v >> (8 * j)) & 0xFF
    # expected: every byte of every non-identity dst cluster in period 0
    ident_dst = {K["dst_clusters"][0] for K in d["components"] if K["identity"]}     # canonical indices
    count = 0
    for f, w in enumerate(widths):
        if cdst[f] in ident_dst:
            continue
        for r in range(32):
            for j in range(w):
                src_local = r * ss[f] + os_[f] + j
                dst_local = r * sd[f] + od[f] + j
                assert seen[(cdst[f], dst_local)] == tag(csrc[f], src_local), (f, r, j)
                count += 1
    assert count == len(seen)


def test_byte_group_plans_cover_every_byte():
    _check_byte_groups([1] * 24 + [8], [0] * 25, list(range(25)))          # 1-byte AoS -> SoA
    _check_byte_groups([1] * 24 + [8], list(range(25)), [0] * 25)          # 1-byte SoA -> AoS
    _check_byte_groups([2, 4, 6, 4] * 4, [0] * 16, list(range(16)))        # g = 2
    _check_byte_groups([1, 3, 4, 8] * 4, [0] * 16, list(range(16)))        # odd widths
    rng = random.Random(5)
    for _ in range(30):
        F = rng.randint(2, 10)
        widths = [rng.choice([1, 2, 3, 4, 5, 8]) for _ in range(F)]
        if all(w % 4 == 0 for w in widths):
            widths[0] = 1
        ls = [rng.randrange(F) for _ in range(F)]
        ld = [rng.randrange(F) for _ in range(F)]
        d = A.plan_describe(A.Layout(widths, ls), A.Layout(widths, ld))
        if d["unit"] < 4 and d["byte_groups"]:
            _check_byte_groups(widths, ls, ld)


# ---------------------------------------------------------------- generalised layouts (N4)

def _rand_general(rng, F):
    widths = [rng.choice([1, 2, 3, 4, 6, 8, 12]) for _ in range(F)]
    labels = [rng.randrange(F) for _ in range(F)]
    cb = {lab: rng.choice([1, 1, 2, 4, 8, 16, 32]) for lab in set(labels)}
    return widths, labels, [cb[l] for l in labels], rng.random() < 0.5


def test_generalised_descriptor_matches_oracle():
    rng = random.Random(13)
    for _ in range(200):
        F = rng.randint(1, 10)
        widths, labels, blocks, aligned = _rand_general(rng, F)
        L = A.Layout(widths, labels, blocks=blocks, aligned=aligned)
        for n in (0, 1, 7, 33, 1000):
            d = O.field_addresses_ex(widths, labels, n, blocks, aligned)
            assert L.nbytes(n) == d["total"]
            for f in range(F):
                assert L.field_address_ex(f, n) == (d["base"][f], d["stride"][f], d["offset"][f], d["block"][f])
        s = L.to_string()
        names = [f"f{i}" for i in range(F)]
        assert A.Layout.from_string(s, names, widths).to_string() == s
    with pytest.raises(A.AdhaError):
        A.Layout([4, 4], [0, 0], blocks=[2, 4])          # one block per cluster
    with pytest.raises(A.AdhaError):
        A.Layout([4], [0], blocks=[3])
    names = ["a", "b", "c"]
    L = A.Layout.from_string("aligned:{a,b}@8|{c}", names, [1, 4, 2])
    assert L.field_address_ex(1, 10) == (0, 8, 4, 8) and L.to_string() == "aligned:{a,b}@8|{c}"


def _gen_plan_checks(widths, ls, bs, als, ld, bd, ald):
    """Unit-mode plan table of generalised layouts: every unit of one period moved exactly once,
    to the generalised element address; padding units never written."""
    Ls = A.Layout(widths, ls, blocks=bs, aligned=als)
    Ld = A.Layout(widths, ld, blocks=bd, aligned=ald)
    d = A.plan_describe(Ls, Ld)
    assert d["tiled"], d
    if d["byte_groups"]:
        return d
    g = d["unit"]
    from tests.test_oracle_remap import clusters_in_order
    cs, cd = clusters_in_order(ls), clusters_in_order(ld)
    csrc = {f: k for k, c in enumerate(cs) for f in c}
    cdst = {f: k for k, c in enumerate(cd) for f in c}
    S = O.field_addresses_ex(widths, ls, 32, bs, als)
    D = O.field_addresses_ex(widths, ld, 32, bd, ald)
    ent_in, ent_out = np.array(d["ent_in"]), np.array(d["ent_out"])
    ent_sc, ent_dc = np.array(d["ent_sc"]), np.array(d["ent_dc"])
    for K in d["components"]:
        if K["identity"]:
            continue
        lo, hi = 32 * K["instr_base"], 32 * (K["instr_base"] + K["n_instr"])
        exp = set()
        for r in range(32):
            for f in K["fields"]:
                for j in range(0, widths[f], g):
                    a_s = O.addr_ex(S, f, r) - int(S["base"][f]) + j
                    a_d = O.addr_ex(D, f, r) - int(D["base"][f]) + j
                    exp.add((a_s // g, a_d // g, csrc[f], cdst[f]))
        got = {(int(a), int(b), d["src_order"][c], d["dst_order"][e])
               for a, b, c, e in zip(ent_in[lo:hi], ent_out[lo:hi], ent_sc[lo:hi], ent_dc[lo:hi])}
        assert got == exp
    return d


def test_generalised_plan_tables():
    _gen_plan_checks([4] * 8, [0] * 8, [1] * 8, False, [0] * 8, [8] * 8, False)            # AoS -> AoSoA8
    _gen_plan_checks([4, 8, 4, 4], [0] * 4, [32] * 4, False, list(range(4)), [1] * 4, False)  # AoSoA32 -> SoA
    _gen_plan_checks([4, 8, 4], list(range(3)), [1] * 3, False, [0] * 3, [1] * 3, True)      # SoA -> aligned AoS
    rng = random.Random(17)
    for _ in range(40):
        F = rng.randint(1, 8)
        widths = [rng.choice([4, 8, 12]) for _ in range(F)]
        w2, ls, bs, als = _rand_general(rng, F)
        _, ld, bd, ald = _rand_general(rng, F)
        _gen_plan_checks(widths, ls, bs, als, ld, bd, ald)


def test_byte_group_packing_is_phase_aware():
    """Byte-group plans are packed for every period phase (a word's bank moves by 8*stride words
    per period): simulated shared-memory wavefronts per load/store instruction stay near 1-2, not
    the 3-4.5 a phase-0-only packing gave (tools/bank_sim.py); plans stay exact (host simulation)."""
    from tools.bank_sim import CASES, make, simulate
    for name, (w, a, b) in CASES.items():
        r = simulate(make(w, a), make(w, b))
        assert r is not None, name
        assert r["ld_wf"] / r["ld_instr"] <= 2.5 and r["st_wf"] / r["st_instr"] <= 3.0, (name, r)
    for w in ([2, 4, 6, 4] * 4, [1] * 24 + [8]):
        F = len(w)
        _check_byte_groups(w, [0] * F, list(range(F)))
        _check_byte_groups(w, list(range(F)), [0] * F)


def test_package_refuses_to_import_without_its_library(tmp_path):
    """No fallback: a copy of the binding next to no libadha.so raises ImportError on import."""
    import shutil
    import subprocess
    import sys
    pkg = tmp_path / "adha_copy"
    pkg.mkdir()
    shutil.copy(os.path.join(ROOT, "paper_1407_4859_b200", "__init__.py"), pkg / "__init__.py")
    out = subprocess.run([sys.executable, "-c", "import adha_copy"], cwd=tmp_path, capture_output=True, text=True)
    assert out.returncode != 0 and "ImportError" in out.stderr and "no fallback" in out.stderr


def test_status_strings_and_version():
    """adha_status_string names every status the header declares (and never returns NULL);
    adha_version is MAJOR*10000 + MINOR*100 + PATCH with MAJOR >= 1 or MINOR >= 1."""
    import re
    text = open(os.path.join(ROOT, "include", "adha.h")).read()
    codes = {int(v): k for k, v in re.findall(r"(ADHA_(?:OK|ERR_[A-Z_]+)) = (\d+)", text)}
    assert len(codes) == 12
    for v, k in codes.items():
        assert A._lib.adha_status_string(v).decode() == k == A.STATUS[v]
    assert A._lib.adha_status_string(999) is not None and A._lib.adha_status_string(-1) is not None
    v = A.version()
    assert v >= 100 and 0 <= v % 100 < 100


# ----------------------------------------------------------------------------- in-place plan (host only)

def _ip(widths, ls, ld, n):
    return A.InplacePlan(A.Layout(widths, ls), A.Layout(widths, ld), n)


@pytest.fixture
def permute_mode(monkeypatch):
    monkeypatch.setenv("ADHA_INPLACE_STAGED_BYTES", "0")


def test_inplace_plan_counts_and_sizes(permute_mode):
    """Host plan of adha_remap_inplace: the buffer needs max(bytes(Ls), bytes(Ld)) (not the sum);
    every body slot of the src layout is content; the permutation closes on src u dst slots
    (moved + fixed = content + junk); the slot size divides every region base of both layouts."""
    widths = [8 if i % 4 == 3 else 4 for i in range(16)]
    rng = random.Random(5)
    for n in (0, 1, 63, 64, 65, 1000, 10_000_000, 12345):
        for ls, ld in [([0] * 16, list(range(16))), (list(range(16)), [0] * 16),
                       ([rng.randrange(5) for _ in range(16)], [rng.randrange(7) for _ in range(16)])]:
            p = _ip(widths, ls, ld, n)
            d = p.describe()
            bs = O.layout_bytes(widths, ls, n)
            bd = O.layout_bytes(widths, ld, n)
            assert p.buffer_bytes == max(bs, bd) == d["buffer_bytes"]
            S, T, u = d["slot_bytes"], d["T"], d["unit"]
            assert u == 4 and S == T * u and S in (256, 512, 1024, 2048, 4096)
            assert d["body_tiles"] == n // T and d["tail_records"] == n % T
            assert d["content_slots"] == (n // T) * 80 // u
            assert d["moved_slots"] + d["fixed_slots"] == d["content_slots"] + d["junk_slots"]
            for lab in (ls, ld):
                base, _, _, _ = O.field_addresses(widths, lab, n)
                assert all(int(b) % S == 0 for b in base)
            assert p.workspace_bytes >= d["segments"] * S


def test_inplace_plan_identity_and_moved_subset(permute_mode):
    widths = [4] * 9
    aosv, soa = [0, 0, 0, 1, 2, 3, 4, 5, 6], list(range(9))
    d = _ip(widths, aosv, aosv, 1 << 16).describe()
    assert d["moved_slots"] == 0 and d["pre_clusters"] == 0 and d["post_clusters"] == 0
    d = _ip(widths, aosv, soa, 1 << 20).describe()     # PAPER.md:113 AoSV -> SoA: only V1..V3 move
    S = d["slot_bytes"]
    # V1..V3's slots move (a couple are fixed points, e.g. V1 of tile 0); the six singletons don't
    assert 0 < d["moved_slots"] <= 3 * 4 * (1 << 20) // S
    assert d["moved_slots"] + d["fixed_slots"] == 9 * 4 * (1 << 20) // S


def test_inplace_plan_staged_mode(monkeypatch):
    """Small buffers (<= ADHA_INPLACE_STAGED_BYTES, 16 MB by default) go through the workspace:
    the workspace holds the dst layout, no slot tables."""
    monkeypatch.delenv("ADHA_INPLACE_STAGED_BYTES", raising=False)
    w = [8 if i % 4 == 3 else 4 for i in range(16)]
    p = _ip(w, [0] * 16, list(range(16)), 100_000)
    d = p.describe()
    assert d["mode"] == "staged" and d["moved_slots"] == 0 and d["segments"] == 0
    assert p.workspace_bytes >= O.layout_bytes(w, list(range(16)), 100_000)
    assert _ip(w, [0] * 16, list(range(16)), 1_000_000).describe()["mode"] == "permute"
    monkeypatch.setenv("ADHA_INPLACE_STAGED_BYTES", "0")
    assert _ip(w, [0] * 16, list(range(16)), 100_000).describe()["mode"] == "permute"


def test_inplace_plan_errors(permute_mode):
    w = [4, 4, 8]
    with pytest.raises(A.AdhaError) as e:
        _ip(w, [0, 0, 0], [0, 1, 2], -1)
    assert e.value.name == "ADHA_ERR_INVALID_ARG"
    with pytest.raises(A.AdhaError) as e:
        A.InplacePlan(A.Layout(w, [0, 0, 0]), A.Layout([4, 4, 4], [0, 1, 2]), 10)
    assert e.value.name == "ADHA_ERR_LAYOUT_MISMATCH"
    with pytest.raises(A.AdhaError) as e:
        A.InplacePlan(A.Layout(w, [0, 0, 0], aligned=True), A.Layout(w, [0, 1, 2]), 10)
    assert e.value.name == "ADHA_ERR_UNSUPPORTED"
    with pytest.raises(A.AdhaError) as e:
        A.InplacePlan(A.Layout(w, [0, 0, 0], blocks=[8, 8, 8]), A.Layout(w, [0, 1, 2]), 10)
    assert e.value.name == "ADHA_ERR_UNSUPPORTED"
    # a record too wide for a 256 / u record tile in shared memory
    with pytest.raises(A.AdhaError) as e:
        _ip([1] * 1000, [0] * 1000, list(range(1000)), 10)
    assert e.value.name == "ADHA_ERR_UNSUPPORTED"


def test_inplace_plan_runs_skip_tile_passes(permute_mode):
    """Runs (fields contiguous in both cluster records) are moved as blocks: a cluster that is one
    run needs no tile rewrite.  K-Means 4xAoS8 -> AoS rewrites only the dst AoS tiles; Medical
    AoS -> AoSV rewrites only the src AoS tiles ({V1,V2,V3} is one run on both sides); SoA -> AoS
    has nothing to rewrite on the src side; identical hybrids nothing at all."""
    km = [4] * 32
    aos8 = [f // 8 for f in range(32)]
    d = _ip(km, aos8, [0] * 32, 1 << 20).describe()
    assert (d["pre_clusters"], d["post_clusters"]) == (0, 1)
    d = _ip(km, [0] * 32, aos8, 1 << 20).describe()
    assert (d["pre_clusters"], d["post_clusters"]) == (1, 0)
    med = [4] * 9
    d = _ip(med, [0] * 9, [0, 0, 0, 1, 2, 3, 4, 5, 6], 1 << 20).describe()
    assert (d["pre_clusters"], d["post_clusters"]) == (1, 0)
    w = [8 if i % 4 == 3 else 4 for i in range(16)]
    d = _ip(w, list(range(16)), [0] * 16, 10_000_000).describe()
    assert (d["pre_clusters"], d["post_clusters"]) == (0, 1)
    # a hybrid whose clusters interleave: {f0,f2} -> {f0,f1,f2} splits into the runs f0 | f2
    d = _ip([4, 4, 4], [0, 1, 0], [0, 0, 0], 4096).describe()
    assert (d["pre_clusters"], d["post_clusters"]) == (1, 1)


@pytest.mark.parametrize("shape", ["C2", "C3", "C3-back", "Medical AoSV->SoA"])
def test_inplace_plan_segments_verified_large(shape, monkeypatch):
    """The parallel cycle decomposition (cut walks advanced 16 at a time per host thread, placed
    by prefix sums; uncut cycles by their smallest slot) checked by the library itself against the
    permutation (ADHA_IP_VERIFY=1) at sizes with hundreds of thousands of slots."""
    monkeypatch.setenv("ADHA_INPLACE_STAGED_BYTES", "0")
    monkeypatch.setenv("ADHA_IP_VERIFY", "1")
    from tests.conftest import golden
    from oracle import planner as P
    w16 = [8 if i % 4 == 3 else 4 for i in range(16)]
    w64 = [8 if i % 4 == 3 else 4 for i in range(64)]
    hyb = P.parse_layout(golden("expected.json")["c3_hybrid"]["value"], {f"f{i}": i for i in range(64)})
    c3 = [0] * 64
    for c, cl in enumerate(hyb):
        for nm in cl:
            c3[int(nm[1:])] = c
    cases = {"C2": (w16, [0] * 16, list(range(16)), 2_000_003), "C3": (w64, list(range(64)), c3, 1_000_003),
             "C3-back": (w64, c3, list(range(64)), 1_000_003),
             "Medical AoSV->SoA": ([4] * 9, [0, 0, 0, 1, 2, 3, 4, 5, 6], list(range(9)), 3_000_001)}
    widths, ls, ld, n = cases[shape]
    d = _ip(widths, ls, ld, n).describe()
    assert d["moved_slots"] > 0 and d["segments"] * 64 >= d["moved_slots"]


def test_remap_chain_route(monkeypatch):
    """adha_remap_chain's routing (host only): C1's tiny chain -> one fused direct launch; with the
    fused tiled chain opted in (ADHA_CHAIN_TILED_BYTES), C4 at 2 GiB and P1/P2 at their bench sizes
    -> one fused tiled launch; a mid-size chain -> one remap per hop; AoSoA-blocked layouts, and
    the default (fused tiled chain off) -> per hop."""
    import os
    monkeypatch.setenv("ADHA_CHAIN_TILED_BYTES", str(64 << 20))
    w9 = [4] * 9
    c4 = [A.Layout(w9, l) for l in ([0] * 9, [0, 0, 0, 1, 2, 3, 4, 5, 6], list(range(9)), [0] * 9)]
    xyz = [A.Layout([4, 4, 4], l) for l in ([0, 0, 0], [0, 1, 2], [0, 0, 0])]
    assert A.remap_chain_route(xyz, 1024) == ("fused_small", 1)
    assert A.remap_chain_route(c4, 2 ** 31 // 36) == ("fused_tiled", 1)
    assert A.remap_chain_route(c4, 300_000) == ("per_hop", 3)
    p1 = [A.Layout(w9, l) for l in ([0] * 9, [0, 0, 0, 1, 2, 3, 4, 5, 6], list(range(9)))]
    assert A.remap_chain_route(p1, 256 ** 3) == ("fused_tiled", 1)
    w32 = [4] * 32
    p2 = [A.Layout(w32, l) for l in (list(range(32)), [i // 8 for i in range(32)], [0] * 32)]
    assert A.remap_chain_route(p2, 2 ** 23) == ("fused_tiled", 1)
    blk = [A.Layout(w9, [0] * 9, blocks=[8] * 9), A.Layout(w9, list(range(9))), A.Layout(w9, [0] * 9)]
    assert A.remap_chain_route(blk, 2 ** 31 // 36) == ("per_hop", 2)
    monkeypatch.delenv("ADHA_CHAIN_TILED_BYTES")
    assert A.remap_chain_route(c4, 2 ** 31 // 36) == ("per_hop", 3)
    assert os.environ.get("ADHA_CHAIN_TILED_BYTES") is None
    with pytest.raises(A.AdhaError):
        A.remap_chain_route([c4[0], A.Layout([4] * 8, [0] * 8)], 10)


def test_routing_thresholds(monkeypatch):
    """The routing the plan reports (remap.cu direct_bytes / merge_bytes, read by adha_remap_plan_describe):
    the direct kernel up to 2 MB of payload, up to 8 MB for plans of >= 16 components (C3's 24); the merged
    plan for multi-component remaps up to a limit set by the src cluster count and identity components;
    ADHA_SMALL_BYTES / ADHA_MERGE_BYTES override them."""
    monkeypatch.delenv("ADHA_SMALL_BYTES", raising=False)
    monkeypatch.delenv("ADHA_MERGE_BYTES", raising=False)
    w16 = [8 if i % 4 == 3 else 4 for i in range(16)]
    d = A.plan_describe(A.Layout.aos(w16), A.Layout.soa(w16))
    assert d["direct_bytes"] == 2 << 20 and d["merge_bytes"] == 0
    w64 = [8 if i % 4 == 3 else 4 for i in range(64)]
    c3 = [0] * 26 + [1] * 10 + [2] * 4 + [3] * 3 + [4, 5, 6, 7, 4] + list(range(8, 8 + 16))
    d = A.plan_describe(A.Layout(w64, list(range(64))), A.Layout(w64, c3))
    assert len(d["components"]) >= 16
    assert d["direct_bytes"] == 8 << 20 and d["merge_bytes"] == 64 << 20
    # merged-plan limit: none for <= 8 src clusters with identity components (Medical AoSV -> SoA),
    # 128 MB for <= 32 src clusters without (K-Means 4xAoS8 -> SoA), 64 MB above 32 (C3 above)
    w9 = [4] * 9
    d = A.plan_describe(A.Layout(w9, [0, 0, 0, 1, 2, 3, 4, 5, 6]), A.Layout(w9, list(range(9))))
    assert any(c["identity"] for c in d["components"]) and d["merge_bytes"] == 2 ** 64 - 1
    w32 = [4] * 32
    d = A.plan_describe(A.Layout(w32, [f // 8 for f in range(32)]), A.Layout(w32, list(range(32))))
    assert not any(c["identity"] for c in d["components"]) and d["merge_bytes"] == 128 << 20
    monkeypatch.setenv("ADHA_SMALL_BYTES", "12345")
    assert A.plan_describe(A.Layout.aos(w16), A.Layout.soa(w16))["direct_bytes"] == 12345
