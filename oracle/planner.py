"""Plain Python oracle for ADHA's two planner passes, ODS and PDL.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Shares no code with the
C++ planner in paper_1407_4859_b200/csrc/.

Every function follows the SPEC.md operation it names, step by step, in the
paper's order (PAPER.md 2 "Overall Framework"):
  ODS   build_affinity_graph -> greedy_cluster -> ods
  PDL   merge_sections, exec_cost, remap_cost, combine_loss,
                         build_run_graph, shortest_plan
  brute force            enumerate_layouts, brute_force_ods, brute_force_plan
                          -- independent exhaustive searches
                         used to pin the greedy / shortest-path results.
Readings: Q11-Q14 (affinity = trip*freq-weighted
co-occurrence, sign rule, Kruskal with inclusive cap, tie-break), Q18 (run
graph over contiguous runs), Q19 (remap cost = bytes/bandwidth + overhead).

Parity notes: exec_cost's model branch is SPEC.md's own ("model
branch invented"); its constants (line bytes and time, throughput, penalty) are
architecture INPUTS, not outputs.  The formula is pinned by SPEC.md:210-212's
worked examples (3000 vs 1000 line times, linearity, partition invariance of
streaming bytes) and by properties of the definition (coalescing penalty ratio,
layout-independent compute term; tests/test_oracle_planner.py); the paper's own
absolute timings (Tables 3-4) are out of scope.
"""
from __future__ import annotations

import itertools
import json
from dataclasses import dataclass, field
from typing import Dict, FrozenSet, List, Optional, Sequence, Tuple


class PlannerError(ValueError):
    """Rejected input (SPEC.md 'errors: ... rejected input')."""


# ----------------------------------------------------------------------------- data model
# SPEC.md:25-63 [TYPE]s


@dataclass(frozen=True)
class Field:
    name: str
    elem_bytes: int
    decl_index: int


@dataclass(frozen=True)
class AccessGroup:
    fields: Tuple[str, ...]
    freq: float
    pattern: str            # "streaming" | "irregular"
    ops: float = 0.0


@dataclass(frozen=True)
class Section:
    id: str
    trip_count: float
    groups: Tuple[AccessGroup, ...]
    allowed_devices: Tuple[str, ...]

    def fields(self) -> FrozenSet[str]:
        out = set()
        for g in self.groups:
            out.update(g.fields)
        return frozenset(out)


@dataclass(frozen=True)
class Device:
    name: str
    line_bytes: int
    line_time_ns: float
    throughput_ops_per_ns: float
    coalescing: bool
    stream_cluster_penalty: float
    cluster_capacity_bytes: int


@dataclass(frozen=True)
class Link:
    src: str
    dst: str
    bandwidth_bytes_per_ns: float
    latency_ns: float


@dataclass
class Architecture:
    devices: List[Device]
    links: List[Link]
    same_device_remap_bandwidth_bytes_per_ns: float
    remap_fixed_overhead_ns: float

    def device(self, name: str) -> Device:
        for d in self.devices:
            if d.name == name:
                return d
        raise PlannerError(f"unknown device {name!r}")


@dataclass
class Program:
    name: str
    record_count: int
    fields: List[Field]
    sections: List[Section]
    order: List[str]

    def field(self, name: str) -> Field:
        for f in self.fields:
            if f.name == name:
                return f
        raise PlannerError(f"undeclared field {name!r}")

    def section(self, sid: str) -> Section:
        for s in self.sections:
            if s.id == sid:
                return s
        raise PlannerError(f"unknown section {sid!r}")

    def elem_bytes(self) -> Dict[str, int]:
        return {f.name: f.elem_bytes for f in self.fields}

    def decl(self) -> Dict[str, int]:
        return {f.name: f.decl_index for f in self.fields}


Profile = Dict[Tuple[str, str, str], float]     # (section id, device, canonical layout) -> ns

# A Layout is a tuple of clusters, each a tuple of field names, in canonical form.
Layout = Tuple[Tuple[str, ...], ...]


# ----------------------------------------------------------------------------- JSON I/O
# SPEC.md:100 (UTF-8 JSON, exact spellings), 248 (profile), 313 (plan), 416 (schema_version)


def program_from_json(obj) -> Program:
    if isinstance(obj, str):
        obj = json.loads(obj)
    fields = [Field(f["name"], int(f["elem_bytes"]), i) for i, f in enumerate(obj["fields"])]
    sections = []
    for s in obj["sections"]:
        groups = tuple(AccessGroup(tuple(g["fields"]), float(g["freq"]), g["pattern"],
                                   float(g.get("ops", 0.0))) for g in s["groups"])
        sections.append(Section(s["id"], float(s["trip_count"]), groups, tuple(s["allowed_devices"])))
    order = list(obj.get("order", [s.id for s in sections]))
    return Program(obj.get("name", "program"), int(obj["record_count"]), fields, sections, order)


def arch_from_json(obj) -> Architecture:
    if isinstance(obj, str):
        obj = json.loads(obj)
    devs = [Device(d["name"], int(d["line_bytes"]), float(d["line_time_ns"]),
                   float(d["throughput_ops_per_ns"]), bool(d["coalescing"]),
                   float(d.get("stream_cluster_penalty", 2.0)), int(d["cluster_capacity_bytes"]))
            for d in obj["devices"]]
    links = [Link(l["from"], l["to"], float(l["bandwidth_bytes_per_ns"]), float(l["latency_ns"]))
             for l in obj.get("links", [])]
    return Architecture(devs, links, float(obj["same_device_remap_bandwidth_bytes_per_ns"]),
                        float(obj["remap_fixed_overhead_ns"]))


def profile_from_json(obj) -> Profile:
    if obj is None:
        return {}
    if isinstance(obj, str):
        obj = json.loads(obj)
    entries = obj["entries"] if isinstance(obj, dict) else obj
    return {(e["section"], e["device"], e["layout"]): float(e["time_ns"]) for e in entries}


# ----------------------------------------------------------------------------- layouts
# SPEC.md:55-58, 76-84 [OP] canonical_layout_string


def canonical(clusters: Sequence[Sequence[str]], decl: Dict[str, int]) -> Layout:
    """Fields in a cluster by decl_index; clusters by minimum decl_index."""
    cs = [tuple(sorted(c, key=lambda n: decl[n])) for c in clusters if len(c)]
    cs.sort(key=lambda c: decl[c[0]])
    return tuple(cs)


def layout_string(l: Layout) -> str:
    """'{f,g,h}|{x}|{y}' -- no whitespace."""
    return "|".join("{" + ",".join(c) + "}" for c in l)


def parse_layout(text: str, decl: Dict[str, int]) -> Layout:
    """Inverse of layout_string; also accepts the paper's Table-2 notation
    'V1,V2,{U1,U2,U3},S' where bare names are singletons."""
    clusters: List[List[str]] = []
    i, n = 0, len(text)
    while i < n:
        ch = text[i]
        if ch in ",| \t":
            i += 1
            continue
        if ch == "{":
            j = text.index("}", i)
            names = [x.strip() for x in text[i + 1:j].split(",") if x.strip()]
            clusters.append(names)
            i = j + 1
        else:
            j = i
            while j < n and text[j] not in ",|{} \t":
                j += 1
            clusters.append([text[i:j]])
            i = j
    seen = [x for c in clusters for x in c]
    if len(seen) != len(set(seen)) or set(seen) != set(decl):
        raise PlannerError(f"layout {text!r} is not a partition of the fields")
    return canonical(clusters, decl)


def cluster_of(l: Layout, name: str) -> Tuple[str, ...]:
    for c in l:
        if name in c:
            return c
    raise PlannerError(f"field {name!r} not in layout")


def cluster_bytes(c: Sequence[str], eb: Dict[str, int]) -> int:
    return sum(eb[n] for n in c)


# ----------------------------------------------------------------------------- ODS
# PAPER.md:40-47


def _w(pattern: str, d: Device) -> float:
    """w_d(pattern): irregular +1; streaming +1 on non-coalescing, -1 on coalescing."""
    if pattern == "irregular":
        return 1.0
    if pattern == "streaming":
        return -1.0 if d.coalescing else 1.0
    raise PlannerError(f"bad pattern {pattern!r}")


def build_affinity_graph(s: Section, d: Device, decl: Dict[str, int]
                         ) -> Tuple[List[str], Dict[Tuple[str, str], float]]:
    """Nodes = fields(s); weight(f,g) = sum over groups G with {f,g} in G of
    trip * freq * w_d(pattern) ("number of common occurrences")."""
    if d.name not in s.allowed_devices:
        raise PlannerError(f"device {d.name!r} not allowed for section {s.id!r}")
    nodes = sorted(s.fields(), key=lambda n: decl[n])
    weights: Dict[Tuple[str, str], float] = {}
    for a_i, a in enumerate(nodes):
        for b in nodes[a_i + 1:]:
            wsum = 0.0
            hit = False
            for g in s.groups:
                if a in g.fields and b in g.fields:
                    wsum += s.trip_count * g.freq * _w(g.pattern, d)
                    hit = True
            if hit:
                weights[(a, b)] = wsum
    return nodes, weights


def greedy_cluster(nodes: Sequence[str], weights: Dict[Tuple[str, str], float], d: Device,
                   eb: Dict[str, int], decl: Dict[str, int]) -> Layout:
    """Kruskal greedy: start from singletons; edges sorted by
    (weight desc, min decl asc, max decl asc); merge the endpoint clusters when weight > 0,
    they differ and the merged bytes <= capacity."""
    for n in nodes:
        if eb[n] > d.cluster_capacity_bytes:
            raise PlannerError(f"field {n!r} ({eb[n]} B) exceeds capacity {d.cluster_capacity_bytes}")
    cl: Dict[str, int] = {n: i for i, n in enumerate(nodes)}
    members: Dict[int, List[str]] = {i: [n] for i, n in enumerate(nodes)}

    def key(e):
        (a, b), w = e
        lo, hi = sorted((decl[a], decl[b]))
        return (-w, lo, hi)

    for (a, b), w in sorted(weights.items(), key=key):
        if not w > 0:
            continue
        ca, cb = cl[a], cl[b]
        if ca == cb:
            continue
        if cluster_bytes(members[ca], eb) + cluster_bytes(members[cb], eb) > d.cluster_capacity_bytes:
            continue
        for n in members[cb]:
            cl[n] = ca
        members[ca].extend(members.pop(cb))
    return canonical(list(members.values()), decl)


def ods(s: Section, d: Device, p: Program) -> Layout:
    """ODS = greedy_cluster(build_affinity_graph(s, d)); untouched program fields become
    singletons."""
    decl, eb = p.decl(), p.elem_bytes()
    nodes, weights = build_affinity_graph(s, d, decl)
    l = greedy_cluster(nodes, weights, d, eb, decl)
    rest = [(f.name,) for f in p.fields if f.name not in s.fields()]
    return canonical(list(l) + rest, decl)


def merge_sections(ss: Sequence[Section]) -> Section:
    """Joined id, trip 1, groups concatenated with freq scaled by member trip, devices
    intersected."""
    if not ss:
        raise PlannerError("merge of no sections")
    groups = []
    for s in ss:
        for g in s.groups:
            groups.append(AccessGroup(g.fields, s.trip_count * g.freq, g.pattern, g.ops))
    allowed = [d for d in ss[0].allowed_devices if all(d in s.allowed_devices for s in ss[1:])]
    if not allowed:
        raise PlannerError("merged sections share no device")
    return Section("+".join(s.id for s in ss), 1.0, tuple(groups), tuple(allowed))


# ----------------------------------------------------------------------------- cost model
# SPEC.md:201-232


def exec_cost(s: Section, l: Layout, d: Device, p: Program, prof: Optional[Profile] = None
              ) -> Tuple[float, float, float, str]:
    """(memory_ns, compute_ns, total_ns, source).  Profile first (PAPER.md:59-60 'tuning
    profile'); else the analytic model of SPEC.md:205-207 (its constants are architecture inputs;
    pinned by SPEC.md:210-212's examples and the tests' invariants)."""
    covered = sorted(x for c in l for x in c)
    if covered != sorted(f.name for f in p.fields):
        raise PlannerError("layout does not span the program fields")
    if prof:
        key = (s.id, d.name, layout_string(l))
        if key in prof:
            return 0.0, 0.0, prof[key], "profile"
    eb = p.elem_bytes()
    memory = 0.0
    compute = 0.0
    for g in s.groups:
        inner = 0.0
        for c in l:
            if not any(x in g.fields for x in c):
                continue
            if g.pattern == "streaming":
                lc = cluster_bytes(c, eb) / d.line_bytes
                if d.coalescing and len(c) > 1:
                    lc = lc * d.stream_cluster_penalty
            else:
                lc = 1.0
            inner += lc * d.line_time_ns
        memory += s.trip_count * g.freq * inner
        compute += s.trip_count * g.freq * g.ops / d.throughput_ops_per_ns
    return memory, compute, memory + compute, "model"


def _link(a: Architecture, d1: str, d2: str) -> Link:
    for l in a.links:
        if (l.src, l.dst) in ((d1, d2), (d2, d1)):
            return l
    raise PlannerError(f"no link between {d1!r} and {d2!r}")


def moved_fields(l1: Layout, d1: str, l2: Layout, d2: str, common: FrozenSet[str]) -> List[str]:
    """same device -> fields whose cluster signature restricted to `common`
    differs; device change -> every common field."""
    if d1 != d2:
        return sorted(common)
    out = []
    for f in common:
        s1 = frozenset(cluster_of(l1, f)) & common
        s2 = frozenset(cluster_of(l2, f)) & common
        if s1 != s2:
            out.append(f)
    return sorted(out)


def remap_cost(l1: Layout, d1: str, l2: Layout, d2: str, common: FrozenSet[str], p: Program,
               a: Architecture) -> Tuple[float, List[str]]:
    """Remap edge weight (PAPER.md:56-57 'based on the number of common fields'):
    bytes(moved) / bandwidth + overhead, 0 when nothing moves (reading Q19)."""
    moved = moved_fields(l1, d1, l2, d2, common)
    eb = p.elem_bytes()
    nbytes = 0.0
    for f in moved:
        nbytes += float(p.record_count) * eb[f]
    if nbytes == 0:
        return 0.0, moved
    if d1 == d2:
        return nbytes / a.same_device_remap_bandwidth_bytes_per_ns + a.remap_fixed_overhead_ns, moved
    lk = _link(a, d1, d2)
    return nbytes / lk.bandwidth_bytes_per_ns + lk.latency_ns, moved


def combine_loss(s1: Section, s2: Section, d: Device, p: Program, prof: Optional[Profile] = None,
                 ods_fn=None) -> float:
    """loss from combining two sections under the merged ODS layout:
    L_m = ods(merge(s1, s2)); loss = [exec(s1, L_m) + exec(s2, L_m)] - [exec(s1, ods(s1)) +
    exec(s2, ods(s2))].  ods_fn(s, d, p) -> Layout replaces the greedy ODS (SPEC.md:237 states
    loss >= 0 when it is the optimal, brute-force ODS)."""
    ods_fn = ods if ods_fn is None else ods_fn
    lm = ods_fn(merge_sections([s1, s2]), d, p)
    merged = exec_cost(s1, lm, d, p, prof)[2] + exec_cost(s2, lm, d, p, prof)[2]
    separate = (exec_cost(s1, ods_fn(s1, d, p), d, p, prof)[2]
                + exec_cost(s2, ods_fn(s2, d, p), d, p, prof)[2])
    return merged - separate


# ----------------------------------------------------------------------------- PDL
# PAPER.md:49-61


@dataclass
class RunNode:
    begin: int
    end: int
    device: str
    layout: Layout
    exec_ns: float
    fields: FrozenSet[str] = field(default_factory=frozenset)


def run_node(p: Program, a: Architecture, b: int, e: int, dname: str, prof: Optional[Profile]
             ) -> RunNode:
    secs = [p.section(sid) for sid in p.order[b:e + 1]]
    d = a.device(dname)
    layout = ods(merge_sections(secs), d, p)
    ex = 0.0
    for s in secs:
        ex += exec_cost(s, layout, d, p, prof)[2]
    flds = frozenset().union(*[s.fields() for s in secs])
    return RunNode(b, e, dname, layout, ex, flds)


def build_run_graph(p: Program, a: Architecture, prof: Optional[Profile] = None) -> List[RunNode]:
    """Nodes (b, e, d) for all contiguous runs and devices allowed by every member
    (SPEC.md:273).  Edges are implicit: run (b',e') -> run (b,e) iff e' = b-1."""
    k = len(p.order)
    nodes = []
    for b in range(k):
        for e in range(b, k):
            secs = [p.section(sid) for sid in p.order[b:e + 1]]
            for d in a.devices:
                if all(d.name in s.allowed_devices for s in secs):
                    nodes.append(run_node(p, a, b, e, d.name, prof))
    return nodes


@dataclass
class Plan:
    runs: List[RunNode]
    remaps: List[Tuple[int, List[str], float]]      # (boundary index, moved, cost)
    total_ns: float


def _plan_key(cost: float, runs: Sequence[RunNode]):
    return (cost, len(runs), tuple((r.device, r.begin) for r in runs))


def shortest_plan(p: Program, a: Architecture, prof: Optional[Profile] = None) -> Plan:
    """Shortest SRC->SNK path over the run graph in topological order (by end index);
    ties: fewer runs, then lexicographically smaller (device, begin) sequence."""
    nodes = build_run_graph(p, a, prof)
    k = len(p.order)
    if not any(n.begin == 0 for n in nodes):
        raise PlannerError("no device can run the first section")
    best: Dict[int, Tuple[float, List[RunNode]]] = {}
    order = sorted(range(len(nodes)), key=lambda i: (nodes[i].end, nodes[i].begin))
    for i in order:
        n = nodes[i]
        cands = []
        if n.begin == 0:
            cands.append((n.exec_ns, [n]))
        for j, m in enumerate(nodes):
            if m.end == n.begin - 1 and j in best:
                rc, _ = remap_cost(m.layout, m.device, n.layout, n.device, m.fields & n.fields, p, a)
                cost = best[j][0] + (rc + n.exec_ns)
                cands.append((cost, best[j][1] + [n]))
        if cands:
            best[i] = min(cands, key=lambda c: _plan_key(c[0], c[1]))
    finals = [best[i] for i, n in enumerate(nodes) if n.end == k - 1 and i in best]
    if not finals:
        raise PlannerError("no plan covers the program")
    total, runs = min(finals, key=lambda c: _plan_key(c[0], c[1]))
    return _make_plan(p, a, runs, total)


def _make_plan(p: Program, a: Architecture, runs: List[RunNode], total: float) -> Plan:
    remaps = []
    for r1, r2 in zip(runs, runs[1:]):
        rc, moved = remap_cost(r1.layout, r1.device, r2.layout, r2.device, r1.fields & r2.fields, p, a)
        remaps.append((r2.begin, moved, rc))
    return Plan(runs, remaps, total)


def plan_to_json(plan: Plan, p: Program) -> dict:
    """SPEC.md:313 plan serialisation."""
    return {
        "schema_version": 1,
        "runs": [{"sections": p.order[r.begin:r.end + 1], "device": r.device,
                  "layout": layout_string(r.layout), "exec_ns": r.exec_ns} for r in plan.runs],
        "remaps": [{"boundary": b, "after": p.order[b - 1], "moved": moved, "cost_ns": c}
                   for b, moved, c in plan.remaps],
        "total_ns": plan.total_ns,
    }


# ----------------------------------------------------------------------------- brute force
# SPEC.md:332-359 [OP] enumerate_layouts, brute_force_ods, brute_force_plan


def enumerate_layouts(names: Sequence[str], eb: Dict[str, int], capacity: Optional[int],
                      decl: Dict[str, int]) -> List[Layout]:
    """Every set partition within the byte capacity, each once, canonical (guard: <= 12 fields)."""
    names = sorted(names, key=lambda n: decl[n])
    if len(names) > 12:
        raise PlannerError("enumerate_layouts guard: at most 12 fields (Bell(12) = 4,213,597)")
    out: List[Layout] = []

    def rec(i: int, blocks: List[List[str]]):
        if i == len(names):
            out.append(canonical(blocks, decl))
            return
        n = names[i]
        for blk in blocks:
            if capacity is None or cluster_bytes(blk, eb) + eb[n] <= capacity:
                blk.append(n)
                rec(i + 1, blocks)
                blk.pop()
        if capacity is None or eb[n] <= capacity:
            blocks.append([n])
            rec(i + 1, blocks)
            blocks.pop()

    rec(0, [])
    return out


def brute_force_ods(s: Section, d: Device, p: Program) -> Tuple[Layout, float]:
    """argmin over enumerate_layouts of the model exec_cost; ties by canonical string."""
    decl, eb = p.decl(), p.elem_bytes()
    best = None
    for l in enumerate_layouts([f.name for f in p.fields], eb, d.cluster_capacity_bytes, decl):
        c = exec_cost(s, l, d, p, None)[2]
        key = (c, layout_string(l))
        if best is None or key < best[0]:
            best = (key, l)
    return best[1], best[0][0]


def brute_force_plan(p: Program, a: Architecture, prof: Optional[Profile] = None) -> Plan:
    """Exhaustive minimum over all 2^(k-1) contiguous-run partitions x per-run devices
    (SPEC.md:354), run layouts from greedy ODS."""
    k = len(p.order)
    if k > 6:
        raise PlannerError("brute_force_plan guard: k <= 6")
    best = None
    for cuts in itertools.product([False, True], repeat=k - 1):
        bounds, b = [], 0
        for i, c in enumerate(cuts):
            if c:
                bounds.append((b, i))
                b = i + 1
        bounds.append((b, k - 1))
        choices = []
        for (b, e) in bounds:
            secs = [p.section(sid) for sid in p.order[b:e + 1]]
            choices.append([d.name for d in a.devices if all(d.name in s.allowed_devices for s in secs)])
        for devs in itertools.product(*choices):
            runs = [run_node(p, a, b, e, dn, prof) for (b, e), dn in zip(bounds, devs)]
            total = runs[0].exec_ns
            for r1, r2 in zip(runs, runs[1:]):
                rc, _ = remap_cost(r1.layout, r1.device, r2.layout, r2.device, r1.fields & r2.fields, p, a)
                total = total + (rc + r2.exec_ns)
            key = _plan_key(total, runs)
            if best is None or key < best[0]:
                best = (key, runs, total)
    if best is None:
        raise PlannerError("no feasible plan")
    return _make_plan(p, a, best[1], best[2])
