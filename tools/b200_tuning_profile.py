"""Measure a B200 tuning profile and run PDL on it ("we provide a
tuning profile of the execution times").

For the program's run graph (adha_plan_candidates) every (section, device, layout) triple is timed
on this B200 with the synthetic consumer kernel adha_section_run reading records through that
layout: a streaming group is one streaming pass over the N records with the group's fields, an
irregular group of frequency q is q*N gathers at seeded random record indices.  The remap edge
bandwidth is the measured adha_remap_regions rate of the Medical AoSV -> SoA moved subset
({V1,V2,V3}) and the fixed overhead is measured at small N.  The profile and the
measured architecture are written as JSON; PDL (adha_plan_pdl) is run on them and, for contrast,
on the analytic model alone.

    python tools/b200_tuning_profile.py [program.json] [out.json]
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import paper_1407_4859_b200 as A  # noqa: E402
from adha_inputs import random_bytes  # noqa: E402


def timed(fn, calls=20, reps=3):
    """GPU time of one call of fn in ns: `calls` back-to-back calls captured in one CUDA graph,
    replayed `reps` times between events (the events bracket only device work: no ctypes
    marshalling or launch latency on an idle stream); median over replays / calls.  Falls back to
    `calls` back-to-back enqueues behind a warm-up call when fn cannot be captured."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    ts = []
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(calls):
                fn()
        g.replay()
        torch.cuda.synchronize()
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e6 / calls)
    except RuntimeError:
        torch.cuda.synchronize()
        for _ in range(reps):
            fn()                                   # keeps the stream busy while the rest is enqueued
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(calls):
                fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e6 / calls)
    return statistics.median(ts)


def main():
    prog_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "tests/golden/medical_b200_program.json")
    out_path = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out/b200_tuning_profile.json")
    prog = json.load(open(prog_path))
    arch = json.load(open(os.path.join(ROOT, "tests/golden/b200_arch.json")))
    names = [f["name"] for f in prog["fields"]]
    widths = [int(f["elem_bytes"]) for f in prog["fields"]]
    n = int(prog["record_count"])
    secs = {s["id"]: s for s in prog["sections"]}
    dev = arch["devices"][0]["name"]

    # ---- which (section, device, layout) triples the run graph evaluates
    cands = A.plan_candidates(prog, arch)["runs"]
    need = sorted({(sid, r["device"], r["layout"]) for r in cands for sid in r["sections"]})
    print(f"{len(cands)} run nodes, {len(need)} (section, device, layout) triples to time", flush=True)

    # ---- one buffer per distinct layout, seeded finite fp32 values
    layouts = {}
    vals = torch.from_numpy(random_bytes(1407, n * 4)).view(torch.int32)
    vals = ((vals & 0x007FFFFF) | 0x3F800000).view(torch.float32)      # floats in [1, 2)
    out = torch.empty(4 * n, dtype=torch.float32, device="cuda")
    gen = torch.Generator(device="cuda")
    gen.manual_seed(14074859)
    idx_cache = {}
    profile = []
    for sid, d, lay in need:
        if lay not in layouts:
            L = A.Layout.from_string(lay, names, widths)
            buf = torch.empty(L.nbytes(n), dtype=torch.uint8, device="cuda")
            src_soa = A.Layout.soa(widths)
            soa = torch.empty(src_soa.nbytes(n), dtype=torch.uint8, device="cuda")
            for f in range(len(widths)):
                off, _, _ = src_soa.field_address(f, n)
                soa[off: off + 4 * n].copy_(vals.view(torch.uint8).to("cuda"))
            A.remap(soa, src_soa, buf, L, n)
            del soa
            layouts[lay] = (L, buf)
        L, buf = layouts[lay]
        s = secs[sid]
        total = 0.0
        for g in s["groups"]:
            fidx = [names.index(x) for x in g["fields"]]
            if g["pattern"] == "streaming":
                reps = max(1, round(g["freq"]))
                total += reps * timed(lambda: A.section_run(buf, L, n, fidx, out, n_out=n))
            else:
                m = int(g["freq"] * n)
                if m not in idx_cache:
                    idx_cache[m] = torch.randint(0, n, (m,), device="cuda", dtype=torch.int64, generator=gen)
                idx = idx_cache[m]
                total += timed(lambda: A.section_run(buf, L, n, fidx, out[:m] if m <= out.numel() else out,
                                                     idx=idx, n_out=m))
        profile.append({"section": sid, "device": d, "layout": lay, "time_ns": total})
        print(f"  {sid} {lay:60s} {total / 1e3:9.1f} us", flush=True)

    # ---- remap edge bandwidth: the Medical moved subset AoSV -> SoA via aliased regions
    aosv = A.Layout.from_string("{V1,V2,V3},U1,U2,U3,S,T,interpT", names, widths)
    soa = A.Layout.soa(widths)
    v_reg = torch.empty(12 * n, dtype=torch.uint8, device="cuda")
    singles = [torch.empty(4 * n, dtype=torch.uint8, device="cuda") for _ in range(6)]
    dst_v = [torch.empty(4 * n, dtype=torch.uint8, device="cuda") for _ in range(3)]
    t_moved = timed(lambda: A.remap_regions([v_reg] + singles, aosv, dst_v + singles, soa, n))
    moved_bytes = 12 * n
    bw = moved_bytes / t_moved                     # one-way moved bytes per ns (SPEC.md:217 model)
    small = 1 << 14
    t_small = timed(lambda: A.remap_regions([v_reg] + singles, aosv, dst_v + singles, soa, small))
    overhead = max(0.0, t_small - 12 * small / bw)
    arch_meas = json.loads(json.dumps(arch))
    arch_meas["same_device_remap_bandwidth_bytes_per_ns"] = bw
    arch_meas["remap_fixed_overhead_ns"] = overhead
    print(f"remap edge: {moved_bytes / 1e6:.0f} MB moved in {t_moved / 1e3:.1f} us -> {bw:.0f} bytes/ns "
          f"({2 * bw:.0f} GB/s read+write), fixed overhead {overhead / 1e3:.1f} us", flush=True)

    prof_json = {"schema_version": 1, "entries": profile}
    plan = A.plan_pdl(prog, arch_meas, prof_json)
    model_plan = A.plan_pdl(prog, arch)
    result = {
        "what": "B200 tuning profile (adha_section_run timings per run-graph candidate) and the PDL plan it gives",
        "program": os.path.relpath(prog_path, ROOT), "records": n,
        "remap_edge": {"moved_bytes": moved_bytes, "time_ns": t_moved, "bandwidth_bytes_per_ns": bw,
                       "fixed_overhead_ns": overhead},
        "profile": prof_json, "plan_measured": plan, "plan_model_only": model_plan,
    }
    with open(out_path, "w") as fh:
        json.dump(result, fh, indent=1)
    print("PDL on the measured B200 profile:")
    for r in plan["runs"]:
        print(f"  run {r['sections']} on {r['device']}: {r['layout']}  ({r['exec_ns'] / 1e3:.1f} us)")
    for m in plan["remaps"]:
        print(f"  remap after {m['after']}: moved {m['moved']} ({m['cost_ns'] / 1e3:.1f} us)")
    print(f"  total {plan['total_ns'] / 1e3:.1f} us")
    print("PDL on the analytic model only:", [(r["sections"], r["layout"]) for r in model_plan["runs"]])


if __name__ == "__main__":
    main()
