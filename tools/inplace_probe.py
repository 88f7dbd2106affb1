"""Time the in-place remap (adha_remap_inplace) against the out-of-place remap on the same shapes.

    python tools/inplace_probe.py [--reps 10] [--cases C2,C2r,P1,P2,C3s]

Per case: host plan time, device time per in-place run (CUDA events on the stream, median of
reps), the remap-equivalent rate 2*N*R / t, the plan's device traffic / t, and the out-of-place
adha_remap rate for the same pair.  The in-place buffer is max(bytes) instead of the sum.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1407_4859_b200 as A  # noqa: E402
from adha_inputs import config_widths, fill_random_device  # noqa: E402


def c3_labels():
    lab = []
    groups = [range(0, 26), range(26, 36), range(36, 40), (40, 41, 42), (43, 47)]
    cl = {}
    for g, fs in enumerate(groups):
        for f in fs:
            cl[f] = g
    nxt = len(groups)
    for f in range(64):
        if f not in cl:
            cl[f] = nxt
            nxt += 1
    return [cl[f] for f in range(64)]


def cases():
    w16, w64 = config_widths(16), config_widths(64)
    aos16, soa16 = [0] * 16, list(range(16))
    med = [4] * 9
    km = [4] * 32
    return {
        "C2": (w16, aos16, soa16, 10_000_000),
        "C2r": (w16, soa16, aos16, 10_000_000),
        "C5": (w16, aos16, soa16, 107_374_182),
        "P1": (med, [0] * 9, [0, 0, 0, 1, 2, 3, 4, 5, 6], 1 << 24),
        "P1b": (med, [0, 0, 0, 1, 2, 3, 4, 5, 6], list(range(9)), 1 << 24),
        "P2": (km, list(range(32)), [f // 8 for f in range(32)], 1 << 23),
        "P2b": (km, [f // 8 for f in range(32)], [0] * 32, 1 << 23),
        "C3s": (w64, list(range(64)), c3_labels(), 10_000_000),
    }


def time_fn(fn, reps, st):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2], ts[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--cases", default="C2,C2r,P1,P1b,P2,P2b,C3s")
    ap.add_argument("--no-oop", action="store_true")
    ap.add_argument("--kernels", action="store_true", help="per-kernel device times (torch.profiler / CUPTI)")
    a = ap.parse_args()
    st = torch.cuda.current_stream()
    for name in a.cases.split(","):
        widths, ls, ld, n = cases()[name]
        Ls, Ld = A.Layout(widths, ls), A.Layout(widths, ld)
        R = sum(widths)
        t0 = time.perf_counter()
        fwd = A.InplacePlan(Ls, Ld, n)
        plan_ms = (time.perf_counter() - t0) * 1e3
        bwd = A.InplacePlan(Ld, Ls, n)
        d = fwd.describe()
        buf = torch.empty(max(fwd.buffer_bytes, bwd.buffer_bytes), dtype=torch.uint8, device="cuda")
        fill_random_device(buf, 7)
        fwd.upload()
        bwd.upload()
        for _ in range(2):
            A.remap_inplace(buf, fwd)
            A.remap_inplace(buf, bwd)
        torch.cuda.synchronize()
        # alternate directions so each timed run remaps real contents
        ts = []
        for _ in range(a.reps):
            med, _mn = time_fn(lambda: A.remap_inplace(buf, fwd), 1, st)
            ts.append(med)
            A.remap_inplace(buf, bwd)
        ts.sort()
        t = ts[len(ts) // 2]
        kern = None
        if a.kernels:
            from torch.profiler import profile, ProfilerActivity
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                for _ in range(3):          # contents do not change the timing
                    A.remap_inplace(buf, fwd)
                torch.cuda.synchronize()
            kern = {}
            for e in prof.key_averages():
                tot = getattr(e, "device_time_total", None)
                if tot is None:
                    tot = getattr(e, "cuda_time_total", 0)
                if tot and "ip_" in e.key:
                    kern[e.key[:90]] = round(tot / 1e3 / 3, 4)
        out = {"case": name, "n": n, "R": R, "plan_ms": round(plan_ms, 2), "inplace_ms": round(t, 4),
               "remap_equiv_gbs": round(2 * n * R / t / 1e6, 1),
               "traffic_gbs": round(d["traffic_bytes"] / t / 1e6, 1),
               "buffer_gb": round(fwd.buffer_bytes / 1e9, 3),
               "workspace_mb": round(fwd.workspace_bytes / 1e6, 2), "plan": d}
        if kern is not None:
            out["kernel_ms_per_run"] = kern
        del buf
        torch.cuda.empty_cache()
        if not a.no_oop:
            src = torch.empty(Ls.nbytes(n), dtype=torch.uint8, device="cuda")
            dst = torch.empty(Ld.nbytes(n), dtype=torch.uint8, device="cuda")
            fill_random_device(src, 8)
            for _ in range(3):
                A.remap(src, Ls, dst, Ld, n)
            med, _ = time_fn(lambda: A.remap(src, Ls, dst, Ld, n), a.reps, st)
            out["out_of_place_ms"] = round(med, 4)
            out["out_of_place_gbs"] = round(2 * n * R / med / 1e6, 1)
            out["out_of_place_buffer_gb"] = round((Ls.nbytes(n) + Ld.nbytes(n)) / 1e9, 3)
            del src, dst
            torch.cuda.empty_cache()
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
