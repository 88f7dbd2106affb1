"""Per-edge GB/s of the P1/P2/C4 chains (each remap timed alone, burst) next to torch copy_ of the
same N*R bytes, interleaved in one process so drift cancels; with the plan's tile size and
component count.  usage: python tools/edge_probe.py [reps]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1407_4859_b200 as A  # noqa: E402
from adha_inputs import fill_random_device  # noqa: E402
import bench  # noqa: E402

REPS = int(sys.argv[1]) if len(sys.argv) > 1 else 5


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for cfg in ("P1", "P2", "C4", "C2"):
    desc, kind, n, _ = bench.CONFIGS[cfg]
    widths, chain = bench.chain_for(kind)
    R = sum(widths)
    lays = [A.Layout(widths, lab) for lab in chain]
    bufs = [torch.empty(l.nbytes(n), dtype=torch.uint8, device="cuda") for l in lays]
    fill_random_device(bufs[0], 7)
    ca = torch.empty(n * R, dtype=torch.uint8, device="cuda")
    cb = torch.empty_like(ca)
    for k in range(len(chain) - 1):
        d = A.plan_describe(lays[k], lays[k + 1])
        rs, cs = [], []
        for _ in range(REPS):
            rs.append(2 * n * R / timed(lambda: A.remap(bufs[k], lays[k], bufs[k + 1], lays[k + 1], n)) / 1e6)
            cs.append(2 * n * R / timed(lambda: cb.copy_(ca)) / 1e6)
        print(f"{cfg} edge {k}: {lays[k].to_string()[:40]:40s} -> {lays[k + 1].to_string()[:40]:40s} "
              f"remap {statistics.median(rs):6.0f}  copy {statistics.median(cs):6.0f}  "
              f"ratio {statistics.median(rs) / statistics.median(cs):.3f}  T {d['T']} comps {len(d['components'])} "
              f"stage {d['stage_bytes']}", flush=True)
    del bufs, ca, cb
    torch.cuda.empty_cache()
