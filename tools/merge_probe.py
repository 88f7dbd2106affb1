"""Merged vs per-component plan at large N for multi-component layout pairs with few src clusters
(the merge_bytes rule in remap.cu).  GPU time per remap from events over back-to-back calls.
usage: python tools/merge_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1407_4859_b200 as A  # noqa: E402
from adha_inputs import config_widths  # noqa: E402

w16 = config_widths(16)
SHAPES = [
    ("Medical AoSV->SoA (7 src)", [4] * 9, [0, 0, 0, 1, 2, 3, 4, 5, 6], list(range(9))),
    ("Medical SoA->AoSV (9 src)", [4] * 9, list(range(9)), [0, 0, 0, 1, 2, 3, 4, 5, 6]),
    ("K-Means 4xAoS8->SoA (4 src)", [4] * 32, [f // 8 for f in range(32)], list(range(32))),
    ("K-Means AoS->4xAoS8 (1 src)", [4] * 32, [0] * 32, [f // 8 for f in range(32)]),
    ("C2 2xAoS8->SoA (2 src)", w16, [f // 8 for f in range(16)], list(range(16))),
    ("C2 4-cluster hybrid->2-cluster (4 src)", w16, [f // 4 for f in range(16)], [f % 2 for f in range(16)]),
]


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


for mb in (512, 2048):
    for name, w, ls, ld in SHAPES:
        R = sum(w)
        n = (mb << 20) // R
        res = {}
        for tag, env in (("components", "0"), ("merged", str(1 << 62))):
            os.environ["ADHA_MERGE_BYTES"] = env
            Ls, Ld = A.Layout(w, ls), A.Layout(w, ld)
            a = torch.empty(Ls.nbytes(n), dtype=torch.uint8, device="cuda")
            b = torch.empty(Ld.nbytes(n), dtype=torch.uint8, device="cuda")
            res[tag] = timed(lambda: A.remap(a, Ls, b, Ld, n))
            del a, b
        os.environ.pop("ADHA_MERGE_BYTES")
        Ls, Ld = A.Layout(w, ls), A.Layout(w, ld)
        comps = len(A.plan_describe(Ls, Ld)["components"])
        print(f"{name:40s} {mb:5d} MB comps {comps:2d}: per-component {res['components']:8.1f} us "
              f"({2 * n * R / res['components'] / 1e3:5.0f} GB/s)  merged {res['merged']:8.1f} us "
              f"({2 * n * R / res['merged'] / 1e3:5.0f} GB/s)", flush=True)
