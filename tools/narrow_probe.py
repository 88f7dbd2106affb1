"""Narrow fields: GB/s of AoS<->SoA remaps for records whose unit g is 4, 2 or 1 byte."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1407_4859_b200 as A
from adha_inputs import fill_random_device

recs = {
    "g=4  16 fields 4/8 B (R=80)": [8 if i % 4 == 3 else 4 for i in range(16)],
    "g=2  16 fields 2/4/6 B (R=64)": [2, 4, 6, 4] * 4,
    "g=1  16 fields 1/2/3/4/... (R=64)": [1, 3, 4, 8] * 4,
    "g=1  24 x 1-byte + 8 (R=32)": [1] * 24 + [8],
}
N = 20_000_000
a = torch.empty(N * 80 + 65536, dtype=torch.uint8, device="cuda")
b = torch.empty(N * 80 + 65536, dtype=torch.uint8, device="cuda")
fill_random_device(a, 1)


def timed(fn, nbytes, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return nbytes / (e0.elapsed_time(e1) / reps) / 1e6


for name, w in recs.items():
    R = sum(w)
    F = len(w)
    for tag, ls, ld in [("AoS->SoA", [0] * F, list(range(F))), ("SoA->AoS", list(range(F)), [0] * F)]:
        Ls, Ld = A.Layout(w, ls), A.Layout(w, ld)
        d = A.plan_describe(Ls, Ld)
        g = timed(lambda: A.remap(a, Ls, b, Ld, N), 2 * N * R)
        print(f"{name:36s} {tag}: {g:6.0f} GB/s  (unit {d['unit']}, matched {d['matched']}, T {d['T']})")
