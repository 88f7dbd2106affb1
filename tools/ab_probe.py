"""A/B probe with drift cancellation: for each layout pair, alternate the variants of one env knob
inside ONE process (the library reads the knobs per call), several rounds, report medians.
    python tools/ab_probe.py ADHA_TMA_SPLIT 0,4096 [N]"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1407_4859_b200 as A
from adha_inputs import config_widths, fill_random_device

knob = sys.argv[1]
variants = sys.argv[2].split(",")
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40_000_000
w = config_widths(16)
R = sum(w)
pairs = {
    "AoS->AoS": ([0] * 16, [0] * 16),
    "SoA->SoA": (list(range(16)), list(range(16))),
    "AoS->SoA": ([0] * 16, list(range(16))),
    "SoA->AoS": (list(range(16)), [0] * 16),
    "AoS->4xAoS20": ([0] * 16, [i // 4 for i in range(16)]),
}
a = torch.empty(N * R + 65536, dtype=torch.uint8, device="cuda")
b = torch.empty(N * R + 65536, dtype=torch.uint8, device="cuda")
fill_random_device(a, 1)


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return 2 * N * R / (e0.elapsed_time(e1) / reps) / 1e6


import time
soak = float(os.environ.get("SOAK_S", "0"))
if soak > 0:                                       # sustained load first: power cap / clocks settle
    Ls0, Ld0 = A.Layout(w, [0] * 16), A.Layout(w, list(range(16)))
    t_end = time.time() + soak
    while time.time() < t_end:
        for _ in range(20):
            A.remap(a, Ls0, b, Ld0, N)
        torch.cuda.synchronize()
res = {}
copy = []
for rnd in range(5):
    copy.append(timed(lambda: b[: N * R].copy_(a[: N * R])))
    for name, (ls, ld) in pairs.items():
        Ls, Ld = A.Layout(w, ls), A.Layout(w, ld)
        for v in variants:
            os.environ[knob] = v
            res.setdefault((name, v), []).append(timed(lambda: A.remap(a, Ls, b, Ld, N)))
print(f"torch copy_ median {statistics.median(copy):.0f} GB/s")
for name in pairs:
    print(f"{name:14s} " + "  ".join(f"{knob}={v}: {statistics.median(res[(name, v)]):6.0f}" for v in variants))
