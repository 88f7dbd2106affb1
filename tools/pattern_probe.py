"""Which access pattern costs what: time remaps of the C2 record (16 fields, 80 B, N records)
between several layout pairs with CUDA events; compare with torch copy_ of the same bytes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1407_4859_b200 as A
from adha_inputs import config_widths, fill_random_device

N = int(sys.argv[1]) if len(sys.argv) > 1 else 40_000_000
w = config_widths(16)
R = sum(w)
pairs = {
    "AoS->AoS (identity, 1 stream)": ([0] * 16, [0] * 16),
    "SoA->SoA (identity, 16 streams)": (list(range(16)), list(range(16))),
    "AoS->SoA (1 -> 16 streams)": ([0] * 16, list(range(16))),
    "SoA->AoS (16 -> 1 streams)": (list(range(16)), [0] * 16),
    "AoS->4xAoS20 (1 -> 4)": ([0] * 16, [i // 4 for i in range(16)]),
    "4xAoS20->AoS (4 -> 1)": ([i // 4 for i in range(16)], [0] * 16),
    "AoS->2xAoS40 (1 -> 2)": ([0] * 16, [i // 8 for i in range(16)]),
}
a = torch.empty(N * R + 65536, dtype=torch.uint8, device="cuda")
b = torch.empty(N * R + 65536, dtype=torch.uint8, device="cuda")
fill_random_device(a, 1)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ms = timed(lambda: b[: N * R].copy_(a[: N * R]))
print(f"{'torch copy_':34s} {2 * N * R / ms / 1e6:7.0f} GB/s")
for name, (ls, ld) in pairs.items():
    Ls, Ld = A.Layout(w, ls), A.Layout(w, ld)
    ms = timed(lambda: A.remap(a, Ls, b, Ld, N))
    print(f"{name:34s} {2 * N * R / ms / 1e6:7.0f} GB/s")
