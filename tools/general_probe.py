"""GB/s of generalised-layout remaps (AoSoA blocks, C-struct alignment), payload read+write."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1407_4859_b200 as A
from adha_inputs import config_widths, fill_random_device

N = 20_000_000
w16 = config_widths(16)
cases = {
    "AoS -> AoSoA32 (C2 record)": (w16, [0] * 16, None, False, [0] * 16, [32] * 16, False),
    "AoSoA32 -> SoA (C2 record)": (w16, [0] * 16, [32] * 16, False, list(range(16)), None, False),
    "AoS -> AoSoA8 (Medical)": ([4] * 9, [0] * 9, None, False, [0] * 9, [8] * 9, False),
    "SoA -> aligned AoS {1,4,2,8,4,2}": ([1, 4, 2, 8, 4, 2], list(range(6)), None, False, [0] * 6, None, True),
    "aligned AoS -> SoA {1,4,2,8,4,2}": ([1, 4, 2, 8, 4, 2], [0] * 6, None, True, list(range(6)), None, False),
}
buf_a = torch.empty(N * 128 + 65536, dtype=torch.uint8, device="cuda")
buf_b = torch.empty_like(buf_a)
fill_random_device(buf_a, 3)


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


for name, (w, ls, bs, als, ld, bd, ald) in cases.items():
    Ls = A.Layout(w, ls, blocks=bs, aligned=als)
    Ld = A.Layout(w, ld, blocks=bd, aligned=ald)
    ms = timed(lambda: A.remap(buf_a, Ls, buf_b, Ld, N))
    moved = Ls.nbytes(N) + Ld.nbytes(N)       # bytes actually read + written (padding included)
    d = A.plan_describe(Ls, Ld)
    print(f"{name:36s} {moved / ms / 1e6:7.0f} GB/s (bytes incl. padding)  unit {d['unit']} byte_groups {d['byte_groups']}")
