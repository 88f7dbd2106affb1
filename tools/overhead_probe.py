"""Fixed per-launch overhead: fit t(N) = a + N/b for the C2 remap and for torch copy_ (same bytes)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1407_4859_b200 as A
from adha_inputs import config_widths, fill_random_device

w = config_widths(16)
R = 80
Ns = [2_500_000, 5_000_000, 10_000_000, 20_000_000, 40_000_000]
a = torch.empty(max(Ns) * R + 65536, dtype=torch.uint8, device="cuda")
b = torch.empty_like(a)
fill_random_device(a, 1)
La, Ls = A.Layout.aos(w), A.Layout.soa(w)


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3     # us


rows = {"remap": [], "copy": []}
for rnd in range(3):
    for n in Ns:
        rows["remap"].append((n, timed(lambda: A.remap(a, La, b, Ls, n))))
        rows["copy"].append((n, timed(lambda: b[: n * R].copy_(a[: n * R]))))
for k, v in rows.items():
    med = {n: statistics.median([t for m, t in v if m == n]) for n in Ns}
    x = np.array(Ns, float)
    y = np.array([med[n] for n in Ns])
    slope, icpt = np.polyfit(x, y, 1)
    print(f"{k:6s} fixed {icpt:6.1f} us  streaming {2 * R / slope / 1e3:7.0f} GB/s   " +
          "  ".join(f"N={n // 1000000}M:{2 * n * R / med[n] / 1e3:5.0f}" for n in Ns))
