"""Medical moved-subset edge (AoSV -> SoA through aliased regions, only {V1,V2,V3} moves), timed
single-shot (as tools/b200_tuning_profile.py does: host launch latency included) and back to back."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1407_4859_b200 as A

names = ["V1", "V2", "V3", "U1", "U2", "U3", "S", "T", "interpT"]
widths = [4] * 9
aosv = A.Layout.from_string("{V1,V2,V3},U1,U2,U3,S,T,interpT", names, widths)
soa = A.Layout.soa(widths)
for n in (256 ** 3, 1 << 14):
    v_reg = torch.empty(12 * n, dtype=torch.uint8, device="cuda")
    singles = [torch.empty(4 * n, dtype=torch.uint8, device="cuda") for _ in range(6)]
    dst_v = [torch.empty(4 * n, dtype=torch.uint8, device="cuda") for _ in range(3)]
    f = lambda: A.remap_regions([v_reg] + singles, aosv, dst_v + singles, soa, n)
    f()
    torch.cuda.synchronize()
    single = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        single.append(e0.elapsed_time(e1) * 1e3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        f()
    e1.record(); torch.cuda.synchronize()
    b2b = e0.elapsed_time(e1) * 1e3 / 50
    print(f"n={n}: single-shot median {statistics.median(single):.1f} us, back-to-back {b2b:.1f} us "
          f"-> {2 * 12 * n / b2b / 1e3:.0f} GB/s (moved bytes read+write)")
