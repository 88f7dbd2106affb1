"""Host cost per call: adha_remap and adha_remap_regions launched back to back from Python with the
GPU queue kept full (time.perf_counter per call), plus a cProfile of the regions call."""
import os, sys, time, cProfile, pstats
sys.path.insert(0, "/root/repo")
import torch
import paper_1407_4859_b200 as A
names = ["V1", "V2", "V3", "U1", "U2", "U3", "S", "T", "interpT"]
widths = [4] * 9
aosv = A.Layout.from_string("{V1,V2,V3},U1,U2,U3,S,T,interpT", names, widths)
soa = A.Layout.soa(widths)
n = 1 << 14
v_reg = torch.empty(12 * n, dtype=torch.uint8, device="cuda")
singles = [torch.empty(4 * n, dtype=torch.uint8, device="cuda") for _ in range(6)]
dst_v = [torch.empty(4 * n, dtype=torch.uint8, device="cuda") for _ in range(3)]
f = lambda: A.remap_regions([v_reg] + singles, aosv, dst_v + singles, soa, n)
La, Ls = A.Layout.aos(widths), A.Layout.soa(widths)
a = torch.empty(La.nbytes(n), dtype=torch.uint8, device="cuda"); b = torch.empty(Ls.nbytes(n), dtype=torch.uint8, device="cuda")
g = lambda: A.remap(a, La, b, Ls, n)
for fn, name in ((f, "regions"), (g, "remap")):
    for _ in range(20): fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(2000): fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(name, "host us/call", (t1 - t) / 2000 * 1e6, "incl sync", (time.perf_counter() - t) / 2000 * 1e6)
cProfile.run("for _ in range(2000): f()", "/tmp/prof.out")
pstats.Stats("/tmp/prof.out").sort_stats("tottime").print_stats(8)
