"""Host time of the in-place plan (adha_inplace_plan_create) for C3 (50M records, SoA -> 24-cluster hybrid) and C2;
with ADHA_IP_TIMING=1 the library prints its phases.  usage: python tools/inplace_plan_time.py"""
import time, sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1407_4859_b200 as A
import bench
from adha_inputs import config_widths
w = config_widths(64)
c3 = bench.c3_labels()[0]
n = 50_000_000
Ls, Ld = A.Layout(w, list(range(64))), A.Layout(w, c3)
for rep in range(3):
    t = time.perf_counter()
    p = A.InplacePlan(Ls, Ld, n)
    print("C3 plan ms", (time.perf_counter() - t) * 1e3, flush=True)
    del p
w16 = config_widths(16)
for rep in range(2):
    t = time.perf_counter()
    p = A.InplacePlan(A.Layout(w16, [0]*16), A.Layout(w16, list(range(16))), 10_000_000)
    print("C2 plan ms", (time.perf_counter() - t) * 1e3, flush=True)
