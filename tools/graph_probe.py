import os, sys, json
sys.path.insert(0, os.getcwd())
import torch
import paper_1407_4859_b200 as A
from adha_inputs import config_widths
w = config_widths(16)
La, Ls = A.Layout(w, [0]*16), A.Layout(w, list(range(16)))
for n in (10_000, 100_000, 300_000, 1_000_000):
    src = torch.zeros(La.nbytes(n), dtype=torch.uint8, device="cuda")
    dst = torch.zeros(Ls.nbytes(n), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3): A.remap(src, La, dst, Ls, n)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20): A.remap(src, La, dst, Ls, n)
    g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); 
    for _ in range(5): g.replay()
    b.record(); torch.cuda.synchronize()
    t = a.elapsed_time(b) / 100
    # host cost per call: time 200 calls with a deep queue
    import time
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(200): A.remap(src, La, dst, Ls, n)
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(json.dumps({"n": n, "graph_us_per_remap": round(t*1e3, 2), "host_us_per_call": round((t1-t0)/200*1e6, 2), "wall_us_per_call": round((t2-t0)/200*1e6,2)}))
