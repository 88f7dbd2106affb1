"""Single-shot (synchronised, host launch latency included) vs back-to-back per-launch time of
C2 and the P1/P2 chain edges, with tile-order and L2-hint variants."""
import os, sys, statistics
sys.path.insert(0, "/root/repo")
import torch, paper_1407_4859_b200 as A, bench
from adha_inputs import fill_random_device
def run(cfg, k, env):
    desc, kind, n, _ = bench.CONFIGS[cfg]
    w, chain = bench.chain_for(kind)
    Ls, Ld = A.Layout(w, chain[k]), A.Layout(w, chain[k + 1])
    a = torch.empty(Ls.nbytes(n), dtype=torch.uint8, device="cuda"); fill_random_device(a, 3)
    b = torch.empty(Ld.nbytes(n), dtype=torch.uint8, device="cuda")
    R = sum(w)
    for kk, v in env.items(): os.environ[kk] = v
    f = lambda: A.remap(a, Ls, b, Ld, n)
    for _ in range(3): f()
    torch.cuda.synchronize()
    singles = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(); f(); e1.record(); torch.cuda.synchronize()
        singles.append(e0.elapsed_time(e1) * 1e3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): f()
    e1.record(); torch.cuda.synchronize()
    b2b = e0.elapsed_time(e1) * 1e3 / 20
    for kk in env: del os.environ[kk]
    print(f"{cfg}/{k} {env} single med {statistics.median(singles):.1f} us min {min(singles):.1f}  b2b {b2b:.1f} us  -> {2*n*R/b2b/1e3:.0f} GB/s", flush=True)
for env in ({}, {"ADHA_TILE_ORDER": "blocked"}, {"ADHA_L2_HINTS": "3"}, {"ADHA_L2_HINTS": "1"}):
    for cfg, k in (("C2", 0), ("P2", 0), ("P2", 1), ("P1", 1)):
        run(cfg, k, env)
