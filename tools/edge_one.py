"""One chain edge of a bench config, a few times, for ncu.  usage: edge_one.py CFG EDGE"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1407_4859_b200 as A
import bench
cfg, k = sys.argv[1], int(sys.argv[2])
desc, kind, n, _ = bench.CONFIGS[cfg]
w, chain = bench.chain_for(kind)
Ls, Ld = A.Layout(w, chain[k]), A.Layout(w, chain[k + 1])
a = torch.zeros(Ls.nbytes(n), dtype=torch.uint8, device="cuda")
b = torch.zeros(Ld.nbytes(n), dtype=torch.uint8, device="cuda")
for _ in range(4):
    A.remap(a, Ls, b, Ld, n)
torch.cuda.synchronize()
print("ok")
