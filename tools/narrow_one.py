"""One narrow-field remap (24 x 1-byte + 8 B, AoS -> SoA, N = 20M) a few times, for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1407_4859_b200 as A
w = [1] * 24 + [8]
n = 20_000_000
La, Ls = A.Layout.aos(w), A.Layout.soa(w)
a = torch.zeros(La.nbytes(n), dtype=torch.uint8, device="cuda")
b = torch.zeros(Ls.nbytes(n), dtype=torch.uint8, device="cuda")
for _ in range(4):
    A.remap(a, La, b, Ls, n)
torch.cuda.synchronize()
print("ok")
