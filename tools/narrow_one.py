"""One narrow-field remap a few times, for ncu.  usage: narrow_one.py [case]
cases: b24 (24 x 1-byte + 8 B, AoS->SoA), g2a (16 fields 2/4/6/4 B AoS->SoA), g2s (same, SoA->AoS),
       al (SoA -> C-aligned AoS {1,4,2,8,4,2})."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1407_4859_b200 as A
case = sys.argv[1] if len(sys.argv) > 1 else "b24"
n = 20_000_000
if case == "b24":
    w = [1] * 24 + [8]
    Ls, Ld = A.Layout.aos(w), A.Layout.soa(w)
elif case in ("g2a", "g2s"):
    w = [2, 4, 6, 4] * 4
    Ls, Ld = A.Layout.aos(w), A.Layout.soa(w)
    if case == "g2s":
        Ls, Ld = Ld, Ls
else:
    w = [1, 4, 2, 8, 4, 2]
    Ls, Ld = A.Layout.soa(w), A.Layout(w, [0] * 6, aligned=True)
a = torch.zeros(Ls.nbytes(n), dtype=torch.uint8, device="cuda")
b = torch.zeros(Ld.nbytes(n), dtype=torch.uint8, device="cuda")
for _ in range(4):
    A.remap(a, Ls, b, Ld, n)
torch.cuda.synchronize()
print("ok")
