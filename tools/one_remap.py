"""One shape at one payload size, forced onto the tiled kernel, remapped `reps` times: the target of
an `ncu -k regex:remap_tiled -s 2 -c 1` capture of the small / mid-size regime.
usage: python tools/one_remap.py {c2|c3|g2|medv} MB [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("ADHA_SMALL_BYTES", "0")
import torch  # noqa: E402
import paper_1407_4859_b200 as A  # noqa: E402
import bench  # noqa: E402

w16 = [8 if i % 4 == 3 else 4 for i in range(16)]
w64 = [8 if i % 4 == 3 else 4 for i in range(64)]
SH = {"c2": (w16, [0] * 16, list(range(16))), "g2": ([2, 4, 6, 4] * 4, [0] * 16, list(range(16))),
      "medv": ([4] * 9, [0, 0, 0, 1, 2, 3, 4, 5, 6], list(range(9)))}
kind, mb = sys.argv[1], float(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
w, ls, ld = SH[kind] if kind != "c3" else (w64, list(range(64)), bench.c3_labels()[0])
n = max(1, int(mb * 2 ** 20) // sum(w))
Ls, Ld = A.Layout(w, ls), A.Layout(w, ld)
a = torch.zeros(Ls.nbytes(n), dtype=torch.uint8, device="cuda")
b = torch.zeros(Ld.nbytes(n), dtype=torch.uint8, device="cuda")
for _ in range(reps):
    A.remap(a, Ls, b, Ld, n)
torch.cuda.synchronize()
print(kind, mb, "MB", n, "records ok")
