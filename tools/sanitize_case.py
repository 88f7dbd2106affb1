"""Small remaps for compute-sanitizer (one tool per run): tiled kernel forced, several layout
pairs, results checked against the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ADHA_SMALL_BYTES"] = "0"
import numpy as np
import torch
import paper_1407_4859_b200 as A
from adha_inputs import config_widths, field_columns
from oracle import remap as O

cases = [(config_widths(16), [0] * 16, list(range(16)), 4 * 608 + 77),
         ([4] * 9, [0, 0, 0, 1, 2, 3, 4, 5, 6], list(range(9)), 3 * 1344 + 5),
         ([1, 2, 3, 4, 8], [0, 1, 0, 1, 2], [0, 0, 1, 1, 1], 5000),
         ([4] * 32, list(range(32)), [i // 8 for i in range(32)], 3000)]
for w, ls, ld, n in cases:
    cols = field_columns(5, n, w)
    src = O.pack(cols, w, ls, n)
    Ls, Ld = A.Layout(w, ls), A.Layout(w, ld)
    d_src = torch.from_numpy(src).cuda()
    d_dst = torch.full((Ld.nbytes(n),), 0xA5, dtype=torch.uint8, device="cuda")
    A.remap(d_src, Ls, d_dst, Ld, n)
    torch.cuda.synchronize()
    exp = np.full(Ld.nbytes(n), 0xA5, np.uint8)
    O.remap(src, ls, exp, ld, w, n)
    assert np.array_equal(d_dst.cpu().numpy(), exp), (w, ls, ld, n)
print("sanitize case ok")
