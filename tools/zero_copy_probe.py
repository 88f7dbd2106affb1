"""Zero-copy probe: adha_remap with src and dst in PINNED HOST memory (UVA-mapped), i.e. the
remap kernel reads the records over PCIe with TMA and writes them back over PCIe.  Checks
parity against the oracle on a sample and reports GB/s (read+write payload)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1407_4859_b200 as A
from adha_inputs import config_widths, field_columns
from oracle import remap as O

w = config_widths(16)
n = 10_000_000
La, Ls = A.Layout.aos(w), A.Layout.soa(w)
h_src = torch.empty(La.nbytes(n), dtype=torch.uint8).pin_memory()
h_dst = torch.full((Ls.nbytes(n),), 0xA5, dtype=torch.uint8).pin_memory()
cols = field_columns(3, 100_000, w)
small = O.pack(cols, w, [0] * 16, 100_000)
h_src[: small.size].copy_(torch.from_numpy(small))
print("aligned", h_src.data_ptr() % 256, h_dst.data_ptr() % 256)
d_src = torch.empty(La.nbytes(n), dtype=torch.uint8, device="cuda"); d_src.copy_(h_src)
d_dst = torch.empty(Ls.nbytes(n), dtype=torch.uint8, device="cuda")
for mode in ["zero-copy", "host-src", "host-dst", "staged"]:
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    def go():
        if mode == "zero-copy":
            A.remap(h_src.data_ptr(), La, h_dst.data_ptr(), Ls, n, stream=torch.cuda.current_stream())
        elif mode == "host-src":
            A.remap(h_src.data_ptr(), La, d_dst, Ls, n)
        elif mode == "host-dst":
            A.remap(d_src, La, h_dst.data_ptr(), Ls, n)
        else:
            A.remap_host(h_src, La, h_dst, Ls, n, scratch)
    go(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        go()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(mode, f"{2 * n * 80 / ms / 1e6:.1f} GB/s", f"{ms:.2f} ms")
    if mode != "host-src":
        out = O.unpack(h_dst.numpy(), w, list(range(16)), n)
        ok = all(np.array_equal(out[f][:100_000], cols[f]) for f in range(16))
        print(mode, "parity on the first 100k records:", ok)
        h_dst.fill_(0xA5)
