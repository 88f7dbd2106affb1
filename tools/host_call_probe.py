"""Host cost of one Python-level adha_remap call, split into its parts (GPU queue kept full).
usage: python tools/host_call_probe.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes  # noqa: E402
import torch  # noqa: E402
import paper_1407_4859_b200 as A  # noqa: E402
from adha_inputs import config_widths  # noqa: E402


def per_call(fn, k=2000):
    for _ in range(50):
        fn()
    t = time.perf_counter()
    for _ in range(k):
        fn()
    return (time.perf_counter() - t) / k * 1e6


w = config_widths(16)
La, Ls = A.Layout(w, [0] * 16), A.Layout(w, list(range(16)))
n = 1000
src = torch.zeros(La.nbytes(n), dtype=torch.uint8, device="cuda")
dst = torch.zeros(Ls.nbytes(n), dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
raw = st.cuda_stream
out = {
    "current_stream_obj_us": per_call(lambda: torch.cuda.current_stream().cuda_stream),
    "raw_stream_us": per_call(lambda: torch._C._cuda_getCurrentRawStream(torch.cuda.current_device())),
    "data_ptr_x2_us": per_call(lambda: (src.data_ptr(), dst.data_ptr())),
    "nbytes_checks_us": per_call(lambda: (La.nbytes(n), Ls.nbytes(n))),
    "ctypes_adha_remap_us": per_call(lambda: A._lib.adha_remap(src.data_ptr(), La.handle, dst.data_ptr(), Ls.handle, n, raw)),
    "python_remap_us": per_call(lambda: A.remap(src, La, dst, Ls, n)),
}
torch.cuda.synchronize()
print(json.dumps({k: round(v, 2) for k, v in out.items()}))
