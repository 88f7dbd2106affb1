"""Does the allocation kind matter?  C2 remap and copy between torch-allocated buffers vs plain
cudaMalloc buffers (ncu showed every dst write entering L2 compression with a 0 % success rate)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
import torch
import paper_1407_4859_b200 as A
from adha_inputs import config_widths, fill_random_device

N = 10_000_000
w = config_widths(16)
La, Ls = A.Layout.aos(w), A.Layout.soa(w)
nb = max(La.nbytes(N), Ls.nbytes(N))
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
try:
    cudart = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so")
except OSError:
    pass
ta = torch.empty(nb, dtype=torch.uint8, device="cuda")
tb = torch.empty(nb, dtype=torch.uint8, device="cuda")
fill_random_device(ta, 1)
pa, pb = ctypes.c_void_p(), ctypes.c_void_p()
assert cudart.cudaMalloc(ctypes.byref(pa), ctypes.c_size_t(nb)) == 0
assert cudart.cudaMalloc(ctypes.byref(pb), ctypes.c_size_t(nb)) == 0
cudart.cudaMemcpy(pa, ctypes.c_void_p(ta.data_ptr()), ctypes.c_size_t(nb), 3)
torch.cuda.synchronize()


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return 2 * N * 80 / (e0.elapsed_time(e1) / reps) / 1e6


res = {}
for rnd in range(5):
    res.setdefault("torch buffers remap", []).append(timed(lambda: A.remap(ta, La, tb, Ls, N)))
    res.setdefault("cudaMalloc buffers remap", []).append(timed(lambda: A.remap(pa.value, La, pb.value, Ls, N)))
    res.setdefault("torch copy_", []).append(timed(lambda: tb[: N * 80].copy_(ta[: N * 80])))
    res.setdefault("cudaMemcpy D2D (cudaMalloc)", []).append(
        timed(lambda: cudart.cudaMemcpyAsync(pb, pa, ctypes.c_size_t(N * 80), 3, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))))
for k, v in res.items():
    print(f"{k:30s} {statistics.median(v):6.0f} GB/s")
print("PYTORCH_CUDA_ALLOC_CONF =", os.environ.get("PYTORCH_CUDA_ALLOC_CONF"))
