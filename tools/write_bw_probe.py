"""HBM bandwidth by traffic mix on this B200: pure writes (fill_), read+write (copy_), pure reads
(a sum), and a 1:3 read:write mix like the fused chain's (one read pass, three write passes)."""
import torch

n = 8 << 30
a = torch.empty(n, dtype=torch.uint8, device="cuda")
b = torch.empty(n, dtype=torch.uint8, device="cuda")
a.fill_(1)
torch.cuda.synchronize()


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


t = timed(lambda: b.fill_(7))
print(f"write only (fill_ 8 GiB):    {n / t / 1e9:7.0f} GB/s")
import ctypes, glob, os
libs = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + \
       glob.glob("/usr/local/cuda/lib64/libcudart.so*")
rt = ctypes.CDLL(libs[0])
stream = torch.cuda.current_stream().cuda_stream
t = timed(lambda: rt.cudaMemsetAsync(ctypes.c_void_p(b.data_ptr()), 0, ctypes.c_size_t(n), ctypes.c_void_p(stream)))
print(f"write only (cudaMemset 8 GiB): {n / t / 1e9:7.0f} GB/s")
t = timed(lambda: b.copy_(a))
print(f"read+write (copy_ 8 GiB):    {2 * n / t / 1e9:7.0f} GB/s")
a32 = a.view(torch.int32)
t = timed(lambda: torch.sum(a32, dtype=torch.int64))
print(f"read only (sum 8 GiB):       {n / t / 1e9:7.0f} GB/s")
q = n // 4
c = torch.empty(q, dtype=torch.uint8, device="cuda")
def mix():
    c.copy_(a[:q])            # read q, write q
    b[:q].fill_(3)            # write q
    b[q:2 * q].fill_(5)       # write q
t = timed(mix)
print(f"1 read : 3 writes (2 GiB x4): {4 * q / t / 1e9:7.0f} GB/s")
