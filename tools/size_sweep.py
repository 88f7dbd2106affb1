"""C2's remap (16 mixed 4/8-byte fields, AoS->SoA) across record counts: out-of-place adha_remap,
in-place adha_remap_inplace and torch copy_ of the same bytes, back to back with CUDA events.
Shows where launch latency stops mattering and where the kernel reaches the copy ceiling.
usage: python tools/size_sweep.py [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1407_4859_b200 as A  # noqa: E402
from adha_inputs import config_widths, fill_random_device  # noqa: E402

REPS = int(sys.argv[1]) if len(sys.argv) > 1 else 20


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(REPS):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / REPS


w = config_widths(16)
R = sum(w)
La, Ls = A.Layout(w, [0] * 16), A.Layout(w, list(range(16)))
for n in (10_000, 100_000, 300_000, 1_000_000, 3_000_000, 10_000_000, 30_000_000, 100_000_000):
    src = torch.empty(La.nbytes(n), dtype=torch.uint8, device="cuda")
    dst = torch.empty(Ls.nbytes(n), dtype=torch.uint8, device="cuda")
    fill_random_device(src, 3)
    t_oop = timed(lambda: A.remap(src, La, dst, Ls, n))
    t_cp = timed(lambda: dst[: n * R].copy_(src[: n * R]))
    fwd, bwd = A.InplacePlan(La, Ls, n), A.InplacePlan(Ls, La, n)
    del dst
    buf = torch.empty(max(fwd.buffer_bytes, bwd.buffer_bytes), dtype=torch.uint8, device="cuda")
    fwd.upload()
    bwd.upload()
    state = [0]

    def ip():
        A.remap_inplace(buf, fwd if state[0] == 0 else bwd)
        state[0] ^= 1
    t_ip = timed(ip)
    gb = 2 * n * R / 1e9
    print(json.dumps({"n": n, "bytes_moved_GB": round(gb, 4), "remap_ms": round(t_oop, 4),
                      "remap_GBps": round(gb / t_oop * 1e3, 1), "copy_GBps": round(gb / t_cp * 1e3, 1),
                      "remap_over_copy": round(t_cp / t_oop, 3), "inplace_ms": round(t_ip, 4),
                      "inplace_GBps": round(gb / t_ip * 1e3, 1)}), flush=True)
    del src, buf
    torch.cuda.empty_cache()
