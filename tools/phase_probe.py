"""Where does a tile's time go?  Loads the DIAGNOSTIC library (built with -DADHA_PHASE_TIMING by
`python paper_1407_4859_b200/build.py --phase-timing`, never used by the package) and reports the
tiled kernel's clock64() phase sums per tile and consumer warp: wait for the TMA data (`full`),
permutation, output-tile barrier, copy-out; and the producer's wait for a free stage.
usage: python tools/phase_probe.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_1407_4859_b200", "_build", "libadha_phase.so"))
lib.adha_layout_create.argtypes = [ctypes.POINTER(ctypes.c_uint32), ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                                   ctypes.POINTER(ctypes.c_void_p)]
lib.adha_layout_bytes.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_uint64)]
lib.adha_remap.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                           ctypes.c_void_p]
lib.adha_debug_phase.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]


def layout(widths, labels):
    h = ctypes.c_void_p()
    rc = lib.adha_layout_create((ctypes.c_uint32 * len(widths))(*widths), len(widths),
                                (ctypes.c_int32 * len(labels))(*labels), ctypes.byref(h))
    assert rc == 0
    return h


def nbytes(h, n):
    b = ctypes.c_uint64()
    assert lib.adha_layout_bytes(h, n, ctypes.byref(b)) == 0
    return b.value


def phases(reset=True):
    out = (ctypes.c_ulonglong * 8)()
    assert lib.adha_debug_phase(out, 1 if reset else 0) == 0
    return list(out)


w16 = [8 if i % 4 == 3 else 4 for i in range(16)]
cases = [
    ("C2 AoS->SoA", w16, [0] * 16, list(range(16)), 10_000_000),
    ("C2 SoA->AoS", w16, list(range(16)), [0] * 16, 10_000_000),
    ("P2 4xAoS8->AoS", [4] * 32, [i // 8 for i in range(32)], [0] * 32, 2 ** 23),
    ("g2 AoS->SoA (byte groups)", [2, 4, 6, 4] * 4, [0] * 16, list(range(16)), 20_000_000),
    ("b24 SoA->AoS (byte groups)", [1] * 24 + [8], list(range(25)), [0] * 25, 20_000_000),
]
if "--small" in sys.argv:
    # small and mid-size remaps forced onto the tiled kernel: where does the fixed cost go?
    os.environ["ADHA_SMALL_BYTES"] = "0"
    import bench
    c3 = bench.c3_labels()[0]
    w64 = [8 if i % 4 == 3 else 4 for i in range(64)]
    cases = [(f"{nm} {mb} MB", w, ls, ld, max(1, (mb << 20) // sum(w)))
             for nm, w, ls, ld in [("C2 AoS->SoA", w16, [0] * 16, list(range(16))),
                                   ("C3 SoA->hybrid", w64, list(range(64)), c3),
                                   ("g2 AoS->SoA", [2, 4, 6, 4] * 4, [0] * 16, list(range(16))),
                                   ("Medical AoSV->SoA", [4] * 9, [0, 0, 0, 1, 2, 3, 4, 5, 6], list(range(9)))]
             for mb in (1, 32)]
lib.adha_remap_chain.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32,
                                 ctypes.c_int64, ctypes.c_void_p]
if "--chain" in sys.argv:
    # C4's chain AoS -> AoSV -> SoA -> AoS at 2 GiB, per hop or fused (ADHA_CHAIN_TILED_BYTES)
    labs = [[0] * 9, [0, 0, 0, 1, 2, 3, 4, 5, 6], list(range(9)), [0] * 9]
    n = (2 ** 31) // 36
    hs = [layout([4] * 9, l) for l in labs]
    bufs = [torch.empty(nbytes(h, n), dtype=torch.uint8, device="cuda") for h in hs]
    bp = (ctypes.c_void_p * 4)(*[b.data_ptr() for b in bufs])
    lp = (ctypes.c_void_p * 4)(*[h.value for h in hs])
    stream = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        assert lib.adha_remap_chain(bp, lp, 4, n, stream) == 0
    torch.cuda.synchronize()
    phases(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        lib.adha_remap_chain(bp, lp, 4, n, stream)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    p = phases(reset=True)
    tiles = max(1, p[4])
    per = [x / tiles for x in p[:4]]
    print(f"C4 chain ({os.environ.get('ADHA_CHAIN_TILED_BYTES', 'per hop')}): {ms:.3f} ms, {3 * 2 * n * 36 / ms / 1e6:.0f} GB/s; "
          f"per tile & warp (clk): wait_full {per[0]:.0f} permute {per[1]:.0f} barrier {per[2]:.0f} copy_out {per[3]:.0f}; "
          f"producer wait_empty/tile {p[5] / (tiles / 8):.0f} issue/tile {p[6] / (tiles / 8):.0f}", flush=True)
    sys.exit(0)
stream = torch.cuda.current_stream().cuda_stream
for name, w, ls, ld, n in cases:
    Ls, Ld = layout(w, ls), layout(w, ld)
    a = torch.empty(nbytes(Ls, n), dtype=torch.uint8, device="cuda")
    b = torch.empty(nbytes(Ld, n), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        assert lib.adha_remap(a.data_ptr(), Ls, b.data_ptr(), Ld, n, stream) == 0
    torch.cuda.synchronize()
    phases(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 10
    for _ in range(reps):
        lib.adha_remap(a.data_ptr(), Ls, b.data_ptr(), Ld, n, stream)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    p = phases(reset=True)
    tiles = max(1, p[4])                        # summed over the 8 consumer warps
    R = sum(w)
    per = [x / tiles for x in p[:4]]
    tot = sum(per)
    print(f"{name:28s} {2 * n * R / ms / 1e6:6.0f} GB/s  per tile & warp (clk): wait_full {per[0]:7.0f}  "
          f"permute {per[1]:6.0f}  barrier {per[2]:6.0f}  copy_out {per[3]:6.0f}  (sum {tot:6.0f}; "
          f"{100 * per[0] / tot:4.1f}% waiting for data)  producer wait_empty/tile {p[5] / (tiles / 8):7.0f}  "
          f"tails/warp {p[7] / 8 / 148 / reps:6.0f}  tiles/CTA {tiles / 8 / 148 / reps:5.1f}  "
          f"{ms * 1e3:7.1f} us/remap", flush=True)
    del a, b
    torch.cuda.empty_cache()
