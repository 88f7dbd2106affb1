"""Helpers for the GPU parity tests: run the CUDA path through the C ABI binding and
compare with the oracle element by element (small N) or on sampled records (full N)."""
from __future__ import annotations

import numpy as np

SENT = 0xA5


def torch():
    import torch as t
    return t


def to_dev(buf: np.ndarray):
    t = torch()
    return t.from_numpy(buf).to("cuda")


def sentinel_dev(nbytes: int):
    t = torch()
    return t.full((max(nbytes, 1),), SENT, dtype=t.uint8, device="cuda")


def run_remap(A, src_np, Ls, Ld, n):
    """CUDA remap of a host-built src buffer; returns the dst buffer on the host."""
    t = torch()
    src = to_dev(src_np) if src_np.size else t.zeros(1, dtype=t.uint8, device="cuda")
    dst = sentinel_dev(Ld.nbytes(n))
    A.remap(src, Ls, dst, Ld, n)
    t.cuda.synchronize()
    return dst.cpu().numpy()[: Ld.nbytes(n)]


def sample_records(n: int, T: int, k: int = 4096, seed: int = 0) -> np.ndarray:
    """Sampled record indices: random ones plus every edge that matters (first/last records,
    tile boundaries around the start and the end, the tail)."""
    rng = np.random.default_rng(seed)
    picks = set(rng.integers(0, n, size=min(k, n)).tolist())
    for i in list(range(0, min(n, 70))) + list(range(max(0, n - 70), n)):
        picks.add(i)
    tail_lo = (n // T) * T
    for base in (T, 2 * T, tail_lo, (n // T // 2) * T):
        for d in (-2, -1, 0, 1, 2):
            if 0 <= base + d < n:
                picks.add(base + d)
    return np.array(sorted(picks), dtype=np.int64)


def gather_fields_dev(buf, widths, base, stride, offset, recs):
    """Bytes of every field of the sampled records, gathered on the device -> host [k, R]."""
    t = torch()
    r = t.from_numpy(recs).to(buf.device)
    cols = []
    for f, w in enumerate(widths):
        idx = (int(base[f]) + r[:, None] * int(stride[f]) + int(offset[f])
               + t.arange(w, device=buf.device)[None, :])
        cols.append(buf[idx.reshape(-1)].reshape(-1, w))
    return t.cat(cols, 1).cpu().numpy()


def exact_chunked_check(O, src, ls, dst, ld, widths, n, chunk=1 << 22, sent=SENT, check_gaps=True):
    """EVERY payload byte of a full-size device remap against the oracle, by record-range chunks
    (exact by record locality): for records [lo, lo+m) the
    slice of each src region is copied to the host into an m-record instance of the src layout,
    the oracle remaps that instance, and each dst region's slice must equal the oracle's.  The
    bytes between dst regions must still hold the sentinel.  Host memory stays O(chunk)."""
    import os
    t = torch()
    F = len(widths)
    bs, ss, _, _ = O.field_addresses(widths, ls, n)
    bd, sd, _, _ = O.field_addresses(widths, ld, n)
    src_regs = sorted({(int(bs[f]), int(ss[f]), f) for f in range(F)}, key=lambda x: x[0])
    dst_regs = sorted({(int(bd[f]), int(sd[f]), f) for f in range(F)}, key=lambda x: x[0])
    # one representative field per region (the set above may hold several fields per base)
    src_regs = list({b: (b, s, f) for b, s, f in src_regs}.values())
    dst_regs = list({b: (b, s, f) for b, s, f in dst_regs}.values())
    threads = min(16, os.cpu_count() or 1)
    checked = 0
    for lo in range(0, n, chunk):
        m = min(chunk, n - lo)
        cbs, _, _, tot_s = O.field_addresses(widths, ls, m)
        cbd, _, _, tot_d = O.field_addresses(widths, ld, m)
        h = np.zeros(tot_s, np.uint8)
        for b, s, f in src_regs:
            h[cbs[f]: cbs[f] + m * s] = src[b + lo * s: b + (lo + m) * s].cpu().numpy()
        exp = np.zeros(tot_d, np.uint8)
        O.remap(h, ls, exp, ld, widths, m, threads=threads)
        for b, s, f in dst_regs:
            got = dst[b + lo * s: b + (lo + m) * s].cpu().numpy()
            want = exp[cbd[f]: cbd[f] + m * s]
            if not np.array_equal(got, want):
                bad = np.nonzero(got != want)[0]
                raise AssertionError(f"records [{lo}, {lo + m}): dst region at {b} (stride {s}) differs at "
                                     f"{bad.size} bytes, first record {lo + bad[0] // s}")
            checked += got.size
    ends = [(b, b + n * s) for b, s, _ in dst_regs] if check_gaps else []
    for (_, e0), (b1, _) in zip(ends, ends[1:]):
        if b1 > e0:
            assert bool((dst[e0:b1] == sent).all()), f"gap [{e0}, {b1}) overwritten"
    return checked
