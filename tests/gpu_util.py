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
