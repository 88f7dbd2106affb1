"""Counter-based generators for synthetic record data (see package docstring)."""
from __future__ import annotations

from typing import List, Sequence

import numpy as np

SEED_BASE = 14074859          # seed = 14074859 + config index

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 finaliser over uint64 counters (wrapping arithmetic)."""
    z = (x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15))
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def random_bytes(seed: int, nbytes: int, stream: int = 0) -> np.ndarray:
    """nbytes of the splitmix64 stream: 8-byte word k = splitmix64(seed + (stream<<40) + k)."""
    nwords = (nbytes + 7) // 8
    ctr = np.arange(nwords, dtype=np.uint64) + np.uint64((seed + (stream << 40)) & 0xFFFFFFFFFFFFFFFF)
    return splitmix64(ctr).view(np.uint8)[:nbytes].copy()


def _specials32(r: np.ndarray) -> np.ndarray:
    """fp32 special bit patterns chosen by r (uint64 random words)."""
    kind = (r % np.uint64(6)).astype(np.int64)
    payload = ((r >> np.uint64(8)) & np.uint64(0x3FFFFF)).astype(np.uint32)
    payload = np.where(payload == 0, np.uint32(1), payload)
    out = np.empty(r.shape, dtype=np.uint32)
    out[kind == 0] = np.uint32(0x7F800000) | payload[kind == 0]                    # sNaN (quiet bit clear)
    out[kind == 1] = np.uint32(0x7FC00000) | payload[kind == 1]                    # qNaN with payload
    out[kind == 2] = np.uint32(0x7F800000)                                         # +Inf
    out[kind == 3] = np.uint32(0xFF800000)                                         # -Inf
    out[kind == 4] = np.uint32(0x80000000)                                         # -0.0
    out[kind == 5] = np.uint32(0x00000001)                                         # smallest denormal
    sign = ((r >> np.uint64(40)) & np.uint64(1)).astype(np.uint32) << np.uint32(31)
    nan = (kind == 0) | (kind == 1)
    out[nan] |= sign[nan]
    return out


def _specials64(r: np.ndarray) -> np.ndarray:
    kind = (r % np.uint64(6)).astype(np.int64)
    payload = (r >> np.uint64(12)) & np.uint64(0x7FFFFFFFFFFFF)
    payload = np.where(payload == 0, np.uint64(1), payload)
    out = np.empty(r.shape, dtype=np.uint64)
    out[kind == 0] = np.uint64(0x7FF0000000000000) | payload[kind == 0]            # sNaN
    out[kind == 1] = np.uint64(0x7FF8000000000000) | payload[kind == 1]            # qNaN
    out[kind == 2] = np.uint64(0x7FF0000000000000)
    out[kind == 3] = np.uint64(0xFFF0000000000000)
    out[kind == 4] = np.uint64(0x8000000000000000)
    out[kind == 5] = np.uint64(1)
    return out


def field_columns(seed: int, n_records: int, widths: Sequence[int], overlay: bool = True
                  ) -> List[np.ndarray]:
    """Mode A: per-field uint8 columns [N, w_f] of random bits plus the fp-special overlay."""
    cols = []
    for f, w in enumerate(widths):
        b = random_bytes(seed, n_records * w, stream=f + 1).reshape(n_records, w)
        if overlay and w in (4, 8) and n_records > 0:
            sel_words = splitmix64(np.arange(n_records, dtype=np.uint64)
                                   + np.uint64(((seed ^ 0x5DEECE66D) + (f << 36)) & 0xFFFFFFFFFFFFFFFF))
            chosen = (sel_words & np.uint64(15)) == 0                        # 1/16 of the slots
            idx = np.nonzero(chosen)[0]
            if idx.size:
                r = splitmix64(sel_words[idx])
                if w == 4:
                    b[idx] = _specials32(r).view(np.uint8).reshape(-1, 4)
                else:
                    b[idx] = _specials64(r).view(np.uint8).reshape(-1, 8)
        cols.append(np.ascontiguousarray(b))
    return cols


def tagged_columns(n_records: int, widths: Sequence[int]) -> List[np.ndarray]:
    """Mode B: slot (i, f) = little-endian bytes of (i << 12) | f, truncated to w_f bytes."""
    i = np.arange(n_records, dtype=np.uint64)
    cols = []
    for f, w in enumerate(widths):
        tag = (i << np.uint64(12)) | np.uint64(f & 0xFFF)
        b = tag.view(np.uint8).reshape(n_records, 8)
        if w <= 8:
            col = b[:, :w]
        else:
            col = np.concatenate([b, np.full((n_records, w - 8), (f * 7 + 3) & 0xFF, np.uint8)], 1)
        cols.append(np.ascontiguousarray(col))
    return cols


def fill_random_device(t, seed: int) -> None:
    """Fill a CUDA uint8 tensor with seeded random bytes (torch RNG; plumbing, no layout math)."""
    import torch
    g = torch.Generator(device=t.device)
    g.manual_seed(int(seed))
    n = t.numel()
    # int32 draws reinterpreted as bytes, 4 bytes per draw
    words = torch.randint(-(2 ** 31), 2 ** 31 - 1, ((n + 3) // 4,), dtype=torch.int32,
                          device=t.device, generator=g)
    t.copy_(words.view(torch.uint8)[:n])


def config_widths(n_fields: int) -> List[int]:
    """BASELINE 'mixed 4/8-byte' record: w_i = 8 if i % 4 == 3 else 4."""
    return [8 if i % 4 == 3 else 4 for i in range(n_fields)]


def kmeans_widths() -> List[int]:
    """K-Means record: 32 fp32 features (Table 1; reading Q1)."""
    return [4] * 32


def medical_fields():
    """Medical record: the nine Table-2 field names, fp32 each (readings Q1, Q17)."""
    names = ["V1", "V2", "V3", "U1", "U2", "U3", "S", "T", "interpT"]
    return names, [4] * 9
