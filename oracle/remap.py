"""ctypes wrapper around oracle/remap_oracle.c plus numpy pack/unpack helpers.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Nothing here is imported by
the product package.

A layout is given to the oracle as ``(widths, cluster_of)``: ``widths[f]`` is
the byte width of field f (decl_index f) and ``cluster_of[f]`` is any label;
fields with equal labels share a cluster ([TYPE] Layout).  The
oracle re-derives canonical order, strides, offsets and 256-byte-aligned
region bases itself (remap_oracle.c header; SURVEY.md 8(c) reading Q3).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import List, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "remap_oracle.c")
_LIB = os.path.join(_HERE, "liboracle_remap.so")
_lib = None


class _Addr(ctypes.Structure):
    _fields_ = [("base", ctypes.c_uint64), ("stride", ctypes.c_uint64), ("offset", ctypes.c_uint64)]


class _AddrEx(ctypes.Structure):
    _fields_ = [("base", ctypes.c_uint64), ("stride", ctypes.c_uint64), ("offset", ctypes.c_uint64),
                ("block", ctypes.c_uint64), ("width", ctypes.c_uint64), ("region_bytes", ctypes.c_uint64)]


def build(force: bool = False) -> str:
    """Compile the C oracle with plain gcc -O2 (building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-pthread",
                               _SRC, "-o", _LIB])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u8p = ctypes.c_void_p
        i32p = ctypes.POINTER(ctypes.c_int32)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        L.oracle_field_addresses.argtypes = [ctypes.c_int, u32p, i32p, ctypes.c_int64,
                                             ctypes.POINTER(_Addr), ctypes.POINTER(ctypes.c_uint64)]
        L.oracle_field_addresses.restype = ctypes.c_int
        L.oracle_layout_bytes.argtypes = [ctypes.c_int, u32p, i32p, ctypes.c_int64]
        L.oracle_layout_bytes.restype = ctypes.c_uint64
        L.oracle_remap_range.argtypes = [u8p, i32p, u8p, i32p, ctypes.c_int, u32p,
                                         ctypes.c_int64, ctypes.c_int64, ctypes.c_int64]
        L.oracle_remap_range.restype = ctypes.c_int
        L.oracle_remap_threads.argtypes = [u8p, i32p, u8p, i32p, ctypes.c_int, u32p,
                                           ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int]
        L.oracle_remap_threads.restype = ctypes.c_int
        L.oracle_field_addresses_ex.argtypes = [ctypes.c_int, u32p, i32p, i32p, ctypes.c_uint32, ctypes.c_int64,
                                                ctypes.POINTER(_AddrEx), ctypes.POINTER(ctypes.c_uint64)]
        L.oracle_field_addresses_ex.restype = ctypes.c_int
        L.oracle_remap_ex.argtypes = [u8p, i32p, i32p, ctypes.c_uint32, u8p, i32p, i32p, ctypes.c_uint32,
                                      ctypes.c_int, u32p, ctypes.c_int64]
        L.oracle_remap_ex.restype = ctypes.c_int
        _lib = L
    return _lib


def _u32(a) -> ctypes.Array:
    return (ctypes.c_uint32 * len(a))(*[int(x) for x in a])


def _i32(a) -> ctypes.Array:
    return (ctypes.c_int32 * len(a))(*[int(x) for x in a])


def field_addresses(widths: Sequence[int], cluster_of: Sequence[int], n_records: int
                    ) -> Tuple[np.ndarray, np.ndarray, np.ndarray, int]:
    """(base[f], stride[f], offset[f], total_bytes) for an n_records layout instance."""
    F = len(widths)
    out = (_Addr * F)()
    tot = ctypes.c_uint64(0)
    rc = lib().oracle_field_addresses(F, _u32(widths), _i32(cluster_of), int(n_records), out,
                                      ctypes.byref(tot))
    if rc != 0:
        raise ValueError("oracle_field_addresses rejected the layout")
    base = np.array([out[f].base for f in range(F)], dtype=np.int64)
    stride = np.array([out[f].stride for f in range(F)], dtype=np.int64)
    offset = np.array([out[f].offset for f in range(F)], dtype=np.int64)
    return base, stride, offset, int(tot.value)


def layout_bytes(widths: Sequence[int], cluster_of: Sequence[int], n_records: int) -> int:
    return int(lib().oracle_layout_bytes(len(widths), _u32(widths), _i32(cluster_of), int(n_records)))


def _ptr(a: np.ndarray) -> int:
    assert a.dtype == np.uint8 and a.flags.c_contiguous
    return a.ctypes.data


def remap(src: np.ndarray, src_cluster_of: Sequence[int], dst: np.ndarray,
          dst_cluster_of: Sequence[int], widths: Sequence[int], n_records: int,
          lo: int = 0, hi: int | None = None, threads: int = 1) -> None:
    """dst[addr_d(f,i)..+w_f) = src[addr_s(f,i)..+w_f) for i in [lo, hi)."""
    hi = n_records if hi is None else hi
    need_s = layout_bytes(widths, src_cluster_of, n_records)
    need_d = layout_bytes(widths, dst_cluster_of, n_records)
    if src.nbytes < need_s or dst.nbytes < need_d:
        raise ValueError("buffer smaller than the layout")
    if n_records == 0 or hi == lo:
        return
    L = lib()
    if threads <= 1:
        rc = L.oracle_remap_range(_ptr(src), _i32(src_cluster_of), _ptr(dst), _i32(dst_cluster_of),
                                  len(widths), _u32(widths), int(n_records), int(lo), int(hi))
    else:
        rc = L.oracle_remap_threads(_ptr(src), _i32(src_cluster_of), _ptr(dst), _i32(dst_cluster_of),
                                    len(widths), _u32(widths), int(n_records), int(lo), int(hi),
                                    int(threads))
    if rc != 0:
        raise ValueError("oracle_remap rejected its arguments")


def pack(columns: List[np.ndarray], widths: Sequence[int], cluster_of: Sequence[int],
         n_records: int, fill: int = 0xA5) -> np.ndarray:
    """Lay per-field columns (column f: uint8 [N, w_f]) out in the layout; gaps = ``fill``."""
    base, stride, offset, total = field_addresses(widths, cluster_of, n_records)
    buf = np.full(total, fill, dtype=np.uint8)
    for f, w in enumerate(widths):
        if n_records == 0:
            continue
        region = buf[base[f]: base[f] + n_records * stride[f]].reshape(n_records, stride[f])
        region[:, offset[f]: offset[f] + w] = columns[f].reshape(n_records, w)
    return buf


def unpack(buf: np.ndarray, widths: Sequence[int], cluster_of: Sequence[int],
           n_records: int) -> List[np.ndarray]:
    """Per-field columns read back out of a layout buffer."""
    base, stride, offset, _ = field_addresses(widths, cluster_of, n_records)
    cols = []
    for f, w in enumerate(widths):
        if n_records == 0:
            cols.append(np.zeros((0, w), dtype=np.uint8))
            continue
        region = buf[base[f]: base[f] + n_records * stride[f]].reshape(n_records, stride[f])
        cols.append(np.ascontiguousarray(region[:, offset[f]: offset[f] + w]))
    return cols


def payload_mask(widths: Sequence[int], cluster_of: Sequence[int], n_records: int) -> np.ndarray:
    """Boolean mask over the layout buffer: True on bytes that belong to some field."""
    base, stride, offset, total = field_addresses(widths, cluster_of, n_records)
    m = np.zeros(total, dtype=bool)
    for f, w in enumerate(widths):
        if n_records == 0:
            continue
        region = m[base[f]: base[f] + n_records * stride[f]].reshape(n_records, stride[f])
        region[:, offset[f]: offset[f] + w] = True
    return m


# ----------------------------------------------------------------------------- generalised layouts
# (natural alignment, AoSoA blocks; SURVEY.md 8(f) N4 -- see remap_oracle.c header)


def _blocks(blocks, n_fields):
    return _i32a_or_null(blocks, n_fields)


def _i32a_or_null(xs, n):
    if xs is None:
        return None
    assert len(xs) == n
    return _i32(xs)


def field_addresses_ex(widths, cluster_of, n_records, blocks=None, aligned=False):
    """dict of per-field numpy arrays base/stride/offset/block/width/region_bytes, plus total."""
    F = len(widths)
    out = (_AddrEx * F)()
    tot = ctypes.c_uint64(0)
    rc = lib().oracle_field_addresses_ex(F, _u32(widths), _i32(cluster_of), _i32a_or_null(blocks, F),
                                         1 if aligned else 0, int(n_records), out, ctypes.byref(tot))
    if rc != 0:
        raise ValueError("oracle_field_addresses_ex rejected the layout")
    d = {k: np.array([getattr(out[f], k) for f in range(F)], dtype=np.int64)
         for k in ("base", "stride", "offset", "block", "width", "region_bytes")}
    d["total"] = int(tot.value)
    return d


def layout_bytes_ex(widths, cluster_of, n_records, blocks=None, aligned=False):
    return field_addresses_ex(widths, cluster_of, n_records, blocks, aligned)["total"]


def addr_ex(d, f, i):
    """Element address of field f of record(s) i (numpy-vectorised over i)."""
    B = int(d["block"][f])
    return (int(d["base"][f]) + (i // B) * (B * int(d["stride"][f])) + int(d["offset"][f]) * B
            + (i % B) * int(d["width"][f]))


def remap_ex(src, src_cluster_of, dst, dst_cluster_of, widths, n_records, src_blocks=None, src_aligned=False,
             dst_blocks=None, dst_aligned=False):
    F = len(widths)
    need_s = layout_bytes_ex(widths, src_cluster_of, n_records, src_blocks, src_aligned)
    need_d = layout_bytes_ex(widths, dst_cluster_of, n_records, dst_blocks, dst_aligned)
    if src.nbytes < need_s or dst.nbytes < need_d:
        raise ValueError("buffer smaller than the layout")
    if n_records == 0:
        return
    rc = lib().oracle_remap_ex(_ptr(src), _i32(src_cluster_of), _i32a_or_null(src_blocks, F), 1 if src_aligned else 0,
                               _ptr(dst), _i32(dst_cluster_of), _i32a_or_null(dst_blocks, F), 1 if dst_aligned else 0,
                               F, _u32(widths), int(n_records))
    if rc != 0:
        raise ValueError("oracle_remap_ex rejected its arguments")


def pack_ex(columns, widths, cluster_of, n_records, blocks=None, aligned=False, fill=0xA5):
    """Lay per-field columns out in a generalised layout: region bytes that are not payload are 0,
    bytes between regions are `fill`."""
    d = field_addresses_ex(widths, cluster_of, n_records, blocks, aligned)
    buf = np.full(d["total"], fill, dtype=np.uint8)
    for f in range(len(widths)):
        buf[d["base"][f]: d["base"][f] + d["region_bytes"][f]] = 0
    i = np.arange(n_records, dtype=np.int64)
    for f, w in enumerate(widths):
        if n_records == 0:
            continue
        a = addr_ex(d, f, i)
        idx = (a[:, None] + np.arange(w, dtype=np.int64)[None, :]).reshape(-1)
        buf[idx] = columns[f].reshape(-1)
    return buf


def unpack_ex(buf, widths, cluster_of, n_records, blocks=None, aligned=False):
    d = field_addresses_ex(widths, cluster_of, n_records, blocks, aligned)
    i = np.arange(n_records, dtype=np.int64)
    cols = []
    for f, w in enumerate(widths):
        a = addr_ex(d, f, i)
        idx = (a[:, None] + np.arange(w, dtype=np.int64)[None, :]).reshape(-1)
        cols.append(buf[idx].reshape(n_records, w) if n_records else np.zeros((0, w), np.uint8))
    return cols
