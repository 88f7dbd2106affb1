"""paper_1407_4859_b200 -- B200-native ADHA data-layout remap (arXiv 1407.4859).

Thin Python binding over the C ABI in ``include/adha.h`` (``libadha.so``, built
in-tree by ``python paper_1407_4859_b200/build.py`` or ``__graft_entry__.build()``).  Argument marshalling only:
every step of the remap runs in the library's sm_100a kernels, the planner in its
C++ host code.  There is no Python or CPU fallback: importing this package
raises if the library is missing.

    from paper_1407_4859_b200 import Layout, remap
    aos = Layout.aos([4, 4, 4])                      # {x,y,z}
    soa = Layout.soa([4, 4, 4])                      # {x}|{y}|{z}
    remap(src, aos, dst, soa, n_records)             # torch uint8 CUDA tensors
"""
from __future__ import annotations

import ctypes
import json
import os
from typing import List, Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libadha.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_1407_4859_b200/build.py` "
                      "(there is no fallback path)")
_lib = ctypes.CDLL(LIB_PATH)

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_cp = ctypes.c_char_p
_L = ctypes.c_void_p           # adha_layout*

_SIGS = {
    "adha_version": (_i32, []),
    "adha_status_string": (_cp, [ctypes.c_int]),
    "adha_last_error": (_cp, []),
    "adha_free": (None, [_vp]),
    "adha_layout_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_uint32), _i32, ctypes.POINTER(_i32),
                                          ctypes.POINTER(_L)]),
    "adha_layout_create_ex": (ctypes.c_int, [ctypes.POINTER(ctypes.c_uint32), _i32, ctypes.POINTER(_i32),
                                             ctypes.POINTER(_i32), ctypes.c_uint32, ctypes.POINTER(_L)]),
    "adha_layout_field_address_ex": (ctypes.c_int, [_L, _i32, _i64, ctypes.POINTER(_u64), ctypes.POINTER(ctypes.c_uint32),
                                                    ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32)]),
    "adha_layout_from_string": (ctypes.c_int, [_cp, ctypes.POINTER(_cp), ctypes.POINTER(ctypes.c_uint32), _i32,
                                               ctypes.POINTER(_L)]),
    "adha_layout_to_string": (ctypes.c_int, [_L, ctypes.POINTER(_cp), ctypes.c_char_p, ctypes.c_size_t,
                                             ctypes.POINTER(ctypes.c_size_t)]),
    "adha_layout_info": (ctypes.c_int, [_L, ctypes.POINTER(_i32), ctypes.POINTER(_i32), ctypes.POINTER(_u64)]),
    "adha_layout_clusters": (ctypes.c_int, [_L, ctypes.POINTER(_i32)]),
    "adha_layout_bytes": (ctypes.c_int, [_L, _i64, ctypes.POINTER(_u64)]),
    "adha_layout_field_address": (ctypes.c_int, [_L, _i32, _i64, ctypes.POINTER(_u64),
                                                 ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32)]),
    "adha_layout_destroy": (None, [_L]),
    "adha_remap": (ctypes.c_int, [_vp, _L, _vp, _L, _i64, _vp]),
    "adha_remap_regions": (ctypes.c_int, [ctypes.POINTER(_vp), _L, ctypes.POINTER(_vp), _L, _i64, _vp]),
    "adha_remap_chain": (ctypes.c_int, [ctypes.POINTER(_vp), ctypes.POINTER(_L), _i32, _i64, _vp]),
    "adha_remap_chain_route": (ctypes.c_int, [ctypes.POINTER(_L), _i32, _i64, ctypes.POINTER(_i32),
                                              ctypes.POINTER(_i32)]),
    "adha_shard_range": (ctypes.c_int, [_i64, _i32, _i32, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "adha_remap_sharded": (ctypes.c_int, [ctypes.POINTER(_vp), _L, ctypes.POINTER(_vp), _L, _i64, _i32,
                                          ctypes.POINTER(_i32), ctypes.POINTER(_vp)]),
    "adha_remap_host": (ctypes.c_int, [_vp, _L, _vp, _L, _i64, _vp, _u64, _vp]),
    "adha_remap_peer": (ctypes.c_int, [_vp, _L, _i32, _vp, _L, _i32, _i64, _vp]),
    "adha_remap_plan_describe": (ctypes.c_int, [_L, _L, ctypes.POINTER(_vp)]),
    "adha_remap_plan_describe_ex": (ctypes.c_int, [_L, _L, _i32, ctypes.POINTER(_vp)]),
    "adha_plan_ods": (ctypes.c_int, [_cp, _cp, _cp, _cp, ctypes.POINTER(_vp)]),
    "adha_plan_pdl": (ctypes.c_int, [_cp, _cp, _cp, ctypes.POINTER(_vp)]),
    "adha_plan_candidates": (ctypes.c_int, [_cp, _cp, _cp, ctypes.POINTER(_vp)]),
    "adha_section_run": (ctypes.c_int, [_vp, _L, _i64, ctypes.POINTER(_i32), _i32, _vp, _i64, _vp, _vp]),
    "adha_inplace_plan_create": (ctypes.c_int, [_L, _L, _i64, ctypes.POINTER(_vp)]),
    "adha_inplace_plan_info": (ctypes.c_int, [_vp, ctypes.POINTER(_u64), ctypes.POINTER(_u64)]),
    "adha_inplace_plan_describe": (ctypes.c_int, [_vp, ctypes.POINTER(_vp)]),
    "adha_inplace_plan_upload": (ctypes.c_int, [_vp, _vp, _u64, _vp]),
    "adha_remap_inplace": (ctypes.c_int, [_vp, _u64, _vp, _vp, _vp]),
    "adha_inplace_plan_destroy": (None, [_vp]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

STATUS = {0: "ADHA_OK", 1: "ADHA_ERR_INVALID_ARG", 2: "ADHA_ERR_PARSE", 3: "ADHA_ERR_LAYOUT_MISMATCH",
          4: "ADHA_ERR_CAPACITY", 5: "ADHA_ERR_ALIGNMENT", 6: "ADHA_ERR_OVERLAP", 7: "ADHA_ERR_TOO_LARGE",
          8: "ADHA_ERR_CUDA", 9: "ADHA_ERR_OOM", 10: "ADHA_ERR_UNSUPPORTED", 11: "ADHA_ERR_PLANNER"}


class AdhaError(RuntimeError):
    def __init__(self, status: int, detail: str):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{self.name}: {detail}")


def _check(rc: int) -> None:
    if rc != 0:
        raise AdhaError(rc, (_lib.adha_last_error() or b"").decode())


def version() -> int:
    return int(_lib.adha_version())


def _u32a(xs):
    return (ctypes.c_uint32 * len(xs))(*[int(x) for x in xs])


def _i32a(xs):
    return (_i32 * len(xs))(*[int(x) for x in xs])


def _names(names):
    if names is None:
        return None
    arr = (_cp * len(names))(*[n.encode() for n in names])
    return arr


class Layout:
    """Immutable layout descriptor: field widths + a partition into clusters (adha.h)."""

    ALIGNED = 1          # ADHA_LAYOUT_ALIGNED: natural (C-struct) alignment inside records

    def __init__(self, widths: Sequence[int], cluster_of: Sequence[int], names: Optional[Sequence[str]] = None,
                 blocks: Optional[Sequence[int]] = None, aligned: bool = False):
        """blocks[f]: AoSoA block of field f's cluster (1, 2, ..., 32; equal within a cluster);
        aligned: C-struct field alignment (adha_layout_create_ex)."""
        if len(widths) != len(cluster_of):
            raise ValueError("widths and cluster_of differ in length")
        h = _L()
        if blocks is None and not aligned:
            _check(_lib.adha_layout_create(_u32a(widths), len(widths), _i32a(cluster_of), ctypes.byref(h)))
        else:
            if blocks is not None and len(blocks) != len(widths):
                raise ValueError("one block per field")
            _check(_lib.adha_layout_create_ex(_u32a(widths), len(widths), _i32a(cluster_of),
                                              None if blocks is None else _i32a(blocks),
                                              Layout.ALIGNED if aligned else 0, ctypes.byref(h)))
        self._h = h
        self.names = list(names) if names is not None else None

    @classmethod
    def from_string(cls, text: str, names: Sequence[str], widths: Sequence[int]) -> "Layout":
        self = cls.__new__(cls)
        h = _L()
        _check(_lib.adha_layout_from_string(text.encode(), _names(names), _u32a(widths), len(widths),
                                            ctypes.byref(h)))
        self._h = h
        self.names = list(names)
        return self

    @classmethod
    def aos(cls, widths, names=None) -> "Layout":
        return cls(widths, [0] * len(widths), names)

    @classmethod
    def soa(cls, widths, names=None) -> "Layout":
        return cls(widths, list(range(len(widths))), names)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            try:
                _lib.adha_layout_destroy(h)
            except Exception:       # interpreter shutdown: the library may already be gone
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def info(self):
        nf, nc, rb = _i32(), _i32(), _u64()
        _check(_lib.adha_layout_info(self._h, ctypes.byref(nf), ctypes.byref(nc), ctypes.byref(rb)))
        return nf.value, nc.value, rb.value

    @property
    def n_fields(self) -> int:
        return self.info()[0]

    @property
    def n_clusters(self) -> int:
        return self.info()[1]

    @property
    def record_bytes(self) -> int:
        return self.info()[2]

    @property
    def cluster_of(self) -> List[int]:
        n = self.n_fields
        out = (_i32 * n)()
        _check(_lib.adha_layout_clusters(self._h, out))
        return list(out)

    def to_string(self, names: Optional[Sequence[str]] = None) -> str:
        names = names if names is not None else self.names
        need = ctypes.c_size_t()
        _check(_lib.adha_layout_to_string(self._h, _names(names), None, 0, ctypes.byref(need)))
        buf = ctypes.create_string_buffer(need.value + 1)
        _check(_lib.adha_layout_to_string(self._h, _names(names), buf, need.value + 1, ctypes.byref(need)))
        return buf.value.decode()

    def nbytes(self, n_records: int) -> int:
        n = int(n_records)
        cache = self.__dict__.setdefault("_nbytes", {})
        if n not in cache:
            out = _u64()
            _check(_lib.adha_layout_bytes(self._h, n, ctypes.byref(out)))
            if len(cache) > 64:
                cache.clear()
            cache[n] = out.value
        return cache[n]

    def field_address_ex(self, field: int, n_records: int):
        """(region_offset, stride, offset, block) of a field for an n_records instance."""
        r, s, o, b = _u64(), ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32()
        _check(_lib.adha_layout_field_address_ex(self._h, int(field), int(n_records), ctypes.byref(r),
                                                 ctypes.byref(s), ctypes.byref(o), ctypes.byref(b)))
        return r.value, s.value, o.value, b.value

    def field_address(self, field: int, n_records: int):
        """(region_offset, stride, offset) of a field for an n_records instance."""
        r, s, o = _u64(), ctypes.c_uint32(), ctypes.c_uint32()
        _check(_lib.adha_layout_field_address(self._h, int(field), int(n_records), ctypes.byref(r),
                                              ctypes.byref(s), ctypes.byref(o)))
        return r.value, s.value, o.value

    def __repr__(self):
        return f"Layout({self.to_string()})"


def _ptr(x) -> int:
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return int(x.data_ptr())
    if hasattr(x, "ctypes"):                        # numpy array (host buffers)
        return int(x.ctypes.data)
    raise TypeError(f"cannot take a pointer of {type(x)}")


def _stream(stream) -> int:
    if stream is None:
        import torch
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        if raw is not None:         # 0.3 us instead of 3 us for building a Stream object per call
            return int(raw(torch.cuda.current_device()))
        return int(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)


def _nbytes(x) -> Optional[int]:
    if hasattr(x, "numel") and hasattr(x, "element_size"):
        return int(x.numel() * x.element_size())
    if hasattr(x, "nbytes"):
        return int(x.nbytes)
    return None


def _check_size(x, need: int, what: str):
    nb = _nbytes(x)
    if nb is not None and nb < need:
        raise ValueError(f"{what} holds {nb} bytes, layout needs {need}")


def remap(src, src_layout: Layout, dst, dst_layout: Layout, n_records: int, stream=None) -> None:
    """Enqueue dst <- src on `stream` (default: torch's current stream).  adha.h adha_remap."""
    n = int(n_records)
    if n > 0:
        _check_size(src, src_layout.nbytes(n), "src")
        _check_size(dst, dst_layout.nbytes(n), "dst")
    _check(_lib.adha_remap(_ptr(src), src_layout.handle, _ptr(dst), dst_layout.handle, n, _stream(stream)))


def remap_regions(src_regions: Sequence, src_layout: Layout, dst_regions: Sequence, dst_layout: Layout,
                  n_records: int, stream=None) -> None:
    """Remap between per-cluster regions (adha_remap_regions): a dst region that aliases the src
    region of an identical cluster is left in place, so only the changed fields move."""
    s = (_vp * len(src_regions))(*[_ptr(x) for x in src_regions])
    d = (_vp * len(dst_regions))(*[_ptr(x) for x in dst_regions])
    if len(src_regions) != src_layout.n_clusters or len(dst_regions) != dst_layout.n_clusters:
        raise ValueError("one region per cluster")
    _check(_lib.adha_remap_regions(s, src_layout.handle, d, dst_layout.handle, int(n_records), _stream(stream)))


def remap_chain(buffers: Sequence, layouts: Sequence[Layout], n_records: int, stream=None) -> None:
    """buffers[k] (layouts[k]) -> buffers[k+1] (layouts[k+1]) for each k, one stream (adha_remap_chain)."""
    if len(buffers) != len(layouts):
        raise ValueError("one buffer per layout")
    for b, l in zip(buffers, layouts):
        if int(n_records) > 0:
            _check_size(b, l.nbytes(int(n_records)), "buffer")
    bufs = (_vp * len(buffers))(*[_ptr(b) for b in buffers])
    ls = (_L * len(layouts))(*[l.handle for l in layouts])
    _check(_lib.adha_remap_chain(bufs, ls, len(layouts), int(n_records), _stream(stream)))


CHAIN_ROUTES = {0: "per_hop", 1: "fused_small", 2: "fused_tiled"}


def remap_chain_route(layouts: Sequence[Layout], n_records: int):
    """(route, launches) adha_remap_chain takes for these layouts and N (disjoint buffers):
    route in CHAIN_ROUTES' values."""
    ls = (_L * len(layouts))(*[l.handle for l in layouts])
    r, k = _i32(), _i32()
    _check(_lib.adha_remap_chain_route(ls, len(layouts), int(n_records), ctypes.byref(r), ctypes.byref(k)))
    return CHAIN_ROUTES[r.value], k.value


def shard_range(n_total: int, n_shards: int, shard: int):
    lo, hi = _i64(), _i64()
    _check(_lib.adha_shard_range(int(n_total), int(n_shards), int(shard), ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def remap_sharded(src_shards: Sequence, src_layout: Layout, dst_shards: Sequence, dst_layout: Layout,
                  n_records_total: int, device_ids: Sequence[int], streams: Sequence) -> None:
    G = len(src_shards)
    if not (len(dst_shards) == len(device_ids) == len(streams) == G):
        raise ValueError("one src, dst, device and stream per shard")
    s = (_vp * G)(*[_ptr(x) for x in src_shards])
    d = (_vp * G)(*[_ptr(x) for x in dst_shards])
    st = (_vp * G)(*[_stream(x) for x in streams])
    _check(_lib.adha_remap_sharded(s, src_layout.handle, d, dst_layout.handle, int(n_records_total), G,
                                   _i32a(device_ids), st))


def remap_peer(src, src_layout: Layout, dst, dst_layout: Layout, n_records: int, stream=None) -> None:
    """Cross-device remap (adha_remap_peer): one kernel on src's device stores the records into
    dst's device over NVLink.  `stream` (default: the current stream of src's device) must
    belong to src's device."""
    import torch
    n = int(n_records)
    if n > 0:
        _check_size(src, src_layout.nbytes(n), "src")
        _check_size(dst, dst_layout.nbytes(n), "dst")
    sdev, ddev = src.device.index, dst.device.index
    if stream is None:
        stream = torch.cuda.current_stream(src.device)
    _check(_lib.adha_remap_peer(_ptr(src), src_layout.handle, sdev, _ptr(dst), dst_layout.handle, ddev, n,
                                _stream(stream)))


def remap_host(src_host, src_layout: Layout, dst_host, dst_layout: Layout, n_records: int, scratch,
               scratch_bytes: Optional[int] = None, stream=None) -> None:
    """Host buffers in, host buffers out, streamed through a device scratch buffer (adha_remap_host)."""
    n = int(n_records)
    if n > 0:
        _check_size(src_host, src_layout.nbytes(n), "src_host")
        _check_size(dst_host, dst_layout.nbytes(n), "dst_host")
    sb = scratch_bytes if scratch_bytes is not None else _nbytes(scratch)
    _check(_lib.adha_remap_host(_ptr(src_host), src_layout.handle, _ptr(dst_host), dst_layout.handle, n,
                                _ptr(scratch), int(sb), _stream(stream)))


def _take_string(p: ctypes.c_void_p) -> str:
    s = ctypes.cast(p, ctypes.c_char_p).value.decode()
    _lib.adha_free(p)
    return s


def plan_describe(src_layout: Layout, dst_layout: Layout, merged: bool = False) -> dict:
    """The compiled remap plan (adha_remap_plan_describe_ex): the component plan, or with
    merged=True the one-component plan used for small and mid-size multi-component remaps."""
    p = _vp()
    _check(_lib.adha_remap_plan_describe_ex(src_layout.handle, dst_layout.handle, 1 if merged else 0, ctypes.byref(p)))
    return json.loads(_take_string(p))


def _js(x) -> bytes:
    return (x if isinstance(x, str) else json.dumps(x)).encode()


def plan_ods(program, arch, section_id: str, device: str) -> str:
    """ODS layout (canonical string) of one section on one device (adha_plan_ods)."""
    p = _vp()
    _check(_lib.adha_plan_ods(_js(program), _js(arch), section_id.encode(), device.encode(), ctypes.byref(p)))
    return _take_string(p)


def plan_pdl(program, arch, profile=None) -> dict:
    """PDL plan as a dict (adha_plan_pdl)."""
    p = _vp()
    _check(_lib.adha_plan_pdl(_js(program), _js(arch), None if profile is None else _js(profile), ctypes.byref(p)))
    return json.loads(_take_string(p))


def plan_candidates(program, arch, profile=None) -> dict:
    """The run graph's nodes (adha_plan_candidates): every contiguous run x device with its ODS
    layout and execution estimate -- the (section, device, layout) triples a profile must cover."""
    p = _vp()
    _check(_lib.adha_plan_candidates(_js(program), _js(arch), None if profile is None else _js(profile),
                                     ctypes.byref(p)))
    return json.loads(_take_string(p))


def section_run(buf, layout: Layout, n_records: int, fields: Sequence[int], out, idx=None, n_out=None,
                stream=None) -> None:
    """Synthetic consumer section (adha_section_run): out[i] = sum_f x_f(r_i)^2 over the listed fp32
    fields, r_i = idx[i] (irregular gather) or i (streaming pass)."""
    n_out = int(n_out if n_out is not None else (idx.numel() if idx is not None else n_records))
    _check(_lib.adha_section_run(_ptr(buf), layout.handle, int(n_records), _i32a(fields), len(fields),
                                 _ptr(idx), n_out, _ptr(out), _stream(stream)))


class InplacePlan:
    """Plan of an in-place remap of an n_records buffer from src_layout to dst_layout
    (adha.h adha_inplace_plan_create; host only).  `buffer_bytes` is what the buffer needs
    (max of both layouts), `workspace_bytes` the device workspace; `upload(workspace)` copies
    the plan's tables there once, then `remap_inplace(buf, plan)` runs it."""

    def __init__(self, src_layout: Layout, dst_layout: Layout, n_records: int):
        h = _vp()
        _check(_lib.adha_inplace_plan_create(src_layout.handle, dst_layout.handle, int(n_records), ctypes.byref(h)))
        self._h = h
        self.src_layout, self.dst_layout, self.n_records = src_layout, dst_layout, int(n_records)
        b, w = _u64(), _u64()
        _check(_lib.adha_inplace_plan_info(h, ctypes.byref(b), ctypes.byref(w)))
        self.buffer_bytes, self.workspace_bytes = b.value, w.value
        self.workspace = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            try:
                _lib.adha_inplace_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    def describe(self) -> dict:
        p = _vp()
        _check(_lib.adha_inplace_plan_describe(self._h, ctypes.byref(p)))
        return json.loads(_take_string(p))

    def upload(self, workspace=None, stream=None):
        """Copy the tables into `workspace` (a uint8 CUDA tensor of >= workspace_bytes; allocated
        on the current device when None) and keep a reference to it."""
        if workspace is None:
            import torch
            workspace = torch.empty(max(self.workspace_bytes, 256), dtype=torch.uint8, device="cuda")
        _check(_lib.adha_inplace_plan_upload(self._h, _ptr(workspace), int(_nbytes(workspace)), _stream(stream)))
        self.workspace = workspace
        return workspace


def remap_inplace(buf, plan: InplacePlan, stream=None) -> None:
    """Enqueue the in-place remap of `buf` (uint8 CUDA tensor of >= plan.buffer_bytes) from the
    plan's src layout to its dst layout (adha_remap_inplace).  Uploads the plan on first use."""
    if plan.workspace is None:
        plan.upload(stream=stream)
    _check(_lib.adha_remap_inplace(_ptr(buf), int(_nbytes(buf)), plan._h, _ptr(plan.workspace), _stream(stream)))


def plan_layouts(plan: dict, field_names: Sequence[str], widths: Sequence[int]) -> List[Layout]:
    """One Layout per run of a PDL plan (adha_plan_pdl output), in execution order.  Consecutive
    runs with different layouts are the plan's remap edges."""
    return [Layout.from_string(r["layout"], field_names, widths) for r in plan["runs"]]


def run_plan_remaps(plan: dict, field_names: Sequence[str], widths: Sequence[int], buffers: Sequence,
                    n_records: int, stream=None) -> List[Layout]:
    """Materialise every run's layout of a PDL plan on the device: buffers[0] holds the records in
    the first run's layout; buffers[k] receives run k's layout (a chain of adha_remap on one
    stream).  Returns the layouts."""
    lays = plan_layouts(plan, field_names, widths)
    if len(buffers) != len(lays):
        raise ValueError("one buffer per run")
    if len(lays) > 1:
        remap_chain(buffers, lays, n_records, stream)
    return lays


__all__ = ["Layout", "AdhaError", "remap", "remap_regions", "remap_chain", "plan_layouts", "run_plan_remaps",
           "plan_candidates", "section_run", "InplacePlan", "remap_inplace", "shard_range", "remap_sharded", "remap_host",
           "plan_describe", "plan_ods", "plan_pdl", "version", "LIB_PATH"]
