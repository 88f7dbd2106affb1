// remap.cu -- host side of the ADHA remap on B200 (sm_100a): plan cache, per-device setup,
// kernel-parameter assembly and launch, and the remap entry points of the C ABI
// (adha_remap, adha_remap_regions, adha_remap_chain, adha_remap_chain_route, adha_remap_sharded,
// adha_remap_peer, adha_remap_plan_describe[_ex]).  Device code: kernels.cuh.
//
// What it computes (adha.h): for all records i and fields f
//     dst[addr_Ld(f,i) .. +w_f) = src[addr_Ls(f,i) .. +w_f)
// as a type-blind copy: integer loads/stores only, never an FP instruction (NaN payloads
// must survive, reading Q6).
//
// Routing per call: the tiled kernel (persistent CTAs, one per SM: a TMA producer warp
// streams src chunks of T-record tiles into shared memory, eight consumer warps permute them
// -- conflict-free 4-byte units, or PRMT byte groups for 1/2-byte units -- and write the dst
// chunks back with 16-byte stores), on the component plan at large N and on the merged
// one-component plan for multi-component remaps up to merge_bytes(); the direct kernel for
// remaps up to direct_bytes(plan) (latency bound) and layouts beyond the tiled limits (> 256
// fields, ...).  adha_remap_chain adds two one-launch routes: the fused direct chain for tiny
// chains and (opt-in) the tiled kernel in chain mode, which keeps each intermediate in L2
// between hops (chain_tiled below).
#include <cuda_runtime.h>

#include <cstdlib>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <tuple>
#include <type_traits>

#include "internal.h"
#include "kernels.cuh"
#include "remap_internal.h"

// ============================================================================ host side

namespace adha {

using namespace dev;

static_assert(sizeof(dev::TiledParams) <= 32764, "tiled kernel parameters exceed the 32764-byte limit");
static_assert(sizeof(dev::EntryTable<dev::CLASS_NENT[3]>) <= sizeof(dev::TableUpload::w) &&
                  sizeof(dev::GroupTable<dev::GCLASS_NG[1]>) <= sizeof(dev::TableUpload::w),
              "a table image must fit one upload kernel's parameters");
static_assert(sizeof(dev::ByteGroup) == 52, "ByteGroup layout");
static_assert(sizeof(dev::NaiveParams) <= 32764, "naive kernel parameters too large");

namespace detail {

typedef void (*TiledLauncher)(dim3, dim3, size_t, cudaStream_t, const TiledParams&, bool);

// Programmatic dependent launch of the remap kernels (ADHA_PDL=0 disables): a remap may start its
// prologue (barrier setup, plan-table copy into shared memory) while the previous kernel in the
// stream drains; its global memory accesses wait for that kernel (griddepcontrol.wait).
bool pdl_enabled() {
    const char* e = std::getenv("ADHA_PDL");
    return !(e && *e == '0');
}

// any kernel taking one parameter struct, with programmatic dependent launch allowed (pdl)
template <typename Prm>
void launch_pdl(void (*kernel)(Prm), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl, const Prm& p) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kernel, p);
}

// Launch with programmatic dependent launch allowed (pdl): the kernel may start while the previous
// kernel in the stream drains; it touches no global memory the previous kernel could write before
// its griddepcontrol.wait (kernels.cuh), only its parameters and its plan table.
template <typename... Args>
void launch_ex(void (*kernel)(Args...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
               const TiledParams& p) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kernel, p);
}

template <typename U, int CLS, bool TMAC>
void launch_tiled(dim3 grid, dim3 block, size_t smem, cudaStream_t st, const TiledParams& p, bool pdl) {
    launch_ex(&remap_tiled_kernel<U, CLASS_NENT[CLS], CLASS_EMAX[CLS], 0, 1, TMAC>, grid, block, smem, st, pdl, p);
}

template <typename U, int CLS, bool TMAC>
const void* tiled_fn() {
    constexpr int NENT = CLASS_NENT[CLS];
    constexpr int EMAX = CLASS_EMAX[CLS];
    return (const void*)&remap_tiled_kernel<U, NENT, EMAX, 0, 1, TMAC>;
}

// fused-chain instantiations (classes 0..2; chain_tiled never picks the largest class)
template <typename U, int CLS>
void launch_chain(dim3 grid, dim3 block, size_t smem, cudaStream_t st, const TiledParams& p, bool pdl) {
    launch_ex(&remap_tiled_kernel<U, CLASS_NENT[CLS], CLASS_EMAX[CLS], 0, 1, false, true>, grid, block, smem, st, pdl, p);
}
template <typename U, int CLS>
const void* chain_fn() {
    return (const void*)&remap_tiled_kernel<U, CLASS_NENT[CLS], CLASS_EMAX[CLS], 0, 1, false, true>;
}
template <typename U>
TiledLauncher pick_chain_cls(int cls, const void** fn) {
    switch (cls) {
        case 0: *fn = chain_fn<U, 0>(); return &launch_chain<U, 0>;
        case 1: *fn = chain_fn<U, 1>(); return &launch_chain<U, 1>;
        default: *fn = chain_fn<U, 2>(); return &launch_chain<U, 2>;
    }
}
TiledLauncher pick_chain(uint32_t unit, int cls, const void** fn) {
    if (unit == 4) return pick_chain_cls<uint32_t>(cls, fn);
    if (unit == 2) return pick_chain_cls<uint16_t>(cls, fn);
    return pick_chain_cls<uint8_t>(cls, fn);
}

// consumer cp.async loader instantiations (4-byte units)
template <int CLS>
void launch_cpa(dim3 grid, dim3 block, size_t smem, cudaStream_t st, const TiledParams& p, bool pdl) {
    launch_ex(&remap_tiled_kernel<uint32_t, CLASS_NENT[CLS], CLASS_EMAX[CLS], 0, 1, false, false, true>, grid, block, smem, st, pdl, p);
}
template <int CLS>
const void* cpa_fn() {
    return (const void*)&remap_tiled_kernel<uint32_t, CLASS_NENT[CLS], CLASS_EMAX[CLS], 0, 1, false, false, true>;
}
TiledLauncher pick_cpa(int cls, const void** fn) {
    switch (cls) {
        case 0: *fn = cpa_fn<0>(); return &launch_cpa<0>;
        case 1: *fn = cpa_fn<1>(); return &launch_cpa<1>;
        case 2: *fn = cpa_fn<2>(); return &launch_cpa<2>;
        default: *fn = cpa_fn<3>(); return &launch_cpa<3>;
    }
}

template <typename U, bool TMAC>
TiledLauncher pick_cls(int cls, const void** fn) {
    switch (cls) {
        case 0: *fn = tiled_fn<U, 0, TMAC>(); return &launch_tiled<U, 0, TMAC>;
        case 1: *fn = tiled_fn<U, 1, TMAC>(); return &launch_tiled<U, 1, TMAC>;
        case 2: *fn = tiled_fn<U, 2, TMAC>(); return &launch_tiled<U, 2, TMAC>;
        default: *fn = tiled_fn<U, 3, TMAC>(); return &launch_tiled<U, 3, TMAC>;
    }
}

template <int GC, bool TMAC>
void launch_groups(dim3 grid, dim3 block, size_t smem, cudaStream_t st, const TiledParams& p, bool pdl) {
    launch_ex(&remap_tiled_kernel<uint8_t, 32, 1, GCLASS_NG[GC], GCLASS_GMAX[GC], TMAC>, grid, block, smem, st, pdl, p);
}
template <int GC, bool TMAC>
const void* groups_fn() {
    return (const void*)&remap_tiled_kernel<uint8_t, 32, 1, GCLASS_NG[GC], GCLASS_GMAX[GC], TMAC>;
}

TiledLauncher pick_groups(int gcls, bool tma, const void** fn) {
    if (tma) {
        if (gcls == 0) { *fn = groups_fn<0, true>(); return &launch_groups<0, true>; }
        *fn = groups_fn<1, true>();
        return &launch_groups<1, true>;
    }
    if (gcls == 0) { *fn = groups_fn<0, false>(); return &launch_groups<0, false>; }
    *fn = groups_fn<1, false>();
    return &launch_groups<1, false>;
}

TiledLauncher pick(uint32_t unit, int cls, bool tma, const void** fn) {
    if (tma) {
        if (unit == 4) return pick_cls<uint32_t, true>(cls, fn);
        if (unit == 2) return pick_cls<uint16_t, true>(cls, fn);
        return pick_cls<uint8_t, true>(cls, fn);
    }
    if (unit == 4) return pick_cls<uint32_t, false>(cls, fn);
    if (unit == 2) return pick_cls<uint16_t, false>(cls, fn);
    return pick_cls<uint8_t, false>(cls, fn);
}

struct PlanCache {
    std::mutex mu;
    std::map<std::tuple<uint64_t, uint64_t, bool>, std::shared_ptr<const RemapPlan>> plans;
    std::set<std::tuple<int, const void*>> attr_done;
    std::map<int, int> sm_count;
};
PlanCache& cache() {
    static PlanCache c;
    return c;
}

std::shared_ptr<const RemapPlan> get_plan(const Layout& ls, const Layout& ld, bool merged = false) {
    PlanCache& c = cache();
    std::lock_guard<std::mutex> g(c.mu);
    auto key = std::make_tuple(ls.id, ld.id, merged);
    auto it = c.plans.find(key);
    if (it != c.plans.end()) return it->second;
    if (c.plans.size() > 4096) c.plans.clear();
    auto p = std::make_shared<const RemapPlan>(compile_plan(ls, ld, merged));
    c.plans.emplace(key, p);
    return p;
}

adha_status cuda_fail(cudaError_t e, const char* what) {
    return fail(ADHA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Device copies of the plan tables (EntryTable / GroupTable images, <= 25 KB each).  The tiled
// kernel copies its table from here into shared memory with coalesced 16-byte loads; passing it
// in the kernel parameters instead cost a larger launch (~30 KB of parameters: +2.5 us) and
// serialised lane-divergent constant-bank loads.  A table is uploaded once per (key, device):
// synchronously on an internal stream at its first use, or -- when the caller's stream is being
// captured into a CUDA graph -- by a small kernel in the captured stream itself (the graph then
// re-uploads on every replay; the copy is not marked resident, so the next uncaptured call
// uploads it for good).  Memory: a 4 MB static __device__ arena per device, then 4 MB cudaMalloc
// chunks; all live as long as the process (a table is never freed: in-flight kernels may still
// read it).
__device__ __align__(256) uint8_t g_plan_tables[4u << 20];   // ~160 plan tables per device

struct TableStore {
    std::mutex mu;
    struct Entry { const void* dptr; bool ready; };
    std::map<std::pair<std::string, int>, Entry> tables;
    struct Chunk { uint8_t* base; size_t used, size; };
    std::map<int, Chunk> chunk;
    std::map<int, cudaStream_t> upload_stream;
};
TableStore& tables() {
    static TableStore t;
    return t;
}

adha_status device_table(const std::string& key, const std::vector<uint32_t>& img, cudaStream_t st,
                         uint64_t* out, bool* enqueued) {
    *enqueued = false;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    TableStore& T = tables();
    std::lock_guard<std::mutex> g(T.mu);
    auto it = T.tables.find({key, dev});
    if (it != T.tables.end() && it->second.ready) {
        *out = (uint64_t)(uintptr_t)it->second.dptr;
        return ADHA_OK;
    }
    const size_t bytes = (img.size() * 4 + 15) / 16 * 16;
    if (bytes > sizeof(TableUpload::w)) return fail(ADHA_ERR_UNSUPPORTED, "plan table too large");
    const void* dptr = nullptr;
    if (it != T.tables.end()) {
        dptr = it->second.dptr;
    } else {
        TableStore::Chunk& C = T.chunk[dev];
        if (!C.base) {
            // the first chunk is the module's static arena: no allocation, so a first call
            // inside CUDA-graph capture works too
            void* a = nullptr;
            e = cudaGetSymbolAddress(&a, g_plan_tables);
            if (e != cudaSuccess) return cuda_fail(e, "cudaGetSymbolAddress (plan tables)");
            C = {static_cast<uint8_t*>(a), 0, sizeof(g_plan_tables)};
        }
        if (C.used + bytes > C.size) {
            void* m = nullptr;
            e = cudaMalloc(&m, 4u << 20);
            if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc (plan tables)");
            C = {static_cast<uint8_t*>(m), 0, 4u << 20};
        }
        dptr = C.base + C.used;
        C.used += (bytes + 255) / 256 * 256;
        it = T.tables.emplace(std::make_pair(key, dev), TableStore::Entry{dptr, false}).first;
    }
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    e = cudaStreamIsCapturing(st, &cs);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamIsCapturing");
    if (cs != cudaStreamCaptureStatusNone) {
        auto U = std::make_unique<TableUpload>();
        std::memset(U.get(), 0, sizeof(TableUpload));
        std::memcpy(U->w, img.data(), img.size() * 4);
        U->dst = (uint64_t)(uintptr_t)dptr;
        U->n16 = (uint32_t)(bytes / 16);
        table_upload_kernel<<<1, 256, 0, st>>>(*U);
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "table_upload_kernel launch");
        *enqueued = true;                  // the remap that reads it must not launch early (no PDL)
    } else {
        cudaStream_t& us = T.upload_stream[dev];
        if (!us && (e = cudaStreamCreateWithFlags(&us, cudaStreamNonBlocking)) != cudaSuccess)
            return cuda_fail(e, "cudaStreamCreateWithFlags");
        e = cudaMemcpyAsync(const_cast<void*>(dptr), img.data(), img.size() * 4, cudaMemcpyHostToDevice, us);
        if (e == cudaSuccess) e = cudaStreamSynchronize(us);
        if (e != cudaSuccess) return cuda_fail(e, "plan table upload");
        it->second.ready = true;
    }
    *out = (uint64_t)(uintptr_t)dptr;
    return ADHA_OK;
}

// per-device setup: SM count and the kernel's dynamic shared memory opt-in
adha_status device_setup(const void* fn, int* n_sm, int threads = NTHREADS) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    PlanCache& c = cache();
    std::lock_guard<std::mutex> g(c.mu);
    auto it = c.sm_count.find(dev);
    if (it == c.sm_count.end()) {
        int sms = 0;
        e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
        it = c.sm_count.emplace(dev, sms).first;
    }
    *n_sm = it->second;
    if (fn && !c.attr_done.count({dev, fn})) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
        cudaFuncAttributes fa;
        e = cudaFuncGetAttributes(&fa, fn);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncGetAttributes");
        if (fa.maxThreadsPerBlock < threads)       // register budget regression guard
            return fail(ADHA_ERR_UNSUPPORTED, "remap_tiled_kernel uses " + std::to_string(fa.numRegs) +
                                                  " registers: cannot launch " + std::to_string(threads) + " threads");
        c.attr_done.insert({dev, fn});
    }
    return ADHA_OK;
}

// Direct global->global kernel: the fallback beyond the tiled kernel's limits, and the
// latency path for small remaps (a handful of KB, where one launch with small parameters
// and one load/store per unit beats staging through shared memory).
// a dst cluster whose region IS the region of its src cluster (adha_remap_regions aliasing, only
// accepted for identity components): nothing moves there, so the direct path leaves its fields
// and its region alone (adha.h: "left untouched")
inline bool aliased(const uint8_t* src, const Layout& ls, const std::vector<uint64_t>& bs, const uint8_t* dst,
                    const Layout& ld, const std::vector<uint64_t>& bd, int f) {
    return (uintptr_t)src + bs[ls.cluster[f]] == (uintptr_t)dst + bd[ld.cluster[f]];
}

template <int NF>
adha_status launch_naive_t(const uint8_t* src, const Layout& ls, const std::vector<uint64_t>& bs, uint8_t* dst,
                           const Layout& ld, const std::vector<uint64_t>& bd, int64_t lo, int64_t hi,
                           cudaStream_t st) {
    int n_sm = 0;
    adha_status s = device_setup(nullptr, &n_sm);
    if (s != ADHA_OK) return s;
    std::vector<int> moved;
    for (int f = 0; f < ls.n_fields; ++f)
        if (!aliased(src, ls, bs, dst, ld, bd, f)) moved.push_back(f);
    auto P = std::make_unique<NaiveParamsT<NF>>();
    for (size_t f0 = 0; f0 < moved.size(); f0 += NF) {
        std::memset(P.get(), 0, sizeof(NaiveParamsT<NF>));
        P->src = (uint64_t)(uintptr_t)src;
        P->dst = (uint64_t)(uintptr_t)dst;
        P->n_records = hi - lo;
        P->lo = lo;
        const int nf = (int)std::min<size_t>(NF, moved.size() - f0);
        P->n_fields = (uint32_t)nf;
        for (int k = 0; k < nf; ++k) {
            const int f = moved[f0 + k];
            const int cs = ls.cluster[f], cd = ld.cluster[f];
            uint32_t sbl = 0, dbl = 0;
            while ((1u << sbl) < ls.block[cs]) ++sbl;
            while ((1u << dbl) < ld.block[cd]) ++dbl;
            P->f[k] = {bs[cs], bd[cd], (uint32_t)ls.stride[cs], (uint32_t)ld.stride[cd], ls.offset[f], ld.offset[f],
                       ls.width[f], sbl | (dbl << 8)};
        }
        const int64_t total = (hi - lo) * (int64_t)nf;
        const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, (int64_t)n_sm * 16));
        launch_pdl(&remap_naive_kernel<NF>, dim3((unsigned)blocks), dim3(256), 0, st, pdl_enabled(), *P);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "remap_naive_kernel launch");
    }
    return ADHA_OK;
}

adha_status launch_naive(const uint8_t* src, const Layout& ls, const std::vector<uint64_t>& bs, uint8_t* dst,
                         const Layout& ld, const std::vector<uint64_t>& bd, int64_t lo, int64_t hi,
                         cudaStream_t st) {
    // dst clusters with padding or AoSoA blocks: zero their regions first (the copy fills the
    // payload); an aliased cluster is the caller's src data and is not touched
    ZeroParams Z;
    std::memset(&Z, 0, sizeof Z);
    for (int c = 0; c < ld.n_clusters(); ++c) {
        if (ld.stride[c] == ld.payload(c) && ld.block[c] == 1) continue;
        if (aliased(src, ls, bs, dst, ld, bd, ld.members[c][0])) continue;
        if (Z.n == ZMAX) {
            zero_kernel<<<256, 256, 0, st>>>(Z);
            Z.n = 0;
        }
        Z.ptr[Z.n] = (uint64_t)(uintptr_t)dst + bd[c];
        Z.bytes[Z.n] = ld.region_bytes(c, hi);
        ++Z.n;
    }
    if (Z.n) {
        zero_kernel<<<256, 256, 0, st>>>(Z);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "zero_kernel launch");
    }
    if (ls.n_fields <= SMALL_NF) return launch_naive_t<SMALL_NF>(src, ls, bs, dst, ld, bd, lo, hi, st);
    return launch_naive_t<MAXF>(src, ls, bs, dst, ld, bd, lo, hi, st);
}

uint64_t small_bytes() {
    const char* e = std::getenv("ADHA_SMALL_BYTES");   // read per call: tests switch the path
    return e && *e ? (uint64_t)std::strtoull(e, nullptr, 10) : (uint64_t)(64u << 10);
}

// Payload up to which a remap takes the direct kernel instead of the tiled one.  The tiled kernel
// has a fixed cost per launch (pipeline fill, table copy, tails: 4-6 us for one component, 4.6 us
// for Medical's 7 on the merged plan, 9-10 us for C3's 24, replayed back to back with
// programmatic dependent launch; tools/small_path_probe.py, profiles/r02ax_small_path.log) while
// the direct kernel streams at ~1 TB/s for 4-byte units and ~0.3-0.5 TB/s for 1-/2-byte units
// after ~2 us.  Crossovers measured on B200: 1-4 MB below 16 components (4 MB: K-Means
// SoA->AoS 6.3 vs 8.3 us tiled vs direct, C2 6.0 vs 5.4), 8-16 MB for C3's 24 components.
// ADHA_SMALL_BYTES, when set, overrides this (tests force either path with it).
uint64_t direct_bytes(const RemapPlan& p) {
    const char* e = std::getenv("ADHA_SMALL_BYTES");
    if (e && *e) return (uint64_t)std::strtoull(e, nullptr, 10);
    return p.comps.size() >= 16 ? (8ull << 20) : (2ull << 20);
}


// Payload up to which a multi-component remap uses the merged plan (ADHA_MERGE_BYTES overrides;
// 0 disables).  Per-component tiles keep every tile near 48 KB at large N; at small and mid N
// they leave a CTA one short tile per component, each paying the pipeline's latency.  A merged
// tile carries one chunk per src cluster, so with many src clusters its chunks get small and the
// TMA unit's cost per bulk copy binds (profiles/r02aa_pieces.log): 64 MB for > 32 src clusters,
// 128 MB otherwise -- and no limit for <= 8 src clusters when the component plan has identity
// components (singleton clusters on both sides), whose separate copy-through tiles lose to whole-
// record tiles at any size.  Measured on B200 (profiles/r02ax_small_path.log, r02bf_small.log,
// r02bh_merge_probe.log): C3's SoA -> hybrid (64 src clusters) 32 MB 30.9 us merged vs 46.9 per
// component, 128 MB 89.1 vs 71.8; hybrid -> SoA (24) 128 MB 66.8 vs 74.7, 512 MB 195.8 vs 188.9;
// Medical AoSV -> SoA (7, six identity components) 2 GB 655 vs 671 us, SoA -> AoSV 653 vs 683;
// without identity components (K-Means 4xAoS8 -> SoA, C2 2xAoS8 -> SoA) 2 GB merged is 1-2 %
// slower.
uint64_t merge_bytes(const RemapPlan& p) {
    const char* e = std::getenv("ADHA_MERGE_BYTES");
    if (e && *e) return (uint64_t)std::strtoull(e, nullptr, 10);
    const size_t ns = p.src_order.size();
    bool identity = false;
    for (const auto& K : p.comps) identity = identity || K.identity;
    if (ns <= 8 && identity) return ~0ull;
    return ns > 32 ? (64ull << 20) : (128ull << 20);
}

adha_status validate(const void* src, const adha_layout* hs, const void* dst, const adha_layout* hd, int64_t n,
                     Checked* out, bool device_buffers) {
    if (!hs || !hd) return fail(ADHA_ERR_INVALID_ARG, "null layout");
    if (n < 0) return fail(ADHA_ERR_INVALID_ARG, "n_records < 0");
    const Layout& ls = hs->L;
    const Layout& ld = hd->L;
    if (ls.n_fields != ld.n_fields) return fail(ADHA_ERR_LAYOUT_MISMATCH, "layouts differ in field count");
    for (int f = 0; f < ls.n_fields; ++f)
        if (ls.width[f] != ld.width[f])
            return fail(ADHA_ERR_LAYOUT_MISMATCH, "field " + std::to_string(f) + " differs in width");
    if (!ls.region_bases(n, out->bs, &out->bytes_s) || !ld.region_bases(n, out->bd, &out->bytes_d))
        return fail(ADHA_ERR_TOO_LARGE, "N * record bytes overflows");
    if (n == 0) return ADHA_OK;
    if (!src || !dst) return fail(ADHA_ERR_INVALID_ARG, "null buffer");
    if (device_buffers && (((uintptr_t)src & 255) || ((uintptr_t)dst & 255)))
        return fail(ADHA_ERR_ALIGNMENT, "src and dst must be 256-byte aligned");
    const uintptr_t s0 = (uintptr_t)src, s1 = s0 + out->bytes_s, d0 = (uintptr_t)dst, d1 = d0 + out->bytes_d;
    if (s0 < d1 && d0 < s1) return fail(ADHA_ERR_OVERLAP, "src and dst ranges overlap");
    return ADHA_OK;
}

adha_status remap_checked(const uint8_t* src, const Layout& ls, uint8_t* dst, const Layout& ld, int64_t n,
                          const Checked& ck, cudaStream_t st) {
    if (n == 0) return ADHA_OK;
    auto plan = get_plan(ls, ld);
    // Multi-component remaps of up to merge_bytes() run on the merged plan (one component, whole
    // records per tile) unless a dst region aliases its src region (remap_regions: those
    // clusters must stay untouched, which needs their own skipped component).
    // the direct-path threshold is the component plan's (its crossover with the tiled kernel
    // was measured per component count; the merged plan only replaces the tiled side of it)
    const uint64_t thr = (ck.dst_local && ck.src_local) ? direct_bytes(*plan) : small_bytes();
    // (a src in host memory keeps the component plan: its tiles read larger chunks over PCIe)
    if (plan->comps.size() > 1 && ck.src_local && (uint64_t)n * ls.record_bytes <= merge_bytes(*plan)) {
        bool alias = false;
        for (const auto& K : plan->comps)
            alias = alias || (K.identity && (uintptr_t)src + ck.bs[K.src_clusters[0]] ==
                                                (uintptr_t)dst + ck.bd[K.dst_clusters[0]]);
        if (!alias) {
            auto mp = get_plan(ls, ld, true);
            if (mp->tiled) plan = mp;
        }
    }
    // small and mid-size remaps (direct_bytes above) run faster on the direct kernel; a dst in
    // pinned host or peer memory keeps the latency-only threshold (the tiled kernel's 16-byte
    // stores suit PCIe / NVLink writes better than the direct kernel's per-field stores)
    if (!plan->tiled || (uint64_t)n * ls.record_bytes <= thr)
        return launch_naive(src, ls, ck.bs, dst, ld, ck.bd, 0, n, st);

    int n_sm = 0;
    adha_status s = device_setup(nullptr, &n_sm);
    if (s != ADHA_OK) return s;

    auto P = std::make_unique<TiledParams>();
    std::memset(P.get(), 0, sizeof(TiledParams));
    P->src = (uint64_t)(uintptr_t)src;
    P->dst = (uint64_t)(uintptr_t)dst;
    P->n_records = n;
    P->stage_bytes = plan->stage_bytes;
    P->s_in = plan->s_in;
    P->s_out = plan->s_out;
    {
        const char* h = std::getenv("ADHA_L2_HINTS");   // bit 0: loads evict_first, bit 1: stores evict_first
        P->l2_hints = h && *h ? (uint32_t)std::strtoul(h, nullptr, 10) : 0u;
        const char* ts = std::getenv("ADHA_TMA_SPLIT");   // bytes per TMA bulk load (multiple of 16), 0 = whole chunk
        P->tma_split = ts && *ts ? ((uint32_t)std::strtoul(ts, nullptr, 10) & ~15u) : 0u;
        const char* b = std::getenv("ADHA_TILE_ORDER");   // "blocked" | default interleaved
        P->blocked = (b && std::string(b) == "blocked") ? 1u : 0u;
    }
    P->n_comp = (uint32_t)plan->comps.size();
    P->unit = plan->unit;
    int64_t tiles = 0;
    uint32_t sc = 0, dc = 0, fi = 0;
    for (size_t k = 0; k < plan->comps.size(); ++k) {
        const RemapPlan::Comp& K = plan->comps[k];
        CompDesc& D = P->comp[k];
        D.T = call_tile(*plan, (int)k, n, n_sm);
        D.tile_bytes = D.T * K.Rs;
        D.out_bytes = D.T * K.Rd;
        // an identity component whose dst region is its src region moves nothing (NEXT N1)
        const bool skip = K.identity && P->src + ck.bs[K.src_clusters[0]] == P->dst + ck.bd[K.dst_clusters[0]];
        D.flags = (uint16_t)((skip ? CF_SKIP : 0) | (K.zero_out ? CF_ZERO_OUT : 0) | (K.tail_zero ? CF_TAIL_ZERO : 0));
        D.n_tiles = skip ? 0 : n / D.T;
        D.tile_base = tiles;
        tiles += D.n_tiles;
        D.identity = K.identity ? 1 : 0;
        D.instr_base = K.instr_base;
        D.n_instr = K.n_instr;
        // byte-group mode staggers chunk k of a component by 32*k bytes (cumulative: chunk k starts
        // 32 bytes after the end of chunk k-1), so equal offsets in chunks k and k+1..k+3 fall in
        // different banks (see remap_plan.cpp)
        const bool stagger = plan->byte_groups;
        D.sc_lo = (uint16_t)sc;
        uint32_t off = 0, idx = 0;
        for (int c : K.src_clusters) {
            P->srcc[sc++] = {ck.bs[c], (uint32_t)ls.stride[c], off + (stagger ? 32u * idx++ : 0u)};
            off += D.T * (uint32_t)ls.stride[c];
        }
        D.sc_hi = (uint16_t)sc;
        D.dc_lo = (uint16_t)dc;
        off = 0;
        idx = 0;
        for (int c : K.dst_clusters) {
            P->dstc[dc++] = {ck.bd[c], (uint32_t)ld.stride[c], off + (stagger ? 32u * idx++ : 0u)};
            off += D.T * (uint32_t)ld.stride[c];
        }
        D.dc_hi = (uint16_t)dc;
        D.f_lo = (uint16_t)fi;
        fi += (uint32_t)K.fields.size();
        D.f_hi = (uint16_t)fi;
    }
    P->total_tiles = tiles;
    P->n_ent = plan->byte_groups ? plan->n_groups_total : (uint32_t)plan->ent_off.size();
    P->n_srcc = sc;
    P->n_dstc = dc;
    // Write-back mode (unit mode).  TMA bulk stores by a 10th warp when every component with
    // tiles has ONE dst chunk of >= 32 KB per tile and at most 8 src chunks: K-Means SoA->4xAoS8
    // +1.3 %, 4xAoS8->AoS +3 % (profiles/r01_notes.md).  Many small dst chunks queue behind the
    // loads in the per-SM TMA engine (C2 AoS->SoA -26 % if forced) and more src chunks gain
    // nothing (Medical SoA->AoS, 9), so those keep the consumers' STG write-back.  Only for dst
    // in this device's HBM.  ADHA_COPYOUT = stg | tma overrides (tests, A/B).
    {
        const char* cm = std::getenv("ADHA_COPYOUT");
        bool tma = false;
        if (ck.dst_local) {
            if (cm && std::strcmp(cm, "tma") == 0) {
                tma = true;
            } else if (!(cm && std::strcmp(cm, "stg") == 0)) {
                bool any = false;
                tma = true;
                for (size_t k = 0; k < plan->comps.size(); ++k) {
                    if (P->comp[k].n_tiles == 0) continue;
                    any = true;
                    const RemapPlan::Comp& K = plan->comps[k];
                    // byte-group mode: the slower permutation gains more from the overlap (2-byte
                    // SoA->AoS +16 % with 16 src chunks), 25 src chunks lose (1-byte, -6 %)
                    const size_t max_src = plan->byte_groups ? 16 : 8;
                    if (K.dst_clusters.size() != 1 || K.src_clusters.size() > max_src || P->comp[k].out_bytes < 32768)
                        tma = false;
                }
                tma = tma && any;
            }
        }
        P->tma_copy = tma ? 1u : 0u;
    }
    // Loader: the producer warp's TMA bulk copies, or (cpa) the consumers' own cp.async, issued
    // for tile i+s_in right after tile i's output barrier.  Each TMA bulk copy has a fixed cost in
    // the SM's TMA unit, so a tile of >= 32 small src chunks arrives slowly (64 SoA chunks of 640 B:
    // 3.98 vs 6.34 TB/s for one chunk, profiles/r02aa_pieces.log); cp.async does not care about the
    // chunk count but puts the load issue on the consumers, which bind at large N (C5 6 361 vs
    // 6 556 GB/s, profiles/r02ac_loader.log).  So cpa only for >= 32 src chunks per tile up to 24 MB:
    // K-Means SoA->AoS 8 MB 13.2 -> 11.9 us, C3 SoA->hybrid 1 MB 18.8 -> 13.0 us (tiled;
    // r02ac_small_path_cpa.log).  ADHA_LOADER = tma | cpa overrides.
    {
        const char* ld_env = std::getenv("ADHA_LOADER");
        bool cpa = (uint64_t)n * ls.record_bytes <= (24ull << 20);
        bool any = false;
        for (size_t k = 0; k < plan->comps.size(); ++k) {
            if (P->comp[k].n_tiles == 0) continue;
            any = true;
            if (plan->comps[k].src_clusters.size() < 32) cpa = false;
        }
        cpa = cpa && any;
        if (ld_env && std::strcmp(ld_env, "cpa") == 0) cpa = true;
        if (ld_env && std::strcmp(ld_env, "tma") == 0) cpa = false;
        P->cpa = (cpa && !P->tma_copy && !plan->byte_groups && plan->unit == 4) ? 1u : 0u;
    }
    const void* fn = nullptr;
    TiledLauncher launch = plan->byte_groups ? pick_groups(plan->group_class, P->tma_copy != 0, &fn)
                           : P->cpa          ? pick_cpa(plan->table_class, &fn)
                                             : pick(plan->unit, plan->table_class, P->tma_copy != 0, &fn);
    const int threads = P->tma_copy ? NTHREADS_TMA : P->cpa ? NTHREADS_CPA : NTHREADS;
    s = device_setup(fn, &n_sm, threads);
    if (s != ADHA_OK) return s;
    bool enq = false;
    s = device_table("p" + std::to_string(plan->uid), plan->table, st, &P->table, &enq);
    if (s != ADHA_OK) return s;
    const bool pdl = pdl_enabled() && !enq;
    // a tail-only call still needs one CTA per component tail
    const int64_t grid = std::max<int64_t>(std::min<int64_t>((int64_t)plan->comps.size(), n_sm),
                                           std::min<int64_t>(tiles, n_sm));
    launch(dim3((unsigned)std::max<int64_t>(grid, 1)), dim3(threads), plan->smem_bytes, st, *P, pdl);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "remap_tiled_kernel launch");
    return ADHA_OK;
}

}  // namespace detail
}  // namespace adha

using namespace adha;
using namespace adha::detail;

// set by adha_remap_peer around its adha_remap call: dst is another device's memory
static thread_local bool g_dst_remote = false;

extern "C" adha_status adha_remap(const void* src, const adha_layout* hs, void* dst, const adha_layout* hd,
                                  int64_t n, void* stream) {
    clear_error();
    Checked ck;
    adha_status s = validate(src, hs, dst, hd, n, &ck, true);
    if (s != ADHA_OK) return s;
    ck.dst_local = !g_dst_remote;
    return remap_checked((const uint8_t*)src, hs->L, (uint8_t*)dst, hd->L, n, ck, (cudaStream_t)stream);
}

extern "C" adha_status adha_remap_regions(const void* const* src_regions, const adha_layout* hs,
                                          void* const* dst_regions, const adha_layout* hd, int64_t n,
                                          void* stream) {
    clear_error();
    Checked ck;
    // layout checks (buffer checks are per region below)
    adha_status s = validate(nullptr, hs, nullptr, hd, 0, &ck, false);
    if (s != ADHA_OK) return s;
    if (n < 0) return fail(ADHA_ERR_INVALID_ARG, "n_records < 0");
    if (n == 0) return ADHA_OK;
    if (!src_regions || !dst_regions) return fail(ADHA_ERR_INVALID_ARG, "null region array");
    const Layout& ls = hs->L;
    const Layout& ld = hd->L;
    std::vector<uint64_t> tmp;
    if (!ls.region_bases(n, tmp, nullptr) || !ld.region_bases(n, tmp, nullptr))
        return fail(ADHA_ERR_TOO_LARGE, "N * record bytes overflows");
    struct Span { uint64_t lo, hi; int side, c; };
    std::vector<Span> spans;
    ck.bs.assign(ls.n_clusters(), 0);
    ck.bd.assign(ld.n_clusters(), 0);
    for (int c = 0; c < ls.n_clusters(); ++c) {
        const uint64_t a = (uint64_t)(uintptr_t)src_regions[c];
        if (!a) return fail(ADHA_ERR_INVALID_ARG, "null src region " + std::to_string(c));
        if (a & 255) return fail(ADHA_ERR_ALIGNMENT, "src region " + std::to_string(c) + " not 256-byte aligned");
        ck.bs[c] = a;
        spans.push_back({a, a + ls.region_bytes(c, n), 0, c});
    }
    for (int c = 0; c < ld.n_clusters(); ++c) {
        const uint64_t a = (uint64_t)(uintptr_t)dst_regions[c];
        if (!a) return fail(ADHA_ERR_INVALID_ARG, "null dst region " + std::to_string(c));
        if (a & 255) return fail(ADHA_ERR_ALIGNMENT, "dst region " + std::to_string(c) + " not 256-byte aligned");
        ck.bd[c] = a;
        spans.push_back({a, a + ld.region_bytes(c, n), 1, c});
    }
    // a dst region may BE the src region of its cluster only when the plan's component for that
    // pair is an identity (same members, offsets, stride and block, no padding): nothing moves there
    auto plan = get_plan(ls, ld);
    auto identity_pair = [&](int cs, int cd) {
        for (const auto& K : plan->comps)
            if (K.identity && K.src_clusters[0] == cs && K.dst_clusters[0] == cd) return true;
        return false;
    };
    for (size_t i = 0; i < spans.size(); ++i)
        for (size_t j = i + 1; j < spans.size(); ++j) {
            const Span& x = spans[i];
            const Span& y = spans[j];
            if (!(x.lo < y.hi && y.lo < x.hi)) continue;
            if (x.side == 0 && y.side == 0) continue;                  // src regions may share memory
            const bool alias = x.side != y.side && x.lo == y.lo &&
                               identity_pair(x.side == 0 ? x.c : y.c, x.side == 0 ? y.c : x.c);
            if (!alias) return fail(ADHA_ERR_OVERLAP, "regions overlap (only identity clusters may alias)");
        }
    return remap_checked(nullptr, ls, nullptr, ld, n, ck, (cudaStream_t)stream);
}

namespace adha {
namespace detail {
// One launch for a chain of latency-bound hops (every hop <= ADHA_SMALL_BYTES of payload, packed
// unblocked layouts, <= CHAIN_NF fields, <= CHAIN_NH hops, pairwise disjoint buffers).  Returns
// ADHA_ERR_UNSUPPORTED (no error recorded) when the chain does not qualify.
adha_status chain_small(void* const* buffers, const adha_layout* const* layouts, int32_t n_layouts, int64_t n,
                        cudaStream_t st, bool launch = true) {
    const char* e = std::getenv("ADHA_CHAIN_FUSE");
    if ((e && *e == '0') || n <= 0 || n_layouts - 1 > CHAIN_NH) return ADHA_ERR_UNSUPPORTED;
    const Layout& l0 = layouts[0]->L;
    if (l0.n_fields > CHAIN_NF || (uint64_t)n * l0.record_bytes > small_bytes()) return ADHA_ERR_UNSUPPORTED;
    std::vector<Checked> ck(n_layouts - 1);
    for (int32_t k = 0; k + 1 < n_layouts; ++k) {
        adha_status s = validate(buffers[k], layouts[k], buffers[k + 1], layouts[k + 1], n, &ck[k], true);
        if (s != ADHA_OK) return s;
    }
    std::vector<std::pair<uintptr_t, uintptr_t>> ranges;
    for (int32_t k = 0; k < n_layouts; ++k) {
        const Layout& L = layouts[k]->L;
        for (int c = 0; c < L.n_clusters(); ++c)
            if (L.block[c] != 1 || L.stride[c] != L.payload(c)) return ADHA_ERR_UNSUPPORTED;
        const uint64_t bytes = k + 1 < n_layouts ? ck[k].bytes_s : ck[k - 1].bytes_d;
        ranges.push_back({(uintptr_t)buffers[k], (uintptr_t)buffers[k] + bytes});
    }
    for (size_t a = 0; a < ranges.size(); ++a)
        for (size_t b = a + 1; b < ranges.size(); ++b)
            if (ranges[a].first < ranges[b].second && ranges[b].first < ranges[a].second) return ADHA_ERR_UNSUPPORTED;
    if (!launch) return ADHA_OK;
    int n_sm = 0;
    adha_status s = device_setup(nullptr, &n_sm);
    if (s != ADHA_OK) return s;
    auto P = std::make_unique<ChainParams>();
    std::memset(P.get(), 0, sizeof(ChainParams));
    P->n_records = n;
    P->n_fields = (uint32_t)l0.n_fields;
    P->n_hops = (uint32_t)(n_layouts - 1);
    for (int32_t k = 0; k < n_layouts; ++k) P->buf[k] = (uint64_t)(uintptr_t)buffers[k];
    for (int32_t k = 0; k + 1 < n_layouts; ++k) {
        const Layout& ls = layouts[k]->L;
        const Layout& ld = layouts[k + 1]->L;
        for (int f = 0; f < ls.n_fields; ++f) {
            const int cs = ls.cluster[f], cd = ld.cluster[f];
            P->f[k][f] = {ck[k].bs[cs], ck[k].bd[cd], (uint32_t)ls.stride[cs], (uint32_t)ld.stride[cd], ls.offset[f],
                          ld.offset[f], ls.width[f], 0u};
        }
    }
    // ~256 (record, field) items per block and hop: enough blocks to spread the latency
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n * l0.n_fields + 255) / 256, n_sm));
    launch_pdl(&remap_chain_small_kernel, dim3((unsigned)blocks), dim3(256), 0, st, pdl_enabled(), *P);
    cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) return cuda_fail(ce, "remap_chain_small_kernel launch");
    return ADHA_OK;
}

// Payload per hop from which adha_remap_chain runs a chain as ONE fused tiled launch; 0 (the
// default) disables it.  Opt in with ADHA_CHAIN_TILED_BYTES.  Measured on B200 (DESIGN.md 6,
// profiles/r02m_*): on C4 the fused chain moves 8.6 GB through HBM instead of 12.9 and draws
// 2.4 % less power, but takes 2.04 ms against 2.02 per hop -- the SM side (four shared-memory
// passes per byte) binds at that rate, not HBM -- and P2 is 8 % slower.
uint64_t chain_tiled_bytes() {
    const char* e = std::getenv("ADHA_CHAIN_TILED_BYTES");
    if (e && *e) return (uint64_t)std::strtoull(e, nullptr, 10);
    return 0;
}

// A chain of H remaps as ONE launch of the tiled kernel in chain mode (TiledParams::chain):
// component h is hop h's merged plan (every field in one component), all hops share the tile
// size T, and a CTA runs each of its bands through every hop before the next pair of bands, so
// hop h reads hop h-1's output of the band back from L2 while it is still being written to HBM
// (each intermediate is still materialised).  HBM traffic drops from 2H to
// H+1 buffer passes.  Conditions: 2 <= H <= 8, packed unblocked layouts, pairwise disjoint
// buffers, unit mode with one unit size, >= chain_tiled_bytes() per hop and at least two bands
// per SM; returns ADHA_ERR_UNSUPPORTED (no error recorded) otherwise.
adha_status chain_tiled(void* const* buffers, const adha_layout* const* layouts, int32_t n_layouts, int64_t n,
                        cudaStream_t st, bool launch = true) {
    const int H = n_layouts - 1;
    const uint64_t thr = chain_tiled_bytes();
    if (thr == 0 || H < 2 || H > 8 || n <= 0) return ADHA_ERR_UNSUPPORTED;
    const Layout& l0 = layouts[0]->L;
    if ((uint64_t)n * l0.record_bytes < thr) return ADHA_ERR_UNSUPPORTED;
    std::vector<Checked> ck(H);
    for (int h = 0; h < H; ++h) {
        adha_status s = validate(buffers[h], layouts[h], buffers[h + 1], layouts[h + 1], n, &ck[h], true);
        if (s != ADHA_OK) return s;
    }
    std::vector<std::pair<uintptr_t, uintptr_t>> ranges;
    for (int k = 0; k < n_layouts; ++k) {
        const Layout& L = layouts[k]->L;
        for (int c = 0; c < L.n_clusters(); ++c)
            if (L.block[c] != 1 || L.stride[c] != L.payload(c)) return ADHA_ERR_UNSUPPORTED;
        const uint64_t bytes = k < H ? ck[k].bytes_s : ck[H - 1].bytes_d;
        ranges.push_back({(uintptr_t)buffers[k], (uintptr_t)buffers[k] + bytes});
    }
    for (size_t a = 0; a < ranges.size(); ++a)
        for (size_t b = a + 1; b < ranges.size(); ++b)
            if (ranges[a].first < ranges[b].second && ranges[b].first < ranges[a].second) return ADHA_ERR_UNSUPPORTED;
    std::vector<std::shared_ptr<const RemapPlan>> plans;
    uint32_t T = 0, unit = 0, max_w = 0;
    uint64_t n_ent = 0, n_sc = 0, n_dc = 0, n_f = 0, stage = 0;
    for (int h = 0; h < H; ++h) {
        auto pl = get_plan(layouts[h]->L, layouts[h + 1]->L, true);
        if (!pl->tiled || pl->byte_groups || pl->comps.size() != 1) return ADHA_ERR_UNSUPPORTED;
        if (unit && pl->unit != unit) return ADHA_ERR_UNSUPPORTED;
        unit = pl->unit;
        T = T ? std::min(T, pl->comps[0].T_max) : pl->comps[0].T_max;
        max_w = std::max(max_w, pl->comps[0].identity ? 0u : pl->comps[0].n_instr);
        n_ent += pl->ent_off.size();
        n_sc += pl->src_order.size();
        n_dc += pl->dst_order.size();
        n_f += pl->comps[0].fields.size();
        plans.push_back(pl);
    }
    for (int h = 0; h < H; ++h)
        stage = std::max<uint64_t>(stage, (uint64_t)T * std::max(plans[h]->comps[0].Rs, plans[h]->comps[0].Rd));
    stage = (stage + 127) / 128 * 128;
    int cls = -1;
    for (int c = 0; c < 3 && cls < 0; ++c)       // (the kernel runs chain mode up to class 2)
        if (n_ent <= (uint64_t)CLASS_NENT[c] && max_w <= (uint32_t)(NCONS * CLASS_EMAX[c])) cls = c;
    const uint64_t n16 = (n_ent + 15) / 16 * 16;
    const uint64_t tbl = (6 * n16 + 16 * (n_sc + n_dc) + 127) / 128 * 128;
    const uint64_t smem = HDR_BYTES + 128 + 4 * stage + tbl;
    if (cls < 0 || n_sc > MAXC || n_dc > MAXC || n_f > MAXF || stage > STAGE_MAX || smem > 232448)
        return ADHA_ERR_UNSUPPORTED;
    int n_sm = 0;
    adha_status s = device_setup(nullptr, &n_sm);
    if (s != ADHA_OK) {
        if (launch) return s;
        clear_error();          // route query on a host without a device: a B200's 148 SMs
        n_sm = 148;
    }
    const int64_t bands = n / T;
    if (bands < 8 * (int64_t)n_sm) return ADHA_ERR_UNSUPPORTED;      // a group of bands per CTA
    if (!launch) return ADHA_OK;

    auto P = std::make_unique<TiledParams>();
    std::memset(P.get(), 0, sizeof(TiledParams));
    P->n_records = n;
    P->stage_bytes = (uint32_t)stage;
    P->s_in = 2;
    P->s_out = 2;
    P->n_comp = (uint32_t)H;
    P->unit = unit;
    P->chain = (uint32_t)H;
    {
        const char* g = std::getenv("ADHA_CHAIN_GROUP");   // bands per group (1..8)
        const uint32_t gb = g && *g ? (uint32_t)std::strtoul(g, nullptr, 10) : 8u;
        P->chain_group = std::min<uint32_t>(8, std::max<uint32_t>(1, gb));
        const char* ch = std::getenv("ADHA_CHAIN_HINTS");
        P->chain_hints = (ch && *ch == '0') ? 0u : 1u;
    }
    P->total_tiles = bands * H;
    {
        const char* hh = std::getenv("ADHA_L2_HINTS");
        P->l2_hints = hh && *hh ? (uint32_t)std::strtoul(hh, nullptr, 10) : 0u;
    }
    // the table image of class cls: off[NENT] | sc[NENT] | dc[NENT] | fields[MAXF]; hop h's
    // cluster indices are offset by the clusters of hops < h
    const uint32_t NE = (uint32_t)CLASS_NENT[cls];
    std::vector<uint32_t> table((6ull * NE + sizeof(FieldDesc) * MAXF + 3) / 4, 0u);
    uint8_t* img = reinterpret_cast<uint8_t*>(table.data());
    FieldDesc* fds = reinterpret_cast<FieldDesc*>(img + 6ull * NE);
    uint32_t sc = 0, dc = 0, ent = 0, instr = 0, fi = 0;
    for (int h = 0; h < H; ++h) {
        const RemapPlan& pl = *plans[h];
        const RemapPlan::Comp& K = pl.comps[0];
        const Layout& ls = layouts[h]->L;
        const Layout& ld = layouts[h + 1]->L;
        CompDesc& D = P->comp[h];
        D.T = T;
        D.tile_bytes = T * K.Rs;
        D.out_bytes = T * K.Rd;
        D.n_tiles = bands;
        D.tile_base = (int64_t)h * bands;
        D.identity = K.identity ? 1 : 0;
        D.flags = 0;
        D.instr_base = instr;
        D.n_instr = K.n_instr;
        const uint32_t sc0 = sc, dc0 = dc;
        D.sc_lo = (uint16_t)sc;
        uint32_t off = 0;
        for (int c : pl.src_order) {
            P->srcc[sc++] = {(uint64_t)(uintptr_t)buffers[h] + ck[h].bs[c], (uint32_t)ls.stride[c], off};
            off += T * (uint32_t)ls.stride[c];
        }
        D.sc_hi = (uint16_t)sc;
        D.dc_lo = (uint16_t)dc;
        off = 0;
        for (int c : pl.dst_order) {
            P->dstc[dc++] = {(uint64_t)(uintptr_t)buffers[h + 1] + ck[h].bd[c], (uint32_t)ld.stride[c], off};
            off += T * (uint32_t)ld.stride[c];
        }
        D.dc_hi = (uint16_t)dc;
        for (size_t e = 0; e < pl.ent_off.size(); ++e, ++ent) {
            reinterpret_cast<uint32_t*>(img)[ent] = pl.ent_off[e];
            img[4ull * NE + ent] = (uint8_t)(pl.ent_sc[e] + sc0);
            img[5ull * NE + ent] = (uint8_t)(pl.ent_dc[e] + dc0);
        }
        instr += K.n_instr;
        D.f_lo = (uint16_t)fi;
        for (int f : K.fields) {
            FieldDesc d;
            d.sc = (uint8_t)(pl.src_slot[ls.cluster[f]] + sc0);
            d.dc = (uint8_t)(pl.dst_slot[ld.cluster[f]] + dc0);
            d.sbl = d.dbl = 0;
            d.soff = ls.offset[f];
            d.doff = ld.offset[f];
            d.width = ls.width[f];
            fds[fi++] = d;
        }
        D.f_hi = (uint16_t)fi;
    }
    P->n_ent = ent;
    P->n_srcc = sc;
    P->n_dstc = dc;
    const void* fn = nullptr;
    TiledLauncher run = pick_chain(unit, cls, &fn);
    s = device_setup(fn, &n_sm, NTHREADS);
    if (s != ADHA_OK) return s;
    // the chain's table depends only on its hops' plans (and the class)
    std::string key = "c" + std::to_string(cls);
    for (const auto& pl : plans) key += "." + std::to_string(pl->uid);
    bool enq = false;
    s = device_table(key, table, st, &P->table, &enq);
    if (s != ADHA_OK) return s;
    const int64_t grid = std::min<int64_t>(bands, n_sm);
    run(dim3((unsigned)grid), dim3(NTHREADS), smem, st, *P, pdl_enabled() && !enq);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "remap_tiled_kernel (chain) launch");
    return ADHA_OK;
}
}  // namespace detail
}  // namespace adha

extern "C" adha_status adha_remap_chain(void* const* buffers, const adha_layout* const* layouts, int32_t n_layouts,
                                        int64_t n, void* stream) {
    clear_error();
    if (!buffers || !layouts || n_layouts < 2) return fail(ADHA_ERR_INVALID_ARG, "need at least two layouts");
    for (int32_t k = 0; k < n_layouts; ++k)
        if (!layouts[k]) return fail(ADHA_ERR_INVALID_ARG, "null layout");
    const adha_status fused = detail::chain_small(buffers, layouts, n_layouts, n, (cudaStream_t)stream);
    if (fused != ADHA_ERR_UNSUPPORTED) return fused;
    clear_error();
    const adha_status tiled = detail::chain_tiled(buffers, layouts, n_layouts, n, (cudaStream_t)stream);
    if (tiled != ADHA_ERR_UNSUPPORTED) return tiled;
    clear_error();
    for (int32_t k = 0; k + 1 < n_layouts; ++k) {
        adha_status s = adha_remap(buffers[k], layouts[k], buffers[k + 1], layouts[k + 1], n, stream);
        if (s != ADHA_OK) return s;
    }
    return ADHA_OK;
}

extern "C" adha_status adha_remap_chain_route(const adha_layout* const* layouts, int32_t n_layouts, int64_t n,
                                              int32_t* route, int32_t* launches) {
    clear_error();
    if (!layouts || n_layouts < 2 || !route || !launches) return fail(ADHA_ERR_INVALID_ARG, "null argument or < 2 layouts");
    for (int32_t k = 0; k < n_layouts; ++k)
        if (!layouts[k]) return fail(ADHA_ERR_INVALID_ARG, "null layout");
    // disjoint stand-in buffers (256-byte aligned, 16 TB apart): the routing assumes the caller's are
    std::vector<void*> fake(n_layouts);
    for (int32_t k = 0; k < n_layouts; ++k) fake[k] = (void*)(uintptr_t)((uint64_t)(k + 1) << 44);
    adha_status s = detail::chain_small(fake.data(), layouts, n_layouts, n, nullptr, false);
    if (s == ADHA_OK) { *route = 1; *launches = 1; return ADHA_OK; }
    if (s != ADHA_ERR_UNSUPPORTED) return s;
    clear_error();
    s = detail::chain_tiled(fake.data(), layouts, n_layouts, n, nullptr, false);
    if (s == ADHA_OK) { *route = 2; *launches = 1; return ADHA_OK; }
    if (s != ADHA_ERR_UNSUPPORTED) return s;
    clear_error();
    *route = 0;
    *launches = n_layouts - 1;
    return ADHA_OK;
}

extern "C" adha_status adha_remap_sharded(const void* const* src_shards, const adha_layout* hs,
                                          void* const* dst_shards, const adha_layout* hd, int64_t n_total,
                                          int32_t n_shards, const int32_t* device_ids, void* const* streams) {
    clear_error();
    if (!src_shards || !dst_shards || !device_ids || !streams || n_shards < 1)
        return fail(ADHA_ERR_INVALID_ARG, "null argument or n_shards < 1");
    if (n_total < 0) return fail(ADHA_ERR_INVALID_ARG, "n_records_total < 0");
    int prev = 0;
    cudaError_t e = cudaGetDevice(&prev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    adha_status out = ADHA_OK;
    for (int32_t g = 0; g < n_shards && out == ADHA_OK; ++g) {
        int64_t lo = 0, hi = 0;
        adha_shard_range(n_total, n_shards, g, &lo, &hi);
        e = cudaSetDevice(device_ids[g]);
        if (e != cudaSuccess) { out = cuda_fail(e, "cudaSetDevice"); break; }
        out = adha_remap(src_shards[g], hs, dst_shards[g], hd, hi - lo, streams[g]);
        if (out != ADHA_OK) set_error("shard " + std::to_string(g) + ": " + adha_last_error());
    }
    std::string msg = adha_last_error();
    cudaSetDevice(prev);
    if (out != ADHA_OK) set_error(msg);
    return out;
}

// ---------------------------------------------------------------------------- cross-device (N2)
// Push design: the kernel runs on the src device and its copy-out STG.128s address the
// peer's HBM through the unified address space (NVLink 5 / NVSwitch).  Loads stay local
// (TMA bulk copies from local HBM); only the dst bytes cross the link, once.
namespace {

std::mutex g_peer_mu;
std::set<std::pair<int, int>> g_peer_enabled;

adha_status check_device_pointer(const void* p, int device, const char* what) {
    cudaPointerAttributes a{};
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) return cuda_fail(e, "cudaPointerGetAttributes");
    if (a.type != cudaMemoryTypeDevice || a.device != device)
        return fail(ADHA_ERR_INVALID_ARG, std::string(what) + " is not device memory of device " +
                                              std::to_string(device));
    return ADHA_OK;
}

adha_status enable_peer(int from, int to) {
    std::lock_guard<std::mutex> lk(g_peer_mu);
    if (g_peer_enabled.count({from, to})) return ADHA_OK;
    int can = 0;
    cudaError_t e = cudaDeviceCanAccessPeer(&can, from, to);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceCanAccessPeer");
    if (!can)
        return fail(ADHA_ERR_CUDA, "device " + std::to_string(from) + " cannot access device " +
                                       std::to_string(to) + " (no P2P path)");
    e = cudaDeviceEnablePeerAccess(to, 0);           // current device is `from`
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
    } else if (e != cudaSuccess) {
        return cuda_fail(e, "cudaDeviceEnablePeerAccess");
    }
    g_peer_enabled.insert({from, to});
    return ADHA_OK;
}

}  // namespace

extern "C" adha_status adha_remap_peer(const void* src, const adha_layout* hs, int32_t src_device, void* dst,
                                       const adha_layout* hd, int32_t dst_device, int64_t n, void* stream) {
    clear_error();
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    if (src_device < 0 || src_device >= count || dst_device < 0 || dst_device >= count)
        return fail(ADHA_ERR_INVALID_ARG, "device id out of range (" + std::to_string(count) + " devices)");
    int prev = 0;
    e = cudaGetDevice(&prev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    e = cudaSetDevice(src_device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    adha_status out = ADHA_OK;
    if (n > 0 && src && dst) {
        out = check_device_pointer(src, src_device, "src");
        if (out == ADHA_OK) out = check_device_pointer(dst, dst_device, "dst");
    }
    if (out == ADHA_OK && src_device != dst_device) out = enable_peer(src_device, dst_device);
    if (out == ADHA_OK) {
        g_dst_remote = src_device != dst_device;    // no TMA write-back into peer memory
        out = adha_remap(src, hs, dst, hd, n, stream);
        g_dst_remote = false;
    }
    std::string msg = adha_last_error();
    cudaSetDevice(prev);
    if (out != ADHA_OK) set_error(msg);
    return out;
}

#ifdef ADHA_PHASE_TIMING
// diagnostic build only: read (and optionally reset) the tiled kernel's phase counters
extern "C" __attribute__((visibility("default"))) int adha_debug_phase(unsigned long long* out8, int reset) {
    cudaError_t e = cudaMemcpyFromSymbol(out8, adha::dev::g_phase, 8 * sizeof(unsigned long long));
    if (e == cudaSuccess && reset) {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        e = cudaMemcpyToSymbol(adha::dev::g_phase, z, sizeof z);
    }
    return (int)e;
}
#endif

// ---------------------------------------------------------------------------- host end-to-end
extern "C" adha_status adha_remap_plan_describe(const adha_layout* hs, const adha_layout* hd, char** json_out) {
    return adha_remap_plan_describe_ex(hs, hd, 0, json_out);
}

extern "C" adha_status adha_remap_plan_describe_ex(const adha_layout* hs, const adha_layout* hd, int32_t merged,
                                                   char** json_out) {
    clear_error();
    if (!hs || !hd || !json_out) return fail(ADHA_ERR_INVALID_ARG, "null argument");
    if (hs->L.n_fields != hd->L.n_fields) return fail(ADHA_ERR_LAYOUT_MISMATCH, "layouts differ in field count");
    for (int f = 0; f < hs->L.n_fields; ++f)
        if (hs->L.width[f] != hd->L.width[f]) return fail(ADHA_ERR_LAYOUT_MISMATCH, "widths differ");
    auto plan = get_plan(hs->L, hd->L, merged != 0);
    std::string s = describe_plan(*plan, hs->L, hd->L);
    // routing threshold of adha_remap for this pair (device dst): payload <= direct_bytes takes the
    // direct kernel (ADHA_SMALL_BYTES overrides, read now)
    s.pop_back();
    s += ",\"direct_bytes\":" + std::to_string(direct_bytes(*plan)) + ",\"merge_bytes\":" +
         std::to_string(plan->comps.size() > 1 ? merge_bytes(*plan) : 0) + "}";
    *json_out = (char*)std::malloc(s.size() + 1);
    if (!*json_out) return fail(ADHA_ERR_OOM, "out of host memory");
    std::memcpy(*json_out, s.c_str(), s.size() + 1);
    return ADHA_OK;
}
