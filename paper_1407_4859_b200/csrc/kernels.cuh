// kernels.cuh -- device code of the remap (included by remap.cu only): the tiled kernel
// (TMA-staged tiles, shared-memory permutation in unit or byte-group mode, 16-byte copy-out;
// its CHAIN instantiations run a whole PDL chain in one launch), the direct kernel for small
// remaps / layouts beyond the tiled kernel's limits, the fused small-chain kernel, and the zero
// kernel.  Design: remap.cu header comment and DESIGN.md section 6.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "ptx.cuh"
#include "remap_plan.h"

namespace adha {
namespace dev {

using namespace adha::ptx;

// Copy-out plan of one consumer thread for the current component: the thread writes the
// 16-byte vectors b = tid*16 + u*NT*16 (u < nv) of a staged tile (dst chunks packed in
// cluster order).  Vector u lands at dst + gofs[u] + lt * gstep[u] for local tile lt.
// The mapping is the same for every tile of the component, so it is computed once per
// component switch and kept in registers.
constexpr uint32_t PMAX = 4;                   // bulk-load pieces per producer lane per tile
constexpr uint32_t VMAX = 12;                  // 12 * 16 B * 256 threads = 49152 B >= stage_bytes

// dst cluster descriptor c: from the shared-memory copy (dcl != 0, unit mode) or the parameters
struct DstDesc {
    uint64_t region;
    uint32_t stride, smem;
};
__device__ __forceinline__ DstDesc dst_desc(const TiledParams& p, uint32_t dcl, uint32_t c) {
    if (dcl) {
        const uint4 v = lds128(dcl + 16 * c);
        return {(uint64_t)v.x | ((uint64_t)v.y << 32), v.z, v.w};
    }
    return {p.dstc[c].region, p.dstc[c].stride, p.dstc[c].smem};
}

__device__ __forceinline__ uint32_t copy_plan(const TiledParams& p, uint32_t dcl, uint32_t c_lo, uint32_t T,
                                              uint32_t total, uint32_t tid, uint64_t (&gofs)[VMAX],
                                              uint32_t (&gstep)[VMAX]) {
    constexpr uint32_t NT = NCONS * 32;
    uint32_t c = c_lo;
    DstDesc d = dst_desc(p, dcl, c);
    uint32_t cbeg = 0, cend = T * d.stride;
    uint32_t nv = 0;
#pragma unroll
    for (uint32_t u = 0; u < VMAX; ++u) {
        const uint32_t b = tid * 16 + u * NT * 16;
        gofs[u] = 0;
        gstep[u] = 0;
        if (b < total) {
            while (b >= cend) {
                ++c;
                d = dst_desc(p, dcl, c);
                cbeg = cend;
                cend = cbeg + T * d.stride;
            }
            gofs[u] = d.region + (b - cbeg);
            // the per-tile step T*stride is a multiple of 128; its low 7 bits carry the chunk's
            // padding in the output stage / 32 (smem offset - packed offset = 32 * chunk index)
            gstep[u] = (cend - cbeg) | ((d.smem - cbeg) >> 5);
            nv = u + 1;
        }
    }
    return nv;
}

// LDS.128 -> STG.128 of one staged tile, four vectors in flight per step
template <bool HINT>
__device__ __forceinline__ void copy_out(uint8_t* dst, uint32_t sm_base, uint32_t tid, int64_t lt, uint32_t nv,
                                         const uint64_t (&gofs)[VMAX], const uint32_t (&gstep)[VMAX], uint64_t pol) {
    constexpr uint32_t NT = NCONS * 32;
#pragma unroll
    for (uint32_t u0 = 0; u0 < VMAX; u0 += 4) {
        if (u0 < nv) {
            uint4 val[4];
#pragma unroll
            for (uint32_t u = u0; u < u0 + 4 && u < VMAX; ++u)
                if (u < nv) val[u - u0] = lds128(sm_base + tid * 16 + u * NT * 16 + ((gstep[u] & 127u) << 5));
#pragma unroll
            for (uint32_t u = u0; u < u0 + 4 && u < VMAX; ++u)
                if (u < nv) {
                    const uint64_t step = gstep[u] & ~127u;
                    if (HINT) stg128_hint(dst + gofs[u] + (uint64_t)lt * step, val[u - u0], pol);
                    else stg128(dst + gofs[u] + (uint64_t)lt * step, val[u - u0]);
                }
        }
    }
}

// Diagnostic build only (-DADHA_PHASE_TIMING, tools/phase_probe.py): clock64() time per phase of
// the tiled kernel, summed over warps and tiles.  [0] consumer wait on `full`, [1] permutation,
// [2] output-tile barrier, [3] copy-out, [4] consumer tiles, [5] producer wait on `empty`,
// [6] producer issue, [7] tails.  Off in the product library.
#ifdef ADHA_PHASE_TIMING
__device__ unsigned long long g_phase[8];
#define ADHA_PT(...) __VA_ARGS__
#else
#define ADHA_PT(...)
#endif

// Tile order of a CTA: interleaved (t = b, b+G, ...: the GPU sweeps the arrays as one front)
// or blocked (CTA b takes the contiguous range [b*M/G, (b+1)*M/G)).
__device__ __forceinline__ int64_t t_first(const TiledParams& p) {
    return p.blocked ? (int64_t)blockIdx.x * p.total_tiles / gridDim.x : (int64_t)blockIdx.x;
}
__device__ __forceinline__ int64_t t_end(const TiledParams& p) {
    return p.blocked ? (int64_t)(blockIdx.x + 1) * p.total_tiles / gridDim.x : p.total_tiles;
}
__device__ __forceinline__ int64_t t_step(const TiledParams& p) { return p.blocked ? 1 : (int64_t)gridDim.x; }

// Fused chain (p.chain = H hops, component k = hop k, all with the same T and n_tiles = bands):
// CTA b owns bands b, b+G, ... and runs them in groups of p.chain_group bands, hop by hop --
// (j0,h0) (j1,h0) .. (j0,h1) (j1,h1) .. -- so the load of tile (j,h) depends on the store of
// (j,h-1), issued one group earlier.  Hop h-1's output of band j is read back from L2.
//
// TileIter walks a CTA's tiles in either mode without divisions per tile: component k, local
// tile lt, and (chain) dist = tiles since the same band's previous hop (its group's size, <= 8).
struct TileIter {
    int64_t t, lt;          // plain: global tile; both: local tile of component k
    int64_t q0, bands;      // chain: first band index of the group (per-CTA numbering), bands of this CTA
    uint32_t k, dist, bb, gsz;
};
__device__ __forceinline__ int64_t cta_tiles(const TiledParams& p, uint32_t H) {
    if (H) {
        const int64_t nb = p.comp[0].n_tiles;
        const int64_t q = nb > (int64_t)blockIdx.x ? (nb - 1 - (int64_t)blockIdx.x) / gridDim.x + 1 : 0;
        return q * H;
    }
    const int64_t a = t_first(p), e = t_end(p), st = t_step(p);
    return a < e ? (e - a + st - 1) / st : 0;
}
__device__ __forceinline__ void tile_begin(const TiledParams& p, uint32_t H, TileIter& it) {
    it.k = 0;
    it.dist = 0;
    if (H) {
        it.bands = cta_tiles(p, H) / H;
        it.q0 = 0;
        it.bb = 0;
        it.gsz = (uint32_t)min((int64_t)p.chain_group, it.bands);
        it.dist = it.gsz;
        it.lt = (int64_t)blockIdx.x;
    } else {
        it.t = t_first(p);
        while (it.t >= p.comp[it.k].tile_base + p.comp[it.k].n_tiles && it.k + 1 < p.n_comp) ++it.k;
        it.lt = it.t - p.comp[it.k].tile_base;
    }
}
__device__ __forceinline__ void tile_next(const TiledParams& p, uint32_t H, TileIter& it) {
    if (H) {
        if (++it.bb == it.gsz) {
            it.bb = 0;
            if (++it.k == H) {                         // next group of bands
                it.k = 0;
                it.q0 += it.gsz;
                it.gsz = (uint32_t)min((int64_t)p.chain_group, it.bands - it.q0);
                it.dist = it.gsz;
            }
        }
        it.lt = (int64_t)blockIdx.x + (it.q0 + it.bb) * (int64_t)gridDim.x;
    } else {
        it.t += t_step(p);
        while (it.t >= p.comp[it.k].tile_base + p.comp[it.k].n_tiles && it.k + 1 < p.n_comp) ++it.k;
        it.lt = it.t - p.comp[it.k].tile_base;
    }
}

// one 16-byte FieldDesc of the plan table (device memory, read-only)
__device__ __forceinline__ FieldDesc ldg_field(const FieldDesc* f) {
    const uint4 v = ldg_nc128(reinterpret_cast<const uint4*>(f));
    FieldDesc d;
    d.sc = (uint8_t)(v.x & 0xFFu);
    d.dc = (uint8_t)((v.x >> 8) & 0xFFu);
    d.sbl = (uint8_t)((v.x >> 16) & 0xFFu);
    d.dbl = (uint8_t)(v.x >> 24);
    d.soff = v.y;
    d.doff = v.z;
    d.width = v.w;
    return d;
}

// cp.async loader (TiledParams::cpa, the CPA instantiations): loader warp lw of NLOAD copies
// bytes [lw*B/NLOAD, (lw+1)*B/NLOAD) of tile (k, lt)'s packed src chunks (B = tile_bytes) into
// input stage `sb` with 16-byte cp.async, 512 contiguous bytes per warp instruction, then arrives
// on the stage's `full` barrier when its copies land (count NLOAD*32).  Unlike TMA bulk copies,
// the cost does not grow with the number of src chunks (64 SoA chunks of 640 B per tile:
// profiles/r02aa_pieces.log).  Cluster descriptors come from the kernel parameters (uniform per
// warp); (c0, b0) cache this warp's first chunk and its packed begin for component ak.
struct CpaState {
    int ak;
    uint32_t c0, b0;
};
__device__ __forceinline__ void cpa_issue(const TiledParams& p, uint32_t k, int64_t lt, uint32_t sb, uint32_t full,
                                          uint32_t lw, uint32_t lane, CpaState& cs) {
    const CompDesc& K = p.comp[k];
    const uint32_t TV = K.tile_bytes >> 4;
    const uint32_t w0 = (lw * TV / NLOAD) << 4, w1 = ((lw + 1) * TV / NLOAD) << 4;
    if ((int)k != cs.ak) {
        cs.ak = (int)k;
        uint32_t c = K.sc_lo, b = 0;
        for (;;) {
            const uint32_t e = b + K.T * p.srcc[c].stride;
            if (e > w0 || c + 1 >= K.sc_hi) break;
            b = e;
            ++c;
        }
        cs.c0 = c;
        cs.b0 = b;
    }
    uint32_t c = cs.c0, b = cs.b0;
    while (b < w1 && c < K.sc_hi) {
        const ClusterDesc d = p.srcc[c];
        const uint32_t bytes = K.T * d.stride, e = b + bytes;
        const uint32_t lo = max(b, w0), hi = min(e, w1);
        const uint8_t* g = (const uint8_t*)(p.src + d.region + (uint64_t)lt * bytes) - b;
        const uint32_t sm = sb + d.smem - b;
        for (uint32_t o = lo + lane * 16; o < hi; o += 32 * 16) cp_async16(sm + o, g + o);
        b = e;
        ++c;
    }
    cp_async_mbar_arrive_noinc(full);
}

// 9 warps per CTA: the register file is split over the 4 SM sub-partitions (16K registers
// each) and one of them holds 3 warps, so a thread may use at most 16384 / 96 = 168 registers;
// __launch_bounds__(NTHREADS, 1) gives ptxas exactly that budget.
template <int NENT, int NG>
using TableOf = typename std::conditional<(NG > 0), GroupTable<NG>, EntryTable<NENT>>::type;

// NG = 0: unit mode (EntryTable<NENT>, EMAX instructions per warp); NG > 0: byte-group mode
// (GroupTable<NG>, GMAX slots per warp, U = uint8_t for the tails).
// TMAC: a 10th warp writes the permuted tiles back with TMA bulk stores (TiledParams::tma_copy);
// otherwise the consumers write them back with STG.
// CHAIN: the fused-chain instantiations (TiledParams::chain; unit mode, STG write-back); the
// plain ones compile every chain branch away.
// The plan's table (TableOf<NENT, NG>) is read from its device copy at p.table.
// CPA: the cp.async loader instantiations (TiledParams::cpa; 4-byte unit mode, STG write-back):
// NLOAD loader warps replace the TMA producer warp.
template <typename U, int NENT, int EMAX, int NG = 0, int GMAX = 1, bool TMAC = false, bool CHAIN = false,
          bool CPA = false>
__global__ void __launch_bounds__(TMAC ? NTHREADS_TMA : CPA ? NTHREADS_CPA : NTHREADS, 1)
    remap_tiled_kernel(const __grid_constant__ TiledParams p) {
    static_assert(!CHAIN || (NG == 0 && !TMAC), "chain mode: unit mode with STG write-back only");
    static_assert(!CPA || (NG == 0 && !TMAC && !CHAIN), "cp.async loader: unit mode with STG write-back only");
    const TableOf<NENT, NG>& et = *reinterpret_cast<const TableOf<NENT, NG>*>(p.table);
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t sbase = (smem_u32(smem) + 127u) & ~127u;
    const uint32_t full0 = sbase;                      // s_in mbarriers: tile landed
    const uint32_t empty0 = sbase + 8 * MAX_S_IN;      // s_in mbarriers: stage consumed
    const uint32_t in0 = sbase + HDR_BYTES;
    const uint32_t out0 = in0 + p.s_in * p.stage_bytes;

    const uint32_t H = CHAIN ? p.chain : 0u;           // fused chain hops, 0 = plain
    const uint32_t ofull0 = sbase + 16 * MAX_S_IN;     // s_out mbarriers: output tile permuted (tma_copy)
    const uint32_t oempty0 = ofull0 + 8 * S_OUT_MAX;   // s_out mbarriers: output tile read by its bulk store
    const uint32_t stored0 = oempty0 + 8 * S_OUT_MAX;  // 8 mbarriers (chain): tile i's stores are visible
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < p.s_in; ++s) {
            mbar_init(full0 + 8 * s, CPA ? NLOAD * 32 : 1);
            mbar_init(empty0 + 8 * s, NCONS);
        }
        for (uint32_t o = 0; o < S_OUT_MAX; ++o) {
            mbar_init(ofull0 + 8 * o, NCONS * 32);
            mbar_init(oempty0 + 8 * o, 1);
        }
        for (uint32_t o = 0; o < 8; ++o) mbar_init(stored0 + 8 * o, NCONS * 32);
        fence_mbarrier_init();
    }
    __syncthreads();

    if (TMAC && warp == NCONS + 1) {
        // ------------------------------------------------------------ TMA write-back (tma_copy)
        // Lane 0 writes every permuted tile back with one bulk store per dst chunk once the
        // consumers arrive on out_full[o]; tile i-1's buffer is released (out_empty) as soon as its
        // bulk group has finished reading shared memory, so the store overlaps the next
        // permutation.  Chosen per launch for components with one large dst chunk per tile.
        if (lane != 0) return;
        grid_dep_wait();
        const uint64_t pol = policy_evict_first();
        uint32_t i = 0, k = 0;
        int prev_o = -1;
        for (int64_t t = t_first(p), te = t_end(p); t < te; t += t_step(p), ++i) {
            while (t >= p.comp[k].tile_base + p.comp[k].n_tiles) ++k;
            const CompDesc& K = p.comp[k];
            const uint32_t o = p.s_out == 2 ? (i & 1u) : 0u;
            const uint32_t j = p.s_out == 2 ? (i >> 1) : i;
            mbar_wait(ofull0 + 8 * o, j & 1u);
            const uint32_t ob = out0 + o * p.stage_bytes;
            const int64_t lt = t - K.tile_base;
            for (uint32_t c = K.dc_lo; c < K.dc_hi; ++c) {
                const uint32_t bytes = K.T * p.dstc[c].stride;
                uint8_t* g = (uint8_t*)p.dst + p.dstc[c].region + (uint64_t)lt * bytes;
                if (p.l2_hints & 2) bulk_store_hint(g, ob + p.dstc[c].smem, bytes, pol);
                else bulk_store(g, ob + p.dstc[c].smem, bytes);
            }
            bulk_commit();
            if (p.s_out == 2) {
                bulk_wait_read<1>();                       // tile i-1's group has read its buffer
                if (prev_o >= 0) mbar_arrive(oempty0 + 8 * prev_o);
            } else {
                bulk_wait_read<0>();
                mbar_arrive(oempty0 + 8 * o);
            }
            prev_o = (int)o;
        }
        bulk_wait_all();
        return;
    }

    if (CPA && warp >= NCONS) {
        // ------------------------------------------------------------ cp.async loader warps
        // the TMA producer's protocol (empty -> load -> full), the copies split over NLOAD warps
        grid_dep_wait();
        CpaState cs{-1, 0u, 0u};
        uint32_t stage = 0, phase = 0;
        const int64_t nt = cta_tiles(p, 0);
        TileIter it;
        tile_begin(p, 0, it);
        for (int64_t i = 0; i < nt; ++i, tile_next(p, 0, it)) {
            mbar_wait(empty0 + 8 * stage, phase ^ 1);
            cpa_issue(p, it.k, it.lt, in0 + stage * p.stage_bytes, full0 + 8 * stage, warp - NCONS, lane, cs);
            if (++stage == p.s_in) { stage = 0; phase ^= 1; }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        return;
    }
    if (warp == NCONS) {
        // ------------------------------------------------------------ TMA producer
        // Per component, every lane holds up to PMAX bulk-load pieces of the tile (src chunks cut
        // into pieces of at most `split` bytes): smem offset, global offset of tile 0, bytes, and
        // the per-tile global step.  Issue is then one bulk copy per piece per lane, no parameter
        // walks on the critical path (the producer's issue time gates the 2-stage pipeline).
        grid_dep_wait();                                  // (PDL) the previous kernel's writes are visible
        const uint64_t pol = policy_evict_first();        // src is read once: evict it first from L2
        uint32_t psm[PMAX], pbytes[PMAX], pstep[PMAX];
        uint64_t pg[PMAX];
        uint32_t np = 0;
        int kp = -1;
        uint32_t stage = 0, phase = 0, k = 0;
        ADHA_PT(long long pw = 0; long long pi = 0);
        const int64_t nt = cta_tiles(p, H);
        TileIter it;
        tile_begin(p, H, it);
        for (int64_t i = 0; i < nt; ++i, tile_next(p, H, it)) {
            k = it.k;
            const int64_t lt = it.lt;
            const uint32_t dist = it.dist;
            if ((int)k != kp) {
                kp = (int)k;
                const uint32_t T = p.comp[k].T;
                // piece size: the configured split, grown until the tile needs at most 32*PMAX pieces
                uint32_t split = p.tma_split ? p.tma_split : 0xFFFFFFF0u;
                uint32_t pieces;
                for (;;) {
                    pieces = 0;
                    for (uint32_t c = p.comp[k].sc_lo; c < p.comp[k].sc_hi; ++c)
                        pieces += (T * p.srcc[c].stride + split - 1) / split;
                    if (pieces <= 32 * PMAX) break;
                    split = ((split + split / 2) + 15) & ~15u;
                }
                np = 0;
                uint32_t piece = 0;
#pragma unroll 1
                for (uint32_t c = p.comp[k].sc_lo; c < p.comp[k].sc_hi; ++c) {
                    const uint32_t bytes = T * p.srcc[c].stride;
                    for (uint32_t o = 0; o < bytes; o += split, ++piece) {
                        if ((piece & 31) != lane) continue;
#pragma unroll
                        for (uint32_t q = 0; q < PMAX; ++q)
                            if (q == np) {
                                psm[q] = p.srcc[c].smem + o;
                                pg[q] = p.src + p.srcc[c].region + o;
                                pbytes[q] = min(split, bytes - o);
                                pstep[q] = bytes;
                            }
                        ++np;
                    }
                }
            }
            ADHA_PT(const long long pt0 = clock64());
            mbar_wait(empty0 + 8 * stage, phase ^ 1);
            // chain: hop k reads what this CTA's consumers stored for the same band at hop k-1
            // (a ring of 8: consumers finish at most tile i-1 by now, so tile i-dist's phase is the
            // last one completed on its barrier)
            if (H && k > 0) {
                mbar_wait(stored0 + 8 * ((i - dist) & 7), (uint32_t)((i - dist) >> 3) & 1u);
                fence_proxy_async_global();      // the consumers' stores (released to us) -> our TMA load
            }
            ADHA_PT(const long long pt1 = clock64(); pw += pt1 - pt0);
            const uint32_t ib = in0 + stage * p.stage_bytes;
            if (lane == 0) mbar_arrive_expect_tx(full0 + 8 * stage, p.comp[k].tile_bytes);
            __syncwarp();
#pragma unroll
            for (uint32_t q = 0; q < PMAX; ++q) {
                if (q < np) {
                    const void* g = (const void*)(pg[q] + (uint64_t)lt * pstep[q]);
                    if ((p.l2_hints & 1) || (H && p.chain_hints)) bulk_load_hint(ib + psm[q], g, pbytes[q], full0 + 8 * stage, pol);
                    else bulk_load(ib + psm[q], g, pbytes[q], full0 + 8 * stage);
                }
            }
            ADHA_PT(pi += clock64() - pt1);
            if (++stage == p.s_in) { stage = 0; phase ^= 1; }
        }
        ADHA_PT(if (lane == 0) { atomicAdd(&g_phase[5], (unsigned long long)pw); atomicAdd(&g_phase[6], (unsigned long long)pi); });
        return;
    }

    // ---------------------------------------------------------------- consumers
    const uint32_t tid = threadIdx.x;
    // Copy the plan's table into shared memory once per CTA -- unit mode: the entry table
    // (off | sc | dc, the n_ent entries in use); byte-group mode: the ByteGroups in use (13 words
    // each) -- plus the cluster descriptors.  The table comes from its device copy with coalesced
    // 16-byte loads (L2-resident after the first CTAs), overlapped with the producer's first TMA
    // loads; a component switch then reads its lanes' entries with LDS.  (Read from the kernel
    // parameters instead, every lane-divergent index was a serialised constant-bank access: C3's
    // merged plan spent ~17 % of its 1-32 MB launches there, profiles/r02y_*.)
    uint32_t tbl = out0 + p.s_out * p.stage_bytes, scl, dcl, n4 = 0;
    if constexpr (NG == 0) {
        n4 = (p.n_ent + 15) & ~15u;                    // <= NENT (a multiple of 16)
        scl = tbl + 6 * n4;
        const uint4* offv = reinterpret_cast<const uint4*>(et.off);
        const uint4* scv = reinterpret_cast<const uint4*>(et.sc);
        const uint4* dcv = reinterpret_cast<const uint4*>(et.dc);
        for (uint32_t i = tid; i < n4 / 4; i += NCONS * 32) sts128(tbl + 16 * i, ldg_nc128(offv + i));
        for (uint32_t i = tid; i < n4 / 16; i += NCONS * 32) {
            sts128(tbl + 4 * n4 + 16 * i, ldg_nc128(scv + i));
            sts128(tbl + 5 * n4 + 16 * i, ldg_nc128(dcv + i));
        }
    } else {
        const uint32_t gbytes = ((uint32_t)sizeof(ByteGroup) * p.n_ent + 15) & ~15u;   // <= sizeof(et.g)
        const uint4* gv = reinterpret_cast<const uint4*>(et.g);
        for (uint32_t i = tid; i < gbytes / 16; i += NCONS * 32) sts128(tbl + 16 * i, ldg_nc128(gv + i));
        scl = tbl + gbytes;
    }
    dcl = scl + 16 * p.n_srcc;
    {
        const uint4* sv = reinterpret_cast<const uint4*>(p.srcc);
        const uint4* dv = reinterpret_cast<const uint4*>(p.dstc);
        for (uint32_t i = tid; i < p.n_srcc; i += NCONS * 32) sts128(scl + 16 * i, sv[i]);
        for (uint32_t i = tid; i < p.n_dstc; i += NCONS * 32) sts128(dcl + 16 * i, dv[i]);
        named_bar_sync(1, NCONS * 32);
    }
    // (PDL) everything above touched only shared memory, the parameters and the plan table; the
    // tails and the copy-out below read and write the caller's buffers
    grid_dep_wait();
    const uint64_t spol = policy_evict_first();
    const uint64_t kpol = CHAIN ? policy_evict_last() : 0;   // chain: intermediates, read back by the next hop
    uint32_t ioff[EMAX], ooff[EMAX], din[EMAX], dout[EMAX];
    // byte-group mode: per slot j, source words m and output words o of this lane's group
    uint32_t gsrc[GMAX][4], gsst[GMAX][4], gout[GMAX][4], gost[GMAX][4], gsel[GMAX][4][2];
    uint32_t gns[GMAX], gno[GMAX], grho[GMAX], gP = 1;
    uint64_t gofs[VMAX];
    uint32_t gstep[VMAX];
    uint32_t ne = 0, nv = 0;

    ADHA_PT(const long long tt0 = clock64());
    // Tails first: records [n_tiles*T_k, N) of every component.  Plain components spread their
    // tail over the consumer threads of ALL CTAs, four records in flight per thread, while the
    // producer's first tiles are still in flight (one CTA copying a 48 KB tail alone took ~40 us).
    // Components whose dst has padding or AoSoA blocks (CF_TAIL_ZERO) zero their dst tail area
    // first, so their tail belongs to one CTA (zero, barrier, copy).
    {
        const int64_t gid = (int64_t)blockIdx.x * (NCONS * 32) + tid;
        const int64_t gstride = (int64_t)gridDim.x * (NCONS * 32);
        int64_t acc = 0;     // tail items of the previous components: each tail starts where the last ended
        for (uint32_t kk = 0; kk < p.n_comp; ++kk) {
            const CompDesc& K = p.comp[kk];
            if (K.flags & CF_SKIP) continue;
            const int64_t lo = K.n_tiles * (int64_t)K.T;
            const int64_t n_tail = p.n_records - lo;
            if (n_tail <= 0) continue;
            // chain: hop kk's tail reads hop kk-1's tail output, so one CTA runs all hops' tails in order
            const bool own = (K.flags & CF_TAIL_ZERO) != 0 || H;
            const int64_t items = n_tail * (int64_t)(K.f_hi - K.f_lo);
            // (short tails of many components would otherwise all land on the first CTAs)
            const int64_t gfirst = (gid - acc % gstride + gstride) % gstride;
            if (!own) acc += items;
            if (own && gridDim.x - 1 - (H ? 0u : kk % gridDim.x) != blockIdx.x) continue;
            const int64_t first = own ? tid : gfirst, step = own ? (int64_t)(NCONS * 32) : gstride;
            if (own && (K.flags & CF_TAIL_ZERO)) {
                // every dst cluster of the component: bytes [lo*stride, ceil(N/B)*B*stride) := 0
                for (uint32_t f = K.f_lo; f < K.f_hi; ++f) {
                    const FieldDesc fd = ldg_field(et.fields + f);
                    const uint64_t B = 1ull << fd.dbl, st = p.dstc[fd.dc].stride;
                    const uint64_t a0 = p.dst + p.dstc[fd.dc].region + (uint64_t)lo * st;
                    const uint64_t a1 = p.dst + p.dstc[fd.dc].region + ((uint64_t)p.n_records + B - 1) / B * B * st;
                    for (uint64_t a = a0 + (uint64_t)tid * sizeof(U); a < a1; a += NCONS * 32 * sizeof(U))
                        *reinterpret_cast<U*>(a) = U(0);
                }
                named_bar_sync(2, NCONS * 32);
            }
            const int64_t total = items;
            for (int64_t x0 = first; x0 < total; x0 += 4 * step) {
                const U* sp[4];
                U* dp[4];
                uint32_t nu[4];
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const int64_t x = x0 + m * step;
                    nu[m] = 0;
                    if (x < total) {
                        // tails are shorter than a tile (< 16384 records): 32-bit division
                        const uint32_t q = (uint32_t)x / (uint32_t)n_tail;
                        const uint32_t f = K.f_lo + q;
                        const uint64_t r = (uint64_t)(lo + ((uint32_t)x - q * (uint32_t)n_tail));
                        const FieldDesc fd = ldg_field(et.fields + f);
                        const uint64_t ss = p.srcc[fd.sc].stride, ds = p.dstc[fd.dc].stride;
                        sp[m] = (const U*)(p.src + p.srcc[fd.sc].region + (r >> fd.sbl) * (ss << fd.sbl) +
                                           ((uint64_t)fd.soff << fd.sbl) + (r & ((1u << fd.sbl) - 1)) * fd.width);
                        dp[m] = (U*)(p.dst + p.dstc[fd.dc].region + (r >> fd.dbl) * (ds << fd.dbl) +
                                     ((uint64_t)fd.doff << fd.dbl) + (r & ((1u << fd.dbl) - 1)) * fd.width);
                        nu[m] = fd.width / (uint32_t)sizeof(U);
                    }
                }
                const uint32_t mx = max(max(nu[0], nu[1]), max(nu[2], nu[3]));
                for (uint32_t j = 0; j < mx; ++j) {
                    U v[4];
#pragma unroll
                    for (int m = 0; m < 4; ++m)
                        if (j < nu[m]) v[m] = sp[m][j];
#pragma unroll
                    for (int m = 0; m < 4; ++m)
                        if (j < nu[m]) dp[m][j] = v[m];
                }
            }
            if (H) named_bar_sync(2, NCONS * 32);             // hop kk's tail stored before hop kk+1 reads it
        }
    }

    ADHA_PT(long long ph[5] = {0, 0, 0, 0, 0}; ph[4] = clock64() - tt0);
    int k_cur = -1;
    uint32_t stage = 0, phase = 0, oslot = 0, k = 0;
    ADHA_PT(long long ntile = 0);
    constexpr bool tmac = TMAC;      // compile-time: the STG instantiations are the plain kernel
    uint32_t i_t = 0, zeroed = 0;
    const int64_t nt = cta_tiles(p, H);
    TileIter it;
    tile_begin(p, H, it);
    bool stored_pending = false;     // chain: tile i-1's stores not yet fenced and signalled
#ifndef ADHA_PDL_TRIGGER
#define ADHA_PDL_TRIGGER 1
#endif
    if (ADHA_PDL_TRIGGER && nt < ADHA_PDL_TRIGGER) grid_dep_launch();
    for (int64_t i = 0; i < nt; ++i, tile_next(p, H, it)) {
        // (PDL) this CTA's last tile: the next remap in the stream may be scheduled now, so its
        // launch is done by the time SMs free up (its global accesses still wait for this grid)
        if (ADHA_PDL_TRIGGER && i + ADHA_PDL_TRIGGER == nt) grid_dep_launch();
        k = it.k;
        const int64_t lt = it.lt;
        const uint32_t dist = it.dist;
        const uint32_t T = p.comp[k].T;
        if ((int)k != k_cur) {
            // this warp's instructions of component k: i = warp + NCONS*e; lane's unit = entry i*32 + lane
            k_cur = (int)k;
            zeroed = 0;
            if (!tmac) nv = copy_plan(p, dcl, p.comp[k].dc_lo, T, p.comp[k].out_bytes, tid, gofs, gstep);
            if (!tmac && (p.comp[k].flags & CF_ZERO_OUT)) {
                // dst records have padding the permutation never writes: zero both output buffers
                // once for this component (the same positions stay untouched in every tile)
                named_bar_sync(1, NCONS * 32);
                const uint4 z = make_uint4(0u, 0u, 0u, 0u);
                for (uint32_t v = tid * 16; v < p.s_out * p.stage_bytes; v += NCONS * 32 * 16) sts128(out0 + v, z);
                named_bar_sync(1, NCONS * 32);
            }
            if constexpr (NG > 0) {
                // G groups per period -> I instructions of 32 lanes; with I < NCONS the periods are
                // split over P = NCONS / I warps per instruction (slot s -> instruction s % I,
                // periods q = s / I (mod P)).  When NCONS * GMAX slots do not divide evenly by I
                // (GMAX = 2, I = 3, 5, 6, 7) that leaves some warps a slot more than others, so the
                // I x periods (instruction, period) items are cut into NCONS equal contiguous
                // ranges instead -- one per warp, at most two instructions each, periods step 1.
                // grho[j] = first period | end period << 16 of slot j.
                const uint32_t G = p.comp[k].n_instr;
                const uint32_t I = (G + 31) / 32;
                const uint32_t P = T / 32;
                const bool bal = GMAX == 2 && I > 0 && I <= (uint32_t)NCONS && ((uint32_t)(NCONS * GMAX) % I) != 0;
                gP = bal ? 1u : (I ? max(1u, (uint32_t)(NCONS * GMAX) / I) : 1u);
#pragma unroll
                for (int j = 0; j < GMAX; ++j) {
                    gns[j] = gno[j] = 0;
                    grho[j] = 0;
                    uint32_t i, q0, q1;
                    bool ok;
                    if (bal) {
                        const uint32_t items = I * P, lo = warp * items / NCONS, hi = (warp + 1) * items / NCONS;
                        i = lo / P + (uint32_t)j;
                        q0 = j == 0 ? lo - (lo / P) * P : 0u;
                        q1 = hi > i * P ? min(P, hi - i * P) : 0u;
                        ok = i < I && q0 < q1;
                    } else {
                        const uint32_t slot = warp + NCONS * j;
                        ok = I && slot < I * gP;
                        i = ok ? slot % I : 0u;
                        q0 = ok ? slot / I : 0u;
                        q1 = P;
                    }
                    if (ok) {
                        const uint32_t gi = i * 32 + lane;
                        grho[j] = q0 | (q1 << 16);
                        if (gi < G) {
                            // the group from its shared-memory copy (13 words, ByteGroup layout)
                            const uint32_t ga = tbl + (uint32_t)sizeof(ByteGroup) * (p.comp[k].instr_base + gi);
                            uint32_t w[13];
#pragma unroll
                            for (int q = 0; q < 13; ++q) w[q] = lds<uint32_t>(ga + 4 * q);
                            // words: out_off 0-1, src_off 2-3, sel 4-9, out_dc 10, src_sc 11, n_out|n_src 12
                            gno[j] = w[12] & 0xFFu;
                            gns[j] = (w[12] >> 8) & 0xFFu;
#pragma unroll
                            for (int m = 0; m < 4; ++m) {
                                const uint32_t sc = (w[11] >> (8 * m)) & 0xFFu, dc = (w[10] >> (8 * m)) & 0xFFu;
                                const uint32_t out_off = (w[m >> 1] >> (16 * (m & 1))) & 0xFFFFu;
                                const uint32_t src_off = (w[2 + (m >> 1)] >> (16 * (m & 1))) & 0xFFFFu;
                                // sel[m][t] is halfword 3m+t of words 4..9
                                const uint32_t h0 = 3 * m, h1 = 3 * m + 1, h2 = 3 * m + 2;
                                const uint32_t s0 = (w[4 + (h0 >> 1)] >> (16 * (h0 & 1))) & 0xFFFFu;
                                const uint32_t s1 = (w[4 + (h1 >> 1)] >> (16 * (h1 & 1))) & 0xFFFFu;
                                const uint32_t s2 = (w[4 + (h2 >> 1)] >> (16 * (h2 & 1))) & 0xFFFFu;
                                gsrc[j][m] = lds<uint32_t>(scl + 16 * sc + 12) + src_off;
                                gsst[j][m] = 32u * lds<uint32_t>(scl + 16 * sc + 8);
                                gout[j][m] = lds<uint32_t>(dcl + 16 * dc + 12) + out_off;
                                gost[j][m] = 32u * lds<uint32_t>(dcl + 16 * dc + 8);
                                gsel[j][m][0] = s0 | (s1 << 16);
                                gsel[j][m][1] = s2;
                            }
                        }
                    }
                }
            } else {
            const uint32_t W = p.comp[k].n_instr;
            ne = W > warp ? (W - warp + NCONS - 1) / NCONS : 0;
#pragma unroll
            for (int e = 0; e < EMAX; ++e) {
                ioff[e] = ooff[e] = din[e] = dout[e] = 0;
                if ((uint32_t)e < ne) {
                    const uint32_t idx = (p.comp[k].instr_base + warp + NCONS * e) * 32 + lane;
                    const uint32_t v = lds<uint32_t>(tbl + 4 * idx);
                    const uint32_t sc = (uint32_t)lds<uint8_t>(tbl + 4 * n4 + idx);
                    const uint32_t dc = (uint32_t)lds<uint8_t>(tbl + 5 * n4 + idx);
                    const uint32_t s_stride = lds<uint32_t>(scl + 16 * sc + 8), s_smem = lds<uint32_t>(scl + 16 * sc + 12);
                    const uint32_t d_stride = lds<uint32_t>(dcl + 16 * dc + 8), d_smem = lds<uint32_t>(dcl + 16 * dc + 12);
                    ioff[e] = s_smem + (v & 0xFFFFu) * (uint32_t)sizeof(U);
                    ooff[e] = d_smem + (v >> 16) * (uint32_t)sizeof(U);
                    din[e] = 32u * s_stride;
                    dout[e] = 32u * d_stride;
                }
            }
            }
        }
        ADHA_PT(const long long c0 = clock64());
        if (tmac) {
            // output buffer o of this tile: wait until the bulk store of its previous tile read it
            const uint32_t o = p.s_out == 2 ? (i_t & 1u) : 0u;
            const uint32_t j = p.s_out == 2 ? (i_t >> 1) : i_t;
            if (j > 0) mbar_wait(oempty0 + 8 * o, (j - 1) & 1u);
            oslot = o;
            if ((p.comp[k].flags & CF_ZERO_OUT) && !((zeroed >> o) & 1u)) {
                const uint4 z = make_uint4(0u, 0u, 0u, 0u);
                for (uint32_t v = tid * 16; v < p.stage_bytes; v += NCONS * 32 * 16) sts128(out0 + o * p.stage_bytes + v, z);
                named_bar_sync(1, NCONS * 32);
                zeroed |= 1u << o;
            }
        }
        mbar_wait(full0 + 8 * stage, phase);
        ADHA_PT(const long long c1 = clock64(); ph[0] += c1 - c0; ++ntile);
        const uint32_t ib = in0 + stage * p.stage_bytes;
        {
            const uint32_t ob = out0 + oslot * p.stage_bytes;
            if (!tmac && p.s_out == 1) named_bar_sync(1, NCONS * 32);   // previous copy-out done with the buffer
            if (p.comp[k].identity) {
                // same cluster on both sides: the staged chunk is already the output chunk; move it
                // to the output buffer with 16-byte shared copies so the input stage is released as
                // early as after a permutation (holding it through the copy-out starves the loads)
                const uint32_t tb = p.comp[k].tile_bytes;
                uint32_t v = tid * 16;
                for (; v + 3 * NCONS * 32 * 16 < tb; v += 4 * NCONS * 32 * 16) {
                    const uint4 a0 = lds128(ib + v), a1 = lds128(ib + v + NCONS * 32 * 16);
                    const uint4 a2 = lds128(ib + v + 2 * NCONS * 32 * 16), a3 = lds128(ib + v + 3 * NCONS * 32 * 16);
                    sts128(ob + v, a0);
                    sts128(ob + v + NCONS * 32 * 16, a1);
                    sts128(ob + v + 2 * NCONS * 32 * 16, a2);
                    sts128(ob + v + 3 * NCONS * 32 * 16, a3);
                }
                for (; v < tb; v += NCONS * 32 * 16) sts128(ob + v, lds128(ib + v));
            } else if constexpr (NG > 0) {
#pragma unroll
                for (int j = 0; j < GMAX; ++j) {
                    if (gno[j]) {
                        uint32_t q = grho[j] & 0xFFFFu;
                        const uint32_t periods = grho[j] >> 16;      // this slot's end period
                        // two periods per iteration: 8 independent shared loads in flight
                        for (; q + gP < periods; q += 2 * gP) {
                            uint32_t w[2][4];
#pragma unroll
                            for (int h = 0; h < 2; ++h)
#pragma unroll
                                for (int m = 0; m < 4; ++m)
                                    w[h][m] = ((uint32_t)m < gns[j])
                                                  ? lds<uint32_t>(ib + gsrc[j][m] + (q + h * gP) * gsst[j][m]) : 0u;
#pragma unroll
                            for (int h = 0; h < 2; ++h)
#pragma unroll
                                for (int o = 0; o < 4; ++o) {
                                    if ((uint32_t)o < gno[j]) {
                                        const uint32_t a = __byte_perm(w[h][0], w[h][1], gsel[j][o][0] & 0xFFFFu);
                                        const uint32_t b = __byte_perm(w[h][2], w[h][3], gsel[j][o][0] >> 16);
                                        sts(ob + gout[j][o] + (q + h * gP) * gost[j][o], __byte_perm(a, b, gsel[j][o][1]));
                                    }
                                }
                        }
                        for (; q < periods; q += gP) {
                            uint32_t w[4];
#pragma unroll
                            for (int m = 0; m < 4; ++m)
                                w[m] = ((uint32_t)m < gns[j]) ? lds<uint32_t>(ib + gsrc[j][m] + q * gsst[j][m]) : 0u;
#pragma unroll
                            for (int o = 0; o < 4; ++o) {
                                if ((uint32_t)o < gno[j]) {
                                    const uint32_t a = __byte_perm(w[0], w[1], gsel[j][o][0] & 0xFFFFu);
                                    const uint32_t b = __byte_perm(w[2], w[3], gsel[j][o][0] >> 16);
                                    sts(ob + gout[j][o] + q * gost[j][o], __byte_perm(a, b, gsel[j][o][1]));
                                }
                            }
                        }
                    }
                }
            } else {
                const uint32_t periods = T / 32;
#pragma unroll
                for (int e = 0; e < EMAX; ++e) {
                    if ((uint32_t)e < ne) {
                        const uint32_t ia = ib + ioff[e], oa = ob + ooff[e];
                        const uint32_t di = din[e], dO = dout[e];
                        uint32_t q = 0;
                        for (; q + 4 <= periods; q += 4) {
                            const U v0 = lds<U>(ia + (q + 0) * di);
                            const U v1 = lds<U>(ia + (q + 1) * di);
                            const U v2 = lds<U>(ia + (q + 2) * di);
                            const U v3 = lds<U>(ia + (q + 3) * di);
                            sts(oa + (q + 0) * dO, v0);
                            sts(oa + (q + 1) * dO, v1);
                            sts(oa + (q + 2) * dO, v2);
                            sts(oa + (q + 3) * dO, v3);
                        }
                        // the last periods % 4 (short tiles: all of them), loads first as above
                        const uint32_t r = periods - q;
                        if (r) {
                            const U v0 = lds<U>(ia + q * di);
                            const U v1 = r > 1 ? lds<U>(ia + (q + 1) * di) : v0;
                            const U v2 = r > 2 ? lds<U>(ia + (q + 2) * di) : v0;
                            sts(oa + q * dO, v0);
                            if (r > 1) sts(oa + (q + 1) * dO, v1);
                            if (r > 2) sts(oa + (q + 2) * dO, v2);
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty0 + 8 * stage);    // input stage free for the producer
            if (stored_pending) {
                // chain: tile i-1's stores were issued a permutation ago, so this fence rarely waits;
                // then signal that the next hop may load them
                fence_proxy_async_global();
                mbar_arrive(stored0 + 8 * ((uint32_t)(i - 1) & 7u));
                stored_pending = false;
            }
            ADHA_PT(const long long c2 = clock64(); ph[1] += c2 - c1);
            if (tmac) {
                fence_proxy_async_smem();                       // this thread's smem writes -> the bulk store
                mbar_arrive(ofull0 + 8 * oslot);
                ++i_t;
            } else {
                named_bar_sync(1, NCONS * 32);                  // output tile complete
                ADHA_PT(const long long c3 = clock64(); ph[2] += c3 - c2);
                if (H && p.chain_hints)
                    copy_out<true>((uint8_t*)p.dst, ob, tid, lt, nv, gofs, gstep, k + 1 < H ? kpol : spol);
                else if (p.l2_hints & 2) copy_out<true>((uint8_t*)p.dst, ob, tid, lt, nv, gofs, gstep, spol);
                else copy_out<false>((uint8_t*)p.dst, ob, tid, lt, nv, gofs, gstep, spol);
                if (H) {
                    // tile i stored: signal after the next tile's permutation (the fence then finds
                    // the stores done) unless a tile of dist 1 -- a single-band group -- loads them
                    // next, or this is the CTA's last tile
                    if (dist >= 2 && i + 1 < nt) {
                        stored_pending = true;
                    } else {
                        fence_proxy_async_global();
                        mbar_arrive(stored0 + 8 * ((uint32_t)i & 7u));
                    }
                }
                ADHA_PT(ph[3] += clock64() - c3);
                if (p.s_out == 2) oslot ^= 1;
            }
        }
        if (++stage == p.s_in) { stage = 0; phase ^= 1; }
    }
    ADHA_PT(if (lane == 0) {
        for (int i = 0; i < 4; ++i) atomicAdd(&g_phase[i], (unsigned long long)ph[i]);
        atomicAdd(&g_phase[4], (unsigned long long)ntile);
        atomicAdd(&g_phase[7], (unsigned long long)ph[4]);
    });

}

// Upload of a plan table inside a captured stream (remap.cu device_table): the image travels as
// this kernel's parameter and is stored to its device copy.
struct TableUpload {
    uint4 w[1600];        // 25 600 bytes >= the largest EntryTable / GroupTable image
    uint64_t dst;
    uint32_t n16, pad;
};
__global__ void table_upload_kernel(const __grid_constant__ TableUpload u) {
    uint4* d = reinterpret_cast<uint4*>(u.dst);
    for (uint32_t i = threadIdx.x; i < u.n16; i += blockDim.x) d[i] = u.w[i];
}

constexpr int ZMAX = 128;
struct ZeroParams {
    uint32_t n, pad;
    uint64_t ptr[ZMAX];
    uint64_t bytes[ZMAX];
};
// zero whole byte ranges (dst regions with padding, direct path); 16-byte stores where aligned
__global__ void zero_kernel(const __grid_constant__ ZeroParams z) {
    for (uint32_t i = 0; i < z.n; ++i) {
        uint8_t* p = (uint8_t*)z.ptr[i];
        const uint64_t nb = z.bytes[i];
        const uint64_t head = ((16 - ((uintptr_t)p & 15)) & 15) < nb ? ((16 - ((uintptr_t)p & 15)) & 15) : nb;
        const uint64_t nv = (nb - head) / 16;
        for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < nv; k += (uint64_t)gridDim.x * blockDim.x)
            reinterpret_cast<uint4*>(p + head)[k] = make_uint4(0u, 0u, 0u, 0u);
        if (blockIdx.x == 0)
            for (uint64_t k = threadIdx.x; k < head + (nb - head) % 16; k += blockDim.x)
                p[k < head ? k : head + nv * 16 + (k - head)] = 0;
    }
}

template <int NF>
__global__ void remap_naive_kernel(const __grid_constant__ NaiveParamsT<NF> p) {
    // (PDL) the previous kernel's writes first; the next launch may be scheduled once every block
    // of this grid has started (its own accesses wait for this grid to complete)
    grid_dep_wait();
    grid_dep_launch();
    const int64_t n = p.n_records;
    const int64_t total = n * (int64_t)p.n_fields;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t f = (uint32_t)(k / n);
        const int64_t r = p.lo + (k - (int64_t)f * n);
        const NaiveField& fd = p.f[f];
        const uint32_t sbl = fd.pad & 0xFF, dbl = (fd.pad >> 8) & 0xFF;
        const uint64_t ur = (uint64_t)r;
        const uint8_t* s = (const uint8_t*)(p.src + fd.sbase + (ur >> sbl) * ((uint64_t)fd.sstride << sbl) +
                                            ((uint64_t)fd.soff << sbl) + (ur & ((1u << sbl) - 1)) * fd.width);
        uint8_t* d = (uint8_t*)(p.dst + fd.dbase + (ur >> dbl) * ((uint64_t)fd.dstride << dbl) +
                                ((uint64_t)fd.doff << dbl) + (ur & ((1u << dbl) - 1)) * fd.width);
        const uintptr_t a = (uintptr_t)s | (uintptr_t)d | fd.width;
        uint32_t j = 0;
        if ((a & 3) == 0) {
            for (; j < fd.width; j += 4) *reinterpret_cast<uint32_t*>(d + j) = *reinterpret_cast<const uint32_t*>(s + j);
        } else {
            for (; j < fd.width; ++j) d[j] = s[j];
        }
    }
}

__global__ void __launch_bounds__(256) remap_chain_small_kernel(const __grid_constant__ ChainParams p) {
    grid_dep_wait();                     // (PDL) as remap_naive_kernel
    grid_dep_launch();
    const int64_t n = p.n_records;
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t lo = (int64_t)blockIdx.x * per;
    const int64_t m = lo < n ? min(per, n - lo) : 0;
    const int64_t total = m * (int64_t)p.n_fields;
    for (uint32_t h = 0; h < p.n_hops; ++h) {
        const uint8_t* src = (const uint8_t*)p.buf[h];
        uint8_t* dst = (uint8_t*)p.buf[h + 1];
        for (int64_t k = threadIdx.x; k < total; k += blockDim.x) {
            const uint32_t f = (uint32_t)(k / m);
            const uint64_t r = (uint64_t)(lo + (k - (int64_t)f * m));
            const NaiveField& fd = p.f[h][f];
            const uint8_t* s = src + fd.sbase + r * fd.sstride + fd.soff;
            uint8_t* d = dst + fd.dbase + r * fd.dstride + fd.doff;
            uint32_t j = 0;
            if ((((uintptr_t)s | (uintptr_t)d | fd.width) & 3) == 0) {
                for (; j < fd.width; j += 4) *reinterpret_cast<uint32_t*>(d + j) = *reinterpret_cast<const uint32_t*>(s + j);
            } else {
                for (; j < fd.width; ++j) d[j] = s[j];
            }
        }
        __syncthreads();     // hop h's stores by this block are visible to the whole block
    }
}

}  // namespace dev
}  // namespace adha
