// remap.cu -- the ADHA remap on B200 (sm_100a): kernels, launch, and the
// remap entry points of the C ABI.
//
// What it computes (adha.h): for all records i and fields f
//     dst[addr_Ld(f,i) .. +w_f) = src[addr_Ls(f,i) .. +w_f)
// as a type-blind copy: integer loads/stores only, never an FP instruction
// (NaN payloads must survive, reading Q6).
//
// remap_tiled_kernel (the hot path):
//   persistent CTAs, one per SM (1 CTA/SM: ~200 KB of shared memory), 9 warps:
//   * warp 8 (producer): per tile, one TMA bulk copy (cp.async.bulk, SASS
//     UBLKCP) per src cluster chunk into an input stage, completion counted as
//     transaction bytes on the stage's mbarrier; s_in stages in flight;
//   * warps 0-7 (consumers): permute the staged tile into an output buffer with
//     32-bit (or 16/8-bit) shared loads/stores driven by a per-lane table held
//     in registers -- conflict-free by construction for 4-byte units -- then
//     warp 0 writes every dst cluster chunk back with one TMA bulk store each
//     (cp.async.bulk.global.shared::cta) from a double-buffered output stage;
//   * the last CTA finishes the N mod T tail records with plain loads/stores.
// remap_naive_kernel: one thread per (record, field) unit copy; used only for
//   layouts beyond the tiled kernel's limits (more than 256 fields, ...).
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

__device__ __forceinline__ uint32_t copy_plan(const TiledParams& p, uint32_t c_lo, uint32_t T, uint32_t total,
                                              uint32_t tid, uint64_t (&gofs)[VMAX], uint32_t (&gstep)[VMAX]) {
    constexpr uint32_t NT = NCONS * 32;
    uint32_t c = c_lo, cbeg = 0, cend = T * p.dstc[c].stride;
    uint32_t nv = 0;
#pragma unroll
    for (uint32_t u = 0; u < VMAX; ++u) {
        const uint32_t b = tid * 16 + u * NT * 16;
        gofs[u] = 0;
        gstep[u] = 0;
        if (b < total) {
            while (b >= cend) {
                ++c;
                cbeg = cend;
                cend = cbeg + T * p.dstc[c].stride;
            }
            gofs[u] = p.dstc[c].region + (b - cbeg);
            // the per-tile step T*stride is a multiple of 128; its low 7 bits carry the chunk's
            // padding in the output stage / 32 (smem offset - packed offset = 32 * chunk index)
            gstep[u] = (cend - cbeg) | ((p.dstc[c].smem - cbeg) >> 5);
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

// Tile order of a CTA: interleaved (t = b, b+G, ...: the GPU sweeps the arrays as one front)
// or blocked (CTA b takes the contiguous range [b*M/G, (b+1)*M/G)).
__device__ __forceinline__ int64_t t_first(const TiledParams& p) {
    return p.blocked ? (int64_t)blockIdx.x * p.total_tiles / gridDim.x : (int64_t)blockIdx.x;
}
__device__ __forceinline__ int64_t t_end(const TiledParams& p) {
    return p.blocked ? (int64_t)(blockIdx.x + 1) * p.total_tiles / gridDim.x : p.total_tiles;
}
__device__ __forceinline__ int64_t t_step(const TiledParams& p) { return p.blocked ? 1 : (int64_t)gridDim.x; }

// 9 warps per CTA: the register file is split over the 4 SM sub-partitions (16K registers
// each) and one of them holds 3 warps, so a thread may use at most 16384 / 96 = 168 registers;
// __launch_bounds__(NTHREADS, 1) gives ptxas exactly that budget.
template <int NENT, int NG>
using TableOf = typename std::conditional<(NG > 0), GroupTable<NG>, EntryTable<NENT>>::type;

// NG = 0: unit mode (EntryTable<NENT>, EMAX instructions per warp); NG > 0: byte-group mode
// (GroupTable<NG>, GMAX slots per warp, U = uint8_t for the tails).
template <typename U, int NENT, int EMAX, int NG = 0, int GMAX = 1>
__global__ void __launch_bounds__(NTHREADS, 1)
    remap_tiled_kernel(const __grid_constant__ TiledParams p, const __grid_constant__ TableOf<NENT, NG> et) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t sbase = (smem_u32(smem) + 127u) & ~127u;
    const uint32_t full0 = sbase;                      // s_in mbarriers: tile landed
    const uint32_t empty0 = sbase + 8 * MAX_S_IN;      // s_in mbarriers: stage consumed
    const uint32_t in0 = sbase + HDR_BYTES;
    const uint32_t out0 = in0 + p.s_in * p.stage_bytes;

    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < p.s_in; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, NCONS);
        }
        fence_mbarrier_init();
    }
    __syncthreads();

    if (warp == NCONS) {
        // ------------------------------------------------------------ TMA producer
        // Per component, every lane holds up to PMAX bulk-load pieces of the tile (src chunks cut
        // into pieces of at most `split` bytes): smem offset, global offset of tile 0, bytes, and
        // the per-tile global step.  Issue is then one bulk copy per piece per lane, no parameter
        // walks on the critical path (the producer's issue time gates the 2-stage pipeline).
        const uint64_t pol = policy_evict_first();        // src is read once: evict it first from L2
        uint32_t psm[PMAX], pbytes[PMAX], pstep[PMAX];
        uint64_t pg[PMAX];
        uint32_t np = 0;
        int kp = -1;
        uint32_t stage = 0, phase = 0, k = 0;
        for (int64_t t = t_first(p), te = t_end(p); t < te; t += t_step(p)) {
            while (t >= p.comp[k].tile_base + p.comp[k].n_tiles) ++k;
            const int64_t lt = t - p.comp[k].tile_base;
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
            mbar_wait(empty0 + 8 * stage, phase ^ 1);
            if (lane == 0) mbar_arrive_expect_tx(full0 + 8 * stage, p.comp[k].tile_bytes);
            __syncwarp();
            const uint32_t ib = in0 + stage * p.stage_bytes;
#pragma unroll
            for (uint32_t q = 0; q < PMAX; ++q) {
                if (q < np) {
                    const void* g = (const void*)(pg[q] + (uint64_t)lt * pstep[q]);
                    if (p.l2_hints & 1) bulk_load_hint(ib + psm[q], g, pbytes[q], full0 + 8 * stage, pol);
                    else bulk_load(ib + psm[q], g, pbytes[q], full0 + 8 * stage);
                }
            }
            if (++stage == p.s_in) { stage = 0; phase ^= 1; }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    const uint32_t tid = threadIdx.x;
    const uint64_t spol = policy_evict_first();
    uint32_t ioff[EMAX], ooff[EMAX], din[EMAX], dout[EMAX];
    // byte-group mode: per slot j, source words m and output words o of this lane's group
    uint32_t gsrc[GMAX][4], gsst[GMAX][4], gout[GMAX][4], gost[GMAX][4], gsel[GMAX][4][2];
    uint32_t gns[GMAX], gno[GMAX], grho[GMAX], gP = 1;
    uint64_t gofs[VMAX];
    uint32_t gstep[VMAX];
    uint32_t ne = 0, nv = 0;

    // Tails first: records [n_tiles*T_k, N) of every component.  Plain components spread their
    // tail over the consumer threads of ALL CTAs, four records in flight per thread, while the
    // producer's first tiles are still in flight (one CTA copying a 48 KB tail alone took ~40 us).
    // Components whose dst has padding or AoSoA blocks (CF_TAIL_ZERO) zero their dst tail area
    // first, so their tail belongs to one CTA (zero, barrier, copy).
    {
        const int64_t gid = (int64_t)blockIdx.x * (NCONS * 32) + tid;
        const int64_t gstride = (int64_t)gridDim.x * (NCONS * 32);
        for (uint32_t kk = 0; kk < p.n_comp; ++kk) {
            const CompDesc& K = p.comp[kk];
            if (K.flags & CF_SKIP) continue;
            const int64_t lo = K.n_tiles * (int64_t)K.T;
            const int64_t n_tail = p.n_records - lo;
            if (n_tail <= 0) continue;
            const bool own = (K.flags & CF_TAIL_ZERO) != 0;
            if (own && gridDim.x - 1 - (kk % gridDim.x) != blockIdx.x) continue;
            const int64_t first = own ? tid : gid, step = own ? (int64_t)(NCONS * 32) : gstride;
            if (own) {
                // every dst cluster of the component: bytes [lo*stride, ceil(N/B)*B*stride) := 0
                for (uint32_t f = K.f_lo; f < K.f_hi; ++f) {
                    const FieldDesc fd = et.fields[f];
                    const uint64_t B = 1ull << fd.dbl, st = p.dstc[fd.dc].stride;
                    const uint64_t a0 = p.dst + p.dstc[fd.dc].region + (uint64_t)lo * st;
                    const uint64_t a1 = p.dst + p.dstc[fd.dc].region + ((uint64_t)p.n_records + B - 1) / B * B * st;
                    for (uint64_t a = a0 + (uint64_t)tid * sizeof(U); a < a1; a += NCONS * 32 * sizeof(U))
                        *reinterpret_cast<U*>(a) = U(0);
                }
                named_bar_sync(2, NCONS * 32);
            }
            const int64_t total = n_tail * (int64_t)(K.f_hi - K.f_lo);
            for (int64_t x0 = first; x0 < total; x0 += 4 * step) {
                const U* sp[4];
                U* dp[4];
                uint32_t nu[4];
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const int64_t x = x0 + m * step;
                    nu[m] = 0;
                    if (x < total) {
                        const uint32_t f = K.f_lo + (uint32_t)(x / n_tail);
                        const uint64_t r = (uint64_t)(lo + (x % n_tail));
                        const FieldDesc fd = et.fields[f];
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
        }
    }

    int k_cur = -1;
    uint32_t stage = 0, phase = 0, oslot = 0, k = 0;
    for (int64_t t = t_first(p), te = t_end(p); t < te; t += t_step(p)) {
        while (t >= p.comp[k].tile_base + p.comp[k].n_tiles) ++k;
        const int64_t lt = t - p.comp[k].tile_base;
        const uint32_t T = p.comp[k].T;
        if ((int)k != k_cur) {
            // this warp's instructions of component k: i = warp + NCONS*e; lane's unit = entry i*32 + lane
            k_cur = (int)k;
            nv = copy_plan(p, p.comp[k].dc_lo, T, p.comp[k].out_bytes, tid, gofs, gstep);
            if (p.comp[k].flags & CF_ZERO_OUT) {
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
                // periods q = s / I (mod P))
                const uint32_t G = p.comp[k].n_instr;
                const uint32_t I = (G + 31) / 32;
                gP = I ? max(1u, (uint32_t)(NCONS * GMAX) / I) : 1u;
#pragma unroll
                for (int j = 0; j < GMAX; ++j) {
                    gns[j] = gno[j] = 0;
                    grho[j] = 0;
                    const uint32_t slot = warp + NCONS * j;
                    if (I && slot < I * gP) {
                        const uint32_t i = slot % I, gi = i * 32 + lane;
                        grho[j] = slot / I;
                        if (gi < G) {
                            const ByteGroup& gr = et.g[p.comp[k].instr_base + gi];
                            gns[j] = gr.n_src;
                            gno[j] = gr.n_out;
#pragma unroll
                            for (int m = 0; m < 4; ++m) {
                                const ClusterDesc& cs = p.srcc[gr.src_sc[m]];
                                const ClusterDesc& cd = p.dstc[gr.out_dc[m]];
                                gsrc[j][m] = cs.smem + gr.src_off[m];
                                gsst[j][m] = 32u * cs.stride;
                                gout[j][m] = cd.smem + gr.out_off[m];
                                gost[j][m] = 32u * cd.stride;
                                gsel[j][m][0] = (uint32_t)gr.sel[m][0] | ((uint32_t)gr.sel[m][1] << 16);
                                gsel[j][m][1] = gr.sel[m][2];
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
                    const uint32_t v = et.off[idx];
                    const ClusterDesc& cs = p.srcc[et.sc[idx]];
                    const ClusterDesc& cd = p.dstc[et.dc[idx]];
                    ioff[e] = cs.smem + (v & 0xFFFFu) * (uint32_t)sizeof(U);
                    ooff[e] = cd.smem + (v >> 16) * (uint32_t)sizeof(U);
                    din[e] = 32u * cs.stride;
                    dout[e] = 32u * cd.stride;
                }
            }
            }
        }
        mbar_wait(full0 + 8 * stage, phase);
        const uint32_t ib = in0 + stage * p.stage_bytes;
        {
            const uint32_t ob = out0 + oslot * p.stage_bytes;
            if (p.s_out == 1) named_bar_sync(1, NCONS * 32);   // previous copy-out done with the buffer
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
                const uint32_t periods = T / 32;
#pragma unroll
                for (int j = 0; j < GMAX; ++j) {
                    if (gno[j]) {
                        uint32_t q = grho[j];
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
                        for (; q < periods; ++q) sts(oa + q * dO, lds<U>(ia + q * di));
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty0 + 8 * stage);    // input stage free for the producer
            named_bar_sync(1, NCONS * 32);                      // output tile complete
            if (p.l2_hints & 2) copy_out<true>((uint8_t*)p.dst, ob, tid, lt, nv, gofs, gstep, spol);
            else copy_out<false>((uint8_t*)p.dst, ob, tid, lt, nv, gofs, gstep, spol);
            if (p.s_out == 2) oslot ^= 1;
        }
        if (++stage == p.s_in) { stage = 0; phase ^= 1; }
    }

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

}  // namespace dev

// ============================================================================ host side


using namespace dev;

static_assert(sizeof(dev::TiledParams) + sizeof(dev::EntryTable<dev::CLASS_NENT[3]>) <= 32764,
              "tiled kernel parameters exceed the 32764-byte kernel parameter limit");
static_assert(sizeof(dev::TiledParams) + sizeof(dev::GroupTable<dev::GCLASS_NG[1]>) <= 32764,
              "byte-group kernel parameters exceed the 32764-byte kernel parameter limit");
static_assert(sizeof(dev::ByteGroup) == 52, "ByteGroup layout");
static_assert(sizeof(dev::NaiveParams) <= 32764, "naive kernel parameters too large");

namespace {

typedef void (*TiledLauncher)(dim3, dim3, size_t, cudaStream_t, const TiledParams&, const void* table);

template <typename U, int CLS>
void launch_tiled(dim3 grid, dim3 block, size_t smem, cudaStream_t st, const TiledParams& p, const void* table) {
    constexpr int NENT = CLASS_NENT[CLS];
    constexpr int EMAX = CLASS_EMAX[CLS];
    remap_tiled_kernel<U, NENT, EMAX><<<grid, block, smem, st>>>(p, *static_cast<const EntryTable<NENT>*>(table));
}

template <typename U, int CLS>
const void* tiled_fn() {
    constexpr int NENT = CLASS_NENT[CLS];
    constexpr int EMAX = CLASS_EMAX[CLS];
    return (const void*)&remap_tiled_kernel<U, NENT, EMAX>;
}

template <typename U>
TiledLauncher pick_cls(int cls, const void** fn) {
    switch (cls) {
        case 0: *fn = tiled_fn<U, 0>(); return &launch_tiled<U, 0>;
        case 1: *fn = tiled_fn<U, 1>(); return &launch_tiled<U, 1>;
        case 2: *fn = tiled_fn<U, 2>(); return &launch_tiled<U, 2>;
        default: *fn = tiled_fn<U, 3>(); return &launch_tiled<U, 3>;
    }
}

template <int GC>
void launch_groups(dim3 grid, dim3 block, size_t smem, cudaStream_t st, const TiledParams& p, const void* table) {
    constexpr int NG = GCLASS_NG[GC];
    constexpr int GMAX = GCLASS_GMAX[GC];
    remap_tiled_kernel<uint8_t, 32, 1, NG, GMAX><<<grid, block, smem, st>>>(p, *static_cast<const GroupTable<NG>*>(table));
}
template <int GC>
const void* groups_fn() {
    return (const void*)&remap_tiled_kernel<uint8_t, 32, 1, GCLASS_NG[GC], GCLASS_GMAX[GC]>;
}

TiledLauncher pick_groups(int gcls, const void** fn) {
    if (gcls == 0) { *fn = groups_fn<0>(); return &launch_groups<0>; }
    *fn = groups_fn<1>();
    return &launch_groups<1>;
}

TiledLauncher pick(uint32_t unit, int cls, const void** fn) {
    if (unit == 4) return pick_cls<uint32_t>(cls, fn);
    if (unit == 2) return pick_cls<uint16_t>(cls, fn);
    return pick_cls<uint8_t>(cls, fn);
}

struct PlanCache {
    std::mutex mu;
    std::map<std::pair<uint64_t, uint64_t>, std::shared_ptr<const RemapPlan>> plans;
    std::set<std::tuple<int, const void*>> attr_done;
    std::map<int, int> sm_count;
};
PlanCache& cache() {
    static PlanCache c;
    return c;
}

std::shared_ptr<const RemapPlan> get_plan(const Layout& ls, const Layout& ld) {
    PlanCache& c = cache();
    std::lock_guard<std::mutex> g(c.mu);
    auto key = std::make_pair(ls.id, ld.id);
    auto it = c.plans.find(key);
    if (it != c.plans.end()) return it->second;
    if (c.plans.size() > 4096) c.plans.clear();
    auto p = std::make_shared<const RemapPlan>(compile_plan(ls, ld));
    c.plans.emplace(key, p);
    return p;
}

adha_status cuda_fail(cudaError_t e, const char* what) {
    return fail(ADHA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// per-device setup: SM count and the kernel's dynamic shared memory opt-in
adha_status device_setup(const void* fn, int* n_sm) {
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
        if (fa.maxThreadsPerBlock < NTHREADS)      // register budget regression guard
            return fail(ADHA_ERR_UNSUPPORTED, "remap_tiled_kernel uses " + std::to_string(fa.numRegs) +
                                                  " registers: cannot launch " + std::to_string(NTHREADS) + " threads");
        c.attr_done.insert({dev, fn});
    }
    return ADHA_OK;
}

// Direct global->global kernel: the fallback beyond the tiled kernel's limits, and the
// latency path for small remaps (a handful of KB, where one launch with small parameters
// and one load/store per unit beats staging through shared memory).
template <int NF>
adha_status launch_naive_t(const uint8_t* src, const Layout& ls, const std::vector<uint64_t>& bs, uint8_t* dst,
                           const Layout& ld, const std::vector<uint64_t>& bd, int64_t lo, int64_t hi,
                           cudaStream_t st) {
    int n_sm = 0;
    adha_status s = device_setup(nullptr, &n_sm);
    if (s != ADHA_OK) return s;
    auto P = std::make_unique<NaiveParamsT<NF>>();
    for (int f0 = 0; f0 < ls.n_fields; f0 += NF) {
        std::memset(P.get(), 0, sizeof(NaiveParamsT<NF>));
        P->src = (uint64_t)(uintptr_t)src;
        P->dst = (uint64_t)(uintptr_t)dst;
        P->n_records = hi - lo;
        P->lo = lo;
        const int nf = std::min(NF, ls.n_fields - f0);
        P->n_fields = (uint32_t)nf;
        for (int k = 0; k < nf; ++k) {
            const int f = f0 + k;
            const int cs = ls.cluster[f], cd = ld.cluster[f];
            uint32_t sbl = 0, dbl = 0;
            while ((1u << sbl) < ls.block[cs]) ++sbl;
            while ((1u << dbl) < ld.block[cd]) ++dbl;
            P->f[k] = {bs[cs], bd[cd], (uint32_t)ls.stride[cs], (uint32_t)ld.stride[cd], ls.offset[f], ld.offset[f],
                       ls.width[f], sbl | (dbl << 8)};
        }
        const int64_t total = (hi - lo) * (int64_t)nf;
        const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, (int64_t)n_sm * 16));
        remap_naive_kernel<NF><<<(unsigned)blocks, 256, 0, st>>>(*P);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "remap_naive_kernel launch");
    }
    return ADHA_OK;
}

adha_status launch_naive(const uint8_t* src, const Layout& ls, const std::vector<uint64_t>& bs, uint8_t* dst,
                         const Layout& ld, const std::vector<uint64_t>& bd, int64_t lo, int64_t hi,
                         cudaStream_t st) {
    // dst clusters with padding or AoSoA blocks: zero their regions first (the copy fills the payload)
    ZeroParams Z;
    std::memset(&Z, 0, sizeof Z);
    for (int c = 0; c < ld.n_clusters(); ++c) {
        if (ld.stride[c] == ld.payload(c) && ld.block[c] == 1) continue;
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

struct Checked {
    uint64_t bytes_s = 0, bytes_d = 0;
    std::vector<uint64_t> bs, bd;
};

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
    // small remaps (<= ADHA_SMALL_BYTES of payload, 64 KB by default) are latency-bound: direct kernel
    if (!plan->tiled || (uint64_t)n * ls.record_bytes <= small_bytes())
        return launch_naive(src, ls, ck.bs, dst, ld, ck.bd, 0, n, st);

    const void* fn = nullptr;
    TiledLauncher launch = plan->byte_groups ? pick_groups(plan->group_class, &fn)
                                             : pick(plan->unit, plan->table_class, &fn);
    int n_sm = 0;
    adha_status s = device_setup(fn, &n_sm);
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
    // a tail-only call still needs one CTA per component tail
    const int64_t grid = std::max<int64_t>(std::min<int64_t>((int64_t)plan->comps.size(), n_sm),
                                           std::min<int64_t>(tiles, n_sm));
    launch(dim3((unsigned)std::max<int64_t>(grid, 1)), dim3(NTHREADS), plan->smem_bytes, st, *P, plan->table.data());
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "remap_tiled_kernel launch");
    return ADHA_OK;
}

}  // namespace
}  // namespace adha

using namespace adha;

extern "C" adha_status adha_remap(const void* src, const adha_layout* hs, void* dst, const adha_layout* hd,
                                  int64_t n, void* stream) {
    clear_error();
    Checked ck;
    adha_status s = validate(src, hs, dst, hd, n, &ck, true);
    if (s != ADHA_OK) return s;
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
        spans.push_back({a, a + (uint64_t)n * ls.stride[c], 0, c});
    }
    for (int c = 0; c < ld.n_clusters(); ++c) {
        const uint64_t a = (uint64_t)(uintptr_t)dst_regions[c];
        if (!a) return fail(ADHA_ERR_INVALID_ARG, "null dst region " + std::to_string(c));
        if (a & 255) return fail(ADHA_ERR_ALIGNMENT, "dst region " + std::to_string(c) + " not 256-byte aligned");
        ck.bd[c] = a;
        spans.push_back({a, a + (uint64_t)n * ld.stride[c], 1, c});
    }
    for (size_t i = 0; i < spans.size(); ++i)
        for (size_t j = i + 1; j < spans.size(); ++j) {
            const Span& x = spans[i];
            const Span& y = spans[j];
            if (!(x.lo < y.hi && y.lo < x.hi)) continue;
            if (x.side == 0 && y.side == 0) continue;                  // src regions may share memory
            // a dst region may BE the src region of an identical cluster: nothing moves there
            const bool alias = x.side != y.side && x.lo == y.lo &&
                               ls.members[x.side == 0 ? x.c : y.c] == ld.members[x.side == 0 ? y.c : x.c];
            if (!alias) return fail(ADHA_ERR_OVERLAP, "regions overlap (only identical clusters may alias)");
        }
    return remap_checked(nullptr, ls, nullptr, ld, n, ck, (cudaStream_t)stream);
}

extern "C" adha_status adha_remap_chain(void* const* buffers, const adha_layout* const* layouts, int32_t n_layouts,
                                        int64_t n, void* stream) {
    clear_error();
    if (!buffers || !layouts || n_layouts < 2) return fail(ADHA_ERR_INVALID_ARG, "need at least two layouts");
    for (int32_t k = 0; k + 1 < n_layouts; ++k) {
        adha_status s = adha_remap(buffers[k], layouts[k], buffers[k + 1], layouts[k + 1], n, stream);
        if (s != ADHA_OK) return s;
    }
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

// ---------------------------------------------------------------------------- host end-to-end
namespace adha {
namespace {
constexpr int PIPE_SLOTS = 4;        // chunks in flight through the device scratch

struct HostPipe {
    cudaStream_t s[PIPE_SLOTS] = {};
    cudaEvent_t start = nullptr, done[PIPE_SLOTS] = {};
};
std::mutex g_pipe_mu;
std::map<int, HostPipe> g_pipes;

adha_status get_pipe(HostPipe** out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    std::lock_guard<std::mutex> g(g_pipe_mu);
    auto it = g_pipes.find(dev);
    if (it == g_pipes.end()) {
        HostPipe hp;
        for (int i = 0; i < PIPE_SLOTS; ++i) {
            if ((e = cudaStreamCreateWithFlags(&hp.s[i], cudaStreamNonBlocking)) != cudaSuccess)
                return cuda_fail(e, "cudaStreamCreate");
            if ((e = cudaEventCreateWithFlags(&hp.done[i], cudaEventDisableTiming)) != cudaSuccess)
                return cuda_fail(e, "cudaEventCreate");
        }
        if ((e = cudaEventCreateWithFlags(&hp.start, cudaEventDisableTiming)) != cudaSuccess)
            return cuda_fail(e, "cudaEventCreate");
        it = g_pipes.emplace(dev, hp).first;
    }
    *out = &it->second;
    return ADHA_OK;
}
}  // namespace
}  // namespace adha

namespace adha {
namespace {
bool is_pinned_host(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost && a.devicePointer == p;   // pinned and UVA-mapped at the same address
}

uint64_t env_bytes(const char* name, uint64_t dflt) {
    const char* e = std::getenv(name);
    return e && *e ? std::strtoull(e, nullptr, 10) : dflt;
}
}  // namespace
}  // namespace adha

extern "C" adha_status adha_remap_host(const void* src_host, const adha_layout* hs, void* dst_host,
                                       const adha_layout* hd, int64_t n, void* scratch, uint64_t scratch_bytes,
                                       void* stream) {
    clear_error();
    Checked ck;
    adha_status s = validate(src_host, hs, dst_host, hd, n, &ck, false);
    if (s != ADHA_OK) return s;
    if (n == 0) return ADHA_OK;
    const Layout& ls = hs->L;
    const Layout& ld = hd->L;
    cudaStream_t user = (cudaStream_t)stream;
    const bool src_pinned = is_pinned_host(src_host), dst_pinned = is_pinned_host(dst_host);
    const bool aligned = !(((uintptr_t)src_host | (uintptr_t)dst_host) & 255);
    // Modes (ADHA_HOST_MODE = auto | zero | hybrid | staged):
    //   hybrid  the copy engine streams src chunks into the device scratch (one H2D per src region),
    //           the remap kernel of each chunk writes its records straight into the pinned host dst
    //           over PCIe -- both PCIe directions busy, no D2H copies;
    //   zero    one remap kernel reads the pinned host src (TMA over PCIe) and writes the pinned
    //           host dst directly, no scratch at all;
    //   staged  H2D per src region, remap in device memory, D2H per dst region (pageable memory).
    std::string mode = std::getenv("ADHA_HOST_MODE") ? std::getenv("ADHA_HOST_MODE") : "auto";
    if (mode == "auto") mode = (dst_pinned && aligned && scratch) ? "hybrid" : "staged";
    if ((mode == "zero" && !(src_pinned && dst_pinned && aligned)) || (mode == "hybrid" && !(dst_pinned && aligned)))
        mode = "staged";
    if (mode == "zero") return remap_checked((const uint8_t*)src_host, ls, (uint8_t*)dst_host, ld, n, ck, user);

    if (!scratch || ((uintptr_t)scratch & 255)) return fail(ADHA_ERR_ALIGNMENT, "scratch must be 256-byte aligned");
    const bool hybrid = mode == "hybrid";
    // Records stream through the scratch in chunks of nc records (a multiple of 4096, so host
    // region offsets lo*stride stay 16-byte aligned); each chunk is its own layout instance
    // (record locality).  PIPE_SLOTS chunks are in flight on PIPE_SLOTS internal streams.
    int slots = PIPE_SLOTS;
    uint64_t Rs = 0, Rd = 0;                   // bytes per record incl. alignment padding
    for (int c = 0; c < ls.n_clusters(); ++c) Rs += ls.stride[c];
    for (int c = 0; c < ld.n_clusters(); ++c) Rd += ld.stride[c];
    // region alignment (256 B per region) and a partial last AoSoA block (< 32 records)
    const uint64_t pad = 256ull * (ls.n_clusters() + ld.n_clusters() + 2) + 32 * (Rs + Rd);
    const uint64_t R = Rs;
    const uint64_t per_rec = hybrid ? Rs : Rs + Rd;
    uint64_t slot = 0;
    for (; slots >= 1; --slots) {
        slot = (scratch_bytes / slots) & ~uint64_t(255);
        if (slot > pad + 4096 * per_rec) break;
    }
    if (slots < 1) return fail(ADHA_ERR_INVALID_ARG, "scratch too small for a chunk of 4096 records");
    // chunk: ~16 MB (hybrid) / 64 MB (staged), but at least 4 MB per src region so every H2D
    // copy stays large (C3's 64 SoA regions -> 256 MB chunks)
    const uint64_t dflt = std::max<uint64_t>(hybrid ? (16ull << 20) : (64ull << 20), (4ull << 20) * ls.n_clusters());
    const uint64_t chunk_bytes = env_bytes("ADHA_HOST_CHUNK_BYTES", dflt);
    int64_t nc = std::min<int64_t>((int64_t)((slot - pad) / per_rec), (int64_t)std::max<uint64_t>(1, chunk_bytes / R));
    nc = std::max<int64_t>(4096, nc / 4096 * 4096);
    nc = std::min<int64_t>(nc, n);
    std::vector<uint64_t> cbs, cbd;
    uint64_t cbytes_s = 0, cbytes_d = 0;
    ls.region_bases(nc, cbs, &cbytes_s);
    ld.region_bases(nc, cbd, &cbytes_d);
    const uint64_t off_d = align256(cbytes_s);
    if ((hybrid ? cbytes_s : off_d + cbytes_d) > slot) return fail(ADHA_ERR_INVALID_ARG, "scratch too small");

    HostPipe* hp = nullptr;
    if ((s = get_pipe(&hp)) != ADHA_OK) return s;
    cudaError_t e = cudaEventRecord(hp->start, user);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
    for (int i = 0; i < slots; ++i)
        if ((e = cudaStreamWaitEvent(hp->s[i], hp->start, 0)) != cudaSuccess) return cuda_fail(e, "cudaStreamWaitEvent");

    const uint8_t* hsrc = (const uint8_t*)src_host;
    uint8_t* hdst = (uint8_t*)dst_host;
    int64_t k = 0;
    std::vector<uint64_t> ms, md;
    for (int64_t lo = 0; lo < n; lo += nc, ++k) {
        const int64_t m = std::min<int64_t>(nc, n - lo);
        const int i = (int)(k % slots);
        cudaStream_t st = hp->s[i];
        uint8_t* dsrc = (uint8_t*)scratch + (uint64_t)i * slot;
        uint8_t* ddst = dsrc + off_d;
        uint64_t mbs = 0, mbd = 0;
        ls.region_bases(m, ms, &mbs);
        ld.region_bases(m, md, &mbd);
        for (int c = 0; c < ls.n_clusters(); ++c) {
            e = cudaMemcpyAsync(dsrc + ms[c], hsrc + ck.bs[c] + (uint64_t)lo * ls.stride[c], ls.region_bytes(c, m),
                                cudaMemcpyHostToDevice, st);
            if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync H2D");
        }
        Checked cm;
        cm.bs = ms;
        cm.bytes_s = mbs;
        if (hybrid) {
            // dst regions of this chunk inside the host buffer: base_c(N) + lo * stride_c
            cm.bd.resize(ld.n_clusters());
            for (int c = 0; c < ld.n_clusters(); ++c) cm.bd[c] = ck.bd[c] + (uint64_t)lo * ld.stride[c];
            if ((s = remap_checked(dsrc, ls, hdst, ld, m, cm, st)) != ADHA_OK) return s;
        } else {
            cm.bd = md;
            cm.bytes_d = mbd;
            if ((s = remap_checked(dsrc, ls, ddst, ld, m, cm, st)) != ADHA_OK) return s;
            for (int c = 0; c < ld.n_clusters(); ++c) {
                e = cudaMemcpyAsync(hdst + ck.bd[c] + (uint64_t)lo * ld.stride[c], ddst + md[c],
                                    ld.region_bytes(c, m), cudaMemcpyDeviceToHost, st);
                if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync D2H");
            }
        }
    }
    for (int i = 0; i < slots; ++i) {
        if ((e = cudaEventRecord(hp->done[i], hp->s[i])) != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
        if ((e = cudaStreamWaitEvent(user, hp->done[i], 0)) != cudaSuccess) return cuda_fail(e, "cudaStreamWaitEvent");
    }
    return ADHA_OK;
}

extern "C" adha_status adha_remap_plan_describe(const adha_layout* hs, const adha_layout* hd, char** json_out) {
    clear_error();
    if (!hs || !hd || !json_out) return fail(ADHA_ERR_INVALID_ARG, "null argument");
    if (hs->L.n_fields != hd->L.n_fields) return fail(ADHA_ERR_LAYOUT_MISMATCH, "layouts differ in field count");
    for (int f = 0; f < hs->L.n_fields; ++f)
        if (hs->L.width[f] != hd->L.width[f]) return fail(ADHA_ERR_LAYOUT_MISMATCH, "widths differ");
    auto plan = get_plan(hs->L, hd->L);
    std::string s = describe_plan(*plan, hs->L, hd->L);
    *json_out = (char*)std::malloc(s.size() + 1);
    if (!*json_out) return fail(ADHA_ERR_OOM, "out of host memory");
    std::memcpy(*json_out, s.c_str(), s.size() + 1);
    return ADHA_OK;
}
