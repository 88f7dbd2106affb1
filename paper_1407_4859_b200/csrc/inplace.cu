// inplace.cu -- the in-place remap ("in-place"; adha.h adha_remap_inplace):
// the remap of PAPER.md:56-57, 146 with src and dst in ONE buffer of max(bytes(Ls, N),
// bytes(Ld, N)) bytes, so an array that fills most of HBM can still change layout.
//
// Plan (inplace_plan.cpp): S-byte slots, T = S / u records per tile.  Launches, in order:
//   ip_tail_kernel (save)         the last N mod T records -> workspace, packed
//   ip_tile_kernel (step 1)       src tiles of changed clusters of several runs: record-major -> blocked
//   ip_cycle_save_kernel          the last slot of every cycle segment -> workspace
//   ip_cycle_shift_kernel         every slot moves one step along its cycle
//   ip_tile_kernel (step 3)       dst tiles of changed clusters of several runs: blocked -> record-major
//   ip_tail_kernel (restore)      the tail records -> their dst addresses
// Type-blind byte moves throughout (reading Q6): no floating-point instruction.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <set>
#include <string>

#include "inplace_plan.h"

namespace adha {
namespace ipdev {

// (programmatic dependent launch) every in-place kernel waits for the previous kernel's writes
// before its first global access, then lets the next launch be scheduled (its own accesses wait
// for this grid in turn)
__device__ __forceinline__ void ip_pdl_begin() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------------------- tail
__global__ void ip_tail_kernel(uint8_t* __restrict__ buf, const IpTailField* __restrict__ tf, uint32_t nf,
                               int64_t r0, int64_t ntail, uint8_t* __restrict__ tailbuf, uint32_t R, int restore) {
    ip_pdl_begin();
    const int64_t total = ntail * nf;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / nf;
        const IpTailField f = tf[idx % nf];
        const uint64_t i = (uint64_t)(r0 + r);
        uint8_t* t = tailbuf + (uint64_t)r * R + f.toff;
        if (!restore) {
            const uint8_t* s = buf + f.src + i * f.stride_s;
            for (uint32_t b = 0; b < f.width; ++b) t[b] = s[b];
        } else {
            uint8_t* d = buf + f.dst + i * f.stride_d;
            for (uint32_t b = 0; b < f.width; ++b) d[b] = t[b];
        }
    }
}

// ---------------------------------------------------------------------------- tile rewrite
// q = floor(n / d) for n * d < 2^32 with magic = ceil(2^32 / d) (0 encodes d == 1).
__device__ __forceinline__ uint32_t fdiv(uint32_t n, uint32_t magic) { return magic ? __umulhi(n, magic) : n; }

// One tile of cluster c (T records, RA atoms per record, T * stride bytes at base + t*T*stride)
// is rewritten in place between record-major form (atom (r, j) at r * RA + j) and blocked form
// (run b's T * a_b atoms contiguous from T * col_b, record r's atoms at r * a_b; a run is a field
// or several fields contiguous in both records, inplace_plan.h; the kernel calls runs "fields").
// to_blocks: record-major -> blocked (step 1); else blocked -> record-major (step 3).
// The tile is staged in shared memory with padding (one atom per record row, or per field
// block) so that the gather along the other major is (nearly) bank-conflict free, then written
// back with coalesced 16-byte stores.  Atom = 32-bit word when u % 4 == 0, else one byte.
// Loads are issued IP_LB vectors per thread at a time, and the first batch of the CTA's next
// tile is loaded into registers before the gather of the current one, so global loads overlap
// the shared-memory work.  Shared memory: [column table: tab_cap bytes][padded tile].
#ifndef IP_LB
#define IP_LB 2
#endif
#ifndef IP_SKEW
#define IP_SKEW 1
#endif
#ifndef IP_SKEW_ST
#define IP_SKEW_ST 0
#endif

template <typename Atom, bool GROUPED>
__device__ __forceinline__ void ip_scatter(Atom* sa, const uint4 x, uint32_t v, int to_blocks, uint32_t lgT,
                                           const IpPiece& pc, uint32_t padR, const IpCol* tab) {
    constexpr uint32_t APV = 16 / sizeof(Atom);
    const uint32_t i0 = v * APV;
    const uint32_t RA = pc.RA;
    if (to_blocks) {   // record-major input: pad per row (row r starts at r * (RA + padR)); rows run on
                       // across the tiles of a piece
        const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
        if (sizeof(Atom) == 4) {
#if IP_SKEW_ST
            // lanes 8g..8g+7 store their 4 words starting at word g (rotated in registers first), so
            // the 32 lanes of each store hit different banks
            const uint32_t k = (threadIdx.x >> 3) & 3;
            const bool r1 = k & 1, r2 = k & 2;
            const uint32_t t0 = r1 ? w4[1] : w4[0], t1 = r1 ? w4[2] : w4[1], t2 = r1 ? w4[3] : w4[2],
                           t3 = r1 ? w4[0] : w4[3];
            const uint32_t v[4] = {r2 ? t2 : t0, r2 ? t3 : t1, r2 ? t0 : t2, r2 ? t1 : t3};   // v[j] = w4[(j+k)&3]
#pragma unroll
            for (uint32_t j = 0; j < 4; ++j) {
                const uint32_t i = i0 + ((j + k) & 3);
                sa[i + fdiv(i, pc.magic_RA) * padR] = (Atom)v[j];
            }
#else
#pragma unroll
            for (uint32_t j = 0; j < 4; ++j) sa[i0 + j + fdiv(i0 + j, pc.magic_RA) * padR] = (Atom)w4[j];
#endif
        } else {
            const uint32_t r0 = fdiv(i0, pc.magic_RA);
            uint32_t o = i0 + r0 * padR, rr = i0 - r0 * RA;
#pragma unroll
            for (uint32_t j = 0; j < 16; ++j) {
                sa[o] = (Atom)(w4[j >> 2] >> (8 * (j & 3)));
                ++o;
                if (++rr == RA) { rr = 0; o += padR; }
            }
        }
    } else {           // field-blocked input: tile q of the piece at q * TS, padding before each field
                       // block, a multiple of 16 bytes (inplace_plan.cpp choose_padf), so the vector
                       // stays 16-byte aligned: one conflict-free 16-byte store
        const uint32_t q = GROUPED ? fdiv(i0, pc.magic_TRA) : 0;
        const uint32_t i = i0 - q * (RA << lgT);
        const uint32_t o = q * pc.TS + i + reinterpret_cast<const uint32_t*>(tab)[RA + (i >> lgT)];
        *reinterpret_cast<uint4*>(sa + o) = x;
    }
}

template <typename Atom, bool GROUPED>
__device__ __forceinline__ uint4 ip_gather(const Atom* sa, uint32_t v, int to_blocks, uint32_t lgT, const IpPiece& pc,
                                           uint32_t P, const IpCol* tab) {
    constexpr uint32_t APV = 16 / sizeof(Atom);
    const uint32_t RA = pc.RA;
    uint32_t w4[4] = {0, 0, 0, 0};
    const uint32_t o0 = v * APV;
    if (to_blocks) {   // output field-blocked: the vector lies in one column block of tile q
        const uint32_t q = GROUPED ? fdiv(o0, pc.magic_TRA) : 0;
        const uint32_t ot = o0 - q * (RA << lgT);
        const IpCol e = tab[ot >> lgT];
        const uint32_t col = e.col_fp & 0xFFFFu;
        const uint32_t local0 = ot - (col << lgT);
        const uint32_t rq = q << lgT;                  // first record row of tile q
        if (sizeof(Atom) == 4 && e.a == 1) {          // 4 consecutive records of one column
            const uint32_t a0 = (rq + local0) * P + col;
#if IP_SKEW
            // lanes 8g..8g+7 read their 4 rows starting at row g: with an odd pitch the 32 lanes of
            // each read then hit 32 different banks; the values are rotated back in registers
            const uint32_t k = (threadIdx.x >> 3) & 3;
            uint32_t v[4];
#pragma unroll
            for (uint32_t j = 0; j < 4; ++j) v[j] = (uint32_t)sa[a0 + ((j + k) & 3) * P];
            const bool r1 = k & 1, r2 = k & 2;
            const uint32_t t0 = r1 ? v[3] : v[0], t1 = r1 ? v[0] : v[1], t2 = r1 ? v[1] : v[2], t3 = r1 ? v[2] : v[3];
            w4[0] = r2 ? t2 : t0;
            w4[1] = r2 ? t3 : t1;
            w4[2] = r2 ? t0 : t2;
            w4[3] = r2 ? t1 : t3;
#else
#pragma unroll
            for (uint32_t j = 0; j < 4; ++j) w4[j] = (uint32_t)sa[a0 + j * P];
#endif
        } else if (sizeof(Atom) == 4 && e.a == 2) {   // 2 records x 2 atoms
            const uint32_t a0 = (rq + (local0 >> 1)) * P + col;
            w4[0] = (uint32_t)sa[a0];
            w4[1] = (uint32_t)sa[a0 + 1];
            w4[2] = (uint32_t)sa[a0 + P];
            w4[3] = (uint32_t)sa[a0 + P + 1];
        } else {
#pragma unroll
            for (uint32_t j = 0; j < APV; ++j) {
                const uint32_t local = local0 + j;
                const uint32_t r = fdiv(local, e.magic_a);
                const Atom val = sa[(rq + r) * P + col + (local - r * e.a)];
                if (sizeof(Atom) == 4) w4[j] = (uint32_t)val;
                else w4[j >> 2] |= (uint32_t)val << (8 * (j & 3));
            }
        }
    } else {           // output record-major: atom (r', jc), r' = q*T + r <- q*TS + bo(jc) + r*a(jc)
        const uint32_t* bo_a = reinterpret_cast<const uint32_t*>(tab);   // packed bo | a << 17 (see ip_tile_kernel)
        uint32_t r = fdiv(o0, pc.magic_RA);
        uint32_t jc = o0 - r * RA;
        const uint32_t T1 = (1u << lgT) - 1;
#pragma unroll
        for (uint32_t j = 0; j < APV; ++j) {
            const uint32_t e = bo_a[jc];
            const Atom val = GROUPED ? sa[(r >> lgT) * pc.TS + (e & 0x1FFFFu) + (r & T1) * (e >> 17)]
                                     : sa[(e & 0x1FFFFu) + r * (e >> 17)];
            if (sizeof(Atom) == 4) w4[j] = (uint32_t)val;
            else w4[j >> 2] |= (uint32_t)val << (8 * (j & 3));
            if (++jc == RA) { jc = 0; ++r; }
        }
    }
    return make_uint4(w4[0], w4[1], w4[2], w4[3]);
}

// MINB: 8 resident CTAs (32 registers) for small pieces, where occupancy hides the load latency;
// 1 for large pieces (fewer CTAs fit anyway; the register budget then goes to the address math).
template <typename Atom, int to_blocks, bool GROUPED, int MINB>
__global__ void __launch_bounds__(256, MINB) ip_tile_kernel(uint8_t* __restrict__ buf, const IpPiece* __restrict__ cl,
                                                      const IpCol* __restrict__ cols, uint32_t ncl, uint64_t m,
                                                      uint32_t T, uint32_t tab_cap) {
    ip_pdl_begin();
    extern __shared__ __align__(16) uint8_t sm[];
    IpCol* tab = reinterpret_cast<IpCol*>(sm);
    Atom* sa = reinterpret_cast<Atom*>(sm + tab_cap);
    const uint32_t lgT = 31 - __clz(T);
    const uint32_t tid = threadIdx.x, nt = blockDim.x;
    uint4 x[IP_LB];
    uint32_t cur_c = 0xFFFFFFFFu;

    auto load_batch0 = [&](const uint8_t* gp, uint32_t nvec) {
        const uint4* g4 = reinterpret_cast<const uint4*>(gp);
#pragma unroll
        for (uint32_t k = 0; k < IP_LB; ++k)
            if (tid + k * nt < nvec) x[k] = g4[tid + k * nt];
    };
    auto load_table = [&](uint32_t c, const IpPiece& d) {   // cluster descriptor's column table -> smem
        if (c == cur_c) return;
        if (to_blocks) {
            for (uint32_t j = tid; j < d.RA; j += nt) tab[j] = cols[d.col_off + j];
        } else {        // field-blocked -> record-major needs only bo and a: one packed word per column
            uint32_t* bo_a = reinterpret_cast<uint32_t*>(tab);   // [RA] bo | a << 17, then [RA] padding
            for (uint32_t j = tid; j < d.RA; j += nt) {
                const IpCol e = cols[d.col_off + j];
                bo_a[j] = e.bo | (e.a << 17);
                bo_a[d.RA + j] = e.col_fp >> 16;
            }
        }
        cur_c = c;
        __syncthreads();
    };
    // one piece: batch 0 is in registers; scatter into the padded tile, prefetch the next piece's
    // batch 0, gather in output order, write back with 16-byte stores
    auto body = [&](const IpPiece& pc, uint8_t* g, uint32_t nvec, auto&& prefetch_next) {
        const uint32_t RA = pc.RA;
        const uint32_t padR = sizeof(Atom) == 4 ? ((RA & 1) ? 0 : 1) : 4;   // row padding (odd word pitch)
        const uint32_t P = RA + padR;
        const uint4* g4 = reinterpret_cast<const uint4*>(g);
        for (uint32_t b0 = 0; b0 < nvec; b0 += IP_LB * nt) {
            if (b0) {
#pragma unroll
                for (uint32_t k = 0; k < IP_LB; ++k)
                    if (b0 + tid + k * nt < nvec) x[k] = g4[b0 + tid + k * nt];
            }
#pragma unroll
            for (uint32_t k = 0; k < IP_LB; ++k) {
                const uint32_t v = b0 + tid + k * nt;
                if (v < nvec) ip_scatter<Atom, GROUPED>(sa, x[k], v, to_blocks, lgT, pc, padR, tab);
            }
        }
        __syncthreads();
        prefetch_next();   // no other CTA writes the next piece
        uint4* o4 = reinterpret_cast<uint4*>(g);
        for (uint32_t v = tid; v < nvec; v += nt) o4[v] = ip_gather<Atom, GROUPED>(sa, v, to_blocks, lgT, pc, P, tab);
        __syncthreads();
    };

    if constexpr (!GROUPED) {
        // one tile per piece: tile p = (c, t) with p = c * m + t, stepping by gridDim.x
        uint32_t c = (uint32_t)(blockIdx.x / m);
        uint64_t t = blockIdx.x - (uint64_t)c * m;
        const uint64_t step_c = gridDim.x / m, step_t = gridDim.x - step_c * m;
        auto advance = [&](uint32_t& cc, uint64_t& tt) {
            cc += (uint32_t)step_c;
            tt += step_t;
            if (tt >= m) { tt -= m; ++cc; }
        };
        if (c < ncl) {
            const IpPiece d = cl[c];
            load_batch0(buf + d.base + t * (uint64_t)T * d.stride, T * d.stride >> 4);
        }
        for (; c < ncl; advance(c, t)) {
            const IpPiece pc = cl[c];
            load_table(c, pc);
            body(pc, buf + pc.base + t * (uint64_t)T * pc.stride, T * pc.stride >> 4, [&] {
                uint32_t cn = c;
                uint64_t tn = t;
                advance(cn, tn);
                if (cn < ncl) {
                    const IpPiece pn = cl[cn];
                    load_batch0(buf + pn.base + tn * (uint64_t)T * pn.stride, T * pn.stride >> 4);
                }
            });
        }
    } else {
        // pieces of g_c tiles: piece (c, t) covers tiles [t*g_c, min((t+1)*g_c, m)) of cluster c;
        // a CTA steps by gridDim.x pieces (piece counts differ between clusters)
        uint32_t c = 0;
        uint64_t t = blockIdx.x;
        auto normalize = [&](uint32_t& cc, uint64_t& tt) {
            while (cc < ncl) {
                const uint64_t np = cl[cc].pieces;
                if (tt < np) break;
                tt -= np;
                ++cc;
            }
        };
        auto piece_vecs = [&](const IpPiece& d, uint64_t tt) {
            const uint64_t t0 = tt * d.g;
            return (uint32_t)(m - t0 < d.g ? m - t0 : d.g) * T * d.stride >> 4;
        };
        normalize(c, t);
        if (c < ncl) {
            const IpPiece d = cl[c];
            load_batch0(buf + d.base + t * d.g * (uint64_t)T * d.stride, piece_vecs(d, t));
        }
        for (; c < ncl; t += gridDim.x, normalize(c, t)) {
            const IpPiece pc = cl[c];
            load_table(c, pc);
            body(pc, buf + pc.base + t * pc.g * (uint64_t)T * pc.stride, piece_vecs(pc, t), [&] {
                uint32_t cn = c;
                uint64_t tn = t + gridDim.x;
                normalize(cn, tn);
                if (cn < ncl) {
                    const IpPiece pn = cl[cn];
                    load_batch0(buf + pn.base + tn * pn.g * (uint64_t)T * pn.stride, piece_vecs(pn, tn));
                }
            });
        }
    }
}

// ---------------------------------------------------------------------------- cycles
// A group of G lanes walks one segment.  Lane l owns 16-byte vectors l, l + G, ... of every
// slot, so each location is loaded and stored by the same thread, in program order: no
// cross-lane ordering is needed.  Content at x_j moves to x_{j+1}; the segment's last slot was
// saved by ip_cycle_save_kernel, its first slot receives the predecessor segment's saved slot.
template <uint32_t S>
__global__ void __launch_bounds__(256) ip_cycle_save_kernel(uint8_t* __restrict__ buf, const uint32_t* __restrict__ seq,
                                                            const IpSeg* __restrict__ segs, uint32_t nseg,
                                                            uint8_t* __restrict__ save) {
    ip_pdl_begin();
    constexpr uint32_t V = S / 16, G = V < 32 ? V : 32, VPL = V / G;
    const uint32_t lane = threadIdx.x % G;
    const uint64_t g0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / G;
    const uint64_t ng = (uint64_t)gridDim.x * blockDim.x / G;
    const uint4* b4 = reinterpret_cast<const uint4*>(buf);
    uint4* s4 = reinterpret_cast<uint4*>(save);
    for (uint64_t s = g0; s < nseg; s += ng) {
        const IpSeg sg = segs[s];
        const uint64_t x = seq[sg.start + sg.len - 1];
#pragma unroll
        for (uint32_t i = 0; i < VPL; ++i) s4[s * V + lane + i * G] = b4[x * V + lane + i * G];
    }
}

template <uint32_t S>
__global__ void __launch_bounds__(256) ip_cycle_shift_kernel(uint8_t* buf, const uint32_t* __restrict__ seq,
                                                             const IpSeg* __restrict__ segs, uint32_t nseg,
                                                             const uint8_t* __restrict__ save) {
    ip_pdl_begin();
    constexpr uint32_t V = S / 16, G = V < 32 ? V : 32, VPL = V / G;
#ifndef IP_SHIFT_VEC
#define IP_SHIFT_VEC 8
#endif
    constexpr uint32_t B = VPL >= IP_SHIFT_VEC ? 1 : IP_SHIFT_VEC / VPL;   // slots per batch (IP_SHIFT_VEC vectors in flight per lane)
    const uint32_t lane = threadIdx.x % G;
    const uint64_t g0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / G;
    const uint64_t ng = (uint64_t)gridDim.x * blockDim.x / G;
    uint4* b4 = reinterpret_cast<uint4*>(buf);
    const uint4* s4 = reinterpret_cast<const uint4*>(save);
    for (uint64_t s = g0; s < nseg; s += ng) {
        const IpSeg sg = segs[s];
        const uint32_t* x = seq + sg.start;
        int32_t j = (int32_t)sg.len - 1;                // next destination index
        while (j >= 1) {
            const int32_t nb = j < (int32_t)B ? j : (int32_t)B;
            uint4 r[B * VPL];
#pragma unroll
            for (uint32_t b = 0; b < B; ++b)
                if ((int32_t)b < nb) {
                    const uint64_t src = x[j - 1 - (int32_t)b];
#pragma unroll
                    for (uint32_t i = 0; i < VPL; ++i) r[b * VPL + i] = b4[src * V + lane + i * G];
                }
#pragma unroll
            for (uint32_t b = 0; b < B; ++b)
                if ((int32_t)b < nb) {
                    const uint64_t dst = x[j - (int32_t)b];
#pragma unroll
                    for (uint32_t i = 0; i < VPL; ++i) b4[dst * V + lane + i * G] = r[b * VPL + i];
                }
            j -= nb;
        }
        const uint64_t x0 = x[0];
#pragma unroll
        for (uint32_t i = 0; i < VPL; ++i) b4[x0 * V + lane + i * G] = s4[(uint64_t)sg.pred * V + lane + i * G];
    }
}

}  // namespace ipdev

namespace {

bool ip_pdl() {
    const char* e = std::getenv("ADHA_PDL");
    return !(e && *e == '0');
}
// cudaLaunchKernelExC with programmatic dependent launch allowed (ADHA_PDL=0: plain launch)
cudaError_t ip_launch(const void* fn, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = ip_pdl() ? 1 : 0;
    return cudaLaunchKernelExC(&cfg, fn, args);
}

adha_status cuda_err(cudaError_t e, const char* what) {
    return fail(ADHA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// calls f(save kernel, shift kernel) instantiated for slot size S
template <typename F>
adha_status with_cycle_kernels(uint32_t S, F&& f) {
    switch (S) {
        case 256: f(ipdev::ip_cycle_save_kernel<256>, ipdev::ip_cycle_shift_kernel<256>); break;
        case 512: f(ipdev::ip_cycle_save_kernel<512>, ipdev::ip_cycle_shift_kernel<512>); break;
        case 1024: f(ipdev::ip_cycle_save_kernel<1024>, ipdev::ip_cycle_shift_kernel<1024>); break;
        case 2048: f(ipdev::ip_cycle_save_kernel<2048>, ipdev::ip_cycle_shift_kernel<2048>); break;
        case 4096: f(ipdev::ip_cycle_save_kernel<4096>, ipdev::ip_cycle_shift_kernel<4096>); break;
        default: return fail(ADHA_ERR_UNSUPPORTED, "slot size");
    }
    return ADHA_OK;
}

std::mutex g_attr_mu;
std::set<std::pair<int, const void*>> g_attr_done;

adha_status smem_optin(int dev, const void* fn) {
    std::lock_guard<std::mutex> g(g_attr_mu);
    if (g_attr_done.count({dev, fn})) return ADHA_OK;
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, fn);
    if (e != cudaSuccess) return cuda_err(e, "cudaFuncGetAttributes");
    // opt-in limit per block (227 KB on sm_100) minus the kernel's static shared memory
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448 - (int)fa.sharedSizeBytes);
    if (e != cudaSuccess) return cuda_err(e, "cudaFuncSetAttribute");
    g_attr_done.insert({dev, fn});
    return ADHA_OK;
}

adha_status launch_tiles(const InplacePlan& P, uint8_t* buf, const uint8_t* ws, bool post, int dev, int sms,
                         cudaStream_t st) {
    const auto& v = post ? P.post : P.pre;
    if (v.empty() || P.m == 0) return ADHA_OK;
    const IpPiece* tab = reinterpret_cast<const IpPiece*>(ws + P.ws_pieces) + (post ? P.pre.size() : 0);
    const IpCol* cols = reinterpret_cast<const IpCol*>(ws + P.ws_cols);
    const uint32_t tab_cap = (P.max_tab + 15) & ~15u;
    const uint32_t smem = tab_cap + P.max_tile;
    bool grouped = false;
    for (const IpPiece& pc : v) grouped = grouped || pc.g > 1;
    const bool small = 8ull * (smem + 1024) <= 232448;   // 8 CTAs of this size fit in one SM
    using K = void (*)(uint8_t*, const IpPiece*, const IpCol*, uint32_t, uint64_t, uint32_t, uint32_t);
    // [word atoms?][post?][grouped?][small?]
    static const K table[2][2][2][2] = {
        {{{ipdev::ip_tile_kernel<uint8_t, 1, false, 1>, ipdev::ip_tile_kernel<uint8_t, 1, false, 8>},
          {ipdev::ip_tile_kernel<uint8_t, 1, true, 1>, ipdev::ip_tile_kernel<uint8_t, 1, true, 8>}},
         {{ipdev::ip_tile_kernel<uint8_t, 0, false, 1>, ipdev::ip_tile_kernel<uint8_t, 0, false, 8>},
          {ipdev::ip_tile_kernel<uint8_t, 0, true, 1>, ipdev::ip_tile_kernel<uint8_t, 0, true, 8>}}},
        {{{ipdev::ip_tile_kernel<uint32_t, 1, false, 1>, ipdev::ip_tile_kernel<uint32_t, 1, false, 8>},
          {ipdev::ip_tile_kernel<uint32_t, 1, true, 1>, ipdev::ip_tile_kernel<uint32_t, 1, true, 8>}},
         {{ipdev::ip_tile_kernel<uint32_t, 0, false, 1>, ipdev::ip_tile_kernel<uint32_t, 0, false, 8>},
          {ipdev::ip_tile_kernel<uint32_t, 0, true, 1>, ipdev::ip_tile_kernel<uint32_t, 0, true, 8>}}}};
    const void* fn = (const void*)table[P.u % 4 == 0][post][grouped][small];
    adha_status s = smem_optin(dev, fn);
    if (s != ADHA_OK) return s;
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, smem);
    if (e != cudaSuccess) return cuda_err(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
    uint64_t pieces = 0;
    for (const IpPiece& pc : v) pieces += pc.pieces;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(pieces, (uint64_t)sms * std::max(occ, 1)));
    uint32_t ncl = (uint32_t)v.size(), T = P.T;
    uint64_t m = (uint64_t)P.m;
    void* args[] = {&buf, (void*)&tab, (void*)&cols, &ncl, &m, &T, (void*)&tab_cap};
    e = ip_launch(fn, dim3(grid), dim3(256), args, smem, st);
    return e == cudaSuccess ? ADHA_OK : cuda_err(e, "ip_tile_kernel launch");
}

adha_status launch_tail(const InplacePlan& P, uint8_t* buf, uint8_t* ws, bool restore, cudaStream_t st) {
    if (P.tail == 0) return ADHA_OK;
    const uint32_t nf = (uint32_t)P.tail_fields.size();
    const int64_t work = P.tail * nf;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 1024));
    const IpTailField* tf = reinterpret_cast<const IpTailField*>(ws + P.ws_tailf);
    int64_t r0 = P.m * (int64_t)P.T, ntail = P.tail;
    uint8_t* tailbuf = ws + P.ws_tail;
    uint32_t nfv = nf, R = (uint32_t)P.ls.record_bytes;
    int rs = restore ? 1 : 0;
    void* args[] = {&buf, (void*)&tf, &nfv, &r0, &ntail, &tailbuf, &R, &rs};
    cudaError_t e = ip_launch((const void*)&ipdev::ip_tail_kernel, dim3(grid), dim3(256), args, 0, st);
    return e == cudaSuccess ? ADHA_OK : cuda_err(e, "ip_tail_kernel launch");
}

}  // namespace
}  // namespace adha

using namespace adha;

extern "C" adha_status adha_inplace_plan_upload(adha_inplace_plan* h, void* workspace, uint64_t workspace_bytes,
                                                void* stream) {
    clear_error();
    if (!h) return fail(ADHA_ERR_INVALID_ARG, "null plan");
    InplacePlan& P = h->P;
    if (!workspace) return fail(ADHA_ERR_INVALID_ARG, "null workspace");
    if ((uintptr_t)workspace & 255) return fail(ADHA_ERR_ALIGNMENT, "workspace must be 256-byte aligned");
    if (workspace_bytes < P.ws_bytes)
        return fail(ADHA_ERR_INVALID_ARG, "workspace holds " + std::to_string(workspace_bytes) + " bytes, plan needs " +
                                              std::to_string(P.ws_bytes));
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_err(e, "cudaGetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t* ws = (uint8_t*)workspace;
    std::vector<IpPiece> pieces(P.pre);
    pieces.insert(pieces.end(), P.post.begin(), P.post.end());
    struct Part { uint64_t off; const void* src; size_t bytes; };
    const Part parts[] = {{P.ws_pieces, pieces.data(), pieces.size() * sizeof(IpPiece)},
                          {P.ws_cols, P.cols.data(), P.cols.size() * sizeof(IpCol)},
                          {P.ws_tailf, P.tail_fields.data(), P.tail_fields.size() * sizeof(IpTailField)},
                          {P.ws_seq, P.seq.data(), P.seq.size() * sizeof(uint32_t)},
                          {P.ws_segs, P.segs.data(), P.segs.size() * sizeof(IpSeg)}};
    for (const Part& q : parts) {
        if (!q.bytes) continue;
        e = cudaMemcpyAsync(ws + q.off, q.src, q.bytes, cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) return cuda_err(e, "cudaMemcpyAsync (plan upload)");
    }
    // `pieces` is a temporary: make sure its copy has left host memory before returning
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_err(e, "cudaStreamSynchronize (plan upload)");
    P.uploaded = workspace;
    P.uploaded_device = dev;
    return ADHA_OK;
}

extern "C" adha_status adha_remap_inplace(void* buf, uint64_t buf_bytes, const adha_inplace_plan* h,
                                          void* workspace, void* stream) {
    clear_error();
    if (!h) return fail(ADHA_ERR_INVALID_ARG, "null plan");
    const InplacePlan& P = h->P;
    if (P.n == 0) return ADHA_OK;
    if (!buf || !workspace) return fail(ADHA_ERR_INVALID_ARG, "null buffer or workspace");
    if ((uintptr_t)buf & 255) return fail(ADHA_ERR_ALIGNMENT, "buffer must be 256-byte aligned");
    const uint64_t need = std::max(P.bytes_s, P.bytes_d);
    if (buf_bytes < need)
        return fail(ADHA_ERR_INVALID_ARG, "buffer holds " + std::to_string(buf_bytes) + " bytes, the remap needs " +
                                              std::to_string(need) + " (max of both layouts)");
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_err(e, "cudaGetDevice");
    if (P.uploaded != workspace || P.uploaded_device != dev)
        return fail(ADHA_ERR_INVALID_ARG, "plan not uploaded to this workspace on this device (adha_inplace_plan_upload)");
    const uintptr_t b0 = (uintptr_t)buf, b1 = b0 + need, w0 = (uintptr_t)workspace, w1 = w0 + P.ws_bytes;
    if (b0 < w1 && w0 < b1) return fail(ADHA_ERR_OVERLAP, "workspace overlaps the buffer");
    int sms = 148;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return cuda_err(e, "cudaDeviceGetAttribute");
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t* b = (uint8_t*)buf;
    uint8_t* ws = (uint8_t*)workspace;
    if (P.staged) {   // small buffer: out-of-place remap into the workspace, then copy back
        // adha_layout is {Layout L}: the plan's own layout copies serve as handles
        const adha_layout* hs = reinterpret_cast<const adha_layout*>(&P.ls);
        const adha_layout* hd = reinterpret_cast<const adha_layout*>(&P.ld);
        adha_status s = adha_remap(b, hs, ws + P.ws_stage, hd, P.n, stream);
        if (s != ADHA_OK) return s;
        e = cudaMemcpyAsync(b, ws + P.ws_stage, P.bytes_d, cudaMemcpyDeviceToDevice, st);
        return e == cudaSuccess ? ADHA_OK : cuda_err(e, "cudaMemcpyAsync (staged in-place remap)");
    }
    adha_status s = launch_tail(P, b, ws, false, st);
    if (s != ADHA_OK) return s;
    s = launch_tiles(P, b, ws, false, dev, sms, st);
    if (s != ADHA_OK) return s;
    if (!P.segs.empty()) {
        const uint32_t nseg = (uint32_t)P.segs.size();
        const uint32_t G = std::min<uint32_t>(32, P.S / 16);
        const uint64_t groups_per_block = 256 / G;
        const unsigned grid =
            (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nseg + groups_per_block - 1) / groups_per_block,
                                                               (uint64_t)sms * 8));
        const uint32_t* seq = reinterpret_cast<const uint32_t*>(ws + P.ws_seq);
        const IpSeg* segs = reinterpret_cast<const IpSeg*>(ws + P.ws_segs);
        uint8_t* save = ws + P.ws_save;
        s = with_cycle_kernels(P.S, [&](auto save_k, auto shift_k) {
            uint32_t nsg = nseg;
            void* args[] = {&b, (void*)&seq, (void*)&segs, &nsg, &save};
            e = ip_launch((const void*)save_k, dim3(grid), dim3(256), args, 0, st);
            if (e == cudaSuccess) e = ip_launch((const void*)shift_k, dim3(grid), dim3(256), args, 0, st);
        });
        if (s != ADHA_OK) return s;
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_err(e, "ip_cycle kernels launch");
    }
    s = launch_tiles(P, b, ws, true, dev, sms, st);
    if (s != ADHA_OK) return s;
    return launch_tail(P, b, ws, true, st);
}
