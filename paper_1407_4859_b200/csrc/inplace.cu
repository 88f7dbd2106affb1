// inplace.cu -- the in-place remap ("in-place"; adha.h adha_remap_inplace):
// the remap of PAPER.md:56-57, 146 with src and dst in ONE buffer of max(bytes(Ls, N),
// bytes(Ld, N)) bytes, so an array that fills most of HBM can still change layout.
//
// Plan (inplace_plan.cpp): S-byte slots, T = S / u records per tile.  Launches, in order:
//   ip_tail_kernel (save)         the last N mod T records -> workspace, packed
//   ip_transpose_kernel (step 1)  src tiles of changed clusters: record-major -> unit-columns
//   ip_cycle_save_kernel          the last slot of every cycle segment -> workspace
//   ip_cycle_shift_kernel         every slot moves one step along its cycle
//   ip_transpose_kernel (step 3)  dst tiles of changed clusters: unit-columns -> record-major
//   ip_tail_kernel (restore)      the tail records -> their dst addresses
// Type-blind byte moves throughout (reading Q6): no floating-point instruction.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <set>
#include <string>

#include "inplace_plan.h"

namespace adha {
namespace ipdev {

// ---------------------------------------------------------------------------- tail
__global__ void ip_tail_kernel(uint8_t* __restrict__ buf, const IpTailField* __restrict__ tf, uint32_t nf,
                               int64_t r0, int64_t ntail, uint8_t* __restrict__ tailbuf, uint32_t R, int restore) {
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

// ---------------------------------------------------------------------------- tile transpose
// A tile of cluster c: T records x K byte-units of u bytes, T * K * u bytes at
// base + t * T * stride.  to_cols: record-major (r, k) -> unit-column-major (k, r); else back.
// Staged in shared memory with one padding word per line so that the gather is (nearly)
// bank-conflict free; written back with coalesced 32-bit stores.  Atom = the element moved:
// 32-bit words when u % 4 == 0, bytes otherwise.
template <typename Atom>
__global__ void __launch_bounds__(256) ip_transpose_kernel(uint8_t* __restrict__ buf, const IpPiece* __restrict__ cl,
                                                           uint32_t ncl, uint64_t m, uint32_t T, uint32_t u,
                                                           int to_cols) {
    extern __shared__ __align__(16) uint8_t sm[];
    Atom* sa = reinterpret_cast<Atom*>(sm);
    constexpr uint32_t PER_WORD = 4 / sizeof(Atom);
    const uint32_t A = u / sizeof(Atom);                 // atoms per unit
    const uint32_t lgT = 31 - __clz(T);
    const uint64_t total = (uint64_t)ncl * m;
    for (uint64_t p = blockIdx.x; p < total; p += gridDim.x) {
        const uint32_t c = (uint32_t)(p / m);
        const uint64_t t = p - (uint64_t)c * m;
        const IpPiece pc = cl[c];
        const uint32_t K = pc.K;
        const uint32_t RA = K * A, CA = T * A;           // atoms per record row / per unit column
        const uint32_t lineA = to_cols ? RA : CA;
        const uint32_t pitch = lineA + (sizeof(Atom) == 4 ? ((lineA & 1) ? 0 : 1) : 4);
        uint8_t* g = buf + pc.base + t * (uint64_t)T * pc.stride;
        const uint32_t bytes = T * pc.stride;
        // load: 16-byte vectors, scattered into padded lines
        const uint4* g4 = reinterpret_cast<const uint4*>(g);
        for (uint32_t v = threadIdx.x; v < bytes / 16; v += blockDim.x) {
            const uint4 x = g4[v];
            const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
            const uint32_t a0 = v * (16 / sizeof(Atom));
#pragma unroll
            for (uint32_t j = 0; j < 16 / sizeof(Atom); ++j) {
                const uint32_t a = a0 + j;
                const uint32_t line = a / lineA, col = a - line * lineA;
                Atom val;
                if (sizeof(Atom) == 4) val = (Atom)w4[j];
                else val = (Atom)(w4[j / 4] >> (8 * (j % 4)));
                sa[line * pitch + col] = val;
            }
        }
        __syncthreads();
        // store: output word w = atoms 4w/size .. ; output order is the other major
        uint32_t* g32 = reinterpret_cast<uint32_t*>(g);
        for (uint32_t w = threadIdx.x; w < bytes / 4; w += blockDim.x) {
            uint32_t out = 0;
#pragma unroll
            for (uint32_t j = 0; j < PER_WORD; ++j) {
                const uint32_t o = w * PER_WORD + j;
                const uint32_t a = o % A, ku = o / A;    // ku: unit index in output order
                uint32_t line, col;
                if (to_cols) {   // output (k, r): ku = k * T + r; input row r, column k*A + a
                    const uint32_t k = ku >> lgT, r = ku & (T - 1);
                    line = r;
                    col = k * A + a;
                } else {         // output (r, k): ku = r * K + k; input column k, row r*A + a
                    const uint32_t r = ku / K, k = ku - r * K;
                    line = k;
                    col = r * A + a;
                }
                const Atom val = sa[line * pitch + col];
                if (sizeof(Atom) == 4) out = (uint32_t)val;
                else out |= (uint32_t)val << (8 * j);
            }
            g32[w] = out;
        }
        __syncthreads();
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
    constexpr uint32_t V = S / 16, G = V < 32 ? V : 32, VPL = V / G;
    constexpr uint32_t B = VPL >= 8 ? 1 : 8 / VPL;     // slots per batch (8 vectors in flight per lane)
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

adha_status cuda_err(cudaError_t e, const char* what) {
    return fail(ADHA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
adha_status launch_cycles(uint32_t S, int blocks, cudaStream_t st, F&& f) {
    switch (S) {
        case 256: f(ipdev::ip_cycle_save_kernel<256>, ipdev::ip_cycle_shift_kernel<256>); break;
        case 512: f(ipdev::ip_cycle_save_kernel<512>, ipdev::ip_cycle_shift_kernel<512>); break;
        case 1024: f(ipdev::ip_cycle_save_kernel<1024>, ipdev::ip_cycle_shift_kernel<1024>); break;
        case 2048: f(ipdev::ip_cycle_save_kernel<2048>, ipdev::ip_cycle_shift_kernel<2048>); break;
        case 4096: f(ipdev::ip_cycle_save_kernel<4096>, ipdev::ip_cycle_shift_kernel<4096>); break;
        default: return fail(ADHA_ERR_UNSUPPORTED, "slot size");
    }
    (void)blocks;
    (void)st;
    return ADHA_OK;
}

std::mutex g_attr_mu;
std::set<std::pair<int, const void*>> g_attr_done;

adha_status smem_optin(int dev, const void* fn) {
    std::lock_guard<std::mutex> g(g_attr_mu);
    if (g_attr_done.count({dev, fn})) return ADHA_OK;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e != cudaSuccess) return cuda_err(e, "cudaFuncSetAttribute");
    g_attr_done.insert({dev, fn});
    return ADHA_OK;
}

adha_status launch_transpose(const InplacePlan& P, uint8_t* buf, const uint8_t* ws, bool post, int dev, int sms,
                             cudaStream_t st) {
    const auto& v = post ? P.post : P.pre;
    if (v.empty() || P.m == 0) return ADHA_OK;
    const IpPiece* tab = reinterpret_cast<const IpPiece*>(ws + P.ws_pieces) + (post ? P.pre.size() : 0);
    const uint32_t smem = (P.max_piece + 15) & ~15u;
    const void* fn = P.u % 4 == 0 ? (const void*)ipdev::ip_transpose_kernel<uint32_t>
                                  : (const void*)ipdev::ip_transpose_kernel<uint8_t>;
    adha_status s = smem_optin(dev, fn);
    if (s != ADHA_OK) return s;
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, smem);
    if (e != cudaSuccess) return cuda_err(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
    const uint64_t pieces = (uint64_t)v.size() * (uint64_t)P.m;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(pieces, (uint64_t)sms * std::max(occ, 1)));
    if (P.u % 4 == 0)
        ipdev::ip_transpose_kernel<uint32_t><<<grid, 256, smem, st>>>(buf, tab, (uint32_t)v.size(), (uint64_t)P.m,
                                                                     P.T, P.u, post ? 0 : 1);
    else
        ipdev::ip_transpose_kernel<uint8_t><<<grid, 256, smem, st>>>(buf, tab, (uint32_t)v.size(), (uint64_t)P.m,
                                                                    P.T, P.u, post ? 0 : 1);
    e = cudaGetLastError();
    return e == cudaSuccess ? ADHA_OK : cuda_err(e, "ip_transpose_kernel launch");
}

adha_status launch_tail(const InplacePlan& P, uint8_t* buf, uint8_t* ws, bool restore, cudaStream_t st) {
    if (P.tail == 0) return ADHA_OK;
    const uint32_t nf = (uint32_t)P.tail_fields.size();
    const int64_t work = P.tail * nf;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 1024));
    ipdev::ip_tail_kernel<<<grid, 256, 0, st>>>(buf, reinterpret_cast<const IpTailField*>(ws + P.ws_tailf), nf,
                                                P.m * (int64_t)P.T, P.tail, ws + P.ws_tail,
                                                (uint32_t)P.ls.record_bytes, restore ? 1 : 0);
    cudaError_t e = cudaGetLastError();
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
    adha_status s = launch_tail(P, b, ws, false, st);
    if (s != ADHA_OK) return s;
    s = launch_transpose(P, b, ws, false, dev, sms, st);
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
        s = launch_cycles(P.S, (int)grid, st, [&](auto save_k, auto shift_k) {
            save_k<<<grid, 256, 0, st>>>(b, seq, segs, nseg, save);
            shift_k<<<grid, 256, 0, st>>>(b, seq, segs, nseg, save);
        });
        if (s != ADHA_OK) return s;
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_err(e, "ip_cycle kernels launch");
    }
    s = launch_transpose(P, b, ws, true, dev, sms, st);
    if (s != ADHA_OK) return s;
    return launch_tail(P, b, ws, true, st);
}
