// remap_host.cu -- adha_remap_host: the remap of HOST buffers through the current device
// (the paper's CPU->GPU remap): hybrid (copy-engine H2D +
// kernel stores into pinned host dst), zero-copy (kernel reads and writes pinned host memory)
// and staged (H2D, remap, D2H) modes; see adha.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "remap_internal.h"

using namespace adha;
using namespace adha::detail;

namespace adha {
namespace {
constexpr int PIPE_SLOTS = 4;        // chunks in flight through the device scratch

struct HostPipe {
    cudaStream_t s[PIPE_SLOTS] = {};
    cudaEvent_t start = nullptr, done[PIPE_SLOTS] = {};
    std::mutex* mu = nullptr;      // held while one call enqueues (the events are shared state)
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
        hp.mu = new std::mutex();      // lives as long as the process, like the pipe's streams
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
    // auto: zero-copy when both sides are pinned and the src has many regions -- one H2D copy per
    // src region and chunk then costs more than the kernel's own TMA reads over PCIe (C3, 64 SoA
    // regions: zero 81.0 GB/s, hybrid 69.1, staged 63.1; C2, one AoS region: hybrid 88, zero 80;
    // profiles/r02f_e2e_c3.log); else hybrid with a pinned dst, else staged
    if (mode == "auto")
        mode = (src_pinned && dst_pinned && aligned && ls.n_clusters() >= 16) ? "zero"
               : (dst_pinned && aligned && scratch)                           ? "hybrid"
                                                                              : "staged";
    if ((mode == "zero" && !(src_pinned && dst_pinned && aligned)) || (mode == "hybrid" && !(dst_pinned && aligned)))
        mode = "staged";
    if (mode == "zero") {
        ck.dst_local = false;                // dst is pinned host memory: STG write-back
        ck.src_local = false;
        return remap_checked((const uint8_t*)src_host, ls, (uint8_t*)dst_host, ld, n, ck, user);
    }

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
    // concurrent calls on one device share the pipe's streams and events: enqueue one at a time
    std::lock_guard<std::mutex> pipe_lock(*hp->mu);
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
            cm.dst_local = false;            // the kernel stores into pinned host memory
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

