// copy_probe.cu -- how fast can ANY kernel move bytes HBM -> HBM on this B200?  The remap's
// roofline denominator is torch copy_ (MEASURED_PEAKS.json); this probe times plain copies of
// the same 8 GiB with several access patterns to see whether a pattern beats copy_ (and by how
// much the read/write mix costs against pure reads or pure writes).  Not on the product path.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1407_4859_b200/csrc \
//        tools/copy_probe.cu -o tools/copy_probe && tools/copy_probe [GiB]
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <functional>
#include <cstring>
#include <string>
#include <vector>

#include "ptx.cuh"

using namespace adha::ptx;

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

__device__ __forceinline__ uint4 ldg_nc(const void* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ uint4 ldg_plain(const void* p) {
    uint4 v;
    asm volatile("ld.global.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ void stg_cs(void* p, uint4 v) {
    asm volatile("st.global.cs.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// grid-stride LDG.128 -> STG.128, U vectors in flight per thread.  HINT: 0 plain, 1 ld.nc +
// st.cs, 2 ld.nc + st.global with L2 evict_first
template <int U, int HINT>
__global__ void k_ldg_stg(const uint4* __restrict__ s, uint4* __restrict__ d, size_t nv) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const uint64_t pol = policy_evict_first();
    for (; i + (U - 1) * stride < nv; i += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = HINT ? ldg_nc(s + i + u * stride) : ldg_plain(s + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (HINT == 1) stg_cs(d + i + u * stride, v[u]);
            else if (HINT == 2) stg128_hint(d + i + u * stride, v[u], pol);
            else stg128(d + i + u * stride, v[u]);
        }
    }
    for (; i < nv; i += stride) d[i] = s[i];
}

// CTA-contiguous chunks: CTA b copies chunks b, b+G, ... of CH bytes (blockDim threads, all
// vectors of a chunk loaded before any is stored)
template <int CHV>
__global__ void k_chunk(const uint4* __restrict__ s, uint4* __restrict__ d, size_t nv) {
    constexpr int PER = CHV / 512;
    for (size_t c = blockIdx.x; c * CHV < nv; c += gridDim.x) {
        const size_t b = c * CHV;
        uint4 v[PER];
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const size_t j = b + u * 512 + threadIdx.x;
            if (j < nv) v[u] = ldg_nc(s + j);
        }
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const size_t j = b + u * 512 + threadIdx.x;
            if (j < nv) d[j] = v[u];
        }
    }
}

__global__ void k_read(const uint4* __restrict__ s, size_t nv, uint32_t* out) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    uint32_t acc = 0;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i + 7 * stride < nv; i += 8 * stride) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = ldg_nc(s + i + u * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    for (; i < nv; i += stride) acc ^= s[i].x;
    if (acc == 0x12345678u) out[0] = acc;
}
__global__ void k_write(uint4* __restrict__ d, size_t nv) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nv; i += stride) stg_cs(d + i, make_uint4(0, 0, 0, 0));
}

// TMA both ways: one CTA per SM, S stages of TB bytes; warp 0 lane 0 loads, warp 1 lane 0 stores
// (bulk store, the stage released after its group has read shared memory)
__global__ void k_tma_copy(const uint8_t* s, uint8_t* d, size_t bytes, uint32_t TB, uint32_t S) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const uint32_t base = (smem_u32(sm) + 127u) & ~127u;
    const uint32_t full0 = base, empty0 = base + 8 * 16, buf0 = base + 256;
    if (threadIdx.x == 0) {
        for (uint32_t i = 0; i < S; ++i) {
            mbar_init(full0 + 8 * i, 1);
            mbar_init(empty0 + 8 * i, 1);
        }
        fence_mbarrier_init();
    }
    __syncthreads();
    const size_t nt = (bytes + TB - 1) / TB;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane != 0) return;
    uint32_t st = 0, ph = 0;
    if (warp == 0) {
        for (size_t t = blockIdx.x; t < nt; t += gridDim.x) {
            mbar_wait(empty0 + 8 * st, ph ^ 1);
            const uint32_t nb = (uint32_t)min((size_t)TB, bytes - t * TB);
            mbar_arrive_expect_tx(full0 + 8 * st, nb);
            bulk_load(buf0 + st * TB, s + t * TB, nb, full0 + 8 * st);
            if (++st == S) { st = 0; ph ^= 1; }
        }
    } else if (warp == 1) {
        int prev = -1;
        for (size_t t = blockIdx.x; t < nt; t += gridDim.x) {
            mbar_wait(full0 + 8 * st, ph);
            const uint32_t nb = (uint32_t)min((size_t)TB, bytes - t * TB);
            bulk_store(d + t * TB, buf0 + st * TB, nb);
            bulk_commit();
            bulk_wait_read<1>();
            if (prev >= 0) mbar_arrive(empty0 + 8 * prev);
            prev = (int)st;
            if (++st == S) { st = 0; ph ^= 1; }
        }
        bulk_wait_all();
    }
}

// TMA loads, consumers write back with LDS.128 -> STG.128 (the remap kernel's pattern without
// the permutation): warp 8 lane 0 loads, warps 0-7 copy out
__global__ void __launch_bounds__(288, 1) k_tma_stg(const uint8_t* s, uint8_t* d, size_t bytes, uint32_t TB, uint32_t S) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const uint32_t base = (smem_u32(sm) + 127u) & ~127u;
    const uint32_t full0 = base, empty0 = base + 8 * 16, buf0 = base + 256;
    if (threadIdx.x == 0) {
        for (uint32_t i = 0; i < S; ++i) {
            mbar_init(full0 + 8 * i, 1);
            mbar_init(empty0 + 8 * i, 8);
        }
        fence_mbarrier_init();
    }
    __syncthreads();
    const size_t nt = bytes / TB;     // whole tiles only (bytes is a multiple of TB here)
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t st = 0, ph = 0;
    if (warp == 8) {
        if (lane) return;
        for (size_t t = blockIdx.x; t < nt; t += gridDim.x) {
            mbar_wait(empty0 + 8 * st, ph ^ 1);
            mbar_arrive_expect_tx(full0 + 8 * st, TB);
            bulk_load(buf0 + st * TB, s + t * TB, TB, full0 + 8 * st);
            if (++st == S) { st = 0; ph ^= 1; }
        }
        return;
    }
    for (size_t t = blockIdx.x; t < nt; t += gridDim.x) {
        mbar_wait(full0 + 8 * st, ph);
        const uint32_t b = buf0 + st * TB;
        uint8_t* g = d + t * TB;
        for (uint32_t v = threadIdx.x * 16; v < TB; v += 4 * 256 * 16) {
            uint4 x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (v + u * 4096 < TB) x[u] = lds128(b + v + u * 4096);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (v + u * 4096 < TB) stg128(g + v + u * 4096, x[u]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8 * st);
        if (++st == S) { st = 0; ph ^= 1; }
    }
}

// Phased copy: every CTA (one per SM, cooperative launch) loads TB bytes, grid barrier, stores
// them, grid barrier: HBM sees long all-read then all-write phases instead of a mix.
__device__ unsigned int g_bar;
__device__ __forceinline__ void grid_bar(unsigned int target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(&g_bar, 1u);
        unsigned int spins = 0;
        while (*(volatile unsigned int*)&g_bar < target && ++spins < (1u << 26)) {
        }
        __threadfence();
    }
    __syncthreads();
}
__global__ void k_phased(const uint8_t* s, uint8_t* d, size_t bytes, uint32_t TB, unsigned int bar0) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const uint32_t base = (smem_u32(sm) + 127u) & ~127u;
    const uint32_t full = base, buf0 = base + 256;
    if (threadIdx.x == 0) {
        mbar_init(full, 1);
        fence_mbarrier_init();
    }
    __syncthreads();
    const size_t nt = (bytes + TB - 1) / TB;
    const size_t rounds = (nt + gridDim.x - 1) / gridDim.x;
    unsigned int gen = bar0;
    for (size_t r = 0; r < rounds; ++r) {
        const size_t t = r * gridDim.x + blockIdx.x;
        const uint32_t nb = t < nt ? (uint32_t)min((size_t)TB, bytes - t * TB) : 0u;
        if (threadIdx.x == 0 && nb) {
            mbar_arrive_expect_tx(full, nb);
            bulk_load(buf0, s + t * TB, nb, full);
        }
        if (nb) mbar_wait(full, (uint32_t)(r & 1));
        gen += gridDim.x;
        grid_bar(gen);
        if (threadIdx.x == 0 && nb) {
            bulk_store(d + t * TB, buf0, nb);
            bulk_commit();
            bulk_wait_all();
        }
        gen += gridDim.x;
        grid_bar(gen);
    }
}


// Many-region tiles: a stage of TB bytes arrives as P bulk copies of TB/P bytes from P regions
// (region j = [j*bytes/P, (j+1)*bytes/P), like an SoA src of P fields); warp 8's lanes issue the
// copies, warps 0-7 write the stage back with LDS.128 -> STG.128 (contiguous dst).  Measures
// what the per-copy cost of the TMA unit does to a tile of many small chunks.
__global__ void __launch_bounds__(288, 1) k_pieces(const uint8_t* s, uint8_t* d, size_t bytes, uint32_t TB, uint32_t S,
                                                   uint32_t P) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const uint32_t base = (smem_u32(sm) + 127u) & ~127u;
    const uint32_t full0 = base, empty0 = base + 8 * 16, buf0 = base + 256;
    if (threadIdx.x == 0) {
        for (uint32_t i = 0; i < S; ++i) {
            mbar_init(full0 + 8 * i, 1);
            mbar_init(empty0 + 8 * i, 8);
        }
        fence_mbarrier_init();
    }
    __syncthreads();
    const uint32_t pb = TB / P;                 // bytes per piece (multiple of 16)
    const size_t region = bytes / P;            // bytes per region
    const size_t nt = region / pb;              // tiles
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t st = 0, ph = 0;
    if (warp == 8) {
        for (size_t t = blockIdx.x; t < nt; t += gridDim.x) {
            mbar_wait(empty0 + 8 * st, ph ^ 1);
            if (lane == 0) mbar_arrive_expect_tx(full0 + 8 * st, pb * P);
            __syncwarp();
            for (uint32_t j = lane; j < P; j += 32)
                bulk_load(buf0 + st * TB + j * pb, s + j * region + t * pb, pb, full0 + 8 * st);
            if (++st == S) { st = 0; ph ^= 1; }
        }
        return;
    }
    for (size_t t = blockIdx.x; t < nt; t += gridDim.x) {
        mbar_wait(full0 + 8 * st, ph);
        const uint32_t b = buf0 + st * TB;
        uint8_t* g = d + t * TB;
        for (uint32_t v = threadIdx.x * 16; v < TB; v += 4 * 256 * 16) {
            uint4 x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (v + u * 4096 < TB) x[u] = lds128(b + v + u * 4096);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (v + u * 4096 < TB) stg128(g + v + u * 4096, x[u]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8 * st);
        if (++st == S) { st = 0; ph ^= 1; }
    }
}

// The same tiles loaded by the consumer warps themselves with cp.async (LDGSTS, 16 B per lane):
// tile i+S-1 is issued before tile i is written back, S-stage ring, cp.async.wait_group.
__global__ void __launch_bounds__(256, 1) k_pieces_ldgsts(const uint8_t* s, uint8_t* d, size_t bytes, uint32_t TB,
                                                          uint32_t S, uint32_t P) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const uint32_t buf0 = (smem_u32(sm) + 127u) & ~127u;
    const uint32_t pb = TB / P;
    const size_t region = bytes / P;
    const size_t nt = region / pb;
    const uint32_t vpp = pb / 16;               // 16-byte vectors per piece
    auto issue = [&](size_t t, uint32_t stg) {
        if (t < nt)
            for (uint32_t v = threadIdx.x; v < TB / 16; v += 256) {
                const uint32_t j = v / vpp, o = (v - j * vpp) * 16;
                const uint8_t* src = s + j * region + t * pb + o;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(buf0 + stg * TB + j * pb + o), "l"(src)
                             : "memory");
            }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    size_t t = blockIdx.x;
    for (uint32_t k = 0; k + 1 < S; ++k) issue(t + k * gridDim.x, k);
    uint32_t st = 0;
    for (; t < nt; t += gridDim.x) {
        issue(t + (S - 1) * (size_t)gridDim.x, (st + S - 1) % S);
        if (S == 2) asm volatile("cp.async.wait_group 1;" ::: "memory");
        else asm volatile("cp.async.wait_group 2;" ::: "memory");
        __syncthreads();
        const uint32_t b = buf0 + st * TB;
        uint8_t* g = d + t * TB;
        for (uint32_t v = threadIdx.x * 16; v < TB; v += 256 * 16) stg128(g + v, lds128(b + v));
        __syncthreads();
        st = (st + 1) % S;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
}

static float time_it(cudaStream_t st, int reps, const std::function<void()>& f) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    f();
    f();
    CK(cudaStreamSynchronize(st));
    CK(cudaEventRecord(a, st));
    for (int i = 0; i < reps; ++i) f();
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms / reps;
}

int main(int argc, char** argv) {
    const double gib = argc > 1 ? atof(argv[1]) : 8.0;
    const size_t bytes = ((size_t)(gib * (1ull << 30))) & ~(size_t)((1 << 16) - 1);
    const size_t nv = bytes / 16;
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    uint8_t *s, *d;
    uint32_t* junk;
    CK(cudaMalloc(&s, bytes));
    CK(cudaMalloc(&d, bytes));
    CK(cudaMalloc(&junk, 64));
    CK(cudaMemset(s, 1, bytes));
    CK(cudaMemset(d, 2, bytes));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    const int reps = 10;
    auto rw = [&](float ms) { return 2.0 * bytes / (ms * 1e-3) / 1e9; };
    auto one = [&](float ms) { return 1.0 * bytes / (ms * 1e-3) / 1e9; };
    printf("bytes per buffer %zu, SMs %d\n", bytes, sms);

    if (argc > 2 && std::string(argv[2]) == "h2d") {
        // H2D of 256 MB as one copy, and as P copies of 256/P MB from P regions 4 GB/P apart (an
        // SoA chunk of adha_remap_host)
        const size_t chunk = 256u << 20, hbytes = 1ull << 32;
        uint8_t* h = nullptr;
        CK(cudaMallocHost(&h, hbytes));
        memset(h, 3, hbytes);
        for (int P : {1, 16, 64, 256}) {
            const size_t piece = chunk / P, stride = hbytes / P;
            std::vector<void*> dsts(P), srcs(P);
            std::vector<size_t> sizes(P, piece);
            for (int j = 0; j < P; ++j) { dsts[j] = d + j * piece; srcs[j] = h + j * stride; }
            float ms = time_it(st, 5, [&] {
                for (int j = 0; j < P; ++j) CK(cudaMemcpyAsync(dsts[j], srcs[j], piece, cudaMemcpyHostToDevice, st));
            });
            printf("H2D 256 MB as %3d copies of %7zu B: %7.3f ms %6.1f GB/s\n", P, piece, ms, chunk / (ms * 1e-3) / 1e9);
        }
        CK(cudaFreeHost(h));
        return 0;
    }
    if (argc > 2 && std::string(argv[2]) == "pieces") {
        for (uint32_t TB : {40960u, 32768u}) {
            for (uint32_t S : {2u, 3u}) {
                const size_t smb = 256 + 128 + (size_t)S * TB;
                if (smb > 232448) continue;
                CK(cudaFuncSetAttribute(k_pieces, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
                CK(cudaFuncSetAttribute(k_pieces_ldgsts, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
                for (uint32_t P : {1u, 8u, 16u, 32u, 64u, 80u}) {
                    if (TB % (P * 16)) continue;
                    float ms = time_it(st, reps, [&] { k_pieces<<<sms, 288, smb, st>>>(s, d, bytes, TB, S, P); });
                    const size_t moved = (bytes / P / (TB / P)) * TB;
                    printf("TMA %2u pieces of %5u B, tile %u KB x %u stages   %8.3f ms %7.0f GB/s\n", P, TB / P, TB >> 10, S, ms,
                           2.0 * moved / (ms * 1e-3) / 1e9);
                    ms = time_it(st, reps, [&] { k_pieces_ldgsts<<<sms, 256, smb, st>>>(s, d, bytes, TB, S, P); });
                    printf("LDGSTS %2u pieces of %5u B, tile %u KB x %u stages %8.3f ms %7.0f GB/s\n", P, TB / P, TB >> 10, S, ms,
                           2.0 * moved / (ms * 1e-3) / 1e9);
                }
            }
        }
        return 0;
    }


    for (int pass = 0; pass < 2; ++pass) {
        printf("---- pass %d\n", pass);
        float ms = time_it(st, reps, [&] { CK(cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice, st)); });
        printf("%-44s %8.3f ms %7.0f GB/s\n", "cudaMemcpyAsync D2D (read+write)", ms, rw(ms));
        ms = time_it(st, reps, [&] { CK(cudaMemsetAsync(d, 0, bytes, st)); });
        printf("%-44s %8.3f ms %7.0f GB/s\n", "cudaMemsetAsync (write only)", ms, one(ms));
        for (int bps : {2, 4, 8}) {
            ms = time_it(st, reps, [&] { k_write<<<sms * bps, 512, 0, st>>>((uint4*)d, nv); });
            printf("k_write STG.cs grid %dx512 (write only)%*s %8.3f ms %7.0f GB/s\n", sms * bps, 5, "", ms, one(ms));
            ms = time_it(st, reps, [&] { k_read<<<sms * bps, 512, 0, st>>>((const uint4*)s, nv, junk); });
            printf("k_read LDG.nc x8 grid %dx512 (read only)%*s %8.3f ms %7.0f GB/s\n", sms * bps, 4, "", ms, one(ms));
        }
        for (int bps : {2, 4, 8}) {
            char name[96];
            ms = time_it(st, reps, [&] { k_ldg_stg<4, 0><<<sms * bps, 512, 0, st>>>((const uint4*)s, (uint4*)d, nv); });
            snprintf(name, sizeof name, "ldg/stg x4 plain grid %dx512", sms * bps);
            printf("%-44s %8.3f ms %7.0f GB/s\n", name, ms, rw(ms));
            ms = time_it(st, reps, [&] { k_ldg_stg<8, 1><<<sms * bps, 512, 0, st>>>((const uint4*)s, (uint4*)d, nv); });
            snprintf(name, sizeof name, "ldg.nc/stg.cs x8 grid %dx512", sms * bps);
            printf("%-44s %8.3f ms %7.0f GB/s\n", name, ms, rw(ms));
            ms = time_it(st, reps, [&] { k_ldg_stg<8, 2><<<sms * bps, 512, 0, st>>>((const uint4*)s, (uint4*)d, nv); });
            snprintf(name, sizeof name, "ldg.nc/stg evict_first x8 grid %dx512", sms * bps);
            printf("%-44s %8.3f ms %7.0f GB/s\n", name, ms, rw(ms));
        }
        for (int bps : {2, 4}) {
            char name[96];
            ms = time_it(st, reps, [&] { k_chunk<512 * 8><<<sms * bps, 512, 0, st>>>((const uint4*)s, (uint4*)d, nv); });
            snprintf(name, sizeof name, "chunk 64 KB per CTA step, grid %dx512", sms * bps);
            printf("%-44s %8.3f ms %7.0f GB/s\n", name, ms, rw(ms));
        }
        for (uint32_t TB : {16384u, 32768u, 49152u, 65536u}) {
            for (uint32_t S : {2u, 3u, 4u}) {
                const size_t smb = 256 + 128 + (size_t)S * TB;
                if (smb > 232448) continue;
                CK(cudaFuncSetAttribute(k_tma_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
                ms = time_it(st, reps, [&] { k_tma_copy<<<sms, 64, smb, st>>>(s, d, bytes, TB, S); });
                char name[96];
                snprintf(name, sizeof name, "TMA load + TMA store, %u KB x %u", TB >> 10, S);
                printf("%-44s %8.3f ms %7.0f GB/s\n", name, ms, rw(ms));
                CK(cudaFuncSetAttribute(k_tma_stg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
                ms = time_it(st, reps, [&] { k_tma_stg<<<sms, 288, smb, st>>>(s, d, bytes, TB, S); });
                snprintf(name, sizeof name, "TMA load + LDS/STG, %u KB x %u", TB >> 10, S);
                printf("%-44s %8.3f ms %7.0f GB/s\n", name, ms, rw(ms));
            }
        }
        for (uint32_t TB : {65536u, 131072u, 196608u}) {
            const size_t smb = 256 + 128 + TB;
            CK(cudaFuncSetAttribute(k_phased, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
            unsigned int zero = 0;
            const size_t nt = (bytes + TB - 1) / TB;
            const unsigned int per_call = (unsigned int)(2 * ((nt + sms - 1) / sms) * sms);
            unsigned int gen = 0;
            CK(cudaMemcpyToSymbol(g_bar, &zero, sizeof zero));
            auto f = [&] {
                void* args[] = {(void*)&s, (void*)&d, (void*)&bytes, (void*)&TB, (void*)&gen};
                CK(cudaLaunchCooperativeKernel((void*)k_phased, sms, 128, args, smb, st));
                gen += per_call;
            };
            ms = time_it(st, reps, f);
            char name[96];
            snprintf(name, sizeof name, "phased (grid barrier) %u KB", TB >> 10);
            printf("%-44s %8.3f ms %7.0f GB/s\n", name, ms, rw(ms));
        }
    }
    // correctness of the last copy variant
    std::vector<uint8_t> h(1 << 20);
    CK(cudaMemcpy(h.data(), d + bytes - h.size(), h.size(), cudaMemcpyDeviceToHost));
    size_t bad = 0;
    for (uint8_t x : h) bad += x != 1;
    printf("check: %zu bad bytes in the last MiB\n", bad);
    return 0;
}
