// sections.cu -- synthetic consumer sections read through a layout:
// the device-side half of a B200 tuning profile for PDL.  Not on the remap
// path.  One thread per output: a streaming pass (records 0..n-1, coalescing depends on the
// layout) or an irregular gather (idx[i], one touched line per field cluster).
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "internal.h"

namespace adha {
namespace dev {

constexpr int SECTION_MAXF = 32;

struct SectionField {
    uint64_t base;     // region base + offset of the field (bytes from buf)
    uint32_t stride;   // cluster record bytes
    uint32_t pad;
};

struct SectionParams {
    uint64_t buf;
    const int64_t* idx;
    float* out;
    int64_t n_out;
    uint32_t n_f;
    uint32_t pad;
    SectionField f[SECTION_MAXF];
};

__global__ void section_kernel(const __grid_constant__ SectionParams p) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p.n_out;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = p.idx ? p.idx[i] : i;
        float acc = 0.0f;
        for (uint32_t k = 0; k < p.n_f; ++k) {
            const float v = *reinterpret_cast<const float*>(p.buf + p.f[k].base + (uint64_t)r * p.f[k].stride);
            acc = fmaf(v, v, acc);
        }
        p.out[i] = acc;
    }
}

}  // namespace dev
}  // namespace adha

using namespace adha;
using namespace adha::dev;

extern "C" adha_status adha_section_run(const void* buf, const adha_layout* h, int64_t n_records,
                                        const int32_t* fields, int32_t n_used, const int64_t* idx, int64_t n_out,
                                        float* out, void* stream) {
    clear_error();
    if (!h || !fields || !out || n_records < 0 || n_out < 0) return fail(ADHA_ERR_INVALID_ARG, "bad argument");
    if (n_used < 1 || n_used > SECTION_MAXF) return fail(ADHA_ERR_INVALID_ARG, "1..32 fields per section pass");
    if (n_out == 0) return ADHA_OK;
    if (!buf || ((uintptr_t)buf & 255)) return fail(ADHA_ERR_ALIGNMENT, "buffer must be 256-byte aligned");
    if (!idx && n_out > n_records) return fail(ADHA_ERR_INVALID_ARG, "streaming pass beyond n_records");
    const Layout& L = h->L;
    std::vector<uint64_t> base;
    if (!L.region_bases(n_records, base, nullptr)) return fail(ADHA_ERR_TOO_LARGE, "layout bytes overflow");
    SectionParams P{};
    P.buf = (uint64_t)(uintptr_t)buf;
    P.idx = idx;
    P.out = out;
    P.n_out = n_out;
    P.n_f = (uint32_t)n_used;
    for (int32_t k = 0; k < n_used; ++k) {
        const int32_t f = fields[k];
        if (f < 0 || f >= L.n_fields) return fail(ADHA_ERR_INVALID_ARG, "field index out of range");
        const int32_t c = L.cluster[f];
        if (L.width[f] != 4 || (L.offset[f] & 3) || (L.stride[c] & 3))
            return fail(ADHA_ERR_UNSUPPORTED, "field " + std::to_string(f) + " is not a 4-byte aligned fp32 slot");
        P.f[k] = {base[c] + L.offset[f], (uint32_t)L.stride[c], 0};
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n_out + 255) / 256, (int64_t)sms * 16));
    section_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(P);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(ADHA_ERR_CUDA, std::string("section_kernel launch: ") + cudaGetErrorString(e));
    return ADHA_OK;
}
