// remap_internal.h -- host helpers shared by remap.cu (launch, C ABI) and remap_host.cu
// (host-memory remap): validation, the checked launch, CUDA error mapping.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "internal.h"
#include "remap_plan.h"

namespace adha {
namespace detail {

struct Checked {
    uint64_t bytes_s = 0, bytes_d = 0;
    std::vector<uint64_t> bs, bd;   // region offsets (relative to the buffer pointers)
    bool dst_local = true;          // dst is this device's HBM (not pinned host or peer memory)
    bool src_local = true;          // src is this device's HBM (not pinned host memory)
};

adha_status cuda_fail(cudaError_t e, const char* what);
adha_status validate(const void* src, const adha_layout* hs, const void* dst, const adha_layout* hd, int64_t n,
                     Checked* out, bool device_buffers);
adha_status remap_checked(const uint8_t* src, const Layout& ls, uint8_t* dst, const Layout& ld, int64_t n,
                          const Checked& ck, cudaStream_t st);

}  // namespace detail
}  // namespace adha
