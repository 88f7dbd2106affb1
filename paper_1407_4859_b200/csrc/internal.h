// internal.h -- shared host-side declarations of libadha (not part of the ABI).
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/adha.h"

namespace adha {

// --------------------------------------------------------------------------- errors
void set_error(const std::string& msg);
void clear_error();
adha_status fail(adha_status s, const std::string& msg);

// --------------------------------------------------------------------------- layout
// Canonical descriptor (adha.h "layout descriptor").
struct Layout {
    int32_t n_fields = 0;
    std::vector<uint32_t> width;                 // per field
    std::vector<int32_t> cluster;                // canonical cluster index per field
    std::vector<uint32_t> offset;                // byte offset of the field in its cluster record
    std::vector<uint64_t> stride;                // per cluster: bytes per cluster record
    std::vector<std::vector<int32_t>> members;   // per cluster, in declaration order
    std::vector<uint32_t> block;                 // per cluster: AoSoA block (1 = plain records)
    bool aligned = false;                        // natural (C-struct) alignment inside records
    uint64_t record_bytes = 0;                   // payload bytes per record (sum of widths)
    uint64_t id = 0;                             // process-unique, keys the plan cache

    int32_t n_clusters() const { return (int32_t)stride.size(); }
    // base(c) for an N-record instance; returns false on overflow.
    bool region_bases(int64_t n, std::vector<uint64_t>& base, uint64_t* total) const;
    // bytes of cluster c's region for N records: ceil(N / B) whole blocks of B records
    uint64_t region_bytes(int32_t c, int64_t n) const {
        const uint64_t b = block[c];
        return ((uint64_t)n + b - 1) / b * b * stride[c];
    }
    // byte address of field f of record i inside its region (generalised element address)
    uint64_t local_addr(int32_t f, uint64_t i) const {
        const int32_t c = cluster[f];
        const uint64_t b = block[c];
        return (i / b) * (b * stride[c]) + (uint64_t)offset[f] * b + (i % b) * width[f];
    }
    // payload bytes of cluster c per record (stride minus alignment padding)
    uint64_t payload(int32_t c) const {
        uint64_t s = 0;
        for (int32_t f : members[c]) s += width[f];
        return s;
    }
};

inline uint64_t align256(uint64_t x) { return (x + 255u) & ~uint64_t(255); }

std::unique_ptr<Layout> make_layout(const uint32_t* widths, int32_t n, const int32_t* labels,
                                    const int32_t* block_of = nullptr, bool aligned = false);
std::string layout_string(const Layout& l, const char* const* names);

}  // namespace adha

struct adha_layout {
    adha::Layout L;
};
