// layout.cpp -- the layout descriptor.
//
// A layout is a partition of the fields into clusters (PAPER.md
// Table 2).  Canonical order: clusters by minimum decl index,
// fields by decl index.  Packed cluster records (reading Q2),
// regions in canonical order with 256-byte-aligned bases (reading Q3), element
// address base + i * stride + offset.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <map>
#include <string>
#include <unordered_map>

#include "internal.h"

namespace adha {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
void clear_error() { g_last_error.clear(); }
adha_status fail(adha_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}

static std::atomic<uint64_t> g_next_id{1};

static uint32_t natural_align(uint32_t w) {
    uint32_t a = 1;
    while (a < 8 && w % (a * 2) == 0) a *= 2;
    return a;
}

std::unique_ptr<Layout> make_layout(const uint32_t* widths, int32_t n, const int32_t* labels,
                                    const int32_t* block_of, bool aligned) {
    auto L = std::make_unique<Layout>();
    L->n_fields = n;
    L->aligned = aligned;
    L->width.assign(widths, widths + n);
    L->cluster.assign(n, -1);
    L->offset.assign(n, 0);
    // number clusters by first sight in decl order == by minimum decl index
    std::unordered_map<int32_t, int32_t> seen;
    std::vector<uint32_t> maxa;
    for (int32_t f = 0; f < n; ++f) {
        auto it = seen.find(labels[f]);
        int32_t c;
        if (it == seen.end()) {
            c = (int32_t)L->members.size();
            seen.emplace(labels[f], c);
            L->members.emplace_back();
            L->stride.push_back(0);
            L->block.push_back(block_of ? (uint32_t)block_of[f] : 1u);
            maxa.push_back(1);
        } else {
            c = it->second;
        }
        L->cluster[f] = c;
        if (aligned) {   // C-struct rule: a field starts at a multiple of its natural alignment
            const uint32_t a = natural_align(widths[f]);
            maxa[c] = std::max(maxa[c], a);
            L->stride[c] = (L->stride[c] + a - 1) / a * a;
        }
        L->offset[f] = (uint32_t)L->stride[c];
        L->stride[c] += widths[f];
        L->members[c].push_back(f);
        L->record_bytes += widths[f];
    }
    for (size_t c = 0; c < L->stride.size(); ++c) L->stride[c] = (L->stride[c] + maxa[c] - 1) / maxa[c] * maxa[c];
    L->id = g_next_id.fetch_add(1);
    return L;
}

bool Layout::region_bases(int64_t n, std::vector<uint64_t>& base, uint64_t* total) const {
    const int32_t C = n_clusters();
    base.assign(C, 0);
    const uint64_t N = (uint64_t)n;
    // overflow guard: all regions (whole blocks) + 256 * C must fit in 63 bits
    uint64_t per_rec = 0, per_blk = 0;
    for (int32_t c = 0; c < C; ++c) { per_rec += stride[c]; per_blk += block[c] * stride[c]; }
    if (per_rec != 0 && N > (uint64_t(INT64_MAX) - 256ull * (uint64_t)C - per_blk) / per_rec) return false;
    uint64_t b = 0;
    for (int32_t c = 0; c < C; ++c) {
        if (c > 0) b = align256(b);
        base[c] = b;
        b += region_bytes(c, n);
    }
    if (total) *total = b;
    return true;
}

std::string layout_string(const Layout& l, const char* const* names) {
    std::string s = l.aligned ? "aligned:" : "";
    for (int32_t c = 0; c < l.n_clusters(); ++c) {
        if (c) s += '|';
        s += '{';
        for (size_t k = 0; k < l.members[c].size(); ++k) {
            if (k) s += ',';
            int32_t f = l.members[c][k];
            if (names && names[f]) s += names[f];
            else s += "f" + std::to_string(f);
        }
        s += '}';
        if (l.block[c] > 1) s += "@" + std::to_string(l.block[c]);
    }
    return s;
}

}  // namespace adha

using namespace adha;

extern "C" {

int32_t adha_version(void) { return 100; }  // 0.1.0

const char* adha_status_string(adha_status s) {
    switch (s) {
        case ADHA_OK: return "ADHA_OK";
        case ADHA_ERR_INVALID_ARG: return "ADHA_ERR_INVALID_ARG";
        case ADHA_ERR_PARSE: return "ADHA_ERR_PARSE";
        case ADHA_ERR_LAYOUT_MISMATCH: return "ADHA_ERR_LAYOUT_MISMATCH";
        case ADHA_ERR_CAPACITY: return "ADHA_ERR_CAPACITY";
        case ADHA_ERR_ALIGNMENT: return "ADHA_ERR_ALIGNMENT";
        case ADHA_ERR_OVERLAP: return "ADHA_ERR_OVERLAP";
        case ADHA_ERR_TOO_LARGE: return "ADHA_ERR_TOO_LARGE";
        case ADHA_ERR_CUDA: return "ADHA_ERR_CUDA";
        case ADHA_ERR_OOM: return "ADHA_ERR_OOM";
        case ADHA_ERR_UNSUPPORTED: return "ADHA_ERR_UNSUPPORTED";
        case ADHA_ERR_PLANNER: return "ADHA_ERR_PLANNER";
    }
    return "ADHA_ERR_UNKNOWN";
}

const char* adha_last_error(void) { return g_last_error.c_str(); }

void adha_free(void* p) { std::free(p); }

static adha_status check_widths(const uint32_t* widths, int32_t n) {
    if (!widths) return fail(ADHA_ERR_INVALID_ARG, "field_widths is NULL");
    if (n < 1 || n > ADHA_MAX_FIELDS)
        return fail(ADHA_ERR_INVALID_ARG, "n_fields must be in 1.." + std::to_string(ADHA_MAX_FIELDS));
    for (int32_t f = 0; f < n; ++f)
        if (widths[f] < 1 || widths[f] > ADHA_MAX_FIELD_BYTES)
            return fail(ADHA_ERR_INVALID_ARG, "field " + std::to_string(f) + " has width " +
                                                  std::to_string(widths[f]));
    return ADHA_OK;
}

adha_status adha_layout_create_ex(const uint32_t* widths, int32_t n, const int32_t* cluster_of,
                                  const int32_t* block_of, uint32_t flags, adha_layout** out) {
    clear_error();
    if (!out || !cluster_of) return fail(ADHA_ERR_INVALID_ARG, "null argument");
    adha_status st = check_widths(widths, n);
    if (st != ADHA_OK) return st;
    if (flags & ~uint32_t(ADHA_LAYOUT_ALIGNED)) return fail(ADHA_ERR_INVALID_ARG, "unknown layout flags");
    if (block_of) {
        std::unordered_map<int32_t, int32_t> blk;
        for (int32_t f = 0; f < n; ++f) {
            const int32_t b = block_of[f];
            if (!(b == 1 || b == 2 || b == 4 || b == 8 || b == 16 || b == 32))
                return fail(ADHA_ERR_INVALID_ARG, "block must be 1, 2, 4, 8, 16 or 32");
            auto it = blk.emplace(cluster_of[f], b).first;
            if (it->second != b) return fail(ADHA_ERR_INVALID_ARG, "fields of one cluster need one block size");
        }
    }
    try {
        auto* h = new adha_layout;
        h->L = std::move(*make_layout(widths, n, cluster_of, block_of, (flags & ADHA_LAYOUT_ALIGNED) != 0));
        *out = h;
    } catch (const std::bad_alloc&) {
        return fail(ADHA_ERR_OOM, "out of host memory");
    }
    return ADHA_OK;
}

adha_status adha_layout_create(const uint32_t* widths, int32_t n, const int32_t* cluster_of,
                               adha_layout** out) {
    return adha_layout_create_ex(widths, n, cluster_of, nullptr, 0u, out);
}

adha_status adha_layout_from_string(const char* text, const char* const* names,
                                    const uint32_t* widths, int32_t n, adha_layout** out) {
    clear_error();
    if (!text || !names || !out) return fail(ADHA_ERR_INVALID_ARG, "null argument");
    adha_status st = check_widths(widths, n);
    if (st != ADHA_OK) return st;
    std::map<std::string, int32_t> index;
    for (int32_t f = 0; f < n; ++f) {
        if (!names[f] || !*names[f]) return fail(ADHA_ERR_INVALID_ARG, "empty field name");
        if (!index.emplace(names[f], f).second)
            return fail(ADHA_ERR_INVALID_ARG, std::string("duplicate field name ") + names[f]);
    }
    std::vector<int32_t> label(n, -1);
    std::vector<int32_t> blk(n, 1);
    int32_t next = 0;
    const char* p = text;
    uint32_t flags = 0;
    while (*p == ' ' || *p == '\t') ++p;
    if (std::strncmp(p, "aligned:", 8) == 0) {
        flags |= ADHA_LAYOUT_ALIGNED;
        p += 8;
    }
    // an optional "@B" after a cluster sets its AoSoA block
    auto take_block = [&](int32_t lab) -> adha_status {
        if (*p != '@') return ADHA_OK;
        ++p;
        char* e = nullptr;
        long b = std::strtol(p, &e, 10);
        if (e == p) return fail(ADHA_ERR_PARSE, "missing block size after '@'");
        p = e;
        for (int32_t f = 0; f < n; ++f)
            if (label[f] == lab) blk[f] = (int32_t)b;
        return ADHA_OK;
    };
    auto is_sep = [](char c) { return c == ',' || c == '|' || c == ' ' || c == '\t' || c == '\n'; };
    auto take_name = [&](const char*& q, std::string& nm) {
        const char* s = q;
        while (*q && !is_sep(*q) && *q != '{' && *q != '}' && *q != '@') ++q;
        nm.assign(s, q - s);
    };
    auto assign = [&](const std::string& nm, int32_t lab) -> adha_status {
        auto it = index.find(nm);
        if (it == index.end()) return fail(ADHA_ERR_PARSE, "unknown field name '" + nm + "'");
        if (label[it->second] != -1) return fail(ADHA_ERR_PARSE, "field '" + nm + "' appears twice");
        label[it->second] = lab;
        return ADHA_OK;
    };
    while (*p) {
        if (is_sep(*p)) { ++p; continue; }
        if (*p == '{') {
            ++p;
            int32_t lab = next++;
            int members = 0;
            for (;;) {
                while (*p && is_sep(*p)) ++p;
                if (!*p) return fail(ADHA_ERR_PARSE, "unterminated '{'");
                if (*p == '}') { ++p; break; }
                if (*p == '{') return fail(ADHA_ERR_PARSE, "nested '{'");
                std::string nm;
                take_name(p, nm);
                if ((st = assign(nm, lab)) != ADHA_OK) return st;
                ++members;
            }
            if (members == 0) return fail(ADHA_ERR_PARSE, "empty cluster '{}'");
            if ((st = take_block(lab)) != ADHA_OK) return st;
        } else if (*p == '}') {
            return fail(ADHA_ERR_PARSE, "unbalanced '}'");
        } else {
            std::string nm;
            take_name(p, nm);
            const int32_t lab = next++;
            if ((st = assign(nm, lab)) != ADHA_OK) return st;
            if ((st = take_block(lab)) != ADHA_OK) return st;
        }
    }
    for (int32_t f = 0; f < n; ++f)
        if (label[f] < 0) return fail(ADHA_ERR_PARSE, std::string("field '") + names[f] + "' missing");
    st = adha_layout_create_ex(widths, n, label.data(), blk.data(), flags, out);
    if (st == ADHA_ERR_INVALID_ARG) st = ADHA_ERR_PARSE;
    return st;
}

adha_status adha_layout_to_string(const adha_layout* h, const char* const* names, char* buf,
                                  size_t cap, size_t* needed) {
    clear_error();
    if (!h || !needed) return fail(ADHA_ERR_INVALID_ARG, "null argument");
    std::string s = layout_string(h->L, names);
    *needed = s.size();
    if (buf && cap > 0) {
        size_t k = std::min(cap - 1, s.size());
        std::memcpy(buf, s.data(), k);
        buf[k] = '\0';
    }
    return ADHA_OK;
}

adha_status adha_layout_info(const adha_layout* h, int32_t* n_fields, int32_t* n_clusters,
                             uint64_t* record_bytes) {
    clear_error();
    if (!h) return fail(ADHA_ERR_INVALID_ARG, "null layout");
    if (n_fields) *n_fields = h->L.n_fields;
    if (n_clusters) *n_clusters = h->L.n_clusters();
    if (record_bytes) *record_bytes = h->L.record_bytes;
    return ADHA_OK;
}

adha_status adha_layout_clusters(const adha_layout* h, int32_t* out) {
    clear_error();
    if (!h || !out) return fail(ADHA_ERR_INVALID_ARG, "null argument");
    std::copy(h->L.cluster.begin(), h->L.cluster.end(), out);
    return ADHA_OK;
}

adha_status adha_layout_bytes(const adha_layout* h, int64_t n, uint64_t* out) {
    clear_error();
    if (!h || !out) return fail(ADHA_ERR_INVALID_ARG, "null argument");
    if (n < 0) return fail(ADHA_ERR_INVALID_ARG, "n_records < 0");
    std::vector<uint64_t> base;
    if (!h->L.region_bases(n, base, out)) return fail(ADHA_ERR_TOO_LARGE, "layout bytes overflow");
    return ADHA_OK;
}

adha_status adha_layout_field_address(const adha_layout* h, int32_t f, int64_t n,
                                      uint64_t* region_offset, uint32_t* stride, uint32_t* offset) {
    clear_error();
    if (!h) return fail(ADHA_ERR_INVALID_ARG, "null layout");
    if (f < 0 || f >= h->L.n_fields) return fail(ADHA_ERR_INVALID_ARG, "field index out of range");
    if (n < 0) return fail(ADHA_ERR_INVALID_ARG, "n_records < 0");
    std::vector<uint64_t> base;
    if (!h->L.region_bases(n, base, nullptr)) return fail(ADHA_ERR_TOO_LARGE, "layout bytes overflow");
    int32_t c = h->L.cluster[f];
    if (region_offset) *region_offset = base[c];
    if (stride) *stride = (uint32_t)h->L.stride[c];
    if (offset) *offset = h->L.offset[f];
    return ADHA_OK;
}

adha_status adha_layout_field_address_ex(const adha_layout* h, int32_t f, int64_t n, uint64_t* region_offset,
                                         uint32_t* stride, uint32_t* offset, uint32_t* block) {
    adha_status st = adha_layout_field_address(h, f, n, region_offset, stride, offset);
    if (st == ADHA_OK && block) *block = h->L.block[h->L.cluster[f]];
    return st;
}

void adha_layout_destroy(adha_layout* h) { delete h; }

adha_status adha_shard_range(int64_t n_total, int32_t n_shards, int32_t shard, int64_t* lo,
                             int64_t* hi) {
    clear_error();
    if (!lo || !hi) return fail(ADHA_ERR_INVALID_ARG, "null argument");
    if (n_total < 0 || n_shards < 1 || shard < 0 || shard >= n_shards)
        return fail(ADHA_ERR_INVALID_ARG, "bad shard arguments");
    // floor(g*N/G) without overflow: N = q*G + r
    const int64_t q = n_total / n_shards, r = n_total % n_shards;
    auto bound = [&](int64_t g) { return q * g + (r * g) / n_shards; };
    *lo = bound(shard);
    *hi = bound(shard + 1);
    return ADHA_OK;
}

}  // extern "C"
