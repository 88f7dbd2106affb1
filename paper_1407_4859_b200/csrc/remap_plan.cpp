// remap_plan.cpp -- compiles a (src layout, dst layout) pair into the tiled
// kernel's plan: unit size, tile records T, pipeline
// stages, chunk placement in shared memory and the per-lane permutation table.
//
// Everything here is N-independent; adha_remap fills the N-dependent region
// bases (adha.h "layout descriptor") into the kernel parameters per call.
#include "remap_plan.h"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>

#include "internal.h"
#include "json.h"

namespace adha {

using namespace dev;

static uint32_t env_u32(const char* name, uint32_t dflt) {
    const char* v = std::getenv(name);
    if (!v || !*v) return dflt;
    long x = std::strtol(v, nullptr, 10);
    return x > 0 ? (uint32_t)x : dflt;
}

// Kuhn's augmenting-path matching on the 32x32 support of cnt (left = src bank).
static bool augment(int u, const uint32_t cnt[32][32], int match_r[32], bool seen[32]) {
    for (int v = 0; v < 32; ++v) {
        if (!cnt[u][v] || seen[v]) continue;
        seen[v] = true;
        if (match_r[v] < 0 || augment(match_r[v], cnt, match_r, seen)) {
            match_r[v] = u;
            return true;
        }
    }
    return false;
}

RemapPlan compile_plan(const Layout& ls, const Layout& ld) {
    RemapPlan P;
    const int F = ls.n_fields;
    const uint64_t R = ls.record_bytes;

    // unit g: largest of 4, 2, 1 dividing every width and every offset in both layouts
    uint64_t gall = 0;
    for (int f = 0; f < F; ++f) {
        gall = std::gcd(gall, (uint64_t)ls.width[f]);
        gall = std::gcd(gall, (uint64_t)ls.offset[f]);
        gall = std::gcd(gall, (uint64_t)ld.offset[f]);
    }
    P.unit = (gall % 4 == 0) ? 4 : (gall % 2 == 0) ? 2 : 1;
    const uint32_t g = P.unit;

    auto naive = [&](const std::string& why) {
        P.tiled = false;
        P.why_naive = why;
        return P;
    };
    if (F > MAXF) return naive("more than " + std::to_string(MAXF) + " fields");
    if (ls.n_clusters() > MAXC || ld.n_clusters() > MAXC)
        return naive("more than " + std::to_string(MAXC) + " clusters");
    const uint64_t W = R / g;
    int cls = -1;
    for (int c = 0; c < 4; ++c)
        if (32 * W <= (uint64_t)CLASS_NENT[c] && W <= (uint64_t)NCONS * CLASS_EMAX[c]) { cls = c; break; }
    if (cls < 0) return naive("record of " + std::to_string(W) + " units exceeds the instruction table");
    P.table_class = cls;
    P.n_instr = (uint32_t)W;

    // tile size and stages
    const uint32_t budget = 232448 - HDR_BYTES;  // sm_100 opt-in dynamic shared memory per block
    const uint32_t target = env_u32("ADHA_STAGE_BYTES", 32768);
    uint32_t s_in = std::min<uint32_t>(env_u32("ADHA_STAGES", 4), MAX_S_IN);
    uint64_t T = std::max<uint64_t>(32, (target / (32 * R)) * 32);
    while (T > 32 && T * W > 65536) T -= 32;                       // 16-bit unit offsets
    auto stage_of = [&](uint64_t t) { return ((t * R) + 127) / 128 * 128; };
    while (s_in > 2 && (s_in + S_OUT) * stage_of(T) > budget) --s_in;
    while (T > 32 && (s_in + S_OUT) * stage_of(T) > budget) T -= 32;
    if ((s_in + S_OUT) * stage_of(T) > budget || T * W > 65536)
        return naive("a 32-record tile does not fit in shared memory");
    P.T = (uint32_t)T;
    P.s_in = s_in;
    P.tile_bytes = (uint32_t)(T * R);
    P.stage_bytes = (uint32_t)stage_of(T);
    P.smem_bytes = HDR_BYTES + (s_in + S_OUT) * P.stage_bytes;

    // chunk placement: clusters in canonical order, each T*stride bytes (a multiple of 32)
    uint32_t off = 0;
    for (int c = 0; c < ls.n_clusters(); ++c) { P.src_chunk.push_back(off); off += (uint32_t)(T * ls.stride[c]); }
    off = 0;
    for (int c = 0; c < ld.n_clusters(); ++c) { P.dst_chunk.push_back(off); off += (uint32_t)(T * ld.stride[c]); }

    // the 32*W units of period 0
    struct Unit { uint32_t in, out; uint8_t sc, dc; };
    std::vector<Unit> units;
    units.reserve(32 * W);
    for (uint32_t r = 0; r < 32; ++r)
        for (int f = 0; f < F; ++f) {
            const int cs = ls.cluster[f], cd = ld.cluster[f];
            for (uint32_t j = 0; j < ls.width[f] / g; ++j) {
                uint64_t ib = P.src_chunk[cs] + r * ls.stride[cs] + ls.offset[f] + j * g;
                uint64_t ob = P.dst_chunk[cd] + r * ld.stride[cd] + ld.offset[f] + j * g;
                units.push_back({(uint32_t)(ib / g), (uint32_t)(ob / g), (uint8_t)cs, (uint8_t)cd});
            }
        }

    std::vector<uint32_t> order;   // unit index per (instruction, lane)
    order.reserve(units.size());
    if (g == 4) {
        // decompose the bank multigraph (src bank -> dst bank) into perfect matchings
        std::vector<uint32_t> bucket[32][32];
        uint32_t cnt[32][32] = {};
        for (uint32_t u = 0; u < units.size(); ++u) {
            int bi = units[u].in % 32, bo = units[u].out % 32;
            bucket[bi][bo].push_back(u);
            ++cnt[bi][bo];
        }
        bool ok = true;
        while (order.size() < units.size()) {
            int match_r[32];
            std::fill(match_r, match_r + 32, -1);
            for (int u = 0; u < 32 && ok; ++u) {
                bool seen[32] = {};
                if (!augment(u, cnt, match_r, seen)) ok = false;
            }
            if (!ok) break;
            int sigma[32];
            for (int v = 0; v < 32; ++v) sigma[match_r[v]] = v;
            uint32_t m = UINT32_MAX;
            for (int u = 0; u < 32; ++u) m = std::min(m, cnt[u][sigma[u]]);
            for (uint32_t rep = 0; rep < m; ++rep)
                for (int u = 0; u < 32; ++u) {
                    order.push_back(bucket[u][sigma[u]].back());
                    bucket[u][sigma[u]].pop_back();
                }
            for (int u = 0; u < 32; ++u) cnt[u][sigma[u]] -= m;
        }
        P.matched = ok;
        if (!ok) order.clear();
    }
    if (order.empty()) {
        // destination order: lanes write consecutive units
        std::vector<uint32_t> idx(units.size());
        std::iota(idx.begin(), idx.end(), 0u);
        std::sort(idx.begin(), idx.end(), [&](uint32_t a, uint32_t b) { return units[a].out < units[b].out; });
        order = idx;
    }
    P.ent_off.resize(order.size());
    P.ent_sc.resize(order.size());
    P.ent_dc.resize(order.size());
    for (size_t k = 0; k < order.size(); ++k) {
        const Unit& u = units[order[k]];
        P.ent_off[k] = u.in | (u.out << 16);
        P.ent_sc[k] = u.sc;
        P.ent_dc[k] = u.dc;
    }
    // kernel-parameter image of EntryTable<NENT>: off[NENT] | sc[NENT] | dc[NENT]
    const uint32_t nent = (uint32_t)CLASS_NENT[cls];
    P.table.assign((nent * 6 + 3) / 4, 0u);
    uint8_t* img = reinterpret_cast<uint8_t*>(P.table.data());
    std::memcpy(img, P.ent_off.data(), P.ent_off.size() * 4);
    std::memcpy(img + 4 * nent, P.ent_sc.data(), P.ent_sc.size());
    std::memcpy(img + 5 * nent, P.ent_dc.data(), P.ent_dc.size());
    P.tiled = true;
    return P;
}

std::string describe_plan(const RemapPlan& p, const Layout& ls, const Layout& ld) {
    std::string o = "{";
    o += "\"tiled\":" + std::string(p.tiled ? "true" : "false");
    o += ",\"why_naive\":" + json::quote(p.why_naive);
    o += ",\"unit\":" + std::to_string(p.unit);
    o += ",\"T\":" + std::to_string(p.T);
    o += ",\"s_in\":" + std::to_string(p.s_in);
    o += ",\"s_out\":" + std::to_string(dev::S_OUT);
    o += ",\"stage_bytes\":" + std::to_string(p.stage_bytes);
    o += ",\"tile_bytes\":" + std::to_string(p.tile_bytes);
    o += ",\"smem_bytes\":" + std::to_string(p.smem_bytes);
    o += ",\"n_instr\":" + std::to_string(p.n_instr);
    o += ",\"n_consumer_warps\":" + std::to_string(dev::NCONS);
    o += ",\"table_class\":" + std::to_string(p.table_class);
    o += ",\"table_entries\":" + std::to_string(dev::CLASS_NENT[p.table_class]);
    o += ",\"matched\":" + std::string(p.matched ? "true" : "false");
    auto arr = [&](const char* name, const std::vector<uint32_t>& v) {
        o += ",\"" + std::string(name) + "\":[";
        for (size_t i = 0; i < v.size(); ++i) o += (i ? "," : "") + std::to_string(v[i]);
        o += "]";
    };
    arr("src_chunk", p.src_chunk);
    arr("dst_chunk", p.dst_chunk);
    std::vector<uint32_t> sst, dst, ein, eout, esc, edc;
    for (auto s : ls.stride) sst.push_back((uint32_t)s);
    for (auto s : ld.stride) dst.push_back((uint32_t)s);
    for (size_t k = 0; k < p.ent_off.size(); ++k) {
        ein.push_back(p.ent_off[k] & 0xFFFF);
        eout.push_back(p.ent_off[k] >> 16);
        esc.push_back(p.ent_sc[k]);
        edc.push_back(p.ent_dc[k]);
    }
    arr("src_stride", sst);
    arr("dst_stride", dst);
    arr("ent_in", ein);
    arr("ent_out", eout);
    arr("ent_sc", esc);
    arr("ent_dc", edc);
    o += "}";
    return o;
}

}  // namespace adha
