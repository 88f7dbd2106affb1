// remap_plan.cpp -- compiles a (src layout, dst layout) pair into the tiled
// kernel's plan: unit size, components, tile records T_k,
// pipeline stages and the per-lane permutation table (remap_plan.h).
//
// Everything here is N-independent; adha_remap picks T_k for the call and fills
// the N-dependent region bases (adha.h "layout descriptor") into the parameters.
#include "remap_plan.h"

#include <algorithm>
#include <array>
#include <cstdlib>
#include <climits>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <map>
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

namespace {
struct Unit {
    uint32_t in, out;   // local unit offsets inside period 0 of the src / dst chunk
    uint8_t sc, dc;     // kernel cluster slots
};

// Order the 32*W units of one period into W instructions of 32 lanes.  g = 4: every
// instruction is a perfect matching of src banks to dst banks.  Returns false if the
// decomposition failed (then destination order is used).
bool matched_order(const std::vector<Unit>& units, std::vector<uint32_t>& order) {
    std::vector<uint32_t> bucket[32][32];
    uint32_t cnt[32][32] = {};
    for (uint32_t u = 0; u < units.size(); ++u) {
        const int bi = units[u].in % 32, bo = units[u].out % 32;
        bucket[bi][bo].push_back(u);
        ++cnt[bi][bo];
    }
    while (order.size() < units.size()) {
        int match_r[32];
        std::fill(match_r, match_r + 32, -1);
        for (int u = 0; u < 32; ++u) {
            bool seen[32] = {};
            if (!augment(u, cnt, match_r, seen)) return false;
        }
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
    return true;
}
}  // namespace

static uint8_t log2u(uint32_t b) {
    uint8_t l = 0;
    while ((1u << l) < b) ++l;
    return l;
}

static FieldDesc field_desc(const RemapPlan& P, const Layout& ls, const Layout& ld, int f) {
    FieldDesc d;
    d.sc = (uint8_t)P.src_slot[ls.cluster[f]];
    d.dc = (uint8_t)P.dst_slot[ld.cluster[f]];
    d.sbl = log2u(ls.block[ls.cluster[f]]);
    d.dbl = log2u(ld.block[ld.cluster[f]]);
    d.soff = ls.offset[f];
    d.doff = ld.offset[f];
    d.width = ls.width[f];
    return d;
}

// Reorder a byte group's slots: source word m moves to slot ps[m], output word o to slot po[o];
// the PRMT selectors are re-encoded for the new source slots.
static void permute_group(ByteGroup& g, const int ps[4], const int po[4]) {
    ByteGroup h = g;
    for (int m = 0; m < g.n_src; ++m) {
        h.src_off[ps[m]] = g.src_off[m];
        h.src_sc[ps[m]] = g.src_sc[m];
    }
    int inv[4] = {0, 1, 2, 3};
    for (int m = 0; m < g.n_src; ++m) inv[m] = ps[m];
    for (int o = 0; o < g.n_out; ++o) {
        // decode (source slot, byte) of each output byte, then re-encode with the new slots
        uint32_t s0 = 0, s1 = 0, s2 = 0;
        for (uint32_t j = 0; j < 4; ++j) {
            const uint32_t c = (g.sel[o][2] >> (4 * j)) & 7;
            uint32_t m, by;
            if (c < 4) {
                const uint32_t a = (g.sel[o][0] >> (4 * j)) & 7;
                m = a < 4 ? 0 : 1;
                by = a & 3;
            } else {
                const uint32_t b = (g.sel[o][1] >> (4 * j)) & 7;
                m = b < 4 ? 2 : 3;
                by = b & 3;
            }
            m = (uint32_t)inv[m];
            s0 |= (m == 0 ? by : m == 1 ? 4 + by : 0) << (4 * j);
            s1 |= (m == 2 ? by : m == 3 ? 4 + by : 0) << (4 * j);
            s2 |= (m < 2 ? j : 4 + j) << (4 * j);
        }
        h.out_off[po[o]] = g.out_off[o];
        h.out_dc[po[o]] = g.out_dc[o];
        h.sel[po[o]][0] = (uint16_t)s0;
        h.sel[po[o]][1] = (uint16_t)s1;
        h.sel[po[o]][2] = (uint16_t)s2;
    }
    g = h;
}

uint32_t call_tile(const RemapPlan& p, int k, int64_t n, int n_sm) {
    const uint32_t T = p.comps[k].T_max;
    const int64_t qt = p.tile_quantum;              // 32 records (a period), 128 in byte-group mode
    if (n_sm > 0 && n < (int64_t)T * n_sm) {
        int64_t t = (n + n_sm - 1) / n_sm;
        t = (t + qt - 1) / qt * qt;
        return (uint32_t)std::max<int64_t>(qt, std::min<int64_t>(t, T));
    }
    // Balance the last round: among T_max*3/4 .. T_max (multiples of the quantum) pick the tile
    // size that minimises rounds * T (rounds = ceil(tiles / SMs)), the critical-path records per CTA.
    const char* e = std::getenv("ADHA_BALANCE");
    if (n_sm <= 0 || (e && *e == '0') || p.comps.size() != 1) return T;
    uint32_t best = T;
    int64_t best_cost = INT64_MAX;
    for (int64_t t = T; t >= std::max<int64_t>(qt, (int64_t)T * 3 / 4); t -= qt) {
        const int64_t tiles = n / t, rounds = (tiles + n_sm - 1) / n_sm;
        const int64_t cost = rounds * t;
        if (cost < best_cost) { best_cost = cost; best = (uint32_t)t; }
    }
    return best;
}

RemapPlan compile_plan(const Layout& ls, const Layout& ld, bool merge) {
    static std::atomic<uint64_t> next_uid{1};
    RemapPlan P;
    P.uid = next_uid++;
    P.merged = merge;
    const int F = ls.n_fields;
    const int Cs = ls.n_clusters(), Cd = ld.n_clusters();

    // unit g: largest of 4, 2, 1 dividing every width and every offset in both layouts
    uint64_t gall = 0;
    for (int f = 0; f < F; ++f) {
        gall = std::gcd(gall, (uint64_t)ls.width[f]);
        gall = std::gcd(gall, (uint64_t)ls.offset[f] * ls.block[ls.cluster[f]]);
        gall = std::gcd(gall, (uint64_t)ld.offset[f] * ld.block[ld.cluster[f]]);
    }
    for (int c = 0; c < Cs; ++c) gall = std::gcd(gall, ls.stride[c]);
    for (int c = 0; c < Cd; ++c) gall = std::gcd(gall, ld.stride[c]);
    P.unit = (gall % 4 == 0) ? 4 : (gall % 2 == 0) ? 2 : 1;
    const uint32_t g = P.unit;

    auto naive = [&](const std::string& why) {
        P.tiled = false;
        P.why_naive = why;
        return P;
    };
    if (F > MAXF) return naive("more than " + std::to_string(MAXF) + " fields");
    if (Cs > MAXC || Cd > MAXC) return naive("more than " + std::to_string(MAXC) + " clusters");

    // components: union-find over src clusters [0, Cs) and dst clusters [Cs, Cs + Cd)
    std::vector<int> parent(Cs + Cd);
    std::iota(parent.begin(), parent.end(), 0);
    auto find = [&](int x) {
        while (parent[x] != x) x = parent[x] = parent[parent[x]];
        return x;
    };
    for (int f = 0; f < F; ++f) {
        int a = find(ls.cluster[f]), b = find(Cs + ld.cluster[f]);
        if (a != b) parent[std::max(a, b)] = std::min(a, b);
    }
    // merged plan (small and mid-size remaps): ONE component over all clusters, so a tile carries
    // whole records and a CTA meets a handful of tiles instead of one short tile per component
    if (merge)
        for (int x = 0; x < Cs + Cd; ++x) parent[x] = 0;
    std::map<int, int> comp_of_root;   // ordered by root = min src cluster of the component
    for (int c = 0; c < Cs; ++c) {
        int r = find(c);
        if (!comp_of_root.count(r)) {
            int k = (int)comp_of_root.size();
            comp_of_root[r] = k;
            P.comps.emplace_back();
        }
        P.comps[comp_of_root[r]].src_clusters.push_back(c);
    }
    for (int c = 0; c < Cd; ++c) P.comps[comp_of_root.at(find(Cs + c))].dst_clusters.push_back(c);
    for (int f = 0; f < F; ++f) {
        auto& K = P.comps[comp_of_root.at(find(ls.cluster[f]))];
        K.fields.push_back(f);
        K.R += ls.width[f];
    }
    if ((int)P.comps.size() > MAXK) return naive("more than " + std::to_string(MAXK) + " components");

    // kernel cluster numbering: clusters grouped by component
    P.src_slot.assign(Cs, -1);
    P.dst_slot.assign(Cd, -1);
    for (auto& K : P.comps) {
        for (int c : K.src_clusters) { P.src_slot[c] = (int)P.src_order.size(); P.src_order.push_back(c); }
        for (int c : K.dst_clusters) { P.dst_slot[c] = (int)P.dst_order.size(); P.dst_order.push_back(c); }
        for (int c : K.src_clusters) K.Rs += (uint32_t)ls.stride[c];
        for (int c : K.dst_clusters) {
            K.Rd += (uint32_t)ld.stride[c];
            const bool padded = ld.stride[c] != ld.payload(c);
            K.zero_out = K.zero_out || padded;
            K.tail_zero = K.tail_zero || padded || ld.block[c] > 1;
        }
        // identity: one cluster on each side with byte-identical records and no padding to zero
        if (K.src_clusters.size() == 1 && K.dst_clusters.size() == 1) {
            const int cs = K.src_clusters[0], cd = K.dst_clusters[0];
            bool same = ls.members[cs] == ld.members[cd] && ls.block[cs] == ld.block[cd] &&
                        ls.stride[cs] == ld.stride[cd] && ld.stride[cd] == ld.payload(cd);
            for (int f : ls.members[cs]) same = same && ls.offset[f] == ld.offset[f];
            K.identity = same;
        }
    }

    // unit mode: the consumers copy the entry table (off | sc | dc) and the cluster descriptors
    // into shared memory once per CTA, so a component switch reads its entries with LDS instead of
    // lane-divergent loads (the table itself comes from its device copy, remap.cu device_table)
    {
        uint64_t w = 0;
        for (auto& K : P.comps)
            if (!K.identity) w += K.R / g;
        const uint64_t n4 = (32 * w + 15) / 16 * 16;   // the kernel's copy rounds to 16 entries
        // (beyond the largest table class unit mode is impossible anyway: byte groups or naive)
        if (32 * w <= (uint64_t)CLASS_NENT[3]) P.tbl_bytes = (uint32_t)((6 * n4 + 16ull * (Cs + Cd) + 127) / 128 * 128);
    }
    // tile sizes and stages
    const uint32_t budget = 232448 - HDR_BYTES - 128 - P.tbl_bytes;   // sm_100 opt-in dynamic smem per block
    const uint32_t target = env_u32("ADHA_STAGE_BYTES", 49152);
    const uint32_t t_cap = env_u32("ADHA_TILE_CAP", 16384);
    uint32_t s_in = std::min<uint32_t>(env_u32("ADHA_STAGES", 4), MAX_S_IN);
    const uint32_t S_OUT = std::min<uint32_t>(std::max<uint32_t>(env_u32("ADHA_OUT_BUFFERS", 2), 1), S_OUT_MAX);
    auto round128 = [](uint64_t x) { return (x + 127) / 128 * 128; };
    uint64_t stage = 0;
    for (auto& K : P.comps) {
        const uint64_t Rmax = std::max(K.Rs, K.Rd);
        uint64_t T = std::max<uint64_t>(32, (target / (32ull * Rmax)) * 32);
        T = std::min<uint64_t>(T, std::max<uint32_t>(32, t_cap / 32 * 32));
        K.T_max = (uint32_t)T;
        stage = std::max<uint64_t>(stage, round128(T * Rmax));
    }
    while (s_in > 2 && (s_in + S_OUT) * stage > budget) --s_in;
    if ((s_in + S_OUT) * stage > budget || stage > STAGE_MAX) {
        // shrink the largest tiles until four buffers fit and a tile is at most STAGE_MAX bytes
        const uint64_t cap = std::min<uint64_t>(budget / (s_in + S_OUT) / 128 * 128, STAGE_MAX);
        stage = 0;
        for (auto& K : P.comps) {
            const uint64_t Rmax = std::max(K.Rs, K.Rd);
            uint64_t T = (cap / Rmax) / 32 * 32;
            if (T < 32) return naive("a 32-record tile does not fit in shared memory");
            K.T_max = (uint32_t)std::min<uint64_t>(K.T_max, T);
            stage = std::max<uint64_t>(stage, round128((uint64_t)K.T_max * Rmax));
        }
    }
    P.s_in = s_in;
    P.s_out = S_OUT;
    P.stage_bytes = (uint32_t)stage;
    P.smem_bytes = HDR_BYTES + 128 + (s_in + S_OUT) * P.stage_bytes + P.tbl_bytes;

    // ---- byte-group mode for unit sizes below 4 bytes (see ByteGroup in remap_plan.h)
    const char* bg_env = std::getenv("ADHA_BYTE_GROUPS");
    if (g < 4 && !(bg_env && *bg_env == '0')) {
        struct OW {
            uint16_t out;
            uint8_t dc;
            std::pair<int, uint32_t> src[4];   // (src cluster slot, aligned word offset) per output byte
            uint8_t byte[4];
            std::vector<std::pair<int, uint32_t>> set;   // distinct source words, sorted
        };
        std::vector<ByteGroup> groups;
        std::vector<uint32_t> base(P.comps.size()), count(P.comps.size());
        // chunk stagger (bytes) of every kernel cluster slot: 32 * (index in its component); only its
        // value mod 128 matters for banks because chunk sizes T*stride are multiples of 128
        std::vector<uint32_t> spad(P.src_order.size()), dpad(P.dst_order.size());
        size_t max_chunks = 1;
        for (auto& K : P.comps) {
            for (size_t i = 0; i < K.src_clusters.size(); ++i) spad[P.src_slot[K.src_clusters[i]]] = 32 * i;
            for (size_t i = 0; i < K.dst_clusters.size(); ++i) dpad[P.dst_slot[K.dst_clusters[i]]] = 32 * i;
            max_chunks = std::max(max_chunks, std::max(K.src_clusters.size(), K.dst_clusters.size()));
        }
        std::vector<std::vector<ByteGroup>> cgs(P.comps.size());
        for (size_t ki = 0; ki < P.comps.size(); ++ki) {
            auto& K = P.comps[ki];
            if (K.identity) continue;
            // the output words of one 32-record period with the source word of each byte
            std::vector<OW> ows;
            for (int cd : K.dst_clusters) {
                // which (field, record, byte) lands on every byte of the chunk's 32-record period
                const uint32_t pb = 32 * (uint32_t)ld.stride[cd];
                std::vector<int> pf(pb, -1);
                std::vector<uint32_t> pr(pb, 0), pj(pb, 0);
                for (int f : ld.members[cd])
                    for (uint32_t r = 0; r < 32; ++r)
                        for (uint32_t j = 0; j < ld.width[f]; ++j) {
                            const uint64_t a = ld.local_addr(f, r) + j;
                            pf[a] = f;
                            pr[a] = r;
                            pj[a] = j;
                        }
                for (uint32_t w = 0; w < pb / 4; ++w) {
                    OW o;
                    o.out = (uint16_t)(4 * w);
                    o.dc = (uint8_t)P.dst_slot[cd];
                    bool any = false;
                    for (uint32_t j = 0; j < 4; ++j) {
                        const uint32_t B = 4 * w + j;
                        const int f = pf[B];
                        if (f < 0) {          // padding byte: the zero source (-1), an unloaded slot
                            o.src[j] = {-1, 0};
                            o.byte[j] = 0;
                        } else {
                            any = true;
                            const int cs = ls.cluster[f];
                            const uint64_t local = ls.local_addr(f, pr[B]) + pj[B];
                            o.src[j] = {P.src_slot[cs], (uint32_t)(local & ~uint64_t(3))};
                            o.byte[j] = (uint8_t)(local & 3);
                        }
                        if (std::find(o.set.begin(), o.set.end(), o.src[j]) == o.set.end()) o.set.push_back(o.src[j]);
                    }
                    if (!any) continue;       // all padding: the pre-zeroed output buffer already holds it
                    std::sort(o.set.begin(), o.set.end());
                    ows.push_back(o);
                }
            }
            // greedy grouping: output words sorted by their first source word; a group takes up to
            // 4 output words whose source words together are at most 4 (looked for in a window)
            std::vector<uint32_t> ord(ows.size());
            std::iota(ord.begin(), ord.end(), 0u);
            std::stable_sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) { return ows[a].set < ows[b].set; });
            std::vector<char> used(ows.size(), 0);
            std::vector<ByteGroup> comp_groups;
            const size_t window = 256;
            for (size_t a = 0; a < ord.size(); ++a) {
                if (used[ord[a]]) continue;
                std::vector<uint32_t> members = {ord[a]};
                std::vector<std::pair<int, uint32_t>> uni = ows[ord[a]].set;
                used[ord[a]] = 1;
                for (size_t b = a + 1; b < ord.size() && b < a + window && members.size() < 4; ++b) {
                    const OW& c = ows[ord[b]];
                    if (used[ord[b]]) continue;
                    std::vector<std::pair<int, uint32_t>> u2 = uni;
                    for (auto& x : c.set)
                        if (std::find(u2.begin(), u2.end(), x) == u2.end()) u2.push_back(x);
                    if (u2.size() > 4) continue;
                    uni = u2;
                    members.push_back(ord[b]);
                    used[ord[b]] = 1;
                }
                ByteGroup gr;
                std::memset(&gr, 0, sizeof gr);
                // real source words first, the zero source (padding) last: slots >= n_src read as 0
                std::stable_partition(uni.begin(), uni.end(), [](const std::pair<int, uint32_t>& x) { return x.first >= 0; });
                const size_t n_real = (size_t)std::count_if(uni.begin(), uni.end(),
                                                            [](const std::pair<int, uint32_t>& x) { return x.first >= 0; });
                gr.n_src = (uint8_t)n_real;
                for (size_t m = 0; m < n_real; ++m) {
                    gr.src_sc[m] = (uint8_t)uni[m].first;
                    gr.src_off[m] = (uint16_t)uni[m].second;
                }
                gr.n_out = (uint8_t)members.size();
                for (size_t o = 0; o < members.size(); ++o) {
                    const OW& ow = ows[members[o]];
                    gr.out_off[o] = ow.out;
                    gr.out_dc[o] = ow.dc;
                    uint32_t s0 = 0, s1 = 0, s2 = 0;
                    for (uint32_t j = 0; j < 4; ++j) {
                        const uint32_t m = (uint32_t)(std::find(uni.begin(), uni.end(), ow.src[j]) - uni.begin());
                        const uint32_t by = ow.byte[j];
                        s0 |= (m == 0 ? by : m == 1 ? 4 + by : 0) << (4 * j);
                        s1 |= (m == 2 ? by : m == 3 ? 4 + by : 0) << (4 * j);
                        s2 |= (m < 2 ? j : 4 + j) << (4 * j);
                    }
                    gr.sel[o][0] = (uint16_t)s0;
                    gr.sel[o][1] = (uint16_t)s1;
                    gr.sel[o][2] = (uint16_t)s2;
                }
                comp_groups.push_back(gr);
            }
            cgs[ki] = std::move(comp_groups);
        }
        // instruction order: fill each 32-lane instruction greedily with groups whose source
        // words and output words can be put in slots (the m-th load / o-th store of all lanes)
        // whose banks are still unused in that instruction -- the slot order inside a group is
        // free, so try every permutation of it.  All lanes of an instruction are at the same
        // period q, and a word's bank moves by 8 * stride words per period, so banks are
        // checked at every phase q = 0..3 (the shift pattern repeats with period 4): clusters
        // of stride 2 (mod 4) and 0 (mod 4) in one instruction collide on odd periods otherwise.
        auto sbank = [&](const ByteGroup& x, int m, int q) {
            const uint32_t h = (8u * (uint32_t)ls.stride[P.src_order[x.src_sc[m]]]) & 31u;
            return ((spad[x.src_sc[m]] + x.src_off[m]) / 4 + q * h) % 32;
        };
        auto obank = [&](const ByteGroup& x, int o, int q) {
            const uint32_t h = (8u * (uint32_t)ld.stride[P.dst_order[x.out_dc[o]]]) & 31u;
            return ((dpad[x.out_dc[o]] + x.out_off[o]) / 4 + q * h) % 32;
        };
        // one greedy pass over the remaining groups in `cand` order: picks conflict-free groups
        // (with their slot permutations) until 32 or the candidates run out
        auto greedy = [&](const std::vector<ByteGroup>& cg, const std::vector<size_t>& cand, std::vector<size_t>& pick,
                          std::vector<std::array<int, 8>>& perms) {
            uint32_t used_s[4][4] = {}, used_o[4][4] = {};     // [slot][phase] bank masks
            for (size_t i : cand) {
                if (pick.size() == 32) break;
                const ByteGroup& gr = cg[i];
                int ps[4] = {0, 1, 2, 3}, po[4] = {0, 1, 2, 3};
                bool ok_s = false, ok_o = false;
                do {
                    bool ok = true;
                    for (int m = 0; m < gr.n_src && ok; ++m)
                        for (int q = 0; q < 4 && ok; ++q) ok = !(used_s[ps[m]][q] >> sbank(gr, m, q) & 1u);
                    if (ok) { ok_s = true; break; }
                } while (std::next_permutation(ps, ps + gr.n_src));
                if (!ok_s) continue;
                do {
                    bool ok = true;
                    for (int o = 0; o < gr.n_out && ok; ++o)
                        for (int q = 0; q < 4 && ok; ++q) ok = !(used_o[po[o]][q] >> obank(gr, o, q) & 1u);
                    if (ok) { ok_o = true; break; }
                } while (std::next_permutation(po, po + gr.n_out));
                if (!ok_o) continue;
                for (int m = 0; m < gr.n_src; ++m)
                    for (int q = 0; q < 4; ++q) used_s[ps[m]][q] |= 1u << sbank(gr, m, q);
                for (int o = 0; o < gr.n_out; ++o)
                    for (int q = 0; q < 4; ++q) used_o[po[o]][q] |= 1u << obank(gr, o, q);
                pick.push_back(i);
                perms.push_back({ps[0], ps[1], ps[2], ps[3], po[0], po[1], po[2], po[3]});
            }
        };
        // Dense packing (the fallback when the balanced tables below exceed the largest group table):
        // the largest conflict-free pick of each instruction is topped up with the next groups.
        auto pack = [&](std::vector<ByteGroup> cg, size_t ki) {
            std::vector<ByteGroup> out;
            std::vector<char> taken(cg.size(), 0);
            size_t left = cg.size();
            uint64_t rng = 0x9E3779B97F4A7C15ull ^ (uint64_t)ki;
            while (left) {
                std::vector<size_t> remaining;
                for (size_t i = 0; i < cg.size(); ++i)
                    if (!taken[i]) remaining.push_back(i);
                // natural order first, then seeded shuffles; keep the largest conflict-free pick
                std::vector<size_t> best_pick;
                std::vector<std::array<int, 8>> best_perms;
                std::vector<size_t> cand = remaining;
                for (int attempt = 0; attempt < 24 && best_pick.size() < std::min<size_t>(32, remaining.size()); ++attempt) {
                    if (attempt) {
                        for (size_t i = cand.size(); i > 1; --i) {       // Fisher-Yates with splitmix64
                            rng += 0x9E3779B97F4A7C15ull;
                            uint64_t z = rng;
                            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
                            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
                            z ^= z >> 31;
                            std::swap(cand[i - 1], cand[z % i]);
                        }
                    }
                    std::vector<size_t> pick;
                    std::vector<std::array<int, 8>> perms;
                    greedy(cg, cand, pick, perms);
                    if (pick.size() > best_pick.size()) { best_pick = pick; best_perms = perms; }
                }
                for (size_t t = 0; t < best_pick.size(); ++t) {
                    const auto& pp = best_perms[t];
                    permute_group(cg[best_pick[t]], pp.data(), pp.data() + 4);
                    taken[best_pick[t]] = 1;
                }
                for (size_t i : remaining)
                    if (best_pick.size() < 32 && !taken[i]) { best_pick.push_back(i); taken[i] = 1; }
                for (size_t i : best_pick) out.push_back(cg[i]);
                left -= best_pick.size();
            }
            return out;
        };
        // Packing into exactly I instructions: groups go one by one to the instruction (and slot
        // permutation) that adds the fewest shared-memory wavefronts over the four period phases;
        // lanes an instruction cannot use conflict-free may stay idle (empty groups).  Returns
        // the groups in instruction order and the wavefronts per 4 periods in *cost.
        auto pack_fixed = [&](std::vector<ByteGroup> cg, size_t ki, uint32_t I, uint64_t* cost) {
            uint64_t rng = 0xD1B54A32D192ED03ull ^ (uint64_t)ki ^ ((uint64_t)I << 32);
            std::vector<size_t> order(cg.size());
            std::iota(order.begin(), order.end(), size_t(0));
            std::vector<ByteGroup> best;
            uint64_t best_cost = ~uint64_t(0);
            for (int attempt = 0; attempt < 4; ++attempt) {
                if (attempt) {
                    for (size_t i = order.size(); i > 1; --i) {       // Fisher-Yates with splitmix64
                        rng += 0x9E3779B97F4A7C15ull;
                        uint64_t z = rng;
                        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
                        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
                        z ^= z >> 31;
                        std::swap(order[i - 1], order[z % i]);
                    }
                }
                // per instruction: bank counts [slot][phase][bank] and their maxima [slot][phase]
                std::vector<std::array<uint8_t, 512>> cs(I), co(I);
                std::vector<std::array<uint8_t, 16>> ms(I), mo(I);
                for (uint32_t i = 0; i < I; ++i) { cs[i].fill(0); co[i].fill(0); ms[i].fill(0); mo[i].fill(0); }
                std::vector<std::vector<ByteGroup>> lanes(I);
                bool ok = true;
                for (size_t gi : order) {
                    const ByteGroup& gr = cg[gi];
                    int bi = -1, bps[4] = {0, 1, 2, 3}, bpo[4] = {0, 1, 2, 3};
                    uint32_t bd = ~0u;
                    for (uint32_t i = 0; i < I; ++i) {
                        if (lanes[i].size() >= 32) continue;
                        uint32_t ds = ~0u, dout = ~0u;
                        int ps[4] = {0, 1, 2, 3}, po[4] = {0, 1, 2, 3}, ps_b[4] = {0, 1, 2, 3}, po_b[4] = {0, 1, 2, 3};
                        do {
                            uint32_t d = 0;
                            for (int m = 0; m < gr.n_src; ++m)
                                for (int q = 0; q < 4; ++q)
                                    d += cs[i][(ps[m] * 4 + q) * 32 + sbank(gr, m, q)] >= ms[i][ps[m] * 4 + q];
                            if (d < ds) { ds = d; std::copy(ps, ps + 4, ps_b); }
                        } while (ds && std::next_permutation(ps, ps + gr.n_src));
                        do {
                            uint32_t d = 0;
                            for (int o = 0; o < gr.n_out; ++o)
                                for (int q = 0; q < 4; ++q)
                                    d += co[i][(po[o] * 4 + q) * 32 + obank(gr, o, q)] >= mo[i][po[o] * 4 + q];
                            if (d < dout) { dout = d; std::copy(po, po + 4, po_b); }
                        } while (dout && std::next_permutation(po, po + gr.n_out));
                        // fewest added wavefronts, then the emptier instruction
                        const uint32_t key = ((ds + dout) << 8) | (uint32_t)lanes[i].size();
                        if (key < bd) {
                            bd = key;
                            bi = (int)i;
                            std::copy(ps_b, ps_b + 4, bps);
                            std::copy(po_b, po_b + 4, bpo);
                        }
                    }
                    if (bi < 0) { ok = false; break; }
                    ByteGroup h = gr;
                    permute_group(h, bps, bpo);
                    for (int m = 0; m < h.n_src; ++m)
                        for (int q = 0; q < 4; ++q) {
                            uint8_t& c = cs[bi][(m * 4 + q) * 32 + sbank(h, m, q)];
                            ms[bi][m * 4 + q] = std::max<uint8_t>(ms[bi][m * 4 + q], ++c);
                        }
                    for (int o = 0; o < h.n_out; ++o)
                        for (int q = 0; q < 4; ++q) {
                            uint8_t& c = co[bi][(o * 4 + q) * 32 + obank(h, o, q)];
                            mo[bi][o * 4 + q] = std::max<uint8_t>(mo[bi][o * 4 + q], ++c);
                        }
                    lanes[bi].push_back(h);
                }
                if (!ok) continue;
                uint64_t c = 0;
                for (uint32_t i = 0; i < I; ++i)
                    for (int x = 0; x < 16; ++x) c += ms[i][x] + mo[i][x];
                if (c < best_cost) {
                    best_cost = c;
                    best.clear();
                    ByteGroup idle;
                    std::memset(&idle, 0, sizeof idle);
                    for (uint32_t i = 0; i < I; ++i) {
                        best.insert(best.end(), lanes[i].begin(), lanes[i].end());
                        if (i + 1 < I) best.resize(best.size() + (32 - lanes[i].size()), idle);
                    }
                }
            }
            *cost = best_cost;
            return best;
        };
        {
            // per component: the instruction count with the smallest estimated busiest-warp time;
            // if the tables do not fit the largest group table (GCLASS_NG[1]), the dense packing instead
            groups.clear();
            bool fits = true;
            for (size_t ki = 0; ki < P.comps.size() && fits; ++ki) {
                base[ki] = (uint32_t)groups.size();
                count[ki] = 0;
                if (cgs[ki].empty()) continue;
                // Per tile, the kernel gives instruction i's periods to gP = NCONS*GMAX / I warp
                // slots; the busiest warp holds ceil(I*gP / NCONS) slots of P/gP periods each.
                // Estimated busiest-warp time per period: slots/gP * (wavefronts per instruction-
                // period + an issue term for the PRMT/address work), minimised over I.
                const uint32_t I_min = (uint32_t)((cgs[ki].size() + 31) / 32);
                const uint32_t S = (uint32_t)(NCONS * GCLASS_GMAX[1]);
                std::vector<ByteGroup> v;
                double vt = 1e300;
                // the busiest warp's share of one period's instructions (kernels.cuh: with
                // I <= NCONS not dividing the slots, warps take equal (instruction, period) ranges)
                auto busy = [&](uint32_t I) {
                    if (I <= (uint32_t)NCONS && S % I != 0) return (double)I / NCONS;
                    const uint32_t gP = std::max<uint32_t>(1, S / I);
                    return (double)((I * gP + NCONS - 1) / NCONS) / gP;
                };
                for (uint32_t I = I_min; I <= S; ++I) {
                    const double busiest = busy(I);
                    // same busiest-warp load with more instructions = more room for conflict-free
                    // lanes: only the largest I of each load class is tried
                    if (I < S && busy(I + 1) == busiest) continue;
                    if (busiest * 8.0 >= vt) continue;     // >= 1 load + 1 store wavefront: cannot win
                    uint64_t c = 0;
                    std::vector<ByteGroup> w = pack_fixed(cgs[ki], ki, I, &c);
                    if (w.empty() || groups.size() + w.size() > (size_t)GCLASS_NG[1]) continue;
                    const double t = busiest * ((double)c / (4.0 * I) + 6.0);
                    if (t < vt) { vt = t; v = std::move(w); }
                }
                if (v.empty()) { fits = false; break; }
                count[ki] = (uint32_t)v.size();
                groups.insert(groups.end(), v.begin(), v.end());
            }
            if (!fits || groups.size() > (size_t)GCLASS_NG[1]) {
                groups.clear();
                for (size_t ki = 0; ki < P.comps.size(); ++ki) {
                    base[ki] = (uint32_t)groups.size();
                    std::vector<ByteGroup> v = pack(cgs[ki], ki);
                    count[ki] = (uint32_t)v.size();
                    groups.insert(groups.end(), v.begin(), v.end());
                }
            }
        }
        // class: all groups fit, and every component's slots fit GMAX per warp
        int gcls = -1;
        for (int c = 0; c < 2 && gcls < 0; ++c) {
            if (groups.size() > (size_t)GCLASS_NG[c]) continue;
            bool fits = true;
            for (size_t ki = 0; ki < P.comps.size(); ++ki) {
                const uint32_t I = (count[ki] + 31) / 32;
                if (!I) continue;
                const uint32_t Pq = std::max<uint32_t>(1, (uint32_t)(NCONS * GCLASS_GMAX[c]) / I);
                fits = fits && (I * Pq + NCONS - 1) / NCONS <= (uint32_t)GCLASS_GMAX[c];
            }
            if (fits) gcls = c;
        }
        if (gcls >= 0) {
            // chunk starts at multiples of 128 bytes keep each word's bank a function of its
            // period-0 offset: tiles of 128-record multiples in byte-group mode
            P.tile_quantum = 128;
            uint64_t stage2 = 0;
            for (auto& K : P.comps) {
                K.T_max = std::max<uint32_t>(128, K.T_max / 128 * 128);
                stage2 = std::max<uint64_t>(stage2, (uint64_t)K.T_max * std::max(K.Rs, K.Rd) + 32 * max_chunks);
            }
            stage2 = (stage2 + 127) / 128 * 128;
            // shared-memory copy of the groups in use and of the cluster descriptors (see unit mode)
            const uint32_t bg_tbl = (uint32_t)((((uint64_t)sizeof(ByteGroup) * groups.size() + 15) / 16 * 16 +
                                                16ull * (Cs + Cd) + 127) / 128 * 128);
            if ((P.s_in + P.s_out) * stage2 + bg_tbl > budget + P.tbl_bytes) gcls = -1;
            else {
                P.stage_bytes = (uint32_t)stage2;
                P.tbl_bytes = bg_tbl;
                P.smem_bytes = HDR_BYTES + 128 + (P.s_in + P.s_out) * P.stage_bytes + P.tbl_bytes;
            }
        }
        if (gcls >= 0) {
            for (size_t ki = 0; ki < P.comps.size(); ++ki) {
                P.comps[ki].instr_base = base[ki];
                P.comps[ki].n_instr = count[ki];
                P.comps[ki].n_groups = count[ki];
            }
            const int ng = GCLASS_NG[gcls];
            const size_t bytes = sizeof(ByteGroup) * ng + sizeof(FieldDesc) * MAXF;
            P.table.assign((bytes + 3) / 4, 0u);
            uint8_t* img = reinterpret_cast<uint8_t*>(P.table.data());
            std::memcpy(img, groups.data(), groups.size() * sizeof(ByteGroup));
            FieldDesc* fd = reinterpret_cast<FieldDesc*>(img + sizeof(ByteGroup) * ng);
            int fi = 0;
            for (auto& K : P.comps)
                for (int f : K.fields) fd[fi++] = field_desc(P, ls, ld, f);
            P.byte_groups = true;
            P.n_groups_total = (uint32_t)groups.size();
            P.group_class = gcls;
            P.matched = false;
            P.tiled = true;
            return P;
        }
    }

    // instructions: 32 * W_k units per non-identity component
    uint64_t total_w = 0, max_w = 0;
    for (auto& K : P.comps) {
        if (K.identity) continue;
        total_w += K.R / g;
        max_w = std::max<uint64_t>(max_w, K.R / g);
    }
    int cls = -1;
    for (int c = 0; c < 4; ++c)
        if (32 * total_w <= (uint64_t)CLASS_NENT[c] && max_w <= (uint64_t)NCONS * CLASS_EMAX[c]) { cls = c; break; }
    if (cls < 0) return naive("record of " + std::to_string(total_w) + " units exceeds the instruction table");
    P.table_class = cls;

    P.matched = (g == 4);
    uint32_t instr = 0;
    for (auto& K : P.comps) {
        K.instr_base = instr;
        K.n_instr = 0;
        if (K.identity) continue;
        std::vector<Unit> units;
        for (uint32_t r = 0; r < 32; ++r)
            for (int f : K.fields) {
                const int cs = ls.cluster[f], cd = ld.cluster[f];
                for (uint32_t j = 0; j < ls.width[f] / g; ++j) {
                    const uint64_t ib = ls.local_addr(f, r) + j * g;
                    const uint64_t ob = ld.local_addr(f, r) + j * g;
                    units.push_back({(uint32_t)(ib / g), (uint32_t)(ob / g), (uint8_t)P.src_slot[cs],
                                     (uint8_t)P.dst_slot[cd]});
                }
            }
        std::vector<uint32_t> order;
        if (g == 4 && !matched_order(units, order)) {
            P.matched = false;
            order.clear();
        }
        if (order.empty()) {
            // destination order (by dst cluster, then unit): lanes write consecutive units
            order.resize(units.size());
            std::iota(order.begin(), order.end(), 0u);
            std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
                if (units[a].dc != units[b].dc) return units[a].dc < units[b].dc;
                return units[a].out < units[b].out;
            });
        }
        for (uint32_t idx : order) {
            const Unit& u = units[idx];
            P.ent_off.push_back(u.in | (u.out << 16));
            P.ent_sc.push_back(u.sc);
            P.ent_dc.push_back(u.dc);
        }
        K.n_instr = K.R / g;
        instr += K.n_instr;
    }

    // table image of EntryTable<NENT> (uploaded to device memory once per plan and device, remap.cu
    // device_table): off[NENT] | sc[NENT] | dc[NENT] | fields[MAXF]
    const uint32_t nent = (uint32_t)CLASS_NENT[cls];
    const size_t bytes = 6ull * nent + sizeof(FieldDesc) * MAXF;
    P.table.assign((bytes + 3) / 4, 0u);
    uint8_t* img = reinterpret_cast<uint8_t*>(P.table.data());
    std::memcpy(img, P.ent_off.data(), P.ent_off.size() * 4);
    std::memcpy(img + 4 * nent, P.ent_sc.data(), P.ent_sc.size());
    std::memcpy(img + 5 * nent, P.ent_dc.data(), P.ent_dc.size());
    FieldDesc* fd = reinterpret_cast<FieldDesc*>(img + 6 * nent);
    int fi = 0;
    for (auto& K : P.comps)
        for (int f : K.fields) fd[fi++] = field_desc(P, ls, ld, f);
    P.tiled = true;
    return P;
}

std::string describe_plan(const RemapPlan& p, const Layout& ls, const Layout& ld) {
    std::string o = "{";
    o += "\"tiled\":" + std::string(p.tiled ? "true" : "false");
    o += ",\"why_naive\":" + json::quote(p.why_naive);
    o += ",\"unit\":" + std::to_string(p.unit);
    o += ",\"s_in\":" + std::to_string(p.s_in);
    o += ",\"s_out\":" + std::to_string(p.s_out);
    o += ",\"stage_bytes\":" + std::to_string(p.stage_bytes);
    o += ",\"smem_bytes\":" + std::to_string(p.smem_bytes);
    o += ",\"n_consumer_warps\":" + std::to_string(dev::NCONS);
    o += ",\"table_class\":" + std::to_string(p.table_class);
    o += ",\"table_entries\":" + std::to_string(dev::CLASS_NENT[p.table_class]);
    o += ",\"matched\":" + std::string(p.matched ? "true" : "false");
    o += ",\"byte_groups\":" + std::string(p.byte_groups ? "true" : "false");
    auto arr = [](const std::vector<uint32_t>& v) {
        std::string s = "[";
        for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
        return s + "]";
    };
    auto iarr = [](const std::vector<int>& v) {
        std::string s = "[";
        for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
        return s + "]";
    };
    o += ",\"T\":" + std::to_string(p.comps.empty() ? 0 : p.comps[0].T_max);
    o += ",\"components\":[";
    for (size_t k = 0; k < p.comps.size(); ++k) {
        const auto& K = p.comps[k];
        o += (k ? ",{" : "{");
        o += "\"src_clusters\":" + iarr(K.src_clusters) + ",\"dst_clusters\":" + iarr(K.dst_clusters) +
             ",\"fields\":" + iarr(K.fields) + ",\"R\":" + std::to_string(K.R) + ",\"Rs\":" + std::to_string(K.Rs) +
             ",\"Rd\":" + std::to_string(K.Rd) + ",\"zero_out\":" + (K.zero_out ? "true" : "false") +
             ",\"T\":" + std::to_string(K.T_max) +
             ",\"identity\":" + (K.identity ? "true" : "false") + ",\"instr_base\":" + std::to_string(K.instr_base) +
             ",\"n_instr\":" + std::to_string(K.n_instr) + "}";
    }
    o += "]";
    o += ",\"src_order\":" + iarr(p.src_order) + ",\"dst_order\":" + iarr(p.dst_order);
    std::vector<uint32_t> sst, dst, ein, eout, esc, edc;
    for (auto s : ls.stride) sst.push_back((uint32_t)s);
    for (auto s : ld.stride) dst.push_back((uint32_t)s);
    for (size_t k = 0; k < p.ent_off.size(); ++k) {
        ein.push_back(p.ent_off[k] & 0xFFFF);
        eout.push_back(p.ent_off[k] >> 16);
        esc.push_back(p.ent_sc[k]);
        edc.push_back(p.ent_dc[k]);
    }
    o += ",\"src_stride\":" + arr(sst) + ",\"dst_stride\":" + arr(dst);
    o += ",\"ent_in\":" + arr(ein) + ",\"ent_out\":" + arr(eout) + ",\"ent_sc\":" + arr(esc) + ",\"ent_dc\":" + arr(edc);
    if (p.byte_groups) {
        // [n_out, n_src, out_off x4, out_dc x4, src_off x4, src_sc x4, sel x12] per group
        const int ng = dev::GCLASS_NG[p.group_class];
        const dev::ByteGroup* gr = reinterpret_cast<const dev::ByteGroup*>(p.table.data());
        uint32_t total = 0;
        for (auto& K : p.comps) total = std::max(total, K.instr_base + K.n_groups);
        o += ",\"group_class_size\":" + std::to_string(ng) + ",\"groups\":[";
        for (uint32_t i = 0; i < total; ++i) {
            const dev::ByteGroup& g = gr[i];
            std::vector<uint32_t> v = {g.n_out, g.n_src};
            for (int m = 0; m < 4; ++m) v.push_back(g.out_off[m]);
            for (int m = 0; m < 4; ++m) v.push_back(g.out_dc[m]);
            for (int m = 0; m < 4; ++m) v.push_back(g.src_off[m]);
            for (int m = 0; m < 4; ++m) v.push_back(g.src_sc[m]);
            for (int m = 0; m < 4; ++m)
                for (int t = 0; t < 3; ++t) v.push_back(g.sel[m][t]);
            o += (i ? "," : "") + arr(v);
        }
        o += "]";
    }
    o += "}";
    return o;
}

}  // namespace adha
