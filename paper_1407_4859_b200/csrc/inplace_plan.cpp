// inplace_plan.cpp -- host plan of the in-place remap (adha.h
// adha_inplace_plan_create).  See inplace_plan.h for the three steps.
//
// The remap itself is the one of adha_remap:
//     dst[addr_Ld(f, i) .. + w_f) = src[addr_Ls(f, i) .. + w_f)
// with dst and src the same buffer.  This file computes, once per (Ls, Ld, N), which S-byte
// slot goes where (a permutation of slot indices), its cycles, and the workspace layout.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>

#include "inplace_plan.h"

namespace adha {

namespace {

uint32_t pow2_unit(const Layout& l) {
    uint32_t u = 16;
    for (int32_t f = 0; f < l.n_fields; ++f)
        while (l.width[f] % u) u >>= 1;
    return u;
}

bool same_members(const Layout& a, int32_t ca, const Layout& b, int32_t cb) {
    return a.members[ca] == b.members[cb];
}

// block of a cluster record containing byte offset o (blocks sorted by offset, tiling the record)
const IpBlock& block_at(const std::vector<IpBlock>& blocks, uint32_t o) {
    size_t lo = 0, hi = blocks.size() - 1;
    while (lo < hi) {   // last block with offset <= o
        const size_t mid = (lo + hi + 1) / 2;
        if (blocks[mid].off <= o) lo = mid; else hi = mid - 1;
    }
    return blocks[lo];
}

// Padding between field blocks of a field-blocked tile in shared memory (atoms per field): chosen
// per cluster by simulating the bank conflicts of the field-blocked -> record-major gather
// (ip_gather in inplace.cu: thread v builds output vector v, atoms (r, jc) with 4v + j = r*RA + jc,
// read from bo(jc) + r * a(jc)); candidates are multiples of 16 bytes (the tile is staged with
// 16-byte shared-memory stores) up to 64 bytes per field block.
uint32_t choose_padf(const std::vector<IpBlock>& blocks, uint64_t stride, uint32_t T, uint32_t atom) {
    const uint32_t RA = (uint32_t)(stride / atom);
    const uint32_t APV = 16 / atom;
    const uint64_t natoms = (uint64_t)T * RA;
    std::vector<uint32_t> col(RA), a(RA), fidx(RA);
    uint32_t fi = 0;
    for (const IpBlock& b : blocks) {
        for (uint32_t k = 0; k < b.width / atom; ++k) {
            const uint32_t j = b.off / atom + k;
            col[j] = b.off / atom;
            a[j] = b.width / atom;
            fidx[j] = fi;
        }
        ++fi;
    }
    uint32_t best = 0;
    uint64_t best_cost = ~0ull;
    for (uint32_t padf = 0; padf * atom <= 64; padf += 16 / atom) {
        uint64_t cost = 0;
        for (uint64_t w = 0; w < 8 && (w * 32 + 31) * APV < natoms; ++w) {
            for (uint32_t j = 0; j < APV; ++j) {
                uint32_t words[32];
                int nw = 0;
                uint32_t per_bank[32] = {0};
                for (uint32_t L = 0; L < 32; ++L) {
                    const uint64_t o = (w * 32 + L) * APV + j;
                    const uint32_t r = (uint32_t)(o / RA), jc = (uint32_t)(o % RA);
                    const uint64_t at = (uint64_t)T * col[jc] + (uint64_t)fidx[jc] * padf + (jc - col[jc]) + (uint64_t)r * a[jc];
                    const uint32_t word = (uint32_t)(at * atom / 4);
                    bool seen = false;
                    for (int q = 0; q < nw; ++q) seen = seen || words[q] == word;
                    if (!seen) { words[nw++] = word; ++per_bank[word % 32]; }
                }
                uint32_t mx = 0;
                for (uint32_t b = 0; b < 32; ++b) mx = std::max(mx, per_bank[b]);
                cost += mx;
            }
        }
        if (cost < best_cost) { best_cost = cost; best = padf; }
    }
    return best;
}

uint64_t tile_smem(uint32_t T, uint64_t stride, size_t n_fields, uint32_t atom, uint32_t padf) {
    // staged tile plus its padding: one atom (<= 4 bytes) per record row in record-major form,
    // padf atoms per field block in field-blocked form
    return ((uint64_t)T * stride + std::max<uint64_t>(4ull * T, (uint64_t)n_fields * padf * atom) + 15) & ~15ull;
}

uint64_t table_smem(uint64_t stride, uint32_t atom) { return stride / atom * sizeof(IpCol); }

constexpr uint32_t MAX_PADF_BYTES = 64;

uint64_t smem_need(uint32_t T, uint64_t stride, size_t n_fields, uint32_t atom) {
    // the kernel packs a padded atom index in 17 bits (field-blocked -> record-major table)
    const uint64_t pad_atoms = std::max<uint64_t>(4ull * T, (uint64_t)n_fields * MAX_PADF_BYTES) / atom;
    if ((uint64_t)T * stride / atom + pad_atoms >= (1u << 17)) return ~0ull;
    return tile_smem(T, stride, n_fields, atom, MAX_PADF_BYTES / atom) + table_smem(stride, atom);
}

uint32_t magic(uint32_t d) {   // ceil(2^32 / d); 0 encodes d == 1
    return d <= 1 ? 0u : (uint32_t)(((1ull << 32) + d - 1) / d);
}

#ifndef IP_PIECE_TARGET_BYTES
#define IP_PIECE_TARGET_BYTES 16384
#endif
#ifndef IP_GROUP_MAX_TILE
#define IP_GROUP_MAX_TILE 4096
#endif
constexpr uint64_t IP_PIECE_TARGET = IP_PIECE_TARGET_BYTES;   // bytes: small tiles are grouped up to this
constexpr uint64_t IP_GROUP_TILE = IP_GROUP_MAX_TILE;         // bytes: only tiles this small are grouped
constexpr uint64_t IP_TILE_PREF = 32768;      // bytes: preferred largest rewritten tile

// column table of a cluster record in atoms (word atoms when u % 4 == 0, else bytes); returns the
// shared memory of one piece (g padded tiles)
uint64_t add_cluster(const std::vector<IpBlock>& blocks, uint64_t stride, uint64_t base, uint32_t atom, uint32_t T,
                     uint64_t m, uint32_t padf, std::vector<IpPiece>& out, std::vector<IpCol>& cols) {
    const uint32_t RA = (uint32_t)(stride / atom);
    const uint64_t tile = (uint64_t)T * stride;
    const uint32_t g = tile > IP_GROUP_TILE ? 1u : (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(IP_PIECE_TARGET / tile, m));
    const uint32_t nb = (uint32_t)blocks.size();
    IpPiece pc{};
    pc.base = base;
    pc.g = g;
    pc.pieces = (m + g - 1) / g;
    pc.stride = (uint32_t)stride;
    pc.RA = RA;
    pc.col_off = (uint32_t)cols.size();
    pc.magic_RA = magic(RA);
    pc.magic_TRA = magic(T * RA);
    pc.TS = T * RA + nb * padf;
    out.push_back(pc);
    uint32_t bidx = 0;
    for (const IpBlock& b : blocks) {
        const uint32_t col = b.off / atom, a = b.width / atom;
        for (uint32_t k = 0; k < a; ++k)
            cols.push_back({col | ((bidx * padf) << 16), a, magic(a), T * col + bidx * padf + k});
        ++bidx;
    }
    // blocked: g tiles of TS atoms; record-major: g*T rows with one padding atom (4 bytes) each
    return (std::max<uint64_t>((uint64_t)g * pc.TS * atom, (uint64_t)g * T * (stride + 4)) + 15) & ~15ull;
}

constexpr uint32_t NONE_SLOT = 0xFFFFFFFFu;

// ADHA_IP_TIMING=1: host time of the plan's phases on stderr (tools/inplace_probe.py)
struct PhaseClock {
    bool on;
    std::chrono::steady_clock::time_point t;
    PhaseClock() : on(std::getenv("ADHA_IP_TIMING") && *std::getenv("ADHA_IP_TIMING") == '1'), t(std::chrono::steady_clock::now()) {}
    void lap(const char* what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[ip plan] %-28s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};
thread_local PhaseClock* g_pc = nullptr;
struct PhaseScope {
    PhaseClock pc;
    PhaseScope() { g_pc = &pc; }
    ~PhaseScope() { g_pc = nullptr; }
};
inline void lap(const char* what) { if (g_pc) g_pc->lap(what); }

unsigned plan_threads(uint64_t work) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>({(uint64_t)hw, 32, work / (1u << 16)}));
}

// f(chunk, begin, end) over [0, n) split evenly into nthr chunks, chunk i on thread i
template <typename F>
void parallel_for(unsigned nthr, uint64_t n, F&& f) {
    if (nthr <= 1) { f(0u, (uint64_t)0, n); return; }
    std::vector<std::thread> th;
    for (unsigned i = 0; i < nthr; ++i)
        th.emplace_back([&, i] { f(i, n * i / nthr, n * (i + 1) / nthr); });
    for (auto& t : th) t.join();
}

inline bool is_cut(uint32_t x) {   // pseudo-random 1-in-512 cut points along the cycles
    uint32_t h = x * 0x9E3779B1u;
    h ^= h >> 15;
    h *= 0x85EBCA77u;
    h ^= h >> 13;
    return (h & 511u) == 0;
}

// The permutation's cycles as segments of at most IP_SEG positions.  Cycles are cut at pseudo-
// random cut points (1 in 512 slots); the walk from each cut point to the next one on its cycle
// is independent of the others.  Walking is a chain of dependent random loads of P, so each host
// thread advances WALK_LANES walks in turn (that many cache misses in flight instead of one); the
// walks' positions are then placed in cut order with prefix sums, in parallel.  Cycles without a
// cut point (short ones) are walked afterwards.  Fixed points are dropped.  Entries of P are set
// to NONE_SLOT as they are placed by the cut walks.
constexpr unsigned WALK_LANES = 16;

// `cuts`: the cut points, ascending (content slots x with is_cut(x) that are not fixed points --
// fixed points are NONE_SLOT in P already and counted in p->fixed_slots by the caller).
void build_segments(uvector<uint32_t>& P, uint64_t nslot, unsigned nthr, InplacePlan* p,
                    const std::vector<uint32_t>& cuts) {
    const uint64_t nc = cuts.size();
    // walk from every cut point up to (not including) the next cut point on its cycle
    struct Walked { uint32_t ci, len; uint64_t off; };        // cut index, length, offset in pos
    struct Out { std::vector<uint32_t> pos; std::vector<Walked> w; };
    const unsigned nw = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(nthr, nc));
    std::vector<Out> outs(nw);
    std::vector<uint32_t> len(nc), next_cut(nc);
    parallel_for(nw, nc, [&](unsigned chunk, uint64_t i0, uint64_t i1) {
        Out& o = outs[chunk];
        o.pos.reserve((i1 - i0) * 600);
        o.w.reserve(i1 - i0);
        struct Lane { uint32_t ci, y; std::vector<uint32_t> buf; bool live; };
        Lane lane[WALK_LANES];
        uint64_t next = i0;
        unsigned live = 0;
        auto start = [&](Lane& L) {
            L.live = next < i1;
            if (!L.live) return;
            L.ci = (uint32_t)next++;
            L.y = cuts[L.ci];
            L.buf.clear();
            ++live;
        };
        for (auto& L : lane) { L.buf.reserve(1024); start(L); }
        while (live) {
            for (auto& L : lane) {
                if (!L.live) continue;
                L.buf.push_back(L.y);
                const uint32_t ny = P[L.y];
                P[L.y] = NONE_SLOT;                  // placed (no other walk visits this slot)
                __builtin_prefetch(&P[ny]);
                L.y = ny;
                if (is_cut(ny)) {
                    o.w.push_back({L.ci, (uint32_t)L.buf.size(), (uint64_t)o.pos.size()});
                    o.pos.insert(o.pos.end(), L.buf.begin(), L.buf.end());
                    len[L.ci] = (uint32_t)L.buf.size();
                    next_cut[L.ci] = ny;
                    --live;
                    start(L);
                }
            }
        }
    });
    lap("cut walks");
    // placement in cut order: seq offset and first segment of every walk (prefix sums)
    std::vector<uint64_t> seq_at(nc + 1, 0), seg_at(nc + 1, 0);
    for (uint64_t i = 0; i < nc; ++i) {
        seq_at[i + 1] = seq_at[i] + len[i];
        seg_at[i + 1] = seg_at[i] + (len[i] + IP_SEG - 1) / IP_SEG;
    }
    p->seq.reserve(p->content_slots + p->junk_slots);
    p->seq.resize(seq_at[nc]);
    p->segs.resize(seg_at[nc]);
    parallel_for(nw, nw, [&](unsigned, uint64_t c0, uint64_t c1) {
        for (uint64_t c = c0; c < c1; ++c)
            for (const Walked& w : outs[c].w) {
                const uint32_t* src = outs[c].pos.data() + w.off;
                std::memcpy(p->seq.data() + seq_at[w.ci], src, (size_t)w.len * 4);
                const uint32_t s0 = (uint32_t)seg_at[w.ci], start = (uint32_t)seq_at[w.ci];
                for (uint32_t a = 0, si = s0; a < w.len; a += IP_SEG, ++si)
                    p->segs[si] = {start + a, std::min<uint32_t>(IP_SEG, w.len - a), a ? si - 1 : 0u, 0};
            }
    });
    // the last slot of walk i precedes the first slot of the walk starting at next_cut[i]
    // (after the placement above: the first segment of that walk must exist before its pred is set)
    parallel_for(nw, nc, [&](unsigned, uint64_t i0, uint64_t i1) {
        for (uint64_t i = i0; i < i1; ++i) {
            const uint64_t nxt = (uint64_t)(std::lower_bound(cuts.begin(), cuts.end(), next_cut[i]) - cuts.begin());
            p->segs[seg_at[nxt]].pred = (uint32_t)(seg_at[i + 1] - 1);
        }
    });
    outs.clear();
    lap("placement");
    p->cycles = 0;   // cut walks do not count cycles; the uncut ones below do
    // Cycles with no cut point (shorter ones): the slot with the smallest index leads its cycle.
    // Every thread tests the unplaced slots of its range -- a walk that meets a smaller index
    // stops: not the leader -- and walks the cycles it leads into a local list; P is only read
    // here and the lists are concatenated in range order afterwards.
    struct Cyc { std::vector<uint32_t> pos, len; };
    std::vector<Cyc> cyc(nthr);
    parallel_for(nthr, nslot, [&](unsigned chunk, uint64_t x0, uint64_t x1) {
        Cyc& c = cyc[chunk];
        for (uint64_t x = x0; x < x1; ++x) {
            if (P[x] == NONE_SLOT) continue;
            uint32_t y = P[x];
            while (y != (uint32_t)x && y > (uint32_t)x) y = P[y];
            if (y != (uint32_t)x) continue;          // a smaller slot on the cycle leads it
            const size_t at = c.pos.size();
            y = (uint32_t)x;
            do {
                c.pos.push_back(y);
                y = P[y];
            } while (y != (uint32_t)x);
            c.len.push_back((uint32_t)(c.pos.size() - at));
        }
    });
    for (const Cyc& c : cyc) {
        size_t off = 0;
        for (uint32_t L : c.len) {
            const uint32_t start = (uint32_t)p->seq.size();
            p->seq.insert(p->seq.end(), c.pos.begin() + off, c.pos.begin() + off + L);
            off += L;
            const uint32_t first = (uint32_t)p->segs.size();
            const uint32_t ns = (L + IP_SEG - 1) / IP_SEG;
            for (uint32_t s = 0; s < ns; ++s) {
                const uint32_t a = start + s * IP_SEG;
                p->segs.push_back({a, std::min<uint32_t>(IP_SEG, start + L - a), s == 0 ? first + ns - 1 : first + s - 1, 0});
            }
            ++p->cycles;
        }
    }
    lap("uncut cycles");
    // (P is not consumed by the uncut pass; the caller drops it)
}

// ADHA_IP_VERIFY=1 (tests): the segments against the permutation they were built from -- every
// moved slot once, consecutive positions of a segment consecutive on the cycle, and every
// segment's predecessor ending on the slot whose content its first position receives.
std::string verify_segments(const uvector<uint32_t>& P0, const InplacePlan& p) {
    std::vector<uint8_t> seen(P0.size(), 0);
    for (uint32_t x : p.seq) {
        if (x >= P0.size() || seen[x]) return "slot listed twice or out of range";
        seen[x] = 1;
    }
    for (uint64_t x = 0; x < P0.size(); ++x)
        if (P0[x] != NONE_SLOT && P0[x] != (uint32_t)x && !seen[x]) return "moved slot missing from the segments";
    for (const IpSeg& sg : p.segs) {
        if (sg.len < 1 || sg.len > IP_SEG || (uint64_t)sg.start + sg.len > p.seq.size()) return "segment bounds";
        for (uint32_t k = 0; k + 1 < sg.len; ++k)
            if (P0[p.seq[sg.start + k]] != p.seq[sg.start + k + 1]) return "segment not along its cycle";
        const IpSeg& pr = p.segs.at(sg.pred);
        if (P0[p.seq[pr.start + pr.len - 1]] != p.seq[sg.start]) return "predecessor segment mismatch";
    }
    return "";
}

}  // namespace

adha_status inplace_plan_build(const Layout& ls, const Layout& ld, int64_t n, InplacePlan* p) {
    PhaseScope phase_scope;
    if (n < 0) return fail(ADHA_ERR_INVALID_ARG, "n_records < 0");
    if (ls.n_fields != ld.n_fields) return fail(ADHA_ERR_LAYOUT_MISMATCH, "layouts differ in field count");
    for (int32_t f = 0; f < ls.n_fields; ++f)
        if (ls.width[f] != ld.width[f])
            return fail(ADHA_ERR_LAYOUT_MISMATCH, "field " + std::to_string(f) + " differs in width");
    for (const Layout* l : {&ls, &ld}) {
        if (l->aligned) return fail(ADHA_ERR_UNSUPPORTED, "in-place remap: packed layouts only (no alignment padding)");
        for (uint32_t b : l->block)
            if (b != 1) return fail(ADHA_ERR_UNSUPPORTED, "in-place remap: unblocked layouts only (no AoSoA)");
    }
    p->ls = ls;
    p->ld = ld;
    p->n = n;
    if (!ls.region_bases(n, p->bs, &p->bytes_s) || !ld.region_bases(n, p->bd, &p->bytes_d))
        return fail(ADHA_ERR_TOO_LARGE, "N * record bytes overflows");
    const uint32_t u = pow2_unit(ls);
    p->u = u;
    const uint32_t atom = u % 4 == 0 ? 4 : 1;

    // Small buffers: remap out of place into the workspace and copy back (two launches, a few
    // microseconds) instead of the tile / cycle passes, whose fixed costs dominate there.
    {
        const char* e = std::getenv("ADHA_INPLACE_STAGED_BYTES");
        const uint64_t lim = e && *e ? std::strtoull(e, nullptr, 10) : IP_STAGED_BYTES;
        p->staged = lim > 0 && std::max(p->bytes_s, p->bytes_d) <= lim;
        p->pre.clear(); p->post.clear(); p->cols.clear(); p->seq.clear(); p->segs.clear(); p->tail_fields.clear();
        p->content_slots = p->moved_slots = p->fixed_slots = p->junk_slots = p->cycles = 0;
        if (p->staged) {
            p->S = p->T = 0;
            p->m = 0;
            p->tail = 0;
            p->ws_pieces = p->ws_cols = p->ws_tailf = p->ws_seq = p->ws_segs = p->ws_save = p->ws_tail = 0;
            p->ws_stage = 0;
            p->ws_bytes = std::max<uint64_t>(align256(p->bytes_d), 256);
            p->uploaded = nullptr;
            p->uploaded_device = -1;
            return ADHA_OK;
        }
    }

    // clusters kept as raw slots: same member set in both layouts
    const int32_t Cs = ls.n_clusters(), Cd = ld.n_clusters();
    std::vector<int32_t> twin_s(Cs, -1), twin_d(Cd, -1);
    for (int32_t c = 0; c < Cs; ++c) {
        const int32_t cd = ld.cluster[ls.members[c][0]];
        if (same_members(ls, c, ld, cd)) { twin_s[c] = cd; twin_d[cd] = c; }
    }
    // Runs: maximal sequences of fields that are consecutive in BOTH the src and the dst cluster
    // record (same cluster pair, same order).  A run is contiguous in both records, so a tile's
    // BLOCKED form -- each run's T records contiguous -- holds the same bytes for the run on both
    // sides.  A cluster made of one run is already in blocked form: no tile rewrite for it.
    std::vector<std::vector<IpBlock>> sblk(Cs), dblk(Cd);
    std::vector<int32_t> dpos(ls.n_fields);       // position of each field inside its dst cluster
    for (int32_t c = 0; c < Cd; ++c)
        for (size_t i = 0; i < ld.members[c].size(); ++i) dpos[ld.members[c][i]] = (int32_t)i;
    for (int32_t c = 0; c < Cs; ++c) {
        const auto& mem = ls.members[c];
        for (size_t i = 0; i < mem.size(); ++i) {
            const int32_t f = mem[i], cd = ld.cluster[f];
            const bool cont = i > 0 && ld.cluster[mem[i - 1]] == cd && dpos[mem[i - 1]] + 1 == dpos[f];
            if (cont) {
                sblk[c].back().width += ls.width[f];
            } else {
                sblk[c].push_back({ls.offset[f], ls.width[f], cd, ld.offset[f]});
            }
        }
    }
    for (int32_t c = 0; c < Cs; ++c)
        for (const IpBlock& b : sblk[c]) dblk[b.peer].push_back({b.peer_off, b.width, c, b.off});
    for (auto& v : dblk)
        std::sort(v.begin(), v.end(), [](const IpBlock& x, const IpBlock& y) { return x.off < y.off; });
    auto transposed_s = [&](int32_t c) { return twin_s[c] < 0 && sblk[c].size() > 1; };
    auto transposed_d = [&](int32_t c) { return twin_d[c] < 0 && dblk[c].size() > 1; };

    // slot size: the largest power of two in [256, 4096] dividing every region base whose
    // rewritten tiles stay small (<= IP_TILE_PREF bytes: several CTAs per SM hide the load
    // latency of the tile pass), else the largest whose tiles fit the shared-memory budget
    uint32_t S = 0;
    for (int pass = 0; pass < 2 && !S; ++pass) {
        for (uint32_t cand = 4096; cand >= 256; cand >>= 1) {
            bool ok = true;
            for (uint64_t b : p->bs) ok = ok && (b % cand == 0);
            for (uint64_t b : p->bd) ok = ok && (b % cand == 0);
            const uint32_t T = cand / u;
            auto fits = [&](const Layout& l, int32_t c, size_t nblocks) {
                if (pass == 0 && (uint64_t)T * l.stride[c] > IP_TILE_PREF) return false;
                return smem_need(T, l.stride[c], nblocks, atom) <= IP_MAX_PIECE;
            };
            for (int32_t c = 0; ok && c < Cs; ++c)
                if (transposed_s(c) && !fits(ls, c, sblk[c].size())) ok = false;
            for (int32_t c = 0; ok && c < Cd; ++c)
                if (transposed_d(c) && !fits(ld, c, dblk[c].size())) ok = false;
            if (ok) { S = cand; break; }
        }
    }
    if (!S) return fail(ADHA_ERR_UNSUPPORTED, "in-place remap: a cluster record is too wide for a " +
                                                  std::to_string(256 / u) + "-record tile in shared memory");
    // (region bases are 256-aligned by construction, so only the tile budget can fail)
    p->S = S;
    p->T = S / u;
    const uint32_t T = p->T;
    p->m = n / T;
    p->tail = n - p->m * (int64_t)T;
    const uint64_t m = (uint64_t)p->m;

    p->pre.clear();
    p->post.clear();
    p->cols.clear();
    p->max_tile = p->max_tab = 0;
    if (m > 0) {
        for (int32_t c = 0; c < Cs; ++c)
            if (transposed_s(c)) {
                const uint64_t sm = add_cluster(sblk[c], ls.stride[c], p->bs[c], atom, T, m, 0, p->pre, p->cols);
                p->max_tile = std::max<uint32_t>(p->max_tile, (uint32_t)sm);
                p->max_tab = std::max<uint32_t>(p->max_tab, (uint32_t)table_smem(ls.stride[c], atom));
            }
        for (int32_t c = 0; c < Cd; ++c)
            if (transposed_d(c)) {
                const uint32_t padf = choose_padf(dblk[c], ld.stride[c], T, atom);
                const uint64_t sm = add_cluster(dblk[c], ld.stride[c], p->bd[c], atom, T, m, padf, p->post, p->cols);
                p->max_tile = std::max<uint32_t>(p->max_tile, (uint32_t)sm);
                p->max_tab = std::max<uint32_t>(p->max_tab, (uint32_t)table_smem(ld.stride[c], atom));
            }
    }

    // ---- the slot permutation over U = (src body slots) u (dst body slots)
    const uint64_t total = std::max(p->bytes_s, p->bytes_d);
    const uint64_t nslot = (total + S - 1) / S;
    if (nslot >= 0xFFFFFFFFull) return fail(ADHA_ERR_TOO_LARGE, "in-place remap: more than 2^32 slots");
    constexpr uint32_t NONE = NONE_SLOT;
    uvector<uint32_t> P;
    p->seq.clear();
    p->segs.clear();
    p->content_slots = p->moved_slots = p->fixed_slots = p->junk_slots = p->cycles = 0;
    if (m > 0) {
        const unsigned nthr = plan_threads(nslot);
        P.resize(nslot);                          // uninitialised: every slot is written once below
        // Body slot ranges: src cluster c's m tiles are slots [bs/S, bs/S + m*Ks) and dst cluster
        // c's are [bd/S, bd/S + m*Kd).  The slot map below is a bijection from the src body slots
        // onto the dst body slots (every dst body slot holds one run piece of one src tile), so a
        // slot "receives content" iff it lies in a dst range -- no scattered marking pass needed.
        struct Range { uint64_t lo, hi; };
        std::vector<Range> src_r, dst_r;
        for (int32_t c = 0; c < Cs; ++c) src_r.push_back({p->bs[c] / S, p->bs[c] / S + m * (ls.stride[c] / u)});
        for (int32_t c = 0; c < Cd; ++c) dst_r.push_back({p->bd[c] / S, p->bd[c] / S + m * (ld.stride[c] / u)});
        auto by_lo = [](const Range& a, const Range& b) { return a.lo < b.lo; };
        std::sort(src_r.begin(), src_r.end(), by_lo);
        std::sort(dst_r.begin(), dst_r.end(), by_lo);
        // slots outside every src body range carry no content: NONE (gaps, the src tail)
        parallel_for(nthr, nslot, [&](unsigned, uint64_t x0, uint64_t x1) {
            uint64_t x = x0;
            for (const Range& r : src_r) {
                if (r.hi <= x) continue;
                if (r.lo >= x1) break;
                if (r.lo > x) std::fill(P.begin() + x, P.begin() + r.lo, NONE);
                x = std::max(x, r.hi);
                if (x >= x1) break;
            }
            if (x < x1) std::fill(P.begin() + x, P.begin() + x1, NONE);
        });
        lap("alloc + clear");
        // per src cluster, per unit column k: slots s0 + t*K + k (t < m) -> d0 + t*Kd (+ k when raw)
        struct Col { uint64_t s0, d0; uint32_t K, Kd, k; bool raw; };
        std::vector<Col> colv;
        for (int32_t c = 0; c < Cs; ++c) {
            const uint32_t K = (uint32_t)(ls.stride[c] / u);
            const uint64_t s0 = p->bs[c] / S;
            for (uint32_t k = 0; k < K; ++k) {
                if (twin_s[c] >= 0) {                     // raw slots of an unchanged cluster
                    colv.push_back({s0, p->bd[twin_s[c]] / S, K, K, k, true});
                    continue;
                }
                // slot k of the blocked tile: run b, slot q of its block
                const IpBlock& b = block_at(sblk[c], k * u);
                const uint32_t q = (k * u - b.off) / u;
                const int32_t cd = b.peer;
                colv.push_back({s0, p->bd[cd] / S + b.peer_off / u + q, K, (uint32_t)(ld.stride[cd] / u), k, false});
            }
        }
        // the slot map; fixed points (a slot mapped onto itself: NONE, counted) and the cut points
        // of the cycle decomposition (build_segments) are found on the way
        std::vector<std::vector<uint32_t>> cut_parts(nthr);
        std::vector<uint64_t> fixed_parts(nthr, 0);
        parallel_for(nthr, m, [&](unsigned chunk, uint64_t t0, uint64_t t1) {
            auto& cp = cut_parts[chunk];
            uint64_t fx = 0;
            for (const Col& cv : colv)
                for (uint64_t t = t0; t < t1; ++t) {
                    const uint32_t x = (uint32_t)(cv.s0 + t * cv.K + cv.k);
                    const uint32_t y = (uint32_t)(cv.d0 + t * cv.Kd + (cv.raw ? cv.k : 0));
                    if (x == y) {
                        P[x] = NONE;
                        ++fx;
                        continue;
                    }
                    P[x] = y;
                    if (is_cut(x)) cp.push_back(x);
                }
            fixed_parts[chunk] = fx;
        });
        lap("slot map");
        for (const Range& r : src_r) p->content_slots += r.hi - r.lo;
        // dst-only slots (receive content, old bytes are src tail / gap) and src-only slots (content
        // that no dst slot overwrites), ascending: plain interval differences of the two range lists
        auto minus = [](const std::vector<Range>& A, const std::vector<Range>& B) {
            std::vector<uint32_t> out;
            size_t j = 0;
            for (const Range& a : A) {
                uint64_t x = a.lo;
                while (j < B.size() && B[j].hi <= x) ++j;
                for (size_t k = j; k < B.size() && B[k].lo < a.hi && x < a.hi; ++k) {
                    for (; x < std::min(B[k].lo, a.hi); ++x) out.push_back((uint32_t)x);
                    x = std::max(x, B[k].hi);
                }
                for (; x < a.hi; ++x) out.push_back((uint32_t)x);
            }
            return out;
        };
        const std::vector<uint32_t> free_in = minus(dst_r, src_r), free_out = minus(src_r, dst_r);
        lap("free lists");
        if (free_in.size() != free_out.size()) return fail(ADHA_ERR_UNSUPPORTED, "in-place plan: slot count mismatch");
        // a dst slot whose old bytes are not content (src tail, gap) receives content; its junk goes
        // to a src-only slot (which becomes dst tail / gap): the permutation closes on U
        std::vector<uint32_t> cuts;
        for (size_t i = 0; i < free_in.size(); ++i) {
            P[free_in[i]] = free_out[i];
            if (is_cut(free_in[i])) cuts.push_back(free_in[i]);
        }
        p->junk_slots = free_in.size();
        for (unsigned c = 0; c < nthr; ++c) {
            cuts.insert(cuts.end(), cut_parts[c].begin(), cut_parts[c].end());
            p->fixed_slots += fixed_parts[c];
        }
        std::sort(cuts.begin(), cuts.end());
        lap("cut points");
        const char* ve = std::getenv("ADHA_IP_VERIFY");
        const bool verify = ve && *ve == '1';
        uvector<uint32_t> P0;
        if (verify) P0 = P;
        build_segments(P, nslot, nthr, p, cuts);
        if (verify) {
            const std::string why = verify_segments(P0, *p);
            if (!why.empty()) return fail(ADHA_ERR_PLANNER, "in-place plan verification: " + why);
        }
        p->moved_slots = p->seq.size();
        if (p->seq.size() >= 0xFFFFFFFFull) return fail(ADHA_ERR_TOO_LARGE, "in-place remap: too many slots");
    }

    // ---- tail records [m*T, n): saved packed (declaration order), restored at the end
    p->tail_fields.clear();
    if (p->tail > 0) {
        uint32_t toff = 0;
        for (int32_t f = 0; f < ls.n_fields; ++f) {
            const int32_t cs = ls.cluster[f], cd = ld.cluster[f];
            p->tail_fields.push_back({p->bs[cs] + ls.offset[f], p->bd[cd] + ld.offset[f], (uint32_t)ls.stride[cs],
                                      (uint32_t)ld.stride[cd], ls.width[f], toff});
            toff += ls.width[f];
        }
    }

    // ---- workspace layout
    uint64_t o = 0;
    auto take = [&](uint64_t bytes) { const uint64_t at = o; o = align256(o + bytes); return at; };
    p->ws_pieces = take((p->pre.size() + p->post.size()) * sizeof(IpPiece));
    p->ws_cols = take(p->cols.size() * sizeof(IpCol));
    p->ws_tailf = take(p->tail_fields.size() * sizeof(IpTailField));
    p->ws_seq = take(p->seq.size() * sizeof(uint32_t));
    p->ws_segs = take(p->segs.size() * sizeof(IpSeg));
    p->ws_save = take(p->segs.size() * (uint64_t)S);
    p->ws_tail = take((uint64_t)p->tail * ls.record_bytes);
    p->ws_bytes = std::max<uint64_t>(o, 256);
    p->uploaded = nullptr;
    p->uploaded_device = -1;
    return ADHA_OK;
}

std::string inplace_plan_json(const InplacePlan& p) {
    auto u64 = [](uint64_t v) { return std::to_string(v); };
    std::string s = "{";
    s += "\"n_records\":" + std::to_string(p.n);
    s += std::string(",\"mode\":\"") + (p.staged ? "staged" : "permute") + "\"";
    s += ",\"unit\":" + u64(p.u) + ",\"slot_bytes\":" + u64(p.S) + ",\"T\":" + u64(p.T);
    s += ",\"body_tiles\":" + std::to_string(p.m) + ",\"tail_records\":" + std::to_string(p.tail);
    s += ",\"src_bytes\":" + u64(p.bytes_s) + ",\"dst_bytes\":" + u64(p.bytes_d);
    s += ",\"buffer_bytes\":" + u64(std::max(p.bytes_s, p.bytes_d));
    s += ",\"pre_clusters\":" + u64(p.pre.size()) + ",\"post_clusters\":" + u64(p.post.size());
    s += ",\"tile_smem\":" + u64(p.max_tile + p.max_tab);
    s += ",\"content_slots\":" + u64(p.content_slots) + ",\"moved_slots\":" + u64(p.moved_slots);
    s += ",\"fixed_slots\":" + u64(p.fixed_slots) + ",\"junk_slots\":" + u64(p.junk_slots);
    s += ",\"cycles\":" + u64(p.cycles) + ",\"segments\":" + u64(p.segs.size());
    uint64_t pre_b = 0, post_b = 0;
    for (const auto& x : p.pre) pre_b += (uint64_t)p.m * p.T * x.stride;
    for (const auto& x : p.post) post_b += (uint64_t)p.m * p.T * x.stride;
    // device traffic of one run: read + write of every transposed tile and moved slot
    s += ",\"traffic_bytes\":" + u64(p.staged ? 2 * ((uint64_t)p.n * p.ls.record_bytes + p.bytes_d)
                                             : 2 * (pre_b + post_b + (p.moved_slots + p.segs.size()) * p.S +
                                                    2 * (uint64_t)p.tail * p.ls.record_bytes));
    s += ",\"workspace_bytes\":" + u64(p.ws_bytes);
    s += "}";
    return s;
}

}  // namespace adha

using namespace adha;

extern "C" adha_status adha_inplace_plan_create(const adha_layout* hs, const adha_layout* hd, int64_t n,
                                                adha_inplace_plan** out) {
    clear_error();
    if (!hs || !hd || !out) return fail(ADHA_ERR_INVALID_ARG, "null argument");
    *out = nullptr;
    adha_inplace_plan* h = nullptr;
    try {
        h = new adha_inplace_plan();
        adha_status st = inplace_plan_build(hs->L, hd->L, n, &h->P);
        if (st != ADHA_OK) { delete h; return st; }
    } catch (const std::bad_alloc&) {
        delete h;
        return fail(ADHA_ERR_OOM, "in-place plan: host allocation failed");
    }
    *out = h;
    return ADHA_OK;
}

extern "C" adha_status adha_inplace_plan_info(const adha_inplace_plan* h, uint64_t* buffer_bytes,
                                              uint64_t* workspace_bytes) {
    clear_error();
    if (!h) return fail(ADHA_ERR_INVALID_ARG, "null plan");
    if (buffer_bytes) *buffer_bytes = std::max(h->P.bytes_s, h->P.bytes_d);
    if (workspace_bytes) *workspace_bytes = h->P.ws_bytes;
    return ADHA_OK;
}

extern "C" adha_status adha_inplace_plan_describe(const adha_inplace_plan* h, char** json_out) {
    clear_error();
    if (!h || !json_out) return fail(ADHA_ERR_INVALID_ARG, "null argument");
    const std::string s = inplace_plan_json(h->P);
    char* c = (char*)std::malloc(s.size() + 1);
    if (!c) return fail(ADHA_ERR_OOM, "out of memory");
    std::memcpy(c, s.c_str(), s.size() + 1);
    *json_out = c;
    return ADHA_OK;
}

extern "C" void adha_inplace_plan_destroy(adha_inplace_plan* h) { delete h; }
