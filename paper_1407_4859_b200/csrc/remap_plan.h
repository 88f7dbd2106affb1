// remap_plan.h -- the compiled remap plan for a (src layout, dst layout) pair
// and the kernel-parameter structs it fills.
//
// Tiled kernel model:
//   * components: the fields split into the connected components of the
//     bipartite graph "src cluster -- dst cluster sharing a field".  Each
//     component is an independent remap of its own clusters (record i of a
//     dst cluster depends only on record i of the src clusters of its
//     component), so each gets its own tile size T_k = records per tile;
//   * a tile of component k is T_k consecutive records (T_k a multiple of 32);
//     for every src cluster c of k the tile's records form ONE contiguous chunk
//     of T_k*stride(c) bytes in region c (element address): a tile
//     arrives in shared memory as one TMA bulk copy per src cluster;
//   * in shared memory the tile is permuted by "units" of g bytes (g = 4, 2 or
//     1: the largest of those dividing every width and offset of both layouts)
//     into an output buffer holding one contiguous chunk per dst cluster, which
//     the consumer warps write back with coalesced 16-byte stores;
//   * a period is 32 records: a chunk advances by 32*stride bytes per period,
//     and chunk starts are multiples of 32*stride, so with g = 4 the 4-byte
//     bank of a unit depends only on its offset inside period 0 of its chunk.
//     The 32*W_k units of one period (W_k = R_k/g) are split into W_k warp
//     instructions of 32 lanes: for g = 4 by decomposing the 32x32 bank
//     multigraph into perfect matchings, so every instruction reads 32
//     distinct banks and writes 32 distinct banks (conflict-free LDS and STS by
//     construction, independent of T_k);
//   * identity components (one src cluster == one dst cluster, same fields)
//     skip the permutation: the staged chunk moves to the output buffer with
//     16-byte shared copies (releasing the input stage early) and is written back;
//   * g = 1 or 2 (byte-group mode): a lane assembles up to 4 output WORDS from
//     up to 4 source words with PRMT (ByteGroup below); groups are packed into
//     instructions conflict-free at every period phase where possible
//     (remap_plan.cpp), and chunk starts are staggered by 32 bytes per cluster.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace adha {
namespace dev {

constexpr int NCONS = 8;                       // consumer warps per CTA
constexpr int NTHREADS = (NCONS + 1) * 32;     // + one TMA producer warp
constexpr int NTHREADS_TMA = (NCONS + 2) * 32; // + a TMA write-back warp (tma_copy instantiations)
constexpr int NLOAD = 3;                       // cp.async loader warps (cpa instantiations)
constexpr int NTHREADS_CPA = (NCONS + NLOAD) * 32;
constexpr int MAXC = 128;                      // clusters per side (tiled kernel)
constexpr int MAXF = 256;                      // fields (tiled kernel tail table, naive chunk)
constexpr int MAXK = 64;                       // components
constexpr int S_OUT_MAX = 2;                   // output staging buffers (1 or 2)
constexpr int HDR_BYTES = 1024;                // barrier header at the start of dynamic smem
constexpr int MAX_S_IN = 8;
constexpr uint32_t STAGE_MAX = 12 * 16 * NCONS * 32;   // copy-out covers 12 16-byte vectors per thread

struct alignas(16) ClusterDesc {   // 16-byte aligned: the kernel copies descriptors with 128-bit loads
    uint64_t region;    // region base in the buffer for this N (bytes)
    uint32_t stride;    // bytes per cluster record
    uint32_t smem;      // chunk offset inside its component's staged tile (bytes), for this call's T
};

struct FieldDesc {
    uint8_t sc, dc;       // src / dst cluster (indices into srcc / dstc)
    uint8_t sbl, dbl;     // log2 of the src / dst cluster's AoSoA block
    uint32_t soff, doff;  // byte offset in the src / dst cluster record
    uint32_t width;
};

struct CompDesc {
    int64_t tile_base;    // first global tile index of the component
    int64_t n_tiles;      // floor(N / T)
    uint32_t T;           // records per tile (multiple of 32)
    uint32_t tile_bytes;  // T * (sum of src strides): TMA transaction bytes per tile
    uint32_t out_bytes;   // T * (sum of dst strides): bytes the copy-out writes per tile
    uint16_t sc_lo, sc_hi, dc_lo, dc_hi;   // cluster ranges (clusters are numbered by component)
    uint16_t f_lo, f_hi;                   // field range in the field table
    uint16_t identity;
    uint16_t flags;       // CF_SKIP | CF_ZERO_OUT | CF_TAIL_ZERO
    uint32_t instr_base;  // first instruction (unit mode) / first group (byte-group mode) in the table
    uint32_t n_instr;     // unit mode: W_k = R_k / g; byte-group mode: groups per period
};

constexpr uint16_t CF_SKIP = 1;       // identity component whose dst region IS its src region (nothing moves)
constexpr uint16_t CF_ZERO_OUT = 2;   // dst records have padding: output buffers pre-zeroed at component start
constexpr uint16_t CF_TAIL_ZERO = 4;  // dst padding or AoSoA blocks: tail area zeroed before the tail copy

struct TiledParams {
    uint64_t src;         // base address: src region c starts at src + srcc[c].region
    uint64_t dst;         // base address: dst region c starts at dst + dstc[c].region
    int64_t n_records;
    int64_t total_tiles;  // sum of the components' n_tiles
    uint32_t stage_bytes; // bytes per staging buffer (max tile bytes, rounded to 128)
    uint32_t s_in;        // input pipeline stages
    uint32_t s_out;       // output buffers: 2 = double-buffered, 1 = one buffer + a barrier before reuse
    uint32_t n_comp;
    uint32_t unit;        // g
    uint32_t l2_hints;    // bit 0: TMA loads with L2 evict_first; bit 1: stores with L2 evict_first
    uint32_t blocked;     // 1: CTA b processes a contiguous tile range, 0: tiles b, b+G, b+2G, ...
    uint32_t tma_split;   // 0: one bulk load per src chunk; else pieces of at most this many bytes
    uint32_t tma_copy;    // 1: tiles written back by the write-back warp with TMA bulk stores, else STG by the consumers
    uint32_t n_ent;       // entries used: unit mode 32 * instructions of all components, byte-group mode groups
    uint32_t n_srcc;      // clusters used in srcc / dstc
    uint32_t n_dstc;
    uint32_t chain;       // 0, or H >= 2: a fused chain of H hops (component k = hop k, adha_remap_chain);
                          // every component has the same T and n_tiles (bands); regions are absolute
    uint32_t chain_group; // chain: bands per group (1..8), each group run hop by hop
    uint32_t chain_hints; // chain: 1 = loads evict_first, intermediates stored evict_last, the last hop evict_first
    uint32_t cpa;         // 1: NLOAD loader warps fill the input stages with cp.async (16 B per lane)
                          // instead of the producer warp's TMA bulk copies (the CPA instantiations)
    uint64_t table;       // device address of the plan's table image (EntryTable<NENT> / GroupTable<NG>),
                          // uploaded once per plan and device (remap.cu device_table)
    CompDesc comp[MAXK];
    ClusterDesc srcc[MAXC];
    ClusterDesc dstc[MAXC];
};

// per-(instruction, lane) table: entry i*32+lane of instruction i (instructions of all
// components concatenated); offsets are units inside period 0 of the unit's chunk
template <int NENT>
struct alignas(16) EntryTable {   // 16-byte aligned: copied to shared memory with 128-bit loads
    uint32_t off[NENT];   // src local unit offset (low 16 bits) | dst local unit offset (high 16 bits)
    uint8_t sc[NENT];     // src cluster of the unit
    uint8_t dc[NENT];     // dst cluster of the unit
    FieldDesc fields[MAXF];   // tail table, fields grouped by component
};

// Byte-group mode (g = 1 or 2 layouts): a lane builds up to 4 OUTPUT WORDS of one period from
// up to 4 SOURCE WORDS with PRMT (byte permute) -- 4-byte shared loads/stores instead of one
// shared instruction per byte.  Output words are grouped by identical source-word sets
// (e.g. fields f..f+3 of records r..r+3 in a 1-byte AoS->SoA transpose share the same 4 words).
struct ByteGroup {
    uint16_t out_off[4];   // dst byte offset (multiple of 4) inside period 0 of the word's chunk
    uint16_t src_off[4];   // src byte offset (multiple of 4) inside period 0 of the word's chunk
    uint16_t sel[4][3];    // per output word: A = prmt(w0,w1,sel0), B = prmt(w2,w3,sel1), out = prmt(A,B,sel2)
    uint8_t out_dc[4];     // dst cluster slot of each output word
    uint8_t src_sc[4];     // src cluster slot of each source word
    uint8_t n_out, n_src, pad0, pad1;
};
template <int NG>
struct alignas(16) GroupTable {
    ByteGroup g[NG];
    FieldDesc fields[MAXF];
};
constexpr int GCLASS_NG[2] = {128, 384};
constexpr int GCLASS_GMAX[2] = {1, 2};    // slots per warp: ceil(instructions * period-split / NCONS)

// Table size classes (entries per warp EMAX = instructions per warp per component).
constexpr int CLASS_NENT[4] = {512, 1024, 2048, 3456};
constexpr int CLASS_EMAX[4] = {2, 4, 8, 14};

struct NaiveField {
    uint64_t sbase, dbase;
    uint32_t sstride, dstride, soff, doff, width, pad;
};
template <int NF>
struct NaiveParamsT {
    uint64_t src;
    uint64_t dst;
    int64_t n_records;
    int64_t lo;           // first record
    uint32_t n_fields;
    NaiveField f[NF];
};
using NaiveParams = NaiveParamsT<MAXF>;
constexpr int SMALL_NF = 32;                  // direct kernel with small parameters (latency path)

// Fused small chain (adha_remap_chain when every hop is a latency-bound remap): one launch runs
// every hop; block b owns a contiguous record range in every buffer and a __syncthreads()
// separates the hops, so hop h+1 reads exactly the bytes block b wrote in hop h.
constexpr int CHAIN_NF = 16, CHAIN_NH = 4;
struct ChainParams {
    uint64_t buf[CHAIN_NH + 1];
    int64_t n_records;
    uint32_t n_fields, n_hops;
    NaiveField f[CHAIN_NH][CHAIN_NF];   // per hop; packed, unblocked layouts only (pad = 0)
};
using SmallParams = NaiveParamsT<SMALL_NF>;

}  // namespace dev

// Host-side compiled plan (N-independent; T per call, region bases per call).
struct RemapPlan {
    struct Comp {
        std::vector<int> src_clusters, dst_clusters, fields;   // original (canonical) indices
        uint32_t R = 0;               // payload bytes per record of the component
        uint32_t Rs = 0, Rd = 0;      // src / dst bytes per record (strides, padding included)
        bool zero_out = false, tail_zero = false;
        uint32_t T_max = 0;           // records per tile at full size
        bool identity = false;
        uint32_t instr_base = 0, n_instr = 0;
        uint32_t n_groups = 0;        // byte-group mode: groups of one period
    };
    uint64_t uid = 0;                 // process-unique plan id (key of its device table copies)
    bool tiled = false;
    bool merged = false;              // compiled with every cluster in one component
    std::string why_naive;            // reason when not tiled
    uint32_t unit = 1;                // g
    uint32_t s_in = 0, s_out = 2, stage_bytes = 0;
    uint32_t smem_bytes = 0;
    uint32_t tbl_bytes = 0;           // unit mode: shared-memory copy of the entry table + cluster descriptors
    int table_class = 0;
    bool matched = false;             // conflict-free matching used (g = 4)
    bool byte_groups = false;         // g < 4: PRMT byte-group mode (GroupTable) instead of units
    uint32_t tile_quantum = 32;       // tile sizes are multiples of this many records
    int group_class = 0;
    uint32_t n_groups_total = 0;      // byte-group mode: groups in the table
    std::vector<Comp> comps;
    std::vector<int> src_order, dst_order;   // kernel cluster index -> canonical cluster
    std::vector<int> src_slot, dst_slot;     // canonical cluster -> kernel cluster index
    std::vector<uint32_t> ent_off;           // 32 * sum(W_k) entries (local offsets)
    std::vector<uint8_t> ent_sc, ent_dc;     // kernel cluster indices
    std::vector<uint32_t> table;             // EntryTable<CLASS_NENT[table_class]> / GroupTable image (fields
                                             // filled); the kernels read a device copy of it
};

struct Layout;
// merge: one component over all clusters (the small / mid-size variant, see remap.cu)
RemapPlan compile_plan(const Layout& ls, const Layout& ld, bool merge = false);
std::string describe_plan(const RemapPlan& p, const Layout& ls, const Layout& ld);
// records per tile of component k for an N-record call on n_sm SMs
uint32_t call_tile(const RemapPlan& p, int k, int64_t n, int n_sm);

}  // namespace adha
