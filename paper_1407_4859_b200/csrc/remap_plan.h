// remap_plan.h -- the compiled remap plan for a (src layout, dst layout) pair
// and the kernel-parameter structs it fills.
//
// Tiled kernel model:
//   * a tile is T consecutive records (T a multiple of 32); for every src
//     cluster c the tile's records form ONE contiguous chunk of T*stride(c)
//     bytes in region c (element address), so a tile arrives in
//     shared memory as n_src TMA bulk copies and leaves as n_dst bulk copies;
//   * in shared memory the tile is permuted by "units" of g bytes (g = 4, 2 or
//     1: the largest of those dividing every width and offset of both layouts);
//   * a period is 32 records: every chunk advances by 32*stride bytes per
//     period, a multiple of 128 bytes, so the 4-byte bank of every unit
//     repeats from period to period;  the 32*W units of one period
//     (W = R/g) are split into W warp instructions of 32 lanes.  For g = 4 the
//     split is a decomposition of the 32x32 bank multigraph into perfect
//     matchings (every instruction reads 32 distinct banks and writes 32
//     distinct banks: conflict-free LDS and STS by construction).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace adha {
namespace dev {

constexpr int NCONS = 8;                       // consumer warps per CTA
constexpr int NTHREADS = (NCONS + 1) * 32;     // + one TMA producer warp
constexpr int MAXC = 128;                      // clusters per side (tiled kernel)
constexpr int MAXF = 256;                      // fields (tiled kernel tail table, naive chunk)
constexpr int S_OUT = 2;                       // output staging buffers
constexpr int HDR_BYTES = 1024;                // barrier header at the start of dynamic smem
constexpr int MAX_S_IN = 8;

struct ClusterDesc {
    uint64_t region;    // region base in the buffer for this N (bytes)
    uint32_t stride;    // bytes per cluster record
    uint32_t smem;      // chunk offset inside a staged tile (bytes)
};

struct FieldDesc {
    uint16_t sc, dc;    // src / dst cluster
    uint32_t soff, doff;  // byte offset in the src / dst cluster record
    uint32_t width;
};

struct TiledParams {
    const uint8_t* src;
    uint8_t* dst;
    int64_t n_records;
    int64_t n_tiles;      // full tiles: floor(N / T)
    int64_t tail_lo;      // n_tiles * T
    uint32_t T;
    uint32_t periods;     // T / 32
    uint32_t tile_bytes;  // T * R: TMA transaction bytes per tile
    uint32_t stage_bytes; // tile_bytes rounded up to 128
    uint32_t n_src, n_dst, n_fields;
    uint32_t s_in;        // input pipeline stages
    uint32_t n_instr;     // W = R / g instructions per period
    uint32_t unit;        // g
    ClusterDesc srcc[MAXC];
    ClusterDesc dstc[MAXC];
    FieldDesc fields[MAXF];
};

// per-(instruction, lane) table: entry i*32+lane of instruction i
template <int NENT>
struct EntryTable {
    uint32_t off[NENT];   // src unit offset (low 16 bits) | dst unit offset (high 16 bits), period 0
    uint8_t sc[NENT];     // src cluster of the unit (its period stride is 32*stride)
    uint8_t dc[NENT];     // dst cluster of the unit
};

// Table size classes (entries per warp EMAX = instructions per warp).
constexpr int CLASS_NENT[4] = {512, 1024, 2048, 3584};
constexpr int CLASS_EMAX[4] = {2, 4, 8, 14};

struct NaiveField {
    uint64_t sbase, dbase;
    uint32_t sstride, dstride, soff, doff, width, pad;
};
struct NaiveParams {
    const uint8_t* src;
    uint8_t* dst;
    int64_t n_records;
    int64_t lo;           // first record
    uint32_t n_fields;
    NaiveField f[MAXF];
};

}  // namespace dev

// Host-side compiled plan (N-independent; region bases are filled per call).
struct RemapPlan {
    bool tiled = false;
    std::string why_naive;        // reason when not tiled
    uint32_t unit = 1;            // g
    uint32_t T = 0, s_in = 0, stage_bytes = 0, tile_bytes = 0, n_instr = 0;
    uint32_t smem_bytes = 0;
    int table_class = 0;
    bool matched = false;         // conflict-free matching used (g = 4)
    std::vector<uint32_t> src_chunk, dst_chunk;     // per cluster chunk offsets in a staged tile
    std::vector<uint32_t> ent_off;                  // 32 * n_instr entries
    std::vector<uint8_t> ent_sc, ent_dc;
    std::vector<uint32_t> table;                    // EntryTable<CLASS_NENT[table_class]> image
};

struct Layout;
RemapPlan compile_plan(const Layout& ls, const Layout& ld);
std::string describe_plan(const RemapPlan& p, const Layout& ls, const Layout& ld);

}  // namespace adha
