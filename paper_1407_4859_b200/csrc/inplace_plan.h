// inplace_plan.h -- host plan of the in-place remap (the "in-place" half;
// adha.h adha_inplace_plan_create).  Not part of the ABI.
//
// The buffer is cut into slots of S bytes (S a power of two in [256, 4096] dividing every
// region base of both layouts).  A tile of T = S / u records (u = the largest power of two
// <= 16 dividing every field width) of a cluster with stride s occupies s / u slots.  A RUN is a
// maximal sequence of fields consecutive in both the src and the dst cluster record; in a tile's
// BLOCKED form (AoSoA with block T, one block per run) run b's T values are contiguous, T * w_b
// bytes = w_b / u whole slots:
//   step 1  (tile-local) each src tile of a cluster made of several runs is rewritten in place
//           from record-major to blocked form (a one-run cluster already is);
//   step 2  (slot permutation) every slot moves to the slot its (run, bytes) occupy in the dst
//           layout's blocked form, by following the permutation's cycles (split into segments
//           so that warps work in parallel; the last slot of each segment is saved first);
//   step 3  (tile-local) each dst tile of a cluster made of several runs is rewritten from
//           blocked to record-major form.
// Clusters whose member set is the same in both layouts are moved as raw slots (no rewrite),
// and not at all when their region base is the same (fixed points).  The last N mod T records
// (the tail) are saved to the workspace first and written to their dst positions last.
#pragma once

#include <sys/mman.h>

#include <cstdlib>
#include <memory>
#include <new>
#include <utility>
#include <vector>

namespace adha {
// std::allocator whose default construction leaves trivial values uninitialised: the plan's
// large index arrays (tens of MB at C3's size) are filled in parallel, not zeroed serially first
// Arrays of >= 4 MB are 2 MB-aligned and advised as transparent huge pages: their first touch
// (the parallel fill) then faults 512x fewer pages -- the first plan of a process spent about a
// third of its time in page faults at C3's size.
template <class T>
struct UninitAlloc : std::allocator<T> {
    using std::allocator<T>::allocator;
    template <class U>
    struct rebind { using other = UninitAlloc<U>; };
    T* allocate(size_t n) {
        const size_t bytes = n * sizeof(T);
        if (bytes < (4u << 20)) return std::allocator<T>::allocate(n);
        const size_t huge = 2u << 20, rounded = (bytes + huge - 1) / huge * huge;
        void* p = std::aligned_alloc(huge, rounded);
        if (!p) throw std::bad_alloc();
        madvise(p, rounded, MADV_HUGEPAGE);
        return static_cast<T*>(p);
    }
    void deallocate(T* p, size_t n) {
        if (n * sizeof(T) < (4u << 20)) std::allocator<T>::deallocate(p, n);
        else std::free(p);
    }
    template <class U, class... Args>
    void construct(U* p, Args&&... args) {
        if constexpr (sizeof...(Args) == 0) ::new ((void*)p) U;
        else ::new ((void*)p) U(std::forward<Args>(args)...);
    }
};
template <class T>
using uvector = std::vector<T, UninitAlloc<T>>;
}  // namespace adha

#include <cstdint>
#include <vector>

#include "internal.h"

namespace adha {

struct IpPiece {        // one cluster region rewritten piece by piece (steps 1 and 3)
    uint64_t base;      // region base (bytes from the buffer start)
    uint64_t pieces;    // ceil(m / g): pieces of this cluster
    uint32_t stride;    // cluster record bytes
    uint32_t RA;        // atoms per record (atom = 4 bytes when u % 4 == 0, else 1 byte)
    uint32_t col_off;   // first entry of this cluster in the column table
    uint32_t magic_RA;  // ceil(2^32 / RA) (0 when RA == 1): q = umulhi(n, magic) for n * RA < 2^32
    uint32_t g;         // tiles per piece (small tiles are grouped so that a piece is ~16 KB)
    uint32_t magic_TRA; // ceil(2^32 / (T * RA)) (used when g > 1)
    uint32_t TS;        // atoms of one padded field-blocked tile in shared memory
    uint32_t pad;
};

struct IpCol {          // one atom column j of a cluster record
    uint32_t col_fp;    // first column of j's field (low 16 bits) | padding atoms before its block << 16
    uint32_t a;         // atoms of j's field
    uint32_t magic_a;   // ceil(2^32 / a) (0 when a == 1)
    uint32_t bo;        // shared-memory atom of (record 0, column j) in the padded field-blocked tile:
                        // T * col + padding before the block + (j - col); record r adds r * a
};

struct IpBlock {        // a run of fields contiguous in both the src and the dst cluster record
    uint32_t off;       // byte offset of the run in this side's cluster record
    uint32_t width;     // bytes of the run
    int32_t peer;       // the other side's cluster
    uint32_t peer_off;  // byte offset of the run in the other side's cluster record
};

struct IpTailField {    // one field of the tail records: src/dst element address terms
    uint64_t src;       // base_s(c) + offset_s(f)
    uint64_t dst;       // base_d(c') + offset_d(f)
    uint32_t stride_s, stride_d, width, toff;   // toff: byte offset in a packed tail record
};

struct IpSeg {          // a run of consecutive positions of one cycle
    uint32_t start;     // first index into seq
    uint32_t len;       // positions (>= 1)
    uint32_t pred;      // segment holding the position just before `start` on the cycle
    uint32_t pad;
};

struct InplacePlan {
    Layout ls, ld;
    int64_t n = 0;
    uint32_t u = 0, S = 0, T = 0;
    int64_t m = 0;                       // body tiles (T records each)
    int64_t tail = 0;                    // n - m * T
    uint64_t bytes_s = 0, bytes_d = 0;   // bytes(Ls, n), bytes(Ld, n)
    std::vector<uint64_t> bs, bd;
    std::vector<IpPiece> pre, post;      // step 1 (src clusters), step 3 (dst clusters)
    std::vector<IpCol> cols;             // column tables of pre then post clusters
    uint32_t max_tile = 0;               // shared memory of the largest rewritten tile (with padding)
    uint32_t max_tab = 0;                // shared memory of the largest column table
    uvector<uint32_t> seq;               // slot indices, cycles in order (slot j -> next on its cycle)
    std::vector<IpSeg> segs;
    std::vector<IpTailField> tail_fields;
    // statistics
    uint64_t content_slots = 0, moved_slots = 0, fixed_slots = 0, junk_slots = 0, cycles = 0;
    // workspace layout (byte offsets, each 256-aligned) and total size
    uint64_t ws_pieces = 0, ws_cols = 0, ws_tailf = 0, ws_seq = 0, ws_segs = 0, ws_save = 0, ws_tail = 0, ws_bytes = 0;
    bool staged = false;                 // small buffer: out-of-place remap into the workspace + copy back
    uint64_t ws_stage = 0;
    // upload state (adha_inplace_plan_upload)
    const void* uploaded = nullptr;
    int uploaded_device = -1;
};

// Buffers up to this many bytes are remapped through the workspace (ADHA_INPLACE_STAGED_BYTES).
constexpr uint64_t IP_STAGED_BYTES = 16ull << 20;
// Segment length: positions per segment (a warp group walks one segment).
constexpr uint32_t IP_SEG = 64;
// Largest transposed tile (shared memory of one CTA, with row padding).
constexpr uint32_t IP_MAX_PIECE = 160u * 1024u;

adha_status inplace_plan_build(const Layout& ls, const Layout& ld, int64_t n, InplacePlan* p);
std::string inplace_plan_json(const InplacePlan& p);

}  // namespace adha

struct adha_inplace_plan {
    adha::InplacePlan P;
};
