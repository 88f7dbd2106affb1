/*
 * adha.h -- C ABI of the B200-native ADHA data-layout remap library (libadha.so).
 *
 * ADHA (arXiv 1407.4859, PAPER.md) chooses a data layout per program section:
 * ODS clusters fields by affinity and PDL places REMAP edges
 * between sections whose layouts differ.  At a remap edge the
 * records move from the parent section's layout to the child's ("a remap
 * operation is performed to SOA layout").  This library is that
 * remap on B200 (hand-written sm_100a kernels), the layout descriptor it is
 * addressed by, and the host planner that produces the layouts.
 *
 * Conventions (all functions):
 *   - Plain C types only: sizes are int32_t / int64_t / uint64_t, buffers are
 *     void pointers, a CUDA stream is passed as `void*` holding a
 *     cudaStream_t (NULL = the legacy default stream of the current device).
 *   - Every function returns an adha_status; ADHA_OK = 0.  On failure a
 *     thread-local message is available from adha_last_error().  Nothing is
 *     partially written on a validation error.
 *   - Ownership: layouts are created and destroyed by the caller; device and
 *     host buffers and streams belong to the caller; strings the library
 *     returns through `char**` are freed with adha_free().
 *   - Layout handles are immutable after creation and may be shared between
 *     threads ("immutable after construction").
 */
#ifndef ADHA_H_
#define ADHA_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define ADHA_API __attribute__((visibility("default")))
#else
#define ADHA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum adha_status {
    ADHA_OK = 0,
    ADHA_ERR_INVALID_ARG = 1,      /* null pointer, negative count, bad index          */
    ADHA_ERR_PARSE = 2,            /* malformed layout string or planner JSON          */
    ADHA_ERR_LAYOUT_MISMATCH = 3,  /* src/dst layouts differ in field count or widths  */
    ADHA_ERR_CAPACITY = 4,         /* planner: a field wider than the cluster capacity */
    ADHA_ERR_ALIGNMENT = 5,        /* a device buffer not 256-byte aligned             */
    ADHA_ERR_OVERLAP = 6,          /* src and dst byte ranges overlap                  */
    ADHA_ERR_TOO_LARGE = 7,        /* N * record bytes overflows 2^63                  */
    ADHA_ERR_CUDA = 8,             /* a CUDA runtime call or kernel launch failed      */
    ADHA_ERR_OOM = 9,              /* host allocation failed                           */
    ADHA_ERR_UNSUPPORTED = 10,     /* outside the library's limits (see below)         */
    ADHA_ERR_PLANNER = 11          /* planner rejected the program (no plan/device)    */
} adha_status;

/* Limits. */
#define ADHA_MAX_FIELDS 4096       /* fields per layout                                 */
#define ADHA_MAX_FIELD_BYTES 65536 /* bytes per field                                   */

/* Opaque layout descriptor. */
typedef struct adha_layout adha_layout;

/* ------------------------------------------------------------------ version / errors */

/* Library version as MAJOR*10000 + MINOR*100 + PATCH. */
ADHA_API int32_t adha_version(void);

/* Static name of a status code ("ADHA_OK", ...). Never NULL. */
ADHA_API const char* adha_status_string(adha_status s);

/* Detail of the last failure on the calling thread ("" if none).  Valid until the
 * next adha_* call on this thread. */
ADHA_API const char* adha_last_error(void);

/* Free a string returned by the library through a char** out-parameter. NULL is ok. */
ADHA_API void adha_free(void* p);

/* ------------------------------------------------------------------ layout descriptor
 *
 * A layout is a partition of the record's fields into clusters (SPEC.md:55-58,
 * [TYPE] Layout; Table 2: a cluster of >= 2 fields is an
 * AoS group, a singleton is an SoA array).  Fields are identified by their
 * declaration index 0..n_fields-1 and have a byte width each.
 *
 * Canonical form: clusters ordered by their minimum field index,
 * fields inside a cluster by index.  A cluster record is the packed
 * concatenation of its fields in that order (reading Q2: no padding):
 *     stride(c) = sum of widths in c,  offset(f) = prefix sum inside c.
 * One buffer holds one region per cluster, in canonical order, each region
 * base aligned up to 256 bytes from the buffer start (reading Q3):
 *     base(0) = 0,  base(c) = align256(base(c-1) + N * stride(c-1)),
 *     bytes(L, N) = base(last) + N * stride(last).
 * The element address of field f of record i is
 *     addr(f, i) = base(cluster(f)) + i * stride(cluster(f)) + offset(f).
 * Bytes between regions are never read for meaning nor written by a remap.
 * A handle carries no record count (reading Q4): one handle serves any N.
 */

/* Create a layout from field widths and a cluster label per field.
 *   field_widths[n_fields]      bytes per field, 1..ADHA_MAX_FIELD_BYTES
 *   cluster_of_field[n_fields]  any int32 labels; equal labels = same cluster
 *   out                         receives the new handle (caller destroys it)
 * Errors: INVALID_ARG (null, n_fields outside 1..ADHA_MAX_FIELDS, width 0 or too big). */
ADHA_API adha_status adha_layout_create(const uint32_t* field_widths, int32_t n_fields,
                               const int32_t* cluster_of_field, adha_layout** out);

/* Layout flags for adha_layout_create_ex. */
#define ADHA_LAYOUT_ALIGNED 1u     /* natural (C-struct) alignment inside cluster records */

/* Generalised layouts (beyond the paper, which considers "only AoS and
 * SoA"):
 *   flags & ADHA_LAYOUT_ALIGNED: a field of width w starts at a multiple of a(w), the largest
 *     power of two dividing w (at most 8); a cluster record's stride is rounded up to the
 *     largest a(w) of its fields (the C struct rule);
 *   block_of_field[f] (NULL = all 1): AoSoA block B in {1,2,4,8,16,32}, equal for the fields
 *     of a cluster.  Records are stored in blocks of B, each field's B values contiguous:
 *       addr(f, i) = base + (i / B) * (B * stride) + offset(f) * B + (i % B) * w_f,
 *     and the region holds ceil(N / B) whole blocks.
 * A remap writes 0 into every byte of a dst region that is not a field byte of a record < N
 * (alignment padding, block slots past N).  Strings: "aligned:" prefix, "{a,b}@8" suffix.
 * Errors: as adha_layout_create; INVALID_ARG for a bad block or unequal blocks in a cluster. */
ADHA_API adha_status adha_layout_create_ex(const uint32_t* field_widths, int32_t n_fields,
                                           const int32_t* cluster_of_field, const int32_t* block_of_field,
                                           uint32_t flags, adha_layout** out);

/* Create a layout from its string form.  Accepts the canonical form of
 * SPEC.md:79 "{f,g,h}|{x}|{y}" and the paper's Table-2 notation
 * "V1,V2,V3,{U1,U2,U3},S" where a bare name is a singleton.
 * Whitespace is ignored.  field_names[n_fields] give the names in declaration
 * order; every name must appear exactly once.
 * Errors: INVALID_ARG (null/bad sizes), PARSE (syntax, unknown or repeated name,
 * missing field). */
ADHA_API adha_status adha_layout_from_string(const char* text, const char* const* field_names,
                                    const uint32_t* field_widths, int32_t n_fields,
                                    adha_layout** out);

/* Write the canonical string into buf (always NUL-terminated when cap > 0,
 * truncated if needed).  field_names may be NULL: names are then "f0", "f1", ...
 * *needed receives the full length excluding the NUL.
 * Errors: INVALID_ARG (null layout or needed). */
ADHA_API adha_status adha_layout_to_string(const adha_layout* layout, const char* const* field_names,
                                  char* buf, size_t cap, size_t* needed);

/* Number of fields / clusters, and R = bytes per record (sum of widths). */
ADHA_API adha_status adha_layout_info(const adha_layout* layout, int32_t* n_fields, int32_t* n_clusters,
                             uint64_t* record_bytes);

/* Canonical cluster index of every field (out[n_fields]). */
ADHA_API adha_status adha_layout_clusters(const adha_layout* layout, int32_t* cluster_of_field);

/* bytes(L, N) as defined above.  Errors: INVALID_ARG (N < 0), TOO_LARGE. */
ADHA_API adha_status adha_layout_bytes(const adha_layout* layout, int64_t n_records, uint64_t* out_bytes);

/* Address terms of one field for an N-record instance:
 * region_offset = base(cluster(f)), stride = stride(cluster(f)), offset = offset(f). */
ADHA_API adha_status adha_layout_field_address(const adha_layout* layout, int32_t field, int64_t n_records,
                                      uint64_t* region_offset, uint32_t* stride, uint32_t* offset);

/* As adha_layout_field_address, plus the cluster's AoSoA block (1 for plain records). */
ADHA_API adha_status adha_layout_field_address_ex(const adha_layout* layout, int32_t field, int64_t n_records,
                                                  uint64_t* region_offset, uint32_t* stride, uint32_t* offset,
                                                  uint32_t* block);

/* Destroy a handle.  NULL is ok. */
ADHA_API void adha_layout_destroy(adha_layout* layout);

/* ------------------------------------------------------------------ the remap (hot path)
 *
 * adha_remap computes, for every record i in [0, N) and every field f
 * (PAPER.md:56-57 remap edge, PAPER.md:146 remap operation):
 *     dst[addr_Ld(f, i) .. + w_f) = src[addr_Ls(f, i) .. + w_f)
 * as a type-blind byte copy (NaN payloads, -0, denormals preserved bit for bit,
 * reading Q6).  Bytes of dst outside its regions are not written.
 *
 *   src, dst     DEVICE pointers on the current CUDA device, each 256-byte
 *                aligned, holding bytes(Ls, N) and bytes(Ld, N) bytes; the two
 *                ranges must not overlap (reading Q5: out of place only)
 *   src_layout, dst_layout   same n_fields and the same width per field (Q8)
 *   n_records    N >= 0; N = 0 is a no-op returning ADHA_OK
 *   stream       cudaStream_t (as void*) the kernel is enqueued on
 *
 * Asynchronous: the call enqueues one kernel launch on `stream` and returns.
 * The remap kernels are launched with programmatic dependent launch: a kernel may start
 * its prologue while the previous kernel on `stream` finishes, but it reads and
 * writes the caller's buffers only after that kernel has completed (stream
 * order is unchanged; ADHA_PDL=0 turns it off).
 * The per-call plan travels as kernel parameters; the first tiled remap of a
 * layout pair on a device uploads the plan's permutation table (<= 25 KB) into
 * library-owned device memory (a static 4 MB arena per device, then 4 MB
 * chunks, kept for the process lifetime) with a copy that the call waits for
 * -- or, inside CUDA-graph capture, with a kernel in the captured stream.
 * Launch errors return ADHA_ERR_CUDA; faults during execution surface at the
 * caller's next synchronisation.
 * Errors: INVALID_ARG, LAYOUT_MISMATCH, ALIGNMENT, OVERLAP, TOO_LARGE, CUDA. */
ADHA_API adha_status adha_remap(const void* src, const adha_layout* src_layout,
                       void* dst, const adha_layout* dst_layout,
                       int64_t n_records, void* stream);

/* The remap between layout instances given REGION BY REGION (SURVEY.md 8(f) N1,
 * "moved subset"): src_regions[c] is the device address of src cluster c's region
 * (canonical cluster order), dst_regions[c] likewise.
 * Regions need not be parts of one buffer.  A dst region that is the very same
 * memory as the src region of an IDENTICAL cluster (same fields at the same
 * offsets, same stride and AoSoA block, no alignment padding: the plan's identity
 * component) is left untouched by both kernel paths, bytes past N in its last block
 * included: its records are already in place, so only the fields whose cluster
 * changes move -- the paper's remap cost "based on the number of common fields"
 * (Medical AoSV -> SoA moves only {V1,V2,V3}).
 * Every region must be 256-byte aligned; a region spans its whole blocks
 * (ceil(N / B) * B * stride(c) bytes); dst regions must not overlap each other or
 * any src region except by that exact aliasing (a member-equal cluster that is not
 * an identity -- padded, or another block size -- is OVERLAP).
 * Asynchronous on `stream` like adha_remap.
 * Errors: INVALID_ARG, LAYOUT_MISMATCH, ALIGNMENT, OVERLAP, TOO_LARGE, CUDA. */
ADHA_API adha_status adha_remap_regions(const void* const* src_regions, const adha_layout* src_layout,
                                        void* const* dst_regions, const adha_layout* dst_layout,
                                        int64_t n_records, void* stream);

/* A chain of remaps on one stream (a PDL plan with several remap edges,
 * PAPER.md:146): buffers[k] holds the records in layouts[k];
 * for k = 0..n_layouts-2: remap buffers[k] (layouts[k]) -> buffers[k+1]
 * (layouts[k+1]).  Every intermediate is materialised.  Same rules as adha_remap.
 * Routes (adha_remap_chain_route tells which one a call takes):
 *   1 fused small  every hop <= ADHA_SMALL_BYTES of payload, <= 16 fields, <= 4 hops: ONE
 *                  launch of the direct chain kernel, a block-level barrier between hops
 *                  (ADHA_CHAIN_FUSE=0 disables it);
 *   2 fused tiled  opt-in (ADHA_CHAIN_TILED_BYTES = the payload per hop from which it applies;
 *                  unset or 0 = off): 2..8 hops, unit-mode plans of one unit size, >= eight tile
 *                  bands per SM: ONE launch of the tiled kernel in chain mode -- a CTA runs groups
 *                  of bands through every hop, so hop h reads hop h-1's output back from L2 while
 *                  it is still written to HBM (HBM traffic (H+1) * N * R instead of 2 * H * N * R
 *                  for H hops; about as fast as per hop on B200, whose SM side binds);
 *   0 per hop      one remap per hop, in order, on `stream`.
 * Both fused routes need packed unblocked layouts and pairwise disjoint buffers. */
ADHA_API adha_status adha_remap_chain(void* const* buffers, const adha_layout* const* layouts,
                             int32_t n_layouts, int64_t n_records, void* stream);

/* The route adha_remap_chain takes for these layouts and N with pairwise disjoint buffers:
 * *route = 0 per hop, 1 fused small, 2 fused tiled; *launches = kernel launches of the chain's
 * remap kernels (1 for the fused routes, n_layouts - 1 per hop).  Host only.
 * Errors: INVALID_ARG, LAYOUT_MISMATCH, TOO_LARGE. */
ADHA_API adha_status adha_remap_chain_route(const adha_layout* const* layouts, int32_t n_layouts,
                                          int64_t n_records, int32_t* route, int32_t* launches);

/* Contiguous shard of N records for shard g of G (reading Q10):
 *     lo = floor(g * N / G),  hi = floor((g + 1) * N / G).
 * Errors: INVALID_ARG (N < 0, G < 1, g outside [0, G)). */
ADHA_API adha_status adha_shard_range(int64_t n_total, int32_t n_shards, int32_t shard,
                             int64_t* lo, int64_t* hi);

/* Single-process multi-device remap.  Shard g holds records [lo_g, hi_g) of an
 * N-record array as its own layout instance of n_g = hi_g - lo_g records
 * (src_shards[g] in src_layout, dst_shards[g] in dst_layout, on device
 * device_ids[g]).  Launches adha_remap for every shard on streams[g] (as void*)
 * and restores the caller's current device.  No data crosses devices: record i
 * of the output depends only on record i of the input (record locality), so
 * the shards need no exchange.  Errors: as adha_remap, per shard. */
ADHA_API adha_status adha_remap_sharded(const void* const* src_shards, const adha_layout* src_layout,
                               void* const* dst_shards, const adha_layout* dst_layout,
                               int64_t n_records_total, int32_t n_shards,
                               const int32_t* device_ids, void* const* streams);

/* Cross-device remap fused with the transfer (NEXT N2; the paper's
 * remap edge crosses a device boundary; a device
 * change moves all common fields).  src (bytes(Ls, N), device memory of src_device)
 * is remapped into dst (bytes(Ld, N), device memory of dst_device) by ONE kernel
 * running on src_device whose 16-byte stores go straight into dst_device's HBM over
 * NVLink (peer access is enabled on first use and left enabled): no staging copy, the
 * transfer overlaps the permutation tile by tile.  With src_device == dst_device it is
 * adha_remap.  `stream` (void*, may be NULL) must belong to src_device.  The caller's
 * current device is restored.  Ownership and asynchrony as adha_remap.
 * Errors: as adha_remap; INVALID_ARG (device id out of range, a pointer not device
 * memory of the stated device); CUDA (the two devices cannot access each other). */
ADHA_API adha_status adha_remap_peer(const void* src, const adha_layout* src_layout, int32_t src_device,
                                     void* dst, const adha_layout* dst_layout, int32_t dst_device,
                                     int64_t n_records, void* stream);

/* End-to-end remap of HOST buffers through the current device: src_host holds
 * bytes(Ls, N), dst_host receives bytes(Ld, N) (only payload bytes written).
 * Strategy (ADHA_HOST_MODE = auto | hybrid | zero | staged; auto = zero when both host
 * buffers are pinned, 256-byte aligned and the src layout has >= 16 clusters (many small
 * H2D copies per chunk otherwise), else hybrid when dst_host is pinned, 256-byte aligned host
 * memory and a scratch is given, else staged):
 *   hybrid  record chunks (~16 MB) are copied host->device into `scratch` (one copy per
 *           src region, copy engine) and each chunk's remap kernel stores its records
 *           straight into dst_host over PCIe: H2D of chunk k+1 overlaps the kernel of k;
 *   zero    one remap kernel reads src_host and writes dst_host directly (both pinned);
 *   staged  H2D per src region, remap in `scratch`, D2H per dst region (pageable memory).
 * `scratch` is a DEVICE buffer of scratch_bytes, 256-byte aligned (may be NULL only
 * in zero mode).  Work is enqueued on internal streams ordered after prior work on
 * `stream`; later work on `stream` waits for completion.  Errors: as adha_remap;
 * INVALID_ARG if the scratch cannot hold a chunk of 4096 records. */
ADHA_API adha_status adha_remap_host(const void* src_host, const adha_layout* src_layout,
                            void* dst_host, const adha_layout* dst_layout,
                            int64_t n_records, void* scratch, uint64_t scratch_bytes,
                            void* stream);

/* ------------------------------------------------------------------ in-place remap
 *
 * The remap of adha_remap with src and dst in ONE device buffer (SURVEY.md 8(f) N1,
 * "in-place"; the paper's remap edge, names no storage, reading Q5):
 * after the call the buffer holds the N records in dst_layout,
 *     buf[addr_Ld(f, i) .. + w_f) = (old buf)[addr_Ls(f, i) .. + w_f)   for all i < N, f,
 * and every other byte of the buffer is unspecified.  The buffer needs
 * max(bytes(Ls, N), bytes(Ld, N)) bytes, not their sum, so an array that fills most of HBM
 * can still change layout.  Packed, unblocked layouts only (no ADHA_LAYOUT_ALIGNED, no
 * AoSoA blocks).  Cost: the buffer is cut into S-byte slots (S in 256..4096); tiles of
 * T = S/u records (u = largest power of two <= 16 dividing every width) of each cluster whose
 * member set changes are rewritten in place, every slot is moved along the cycles of a slot
 * permutation, and the dst tiles are rewritten back.  Clusters that keep their member set
 * and their region base move no byte (the moved-subset rule).  Buffers of at
 * most 16 MB (ADHA_INPLACE_STAGED_BYTES at plan creation) are instead remapped out of place
 * into the workspace and copied back ("staged" mode: the workspace then holds bytes(Ld, N)).
 *
 * Usage: plan = create(Ls, Ld, N) [host only]; upload(plan, workspace) once; then
 * adha_remap_inplace(buf, ...) any number of times (each call remaps the buffer's current
 * contents from Ls to Ld).  The workspace (device, 256-byte aligned, plan-sized, see
 * adha_inplace_plan_info) belongs to the plan while it is in use and must not overlap buf; it
 * also holds per-run scratch (saved slots, the tail), so two runs of one plan must not overlap
 * in time: order them on one stream, or give concurrent runs their own plan and workspace.
 * adha_inplace_plan_upload is not thread-safe with respect to other calls on the same plan. */
typedef struct adha_inplace_plan adha_inplace_plan;

/* Host-side plan (slot permutation, its cycles, workspace layout) for an N-record buffer.
 * Errors: INVALID_ARG (null, N < 0), LAYOUT_MISMATCH, TOO_LARGE, UNSUPPORTED (aligned or
 * blocked layout; a changed cluster record too wide for a tile in shared memory), OOM. */
ADHA_API adha_status adha_inplace_plan_create(const adha_layout* src_layout, const adha_layout* dst_layout,
                                              int64_t n_records, adha_inplace_plan** out);

/* buffer_bytes = max(bytes(Ls, N), bytes(Ld, N)); workspace_bytes = device workspace the plan
 * needs (tables, one saved slot per cycle segment, the packed tail records).  Either may be NULL. */
ADHA_API adha_status adha_inplace_plan_info(const adha_inplace_plan* plan, uint64_t* buffer_bytes,
                                            uint64_t* workspace_bytes);

/* JSON statistics of the plan (slot size, tile records, moved / fixed slots, cycles, segments,
 * device traffic of one run); free with adha_free. */
ADHA_API adha_status adha_inplace_plan_describe(const adha_inplace_plan* plan, char** json_out);

/* Copy the plan's tables into `workspace` (device memory of the current device) on `stream`
 * and wait for the copy.  Errors: INVALID_ARG (null, workspace too small), ALIGNMENT, CUDA. */
ADHA_API adha_status adha_inplace_plan_upload(adha_inplace_plan* plan, void* workspace, uint64_t workspace_bytes,
                                              void* stream);

/* Enqueue the in-place remap of `buf` (device, 256-byte aligned, buf_bytes >= buffer_bytes)
 * on `stream` (up to 6 kernel launches; allocates nothing).  Asynchronous like adha_remap.
 * Errors: INVALID_ARG (null, buffer too small, plan not uploaded to this workspace on the
 * current device), ALIGNMENT, OVERLAP (workspace inside the buffer), CUDA. */
ADHA_API adha_status adha_remap_inplace(void* buf, uint64_t buf_bytes, const adha_inplace_plan* plan,
                                        void* workspace, void* stream);

/* Destroy a plan.  NULL is ok. */
ADHA_API void adha_inplace_plan_destroy(adha_inplace_plan* plan);

/* JSON description of the compiled remap plan for a layout pair (tile records,
 * pipeline stages, unit size, per-instruction table, kernel choice) -- for
 * tests and tooling; the hot path never calls it.  Free with adha_free. */
ADHA_API adha_status adha_remap_plan_describe(const adha_layout* src_layout, const adha_layout* dst_layout,
                                     char** json_out);

/* The same for the MERGED plan of the pair (merged != 0: every cluster in one component, the
 * plan adha_remap runs for multi-component remaps of up to ADHA_MERGE_BYTES), or for the
 * component plan (merged == 0, = adha_remap_plan_describe). */
ADHA_API adha_status adha_remap_plan_describe_ex(const adha_layout* src_layout, const adha_layout* dst_layout,
                                               int32_t merged, char** json_out);

/* ------------------------------------------------------------------ planner (host)
 *
 * Inputs are UTF-8 JSON documents in the SPEC.md schemas (schema_version 1):
 *   program  {"record_count", "fields":[{"name","elem_bytes"}], "sections":[{"id",
 *             "trip_count", "allowed_devices", "groups":[{"fields","freq","pattern","ops"}]}],
 *             "order"}
 *   arch     {"devices":[{"name","line_bytes","line_time_ns","throughput_ops_per_ns",
 *             "coalescing","stream_cluster_penalty","cluster_capacity_bytes"}],
 *             "links":[{"from","to","bandwidth_bytes_per_ns","latency_ns"}],
 *             "same_device_remap_bandwidth_bytes_per_ns","remap_fixed_overhead_ns"}
 *   profile  [{"section","device","layout","time_ns"}] or {"entries":[...]}
 */

/* ODS of one section on one device: affinity graph, Kruskal
 * greedy clustering under the device's cluster capacity, untouched fields as
 * singletons.  *layout_out = canonical string (adha_free).
 * Errors: PARSE, PLANNER (unknown section/device, device not allowed),
 * CAPACITY (a field wider than the capacity). */
ADHA_API adha_status adha_plan_ods(const char* program_json, const char* arch_json,
                          const char* section_id, const char* device, char** layout_out);

/* PDL: run graph over contiguous section runs x devices, run
 * layouts from ODS of the merged run, remap edges = moved bytes / bandwidth +
 * overhead, shortest path.  *plan_out = JSON
 * {"runs":[{"sections","device","layout","exec_ns"}],
 *  "remaps":[{"boundary","after","moved","cost_ns"}], "total_ns"}.
 * profile_json may be NULL.  Errors: PARSE, PLANNER, CAPACITY. */
ADHA_API adha_status adha_plan_pdl(const char* program_json, const char* arch_json,
                          const char* profile_json, char** plan_out);

/* The run graph's nodes ([OP] build_run_graph): every contiguous run of
 * sections x every device allowed by all its members, with the run's layout (ODS of the
 * merged run) and its execution estimate under `profile_json` (nullable).
 * *runs_out = {"runs":[{"begin","end","sections","device","layout","exec_ns"}]} (adha_free).
 * Used to know which (section, device, layout) triples a tuning profile must cover
 * (PAPER.md:59-60).  Errors: PARSE, PLANNER, CAPACITY. */
ADHA_API adha_status adha_plan_candidates(const char* program_json, const char* arch_json,
                                          const char* profile_json, char** runs_out);

/* ------------------------------------------------------------------ synthetic consumer sections
 *
 * A section kernel reading records THROUGH a layout, for measuring a B200 tuning profile
 * ("we provide a tuning profile of the execution times").
 * For i in [0, n_out): r = idx ? idx[i] : i;  out[i] = sum over the listed fields f of x_f(r)^2,
 * fields read as fp32 (width 4, 4-byte aligned in the layout) and summed in list order with
 * fused multiply-add.  idx == NULL is a streaming pass over records 0..n_out-1 (a vectorizable
 * section); idx != NULL is an irregular gather (heavy control flow).
 *   buf        DEVICE buffer holding n_records records in `layout` (256-byte aligned)
 *   fields     host array of n_fields_used field indices (1..32)
 *   idx        DEVICE array of n_out record indices in [0, n_records), or NULL
 *   out        DEVICE float array of n_out
 * Asynchronous on `stream`.  Errors: INVALID_ARG, UNSUPPORTED (field not fp32-addressable), CUDA. */
ADHA_API adha_status adha_section_run(const void* buf, const adha_layout* layout, int64_t n_records,
                                      const int32_t* fields, int32_t n_fields_used, const int64_t* idx,
                                      int64_t n_out, float* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ADHA_H_ */
