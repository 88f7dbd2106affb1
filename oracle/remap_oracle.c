/*
 * oracle/remap_oracle.c -- CPU ORACLE FOR THE ADHA LAYOUT REMAP.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1407_4859_b200/) never includes, links or calls it,
 * and this file includes nothing from the product tree.
 *
 * What it computes (SURVEY.md 8(c) c1 -- the plain definition):
 *   for every record i in [0, N) and every field f:
 *     dst[addr_Ld(f,i) .. +w_f) = src[addr_Ls(f,i) .. +w_f)
 *   with the element address of SPEC.md:363 ([OP] simulate_misses):
 *     addr_L(f,i) = base(cluster_L(f)) + i * bytes(cluster_L(f)) + offset(f within cluster)
 *
 * Readings it follows (listed in DESIGN.md "Readings"):
 *   - a layout is a partition of the fields into clusters; canonical order:
 *     clusters by minimum decl_index, fields in a cluster by decl_index
 *     ([TYPE] Layout; Table 2);
 *   - cluster records are packed, no padding: bytes(c) = sum of widths
 *     (reading Q2);
 *   - clusters occupy disjoint regions of one buffer, placed in
 *     canonical cluster order, each region base aligned up to 256 bytes from
 *     the buffer start (reading Q3);  bytes outside regions are never written;
 *   - the remap is a type-blind byte copy (reading Q6): NaN payloads survive.
 *
 * Generalised layouts (beyond the paper, which "consider[s] only
 * AoS and SoA"), in the *_ex functions:
 *   - natural alignment (flags bit 0, C-struct rule): a field of width w starts at a
 *     multiple of a(w) = the largest power of two dividing w, at most 8; the cluster
 *     record stride is rounded up to the largest a(w) of its fields;
 *   - AoSoA blocking: a cluster with block B (1, 2, 4, 8, 16 or 32) stores its records
 *     in blocks of B, each field's B values contiguous inside the block:
 *       addr(f, i) = base + (i / B) * (B * stride) + offset(f) * B + (i % B) * w_f ,
 *     and its region holds ceil(N / B) whole blocks;
 *   - every byte of a dst region that is not a field byte of a record < N (alignment
 *     padding, slots past N in the last block) is written 0.
 *
 * Everything is a plain loop of memcpy, in the order of the definition.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define ORACLE_OK 0
#define ORACLE_BAD 1

/* Per-field addressing derived from (widths, partition) for a layout of N records. */
typedef struct {
    uint64_t base;    /* region base of the field's cluster, bytes from buffer start */
    uint64_t stride;  /* bytes(cluster) = record stride within the region            */
    uint64_t offset;  /* offset of the field inside one cluster record               */
} oracle_addr;

static uint64_t align_up_256(uint64_t x) { return (x + 255u) & ~(uint64_t)255u; }

/*
 * Canonical cluster index of every field.  Fields are visited in decl order
 * (index 0..F-1); the first time a label is seen is at its cluster's minimum
 * decl_index, so numbering clusters in order of first sight sorts clusters by
 * minimum decl_index.  Returns the number of clusters, or -1.
 */
static int canonical_clusters(int n_fields, const int32_t* label, int32_t* canon)
{
    int n_clusters = 0;
    for (int f = 0; f < n_fields; ++f) {
        int found = -1;
        for (int g = 0; g < f; ++g) {
            if (label[g] == label[f]) { found = canon[g]; break; }
        }
        if (found < 0) found = n_clusters++;
        canon[f] = found;
    }
    return n_clusters;
}

/*
 * addr[f] for a layout of n_records records.  Returns the total buffer bytes
 * (end of the last region) in *total_bytes.
 */
int oracle_field_addresses(int n_fields, const uint32_t* widths, const int32_t* cluster_of,
                           int64_t n_records, oracle_addr* addr, uint64_t* total_bytes)
{
    if (n_fields <= 0 || n_records < 0 || !widths || !cluster_of || !addr) return ORACLE_BAD;
    int32_t* canon = (int32_t*)malloc(sizeof(int32_t) * (size_t)n_fields);
    if (!canon) return ORACLE_BAD;
    int n_clusters = canonical_clusters(n_fields, cluster_of, canon);

    uint64_t base = 0;
    for (int c = 0; c < n_clusters; ++c) {
        /* bytes(c) and the offsets of its fields, in decl order (packed) */
        uint64_t stride = 0;
        for (int f = 0; f < n_fields; ++f) {
            if (canon[f] == c) {
                addr[f].offset = stride;
                stride += widths[f];
            }
        }
        if (c > 0) base = align_up_256(base);
        for (int f = 0; f < n_fields; ++f) {
            if (canon[f] == c) {
                addr[f].base = base;
                addr[f].stride = stride;
            }
        }
        base += (uint64_t)n_records * stride;
    }
    if (total_bytes) *total_bytes = base;
    free(canon);
    return ORACLE_OK;
}

uint64_t oracle_layout_bytes(int n_fields, const uint32_t* widths, const int32_t* cluster_of,
                             int64_t n_records)
{
    oracle_addr* a = (oracle_addr*)malloc(sizeof(oracle_addr) * (size_t)n_fields);
    uint64_t total = 0;
    if (a && oracle_field_addresses(n_fields, widths, cluster_of, n_records, a, &total) != ORACLE_OK)
        total = 0;
    free(a);
    return total;
}

/*
 * The remap of records [lo, hi) of an N-record layout instance:
 * for i in [lo, hi): for f: memcpy(dst + addr_d(f,i), src + addr_s(f,i), w_f).
 */
int oracle_remap_range(const uint8_t* src, const int32_t* src_cluster_of,
                       uint8_t* dst, const int32_t* dst_cluster_of,
                       int n_fields, const uint32_t* widths,
                       int64_t n_records, int64_t lo, int64_t hi)
{
    if (!src || !dst || lo < 0 || hi > n_records || lo > hi) return ORACLE_BAD;
    oracle_addr* as = (oracle_addr*)malloc(sizeof(oracle_addr) * (size_t)n_fields);
    oracle_addr* ad = (oracle_addr*)malloc(sizeof(oracle_addr) * (size_t)n_fields);
    int rc = ORACLE_BAD;
    if (as && ad &&
        oracle_field_addresses(n_fields, widths, src_cluster_of, n_records, as, NULL) == ORACLE_OK &&
        oracle_field_addresses(n_fields, widths, dst_cluster_of, n_records, ad, NULL) == ORACLE_OK) {
        for (int64_t i = lo; i < hi; ++i) {
            for (int f = 0; f < n_fields; ++f) {
                const uint8_t* s = src + as[f].base + (uint64_t)i * as[f].stride + as[f].offset;
                uint8_t* d = dst + ad[f].base + (uint64_t)i * ad[f].stride + ad[f].offset;
                memcpy(d, s, widths[f]);
            }
        }
        rc = ORACLE_OK;
    }
    free(as);
    free(ad);
    return rc;
}

int oracle_remap(const uint8_t* src, const int32_t* src_cluster_of,
                 uint8_t* dst, const int32_t* dst_cluster_of,
                 int n_fields, const uint32_t* widths, int64_t n_records)
{
    return oracle_remap_range(src, src_cluster_of, dst, dst_cluster_of, n_fields, widths,
                              n_records, 0, n_records);
}

/*
 * The same loop split into contiguous record ranges over n_threads POSIX
 * threads (record locality: record i of dst depends only on record i of src).
 * Used only to time the oracle on all host cores (bench.py cpu_baseline).
 */
typedef struct {
    const uint8_t* src; const int32_t* sc; uint8_t* dst; const int32_t* dc;
    int n_fields; const uint32_t* widths; int64_t n; int64_t lo, hi; int rc;
} oracle_job;

static void* oracle_worker(void* p)
{
    oracle_job* j = (oracle_job*)p;
    j->rc = oracle_remap_range(j->src, j->sc, j->dst, j->dc, j->n_fields, j->widths, j->n, j->lo, j->hi);
    return NULL;
}

int oracle_remap_threads(const uint8_t* src, const int32_t* src_cluster_of,
                         uint8_t* dst, const int32_t* dst_cluster_of,
                         int n_fields, const uint32_t* widths,
                         int64_t n_records, int64_t lo, int64_t hi, int n_threads)
{
    if (n_threads < 1) n_threads = 1;
    oracle_job* jobs = (oracle_job*)calloc((size_t)n_threads, sizeof(oracle_job));
    pthread_t* th = (pthread_t*)calloc((size_t)n_threads, sizeof(pthread_t));
    if (!jobs || !th) { free(jobs); free(th); return ORACLE_BAD; }
    int64_t span = hi - lo;
    for (int t = 0; t < n_threads; ++t) {
        oracle_job* j = &jobs[t];
        j->src = src; j->sc = src_cluster_of; j->dst = dst; j->dc = dst_cluster_of;
        j->n_fields = n_fields; j->widths = widths; j->n = n_records;
        j->lo = lo + span * t / n_threads;
        j->hi = lo + span * (t + 1) / n_threads;
        pthread_create(&th[t], NULL, oracle_worker, j);
    }
    int rc = ORACLE_OK;
    for (int t = 0; t < n_threads; ++t) {
        pthread_join(th[t], NULL);
        if (jobs[t].rc != ORACLE_OK) rc = ORACLE_BAD;
    }
    free(jobs);
    free(th);
    return rc;
}

/* ------------------------------------------------------------------ generalised layouts */

typedef struct {
    uint64_t base, stride, offset, block, width, region_bytes;
} oracle_addr_ex;

static uint64_t natural_align(uint64_t w)
{
    uint64_t a = 1;
    while (a < 8 && w % (a * 2) == 0) a *= 2;
    return a;
}

/*
 * Generalised addresses.  block_of[f] (NULL = all 1) must be equal for the fields of one
 * cluster; flags bit 0 = natural alignment.  Returns ORACLE_BAD on invalid input.
 */
int oracle_field_addresses_ex(int n_fields, const uint32_t* widths, const int32_t* cluster_of,
                              const int32_t* block_of, uint32_t flags, int64_t n_records,
                              oracle_addr_ex* addr, uint64_t* total_bytes)
{
    if (n_fields <= 0 || n_records < 0 || !widths || !cluster_of || !addr) return ORACLE_BAD;
    int32_t* canon = (int32_t*)malloc(sizeof(int32_t) * (size_t)n_fields);
    if (!canon) return ORACLE_BAD;
    int n_clusters = canonical_clusters(n_fields, cluster_of, canon);
    uint64_t base = 0;
    int rc = ORACLE_OK;
    for (int c = 0; c < n_clusters && rc == ORACLE_OK; ++c) {
        uint64_t run = 0, maxa = 1, blk = 0;
        for (int f = 0; f < n_fields; ++f) {
            if (canon[f] != c) continue;
            uint64_t b = block_of ? (uint64_t)block_of[f] : 1;
            if (blk == 0) blk = b;
            if (b != blk || !(b == 1 || b == 2 || b == 4 || b == 8 || b == 16 || b == 32)) rc = ORACLE_BAD;
            if (flags & 1u) {
                uint64_t a = natural_align(widths[f]);
                if (a > maxa) maxa = a;
                run = (run + a - 1) / a * a;
            }
            addr[f].offset = run;
            addr[f].width = widths[f];
            run += widths[f];
        }
        uint64_t stride = (run + maxa - 1) / maxa * maxa;
        uint64_t nblocks = ((uint64_t)n_records + blk - 1) / blk;
        if (c > 0) base = align_up_256(base);
        for (int f = 0; f < n_fields; ++f) {
            if (canon[f] != c) continue;
            addr[f].base = base;
            addr[f].stride = stride;
            addr[f].block = blk;
            addr[f].region_bytes = nblocks * blk * stride;
        }
        base += nblocks * blk * stride;
    }
    if (total_bytes) *total_bytes = base;
    free(canon);
    return rc;
}

static uint64_t addr_ex(const oracle_addr_ex* a, uint64_t i)
{
    return a->base + (i / a->block) * (a->block * a->stride) + a->offset * a->block + (i % a->block) * a->width;
}

/*
 * Generalised remap of records [lo, hi): dst regions of the records' blocks are first set to
 * zero (all of them when lo == 0 and hi == N), then every field byte is copied.
 */
int oracle_remap_ex(const uint8_t* src, const int32_t* src_cluster_of, const int32_t* src_block_of,
                    uint32_t src_flags, uint8_t* dst, const int32_t* dst_cluster_of,
                    const int32_t* dst_block_of, uint32_t dst_flags, int n_fields, const uint32_t* widths,
                    int64_t n_records)
{
    if (!src || !dst) return ORACLE_BAD;
    oracle_addr_ex* as = (oracle_addr_ex*)malloc(sizeof(oracle_addr_ex) * (size_t)n_fields);
    oracle_addr_ex* ad = (oracle_addr_ex*)malloc(sizeof(oracle_addr_ex) * (size_t)n_fields);
    int rc = ORACLE_BAD;
    if (as && ad &&
        oracle_field_addresses_ex(n_fields, widths, src_cluster_of, src_block_of, src_flags, n_records, as, NULL) ==
            ORACLE_OK &&
        oracle_field_addresses_ex(n_fields, widths, dst_cluster_of, dst_block_of, dst_flags, n_records, ad, NULL) ==
            ORACLE_OK) {
        /* 1. every byte of every dst region := 0 */
        for (int f = 0; f < n_fields; ++f) memset(dst + ad[f].base, 0, ad[f].region_bytes);
        /* 2. the field bytes of every record */
        for (int64_t i = 0; i < n_records; ++i)
            for (int f = 0; f < n_fields; ++f)
                memcpy(dst + addr_ex(&ad[f], (uint64_t)i), src + addr_ex(&as[f], (uint64_t)i), widths[f]);
        rc = ORACLE_OK;
    }
    free(as);
    free(ad);
    return rc;
}
