/*
 * fmgpu.h — C ABI of the B200-native FM-index Occ / backward-search engine.
 *
 * Drop-in boundary for the hot path of the reference package `fmpm`
 * (/root/reference/pkg/src/fmpm).  The reference's only plugin boundary is the
 * per-bucket kernel registry (kernels.py:295-350: `all4(block, prefix_len)`),
 * one 32-byte bucket per call; a GPU launch per ~100 ns of memory work would be
 * pointless, so this ABI replaces the INDEX-LEVEL functions those plugins serve
 * with batched entry points over a device-resident index:
 *
 *   fmg_index_create   <- serialize.py:87-92 bucket records / index.py:24-54
 *   fmg_occ_pair       <- occ.py:59-96   occ_pair_all(index, k-1, l)
 *   fmg_exact*         <- search.py:74-94  exact_search (+ init_interval 50-57,
 *                                          extend_backward 60-71)
 *   fmg_inexact*       <- search.py:97-159 inexact_search
 *   fmg_psi_inverse    <- search.py:172-186 psi_inverse_fused
 *   fmg_locate_rows    <- search.py:189-208 locate_row
 *   fmg_reconstruct_text <- search.py:270-286 reconstruct_reference
 *
 * Conventions
 *   - Plain pointers and sizes only; no C++ or torch types.
 *   - Rows and positions are uint32 (the engine rejects n + 1 >= 2^32 - 1).
 *   - Entry points without the _host suffix take DEVICE pointers and are
 *     asynchronous on `stream` (a cudaStream_t, NULL = legacy default stream);
 *     the caller owns every buffer and synchronises.
 *   - Entry points with the _host suffix take HOST pointers (pinned or pageable)
 *     and return after the results are in host memory.
 *   - Every function returns an fmg_status; the message of the last failure on
 *     the calling thread is available from fmg_last_error().  No exception
 *     crosses this boundary.
 *   - Input errors are reported PER CALL.  _host entry points return
 *     FMG_EINVAL for a bad position or row (the reference raises ValueError,
 *     occ.py:68-79, search.py:199-200).  Device entry points that take a
 *     `status` argument validate on the device and OR error bits into that
 *     caller-owned device word (1 = position / row out of range or pair out
 *     of order, 2 = predecessor walk did not terminate: corrupt index); the
 *     caller zeroes it before the call and reads it after synchronising.
 *     status == NULL makes the call unchecked: bad queries yield zeros and
 *     are not reported.  No state is shared between calls.
 */
#ifndef FMGPU_H
#define FMGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum fmg_status {
  FMG_OK = 0,
  FMG_EINVAL = 1,    /* invalid argument (reference: ValueError)            */
  FMG_ECAPACITY = 2, /* output capacity exceeded                            */
  FMG_ECUDA = 3,     /* CUDA runtime failure; see fmg_last_error()          */
  FMG_ENOMEM = 4,    /* host or device allocation failed                    */
  FMG_EINTERNAL = 5  /* any other internal failure                          */
} fmg_status;

typedef struct fmg_index fmg_index;     /* device-resident index (immutable) */
typedef struct fmg_matches fmg_matches; /* result set of an inexact search   */

/* Thread-local text of the last failure on this thread ("" if none). */
const char* fmg_last_error(void);

/* Number of visible CUDA devices (0 on a host without a GPU). */
int fmg_device_count(int* count);

/* ---------------------------------------------------------------------------
 * Index construction (host, no GPU needed).  Replaces suffix.py:21-71 and
 * index.py:67-101.  fmb_build fills exactly the arrays .fmi v1 stores:
 *   bucket_records: ceil((n+1)/128) x 64 bytes (4 x u64 LE base, 32 B chars)
 *   sa_samples:     n/32 + 1 entries (suffix-array rows 0, 32, 64, ...)
 *   c:              5 entries, c[4] == n
 * `codes` holds n symbol codes in [0, 4) (A, C, G, T).
 * ------------------------------------------------------------------------- */
int fmb_suffix_array(const uint8_t* codes, uint64_t n, uint32_t* sa_out /* n+1 */);
int fmb_build(const uint8_t* codes, uint64_t n, uint8_t* bucket_records, uint64_t* sa_samples,
              uint64_t* c, uint64_t* sentinel_row, int nthreads);
/* Same outputs, built on GPU `device` (prefix doubling + radix sort in HBM,
 * ~36 bytes of device memory per character).  `codes` is a HOST pointer;
 * sa_out (n+1 entries, host) may be NULL. */
int fmb_build_gpu(int device, const uint8_t* codes, uint64_t n, uint8_t* bucket_records,
                  uint64_t* sa_samples, uint64_t* c, uint64_t* sentinel_row, uint32_t* sa_out);

/* ---------------------------------------------------------------------------
 * Device index.
 * fmg_index_create uploads the .fmi bucket records (serialize.py:87-92) to
 * `device` and re-lays them out on the GPU as 32-byte lines of 64 characters,
 * each with its own u32 checkpoint, so every Occ position costs one sector.
 * ------------------------------------------------------------------------- */
int fmg_index_create(int device, const void* bucket_records, uint64_t n_buckets, uint64_t n,
                     uint64_t sentinel_row, const uint64_t c[5], fmg_index** out);
/* Optional index of the REVERSED text (its .fmi bucket records and sentinel
 * row; same n and C).  With it attached, fmg_inexact[_packed] at
 * max_diff = 1 runs the bidirectional engine (identical results, fewer Occ
 * steps: each half of the pattern is matched exactly before the edit is
 * placed in the other half).  No reference counterpart (an engine cache). */
int fmg_index_set_reverse(fmg_index* index, const void* bucket_records, uint64_t n_buckets,
                          uint64_t sentinel_row);
int fmg_index_has_reverse(const fmg_index* index, int* has);
/* Suffix-array samples for locate (index.py:93); count must be n/32 + 1. */
int fmg_index_set_samples(fmg_index* index, const uint64_t* sa_samples, uint64_t count);
/* n, the device ordinal and the device bytes the handle owns. */
int fmg_index_info(const fmg_index* index, uint64_t* n, int* device, uint64_t* device_bytes);
void fmg_index_destroy(fmg_index* index);

/* ---------------------------------------------------------------------------
 * Occ step (occ.py:59-96).  For pair i, kl[2i] = k, kl[2i+1] = l; the eight
 * outputs are Occ(b, k-1) for b = A,C,G,T then Occ(b, l) for b = A,C,G,T.
 * k == 0 means k-1 == -1 and gives zeros (occ.py:74-77).  Requires
 * k <= l + 1 and l <= n.
 * ------------------------------------------------------------------------- */
int fmg_occ_pair(const fmg_index* index, const uint32_t* kl, uint64_t count, uint32_t* out,
                 uint32_t* status, void* stream);
int fmg_occ_pair_host(const fmg_index* index, const uint32_t* kl, uint64_t count, uint32_t* out);

/* ---------------------------------------------------------------------------
 * Exact backward search (search.py:74-94).  Output kl_out[2i] = k,
 * kl_out[2i+1] = l of the interval exact_search returns, INCLUDING the first
 * empty interval (l+1, l) at which the search stopped.
 * General form: codes in [0,4), pattern i = codes[offsets[i] .. offsets[i+1]),
 * every pattern non-empty.  Packed form: fixed length 1 <= m <= 32, pattern i
 * in packed[i], character j in bits 2j..2j+1.
 * ------------------------------------------------------------------------- */
int fmg_exact(const fmg_index* index, const uint8_t* codes, const uint64_t* offsets,
              uint64_t count, uint32_t* kl_out, void* stream);
int fmg_exact_packed(const fmg_index* index, const uint64_t* packed, uint32_t m, uint64_t count,
                     uint32_t* kl_out, void* stream);
int fmg_exact_host(const fmg_index* index, const uint8_t* codes, const uint64_t* offsets,
                   uint64_t count, uint32_t* kl_out);
int fmg_exact_packed_host(const fmg_index* index, const uint64_t* packed, uint32_t m,
                          uint64_t count, uint32_t* kl_out);

/* ---------------------------------------------------------------------------
 * Bounded-difference search (search.py:97-159): every (k, l) reachable with
 * at most `max_diff` skips / inserts / mismatches, deduplicated keeping the
 * smallest difference count, sorted by (k, l, diffs) per pattern.  Patterns
 * as in fmg_exact (device or host pointers respectively).  The result set is
 * owned by an fmg_matches handle; copy it out with fmg_matches_copy.
 * ------------------------------------------------------------------------- */
int fmg_inexact(const fmg_index* index, const uint8_t* codes, const uint64_t* offsets,
                uint64_t count, int max_diff, fmg_matches** out, void* stream);
int fmg_inexact_host(const fmg_index* index, const uint8_t* codes, const uint64_t* offsets,
                     uint64_t count, int max_diff, fmg_matches** out);
/* Whether a bounded-difference call of `count` patterns of at most `max_len`
 * characters would use the reverse index (fmg_index_set_reverse) if one were
 * attached: 1 for the bidirectional engines, 0 when another engine takes the
 * batch (small batches, max_diff != 1, or the flat one-edit engine of
 * HBM-resident indexes, which needs none).  Lets the host skip building and
 * uploading a reverse index nobody reads (13 GB on the device at 3.1 Gbp).
 * May build the index's prefix / k-mer tables (the search needs them anyway). */
int fmg_inexact_wants_reverse(const fmg_index* index, uint64_t count, uint64_t max_len,
                              int max_diff, int* wants);
/* Fixed-length patterns (1 <= m <= 32) packed as in fmg_exact_packed. */
int fmg_inexact_packed(const fmg_index* index, const uint64_t* packed, uint32_t m, uint64_t count,
                       int max_diff, fmg_matches** out, void* stream);
int fmg_inexact_packed_host(const fmg_index* index, const uint64_t* packed, uint32_t m,
                            uint64_t count, int max_diff, fmg_matches** out);
/* Total number of (k, l, diffs) results and the number of patterns. */
int fmg_matches_size(const fmg_matches* m, uint64_t* total, uint64_t* patterns);
/* Occ steps the search executed (work counter, for reporting). */
int fmg_matches_steps(const fmg_matches* m, uint64_t* steps);
/* CSR copy-out: row_offsets has patterns+1 entries; k, l, diffs have `total`.
 * to_host != 0: destination pointers are host memory, else device memory. */
int fmg_matches_copy(const fmg_matches* m, uint64_t* row_offsets, uint32_t* k, uint32_t* l,
                     uint8_t* diffs, int to_host);
/* Releases the result buffers, stream-ordered on the stream the search ran on
 * (that stream must still exist). */
void fmg_matches_free(fmg_matches* m);

/* ---------------------------------------------------------------------------
 * Position recovery.
 * fmg_psi_inverse: for row i, out_sym[i] = BWT symbol at row i and
 * out_row[i] = predecessor row (search.py:172-186); at the sentinel row
 * out_sym = 255 and out_row = 0xFFFFFFFF (the reference returns None).
 * fmg_locate_rows: text position of each row (search.py:189-208); requires
 * fmg_index_set_samples.
 * ------------------------------------------------------------------------- */
int fmg_psi_inverse(const fmg_index* index, const uint32_t* rows, uint64_t count,
                    uint8_t* out_sym, uint32_t* out_row, uint32_t* status, void* stream);
int fmg_locate_rows(const fmg_index* index, const uint32_t* rows, uint64_t count,
                    uint32_t* out_pos, uint32_t* status, void* stream);
int fmg_locate_rows_host(const fmg_index* index, const uint32_t* rows, uint64_t count,
                         uint32_t* out_pos);

/* reconstruct_reference (search.py:270-286): the n text codes (0..3) the
 * index was built from, recovered on the GPU by walking the predecessor cycle
 * from every sampled row in parallel (~32 steps each); requires
 * fmg_index_set_samples.  status bit 2 = corrupt index. */
int fmg_reconstruct_text(const fmg_index* index, uint8_t* codes_out /* device, n */, uint32_t* status,
                         void* stream);
int fmg_reconstruct_text_host(const fmg_index* index, uint8_t* codes_out /* host, n */);

/* ---------------------------------------------------------------------------
 * Bucket-level rank kernels: the reference's per-bucket plugin surface
 * (kernels.py:125-292, count_bucket_* / count_bucket_all4 / mask_bucket) as
 * batched kernels.  blocks: count x 32 packed bytes (128 fields, reference
 * bit order), 32-byte aligned; prefix_lens in [0, 128]; symbols in [0, 4) or
 * NULL for all four counts (out: count x 4 u32 in A, C, G, T order, else
 * count x 1).  method 0 = masked popcount (scalar / bytelut / auto), 1 = the
 * paper's nibble pipeline (PRMT table lookups + SAD; nibble / simd).
 * Device form: device pointers on the CURRENT device, `status` as above.
 * Host forms run on `device` and return FMG_EINVAL for a bad prefix / symbol.
 * fmg_bucket_nibble_trace_host writes 15 u64 per query (KernelTrace,
 * kernels.py:101-115): masked words[4], lookup lo words[4], lookup hi
 * words[4], group SADs (16 bits each), sad_total | raw_count << 32, count.
 * ------------------------------------------------------------------------- */
int fmg_bucket_count(const uint8_t* blocks, const uint32_t* prefix_lens, const uint8_t* symbols,
                     uint64_t count, int method, uint32_t* out, uint32_t* status, void* stream);
int fmg_bucket_count_host(int device, const uint8_t* blocks, const uint32_t* prefix_lens,
                          const uint8_t* symbols, uint64_t count, int method, uint32_t* out);
int fmg_bucket_mask_host(int device, const uint8_t* blocks, const uint32_t* prefix_lens, uint64_t count,
                         uint8_t* out);
int fmg_bucket_nibble_trace_host(int device, const uint8_t* blocks, const uint32_t* prefix_lens,
                                 const uint8_t* symbols, uint64_t count, uint64_t* trace);

/* Blocks until all work the library queued on `stream` has finished. */
int fmg_stream_sync(void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FMGPU_H */
