/*
 * ams_b200.h — C ABI of the B200-native AMS-sort hot path.
 *
 * The reference (`mlpsort`, pure Python) exposes this path only as the
 * Python function
 *     ams_sort(net, data, params, scheme, seed) -> (dict[pe] -> list, reports)
 * (/root/reference/pkg/src/mlpsort/ams.py:271-313).  There is no native
 * FFI in the reference; this header is the boundary a binding would load
 * (ctypes stub in INTEGRATION.md, used by paper_1410_6754_b200/_lib.py).
 * Plain C types only: device buffers are `void*` / `uint64_t*` device
 * pointers, small per-level metadata are host arrays.
 *
 * Every function returns AMS_OK (0) or an error code; ams_last_error()
 * returns the thread-local message.  Error classes follow the reference:
 * AMS_EINVAL maps to Python ValueError (ams.py:45-52, 61-65, 164-165,
 * 186-187, 206-207), AMS_ECUDA / AMS_EINTERNAL to RuntimeError
 * (fastsort.py:128-129, delivery.py:104-105, simnet.py:190-191).
 * Nothing here prints or exits.
 */
#ifndef AMS_B200_H
#define AMS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AMS_OK 0
#define AMS_EINVAL 1
#define AMS_ECUDA 2
#define AMS_ENOMEM 3
#define AMS_EINTERNAL 4

/* Key encodings: kernels compare keys as uint64 after an order-preserving
 * map (uint64: identity, int64: sign flip, float64: sign-flip transform).
 * The reference's keys are Python ints from getrandbits(64)
 * (bench.py:159-164) — AMS_KEY_U64. */
#define AMS_KEY_U64 0
#define AMS_KEY_I64 1
#define AMS_KEY_F64 2

/* Kernel tile (elements per CTA tile in the level kernels) and the
 * largest bucket the CTA-local final sort handles in shared memory. */
#define AMS_TILE 4096
#define AMS_SMEM_SORT_CAP 4096
/* capacity of the fixed-capacity digit cells of the keys-only final sort */
#define AMS_FX_CAP 2048
#define AMS_MAX_BUCKETS 4096

const char* ams_last_error(void);
int ams_version(void);

/* ------------------------------------------------------------------ */
/* Host helpers (no GPU needed).                                       */

/* SeedSpec(master_seed, stream_id).rng() seeding (core.py:62-67): the
 * 32-bit words CPython's random_seed() feeds init_by_array, least
 * significant first; *out_nwords = number of words used (1..4). */
int ams_stream_seed(int64_t master_seed, const char* stream_id, uint32_t out_words[4],
                    int* out_nwords);
/* hashlib.blake2b(msg, digest_size=16).digest() (core.py:64). */
int ams_blake2b_128(const uint8_t* msg, uint64_t len, uint8_t out[16]);
/* sorted(random.Random(seed).sample(range(n), k)) (ams.py:171-173). */
int ams_sample_indices(const uint32_t* seed_words, int nwords, uint64_t n, uint64_t k,
                       uint64_t* out);
/* `count` successive Random(seed).getrandbits(k), 1 <= k <= 64. */
int ams_mt_getrandbits(const uint32_t* seed_words, int nwords, int k, uint64_t count,
                       uint64_t* out);
/* draw_sample (ams.py:157-175) for all groups of one level; see seeds.cpp. */
int ams_draw_sample_positions(int64_t master_seed, const char* stream, int level,
                              int ngroups, const int32_t* group_first, const int32_t* group_npe,
                              const uint64_t* targets, const uint64_t* sizes,
                              const uint64_t* offs, uint64_t capacity, uint64_t* out_idx,
                              uint64_t* out_gpos, uint64_t* out_group_count);
/* scan_groups (ams.py:112-116): AMS_OK if feasible, 1 if not. */
int ams_scan_groups(const uint64_t* sizes, int nb, int r, uint64_t limit,
                    uint64_t* out_boundaries, uint64_t* out_loads, uint64_t* out_max_load);
/* optimal_group_plan (ams.py:119-154). */
int ams_group_plan(const uint64_t* sizes, int nb, int r, uint64_t* out_boundaries,
                   uint64_t* out_loads, uint64_t* out_max_load);
/* Host half of ams_level for all groups of a level (ams.py:231-258 +
 * delivery.py:78-180): plans, next-level member sizes, exchange stats. */
int ams_plan_level(int ngroups, const int32_t* group_npe, const int32_t* group_nb, int r,
                   const uint32_t* seg_hist, int nb_stride, uint64_t* out_boundaries,
                   uint64_t* out_loads, uint64_t* out_max_load, uint64_t* out_new_sizes,
                   uint64_t* out_stats);
/* deliver_deterministic (delivery.py:188-306) for one group: P members in r
 * subgroups, pieces[P][r] = piece sizes; pe0 = first member's PE id (error
 * messages).  Writes the new member sizes [P] and slices {src, dst, len}
 * (src relative to the group's simple layout: subgroup, source member,
 * bucket; dst relative to the group's new member arrays, receivers
 * concatenating by source, simnet.py:324-325); slice_cap >= P*(r+1) is
 * enough.  stats[4] as ams_plan_level (NULL skips).  AMS_EINVAL for a piece
 * above ceil(n/p) (delivery.py:212-217), AMS_EINTERNAL when the residual
 * capacities cannot hold the large pieces (delivery.py:274-276). */
int ams_deliver_deterministic(int P, int r, int pe0, const uint64_t* pieces, uint64_t* out_new_sizes,
                              uint64_t* out_slices, int slice_cap, int* out_nslices,
                              uint64_t* out_stats);
/* deliver_simple_permuted (delivery.py:151-185): as above, subgroup g's
 * sending members enumerated in the Feistel order of stream
 * "{level_stream}/deliver/order-g{g}" (core.py:96-159), level_stream =
 * "{SeedSpec.stream_id}/L{level}-g{first PE of the group}". */
int ams_deliver_permuted(int P, int r, int64_t master_seed, const char* level_stream,
                         const uint64_t* pieces, uint64_t* out_new_sizes, uint64_t* out_slices,
                         int slice_cap, int* out_nslices, uint64_t* out_stats);
/* deliver_randomized (delivery.py:318-436, default delegation factor
 * 309-315): chunking, Feistel delegation, per-holder CPython shuffles;
 * slice_cap >= P*(2r+2) is enough.  Output as ams_deliver_deterministic. */
int ams_deliver_randomized(int P, int r, int64_t master_seed, const char* level_stream,
                           const uint64_t* pieces, uint64_t* out_new_sizes, uint64_t* out_slices,
                           int slice_cap, int* out_nslices, uint64_t* out_stats);

/* ------------------------------------------------------------------ */
/* Device context: one per GPU (one process per GPU).                  */

typedef struct ams_ctx ams_ctx_t;

/* `stream` is a cudaStream_t (NULL = the legacy default stream). */
int ams_ctx_create(int device, void* stream, ams_ctx_t** out);
int ams_ctx_destroy(ams_ctx_t* ctx);
int ams_ctx_set_stream(ams_ctx_t* ctx, void* stream);
/* Number of this library's kernels launched so far on the context. */
uint64_t ams_ctx_launches(const ams_ctx_t* ctx);
int ams_ctx_sync(ams_ctx_t* ctx);

/* Optional per-kernel-category timing: when enabled every launch is
 * bracketed by CUDA events on the context's stream; stats give the summed
 * device milliseconds, algorithmic bytes (keys/values read + written) and
 * launch counts per category. */
#define AMS_KCAT_SAMPLE 0
#define AMS_KCAT_RANK 1
#define AMS_KCAT_CLS 2
#define AMS_KCAT_HIST 3
#define AMS_KCAT_CHUNKSCAN 4
#define AMS_KCAT_CELLBASE 5
#define AMS_KCAT_SCATTER 6
#define AMS_KCAT_RANGES 7
#define AMS_KCAT_FHIST 8
#define AMS_KCAT_FSCATTER 9
#define AMS_KCAT_SMEMSORT 10
#define AMS_KCAT_MAP 11
#define AMS_KCAT_SCATTER_U 12
#define AMS_NUM_KCAT 13
int ams_ctx_set_timing(ams_ctx_t* ctx, int enable);
int ams_ctx_kernel_stats(ams_ctx_t* ctx, double* ms, double* bytes, uint64_t* launches, int ncat);
int ams_ctx_reset_stats(ams_ctx_t* ctx);
/* Timed launches since the last call (timing on): category and start / end
 * in ms from the first launch of each resolved batch (batches are resolved
 * by ams_ctx_kernel_stats / ams_ctx_timeline).  Fills up to cap entries,
 * *count = number available; clears the list. */
int ams_ctx_timeline(ams_ctx_t* ctx, int* cat, float* t0, float* t1, int cap, int* count);

/* K1 — sample gather (draw_sample, ams.py:157-175, data side):
 *   d_out_keys[i] = ordered(src[h_idx[i]]), d_out_pos[i] = h_gpos[i]. */
int ams_level_sample(ams_ctx_t* ctx, const void* src, int key_kind, uint64_t count,
                     const uint64_t* h_idx, const uint64_t* h_gpos, uint64_t* d_out_keys,
                     uint32_t* d_out_pos);

/* K2 — splitter selection (select_splitters ams.py:178-198 via the
 * fast work-inefficient rank sort fastsort.py:57-130): per group g the
 * sample [h_soff[g], h_soff[g+1]) is ranked by counting under
 * (key, pos); splitter i = element of rank (i*S)//nb.  Builds the
 * classifier (sorted splitters + key-range LUT) of each group in the
 * context. */
int ams_level_splitters(ams_ctx_t* ctx, int ngroups, const uint64_t* d_sample_keys,
                        const uint32_t* d_sample_pos, const uint64_t* h_soff,
                        const int32_t* h_nb);
/* Copy group g's splitters to host (parity checks / reports). */
int ams_read_splitters(ams_ctx_t* ctx, int group, uint64_t* keys, uint32_t* pos, int* nspl);

/* K3 — classify + per-tile / per-segment histograms (partition_buckets,
 * ams.py:201-211; histogram allreduce input ams.py:236-237).
 * Segment s = one PE: [h_seg_off[s], +h_seg_len[s]) of `src`, member of
 * group h_seg_group[s] (groups are contiguous runs of segments); element
 * position for tie-breaking = buffer index + h_group_posbase[g].  Blocks
 * until the per-segment histogram is in h_seg_hist_out ([nseg][nb_stride]).
 * track_minmax: record global min/max key (for the final sort's ranges).
 * stable (used by the following ams_level_scatter) = 0 allows any order
 * inside one tile's bucket run: valid only for the last level without
 * values, where only PE membership matters (F7). */
int ams_level_classify(ams_ctx_t* ctx, const void* src, int key_kind, int nseg,
                       const uint64_t* h_seg_off, const uint64_t* h_seg_len,
                       const int32_t* h_seg_group, int ngroups, const int64_t* h_group_posbase,
                       int nb_stride, int track_minmax, int stable, uint32_t* h_seg_hist_out);

/* K4+K6 — stable scatter into (group, source segment, bucket) order
 * (the simple delivery layout: pieces ams.py:240-248, deliver_simple
 * delivery.py:151-180, exchange order simnet.py:324-325, receive concat
 * ams.py:252-256).  Uses the segments of the last ams_level_classify.
 * h_boundaries: [ngroups][r+1] plan boundaries; group g's output begins
 * at dst + h_group_dst_start[g].  vals may be NULL (keys only).
 * Also derives the key bounds of the ngroups*r child groups; children
 * [child_first, child_first + child_count) are this GPU's groups at the
 * next level (all of them on a single GPU). */
int ams_level_scatter(ams_ctx_t* ctx, const void* src, const void* src_vals, int key_kind,
                      void* dst, void* dst_vals, int r, const uint64_t* h_boundaries,
                      const uint64_t* h_group_dst_start, int child_first, int child_count);
/* As ams_level_scatter; flags AMS_SCATTER_BUCKET_MAJOR (keys-only last
 * level, where only PE membership matters: ams.py:310-312) lays
 * every group out bucket by bucket, for ams_final_sort_buckets. */
#define AMS_SCATTER_BUCKET_MAJOR 1
int ams_level_scatter_ex(ams_ctx_t* ctx, const void* src, const void* src_vals, int key_kind,
                         void* dst, void* dst_vals, int r, const uint64_t* h_boundaries,
                         const uint64_t* h_group_dst_start, int child_first, int child_count,
                         int flags);

/* ---- multi-GPU level 1 over NVLink (one process per GPU) ----------------
 * The first level's single group spans every GPU: each GPU
 * scatters its PEs' keys straight into the receive buffers of the GPUs that
 * own the destination groups (Network.exchange, simnet.py:294-335: group g's
 * buffer is the concatenation of the source PEs' pieces in PE order).
 *
 * ams_peer_buffer: library-owned device buffer `slot` (0..7) of at least
 * `bytes`, its address and the 64-byte CUDA IPC handle peers open; *grown = 1
 * when it was (re)allocated, so peers must re-open it.
 * ams_peer_open: map a peer process's buffer (cudaIpcOpenMemHandle with lazy
 * peer access; cached per handle); ams_peer_close_all unmaps them.
 * ams_level_scatter_peers: after ams_level_classify of the local PEs (one
 * group), bucket b of local segment s goes to buffer dst[bucket_dst[b]] at
 * index cell_base[s * nb + b] + its stable rank (values to dst_vals[...]).
 * Also derives the key bounds of children [child_first, child_first +
 * child_count) of the r children (this GPU's next-level groups).  The
 * caller synchronises the GPUs before and after (its barrier). */
int ams_peer_buffer(ams_ctx_t* ctx, int slot, uint64_t bytes, void** dptr, void* ipc_handle, int* grown);
int ams_peer_open(ams_ctx_t* ctx, const void* ipc_handle, void** dptr);
int ams_peer_close_all(ams_ctx_t* ctx);
int ams_level_scatter_peers(ams_ctx_t* ctx, const void* src, const void* src_vals, int key_kind, int ndst,
                            void* const* dst, void* const* dst_vals, const int32_t* bucket_dst,
                            const uint64_t* cell_base, int r, const uint64_t* h_boundaries, int child_first,
                            int child_count);

/* Global min/max key seen by a track_minmax classify (ordered encoding);
 * the multi-rank driver all-reduces them and writes them back before the
 * final sort so every rank's key ranges are true bounds. */
int ams_get_minmax(ams_ctx_t* ctx, uint64_t out[2]);
int ams_set_minmax(ams_ctx_t* ctx, const uint64_t in[2]);

/* K7-K9 — final local sort (ams.py:310-312), stable by key.  Segment s
 * of `src` (ordered keys) is final PE s = child s of the last
 * ams_level_scatter (its key bounds come from there).  Large segments are
 * digit-partitioned into `tmp` and every cell sorted in shared memory into
 * `out` (keys mapped back to `key_kind`).  `src` is clobbered. */
int ams_final_sort(ams_ctx_t* ctx, void* src, void* src_vals, void* tmp, void* tmp_vals,
                   void* out, void* out_vals, int key_kind, int nseg, const uint64_t* h_seg_off,
                   const uint64_t* h_seg_len);
/* Final local sort (keys only) after a bucket-major last level: nbk buckets
 * in output order, bucket i = bk_len[i] keys at bk_off[i], bucket bk_bucket[i]
 * of the last level's group bk_group[i].  Buckets above shared memory are
 * split into fixed-capacity digit cells in one pass (no histogram); cells
 * are sorted in shared memory; overflowing buckets take exact rounds. */
int ams_final_sort_buckets(ams_ctx_t* ctx, void* src, void* tmp, void* out, int key_kind, int nbk,
                           const uint64_t* bk_off, const uint64_t* bk_len, const int32_t* bk_group,
                           const int32_t* bk_bucket);

/* Cells of the final sort that needed another partition round / the LSD
 * fallback, summed since the context was created: out = {overflow, fallback}. */
int ams_final_sort_stats(ams_ctx_t* ctx, uint64_t out[2]);
/* Buckets of bucket-major keys-only last levels that took the fixed-capacity
 * partition, and those of them whose cells overflowed (re-partitioned
 * exactly), summed since the context was created: out = {buckets, overflowed}. */
int ams_final_sort_fixed_stats(ams_ctx_t* ctx, uint64_t out[2]);

/* Plain copy with key mapping (used for the p == 1 / k == 0 edge and the
 * host-buffer end-to-end path). */
int ams_map_keys(ams_ctx_t* ctx, const void* src, void* dst, uint64_t n, int from_kind,
                 int to_kind);


/* ------------------------------------------------------------------ */
/* One-call sort: ams_sort(net, data, params, "simple", seed)           */
/* (ams.py:271-313) on the context's GPU, the whole level loop in C++.  */

#define AMS_MAX_LEVELS 8

/* AmsParams (ams.py:33-65) + SeedSpec (core.py:46-71) + key encoding. */
/* Delivery schemes (delivery.py:439-455 SCHEMES): "simple" (151-180),
 * "deterministic" (188-306, the reference CLI default), "permuted"
 * (183-185) and "randomized" (318-436). */
#define AMS_SCHEME_SIMPLE 0
#define AMS_SCHEME_DETERMINISTIC 1
#define AMS_SCHEME_PERMUTED 2
#define AMS_SCHEME_RANDOMIZED 3
#define AMS_SAMPLE_PARITY 0
#define AMS_SAMPLE_DEVICE 1

typedef struct {
  int levels;                          /* k = len(group_counts) */
  int group_counts[AMS_MAX_LEVELS];    /* r per level; product = p */
  double oversampling;                 /* a; <= 0 selects 1.6*log10(max(n,10)) (ams.py:278-280) */
  int overpartition;                   /* b (reference default 16) */
  double imbalance;                    /* epsilon (reference default 0.2) */
  int64_t master_seed;                 /* SeedSpec.master_seed */
  const char* stream_id;               /* SeedSpec.stream_id, e.g. "algo/rep0" */
  int key_kind;                        /* AMS_KEY_U64 / AMS_KEY_I64 / AMS_KEY_F64 */
  int with_stats;                      /* fill the exchange maxima of the reports */
  int scheme;                          /* AMS_SCHEME_SIMPLE / _DETERMINISTIC / _PERMUTED / _RANDOMIZED */
  int record_holders;                  /* keep, per level and PE, how many splitters were drawn from
                                          the PE (the ledger's extract_by_ranks charge,
                                          fastsort.py:111-130; one small D2H per level) */
  /* Continuation of a sort whose first levels ran elsewhere (multi-GPU:
   * level 1 is the exchange between the GPUs); all zero for a
   * whole sort.  The p PEs of the call are the global PEs [pe_base, pe_base
   * + p) and start as init_groups equal groups at level level_base (0-based
   * index into group_counts, which still lists every level of the sort);
   * the context holds the groups' key bounds (ams_level_scatter_peers /
   * ams_level_scatter leave them).  oversampling must be given (> 0: `a`
   * comes from the global n).  With a non-simple scheme `vals` holds the
   * origin tags of the input (index in the whole sort's input), which break
   * key ties (delivery.py:188-455 can reorder sources); user payloads are
   * not carried in that case and out_vals is unused. */
  int level_base;
  int init_groups;                     /* 0 or 1: one group */
  int pe_base;
  /* AMS_SAMPLE_PARITY (0): sample positions from the reference's seeded
   * streams (CPython MT19937 restated on the host, ams.py:157-175): bucket
   * boundaries equal the reference's.  AMS_SAMPLE_DEVICE (1): the same
   * quota split (ams.py:166-171) with stratified positions drawn on the
   * device (distinct by construction, every element of a PE equally
   * likely) — no host draw; boundaries differ from the reference's, the
   * output and the (1 + eps) bound do not.  Not with record_holders. */
  int sample_mode;
} ams_params_t;

/* One level's report (ams.py:294-308; exchange maxima simnet.py:109-124). */
typedef struct {
  int level, r;
  uint64_t max_load, min_load, sample_size, plan_load, over_budget;
  uint64_t max_words, max_msgs, max_sent_msgs, max_recv_msgs;
} ams_level_report_t;

/* Sort n = sum(pe_sizes) keys (device buffer, PE-major: PE i owns the next
 * pe_sizes[i]) with optional 8-byte payloads into out (+ out_vals): the
 * concatenation of the per-PE outputs of ams_sort.  out_pe_sizes[p] gets
 * the final PE sizes, reports[levels] the level reports (either may be
 * NULL).  Inputs are not modified; the context owns the workspace.  Runs on
 * the context's stream and returns after the last host-side step (the
 * device work may still be in flight). */
int ams_sort_run(ams_ctx_t* ctx, const ams_params_t* params, int p, const uint64_t* pe_sizes,
                 const void* keys, const void* vals, void* out, void* out_vals,
                 uint64_t* out_pe_sizes, ams_level_report_t* reports);
/* Records of the last ams_sort_run, level by level (host arrays; NULL
 * skips a field): group_first/npe [G], sizes_before/new_sizes [P],
 * drawn [G], nb [G], seg_hist [P][nb_stride], boundaries [G][r+1],
 * loads [G][r], max_load [G], stats [G][4] (when has_stats). */
int ams_run_level_dims(ams_ctx_t* ctx, int level, int* r, int* ngroups, int* npe, int* nb_stride,
                       int* has_stats);
int ams_run_level(ams_ctx_t* ctx, int level, int32_t* group_first, int32_t* group_npe,
                  uint64_t* sizes_before, uint64_t* drawn, int32_t* nb, uint32_t* seg_hist,
                  uint64_t* boundaries, uint64_t* loads, uint64_t* max_load, uint64_t* new_sizes,
                  uint64_t* stats);
/* Id of the last ams_sort_run on the context (1, 2, ...); the records of the
 * last 8 runs stay readable by id (run 0 = the last run). */
uint64_t ams_run_id(const ams_ctx_t* ctx);
int ams_run_level_dims_at(ams_ctx_t* ctx, uint64_t run, int level, int* r, int* ngroups, int* npe,
                          int* nb_stride, int* has_stats);
int ams_run_level_at(ams_ctx_t* ctx, uint64_t run, int level, int32_t* group_first, int32_t* group_npe,
                     uint64_t* sizes_before, uint64_t* drawn, int32_t* nb, uint32_t* seg_hist,
                     uint64_t* boundaries, uint64_t* loads, uint64_t* max_load, uint64_t* new_sizes,
                     uint64_t* stats);
/* Per PE [P]: number of that level's splitters drawn from the PE's sample
 * (replaces the holder bookkeeping of extract_by_ranks, fastsort.py:111-130,
 * for CostLedger parity); needs params.record_holders. */
int ams_run_level_holders_at(ams_ctx_t* ctx, uint64_t run, int level, uint32_t* holders);

/* Relayout helpers of the non-simple deliveries for callers that run a
 * level themselves (the multi-GPU drivers): dst[d + i] = src[s + i] for
 * every range {s, d, len} (host array of 3 * nranges u64; values too when
 * given), and dst[i] = start + i. */
int ams_copy_ranges(ams_ctx_t* ctx, const uint64_t* h_ranges, int nranges, const void* src, void* dst,
                    const void* src_vals, void* dst_vals);
int ams_fill_iota(ams_ctx_t* ctx, void* dst, uint64_t n, uint64_t start);

/* ------------------------------------------------------------------ */
/* Single-process multi-device driver: one context   */
/* per entry of devices[] (entries may repeat: several contexts on one   */
/* GPU), each with its own stream; peer access is enabled between        */
/* distinct devices.  PE i lives on context i * G / p, and               */
/* group_counts[0] must be a multiple of G, so only level 1 crosses      */
/* devices: its pieces are stored straight into the owners' receive      */
/* buffers over peer pointers (ams_level_scatter_peers); the later       */
/* levels and the final sort run as ams_sort_run continuations.          */

typedef struct ams_mg ams_mg_t;
int ams_mg_create(const int* devices, int ngpu, ams_mg_t** out);
int ams_mg_destroy(ams_mg_t* mg);
int ams_mg_size(const ams_mg_t* mg);
/* The i-th context (its ams_run_level* records hold the later levels of the
 * PEs that live there; timing; launch counts). */
int ams_mg_ctx(ams_mg_t* mg, int i, ams_ctx_t** out);
/* ams_sort (ams.py:271-313) over G devices: keys[i] / out[i] (and vals /
 * out_vals, simple scheme only; NULL otherwise) are device i's buffers for
 * PEs [i*p/G, (i+1)*p/G), PE-major; out[i] must hold the device's final
 * keys (sum of its out_pe_sizes; at most (1 + eps) n / G, ams.py:258).  The
 * caller's inputs must be ready (no stream is shared with the caller); the
 * call returns when every device has finished.  Results are bit-identical
 * for every G (same logical PEs and seeded streams). */
int ams_mg_sort_run(ams_mg_t* mg, const ams_params_t* params, int p, const uint64_t* pe_sizes,
                    const void* const* keys, const void* const* vals, void* const* out,
                    void* const* out_vals, uint64_t* out_pe_sizes, ams_level_report_t* reports);
/* Level-1 records of the last ams_mg_sort_run (as ams_run_level; one group). */
int ams_mg_level1_dims(const ams_mg_t* mg, int* r, int* p, int* nb_stride);
int ams_mg_level1(const ams_mg_t* mg, uint64_t* sizes_before, uint64_t* drawn, int32_t* nb,
                  uint32_t* seg_hist, uint64_t* boundaries, uint64_t* loads, uint64_t* max_load,
                  uint64_t* new_sizes, uint64_t* stats);

/* ------------------------------------------------------------------ */
/* RLM-sort (recurse-last multiway mergesort, rlm.py:86-132): SURVEY     */
/* section 8(f) row 4.                                                   */

/* deliver_simple (delivery.py:151-180) for one group from its piece sizes
 * [P][r]: the new member sizes (quota slots, delivery.py:78-80) and the
 * exchange stats (NULL skips); the member arrays are consecutive slices of
 * the group's simple layout. */
int ams_deliver_simple(int P, int r, const uint64_t* pieces, uint64_t* out_new_sizes,
                       uint64_t* out_stats);

/* One level's report (rlm.py:118-131). */
typedef struct {
  int level, r;
  uint64_t max_load, min_load;
  uint64_t max_words, max_msgs, max_sent_msgs, max_recv_msgs;
} ams_rlm_report_t;

/* rlm_sort (rlm.py:86-132) of n = sum(pe_sizes) keys (device buffer,
 * PE-major) with LevelPlan(p, group_counts) (rlm.py:22-45; AMS_EINVAL with
 * the reference's messages when the counts do not telescope p) and the
 * delivery `scheme` (AMS_SCHEME_*, streams "{stream_id}/L{lv}-g{lo}/deliver"
 * as rlm.py:101-110).  Writes the concatenation of the per-PE outputs to
 * out; out_origin (optional, u64[n]) gets every output element's index in
 * the input (its Element identity, core.py:19-43); out_vals (with vals) the
 * payloads in output order.  out_pe_sizes[p] and reports[levels] may be
 * NULL.  Cut positions come from an exact device selection (the unique
 * result of multiselect_many, multiselect.py:45-137). */
int ams_rlm_sort_run(ams_ctx_t* ctx, int levels, const int32_t* group_counts, int scheme,
                     int64_t master_seed, const char* stream_id, int key_kind, int p,
                     const uint64_t* pe_sizes, const void* keys, const void* vals, void* out,
                     void* out_origin, void* out_vals, uint64_t* out_pe_sizes,
                     ams_rlm_report_t* reports);
/* Records of the last ams_rlm_sort_run: group_first/npe [G], sizes_before /
 * new_sizes [P], cuts [P][r+1] (_cut_points, rlm.py:53-83), stats [G][4]. */
int ams_rlm_level_dims(ams_ctx_t* ctx, int level, int* r, int* ngroups, int* npe);
int ams_rlm_level(ams_ctx_t* ctx, int level, int32_t* group_first, int32_t* group_npe,
                  uint64_t* sizes_before, uint64_t* cuts, uint64_t* new_sizes, uint64_t* stats);

#ifdef __cplusplus
}
#endif

#endif /* AMS_B200_H */
