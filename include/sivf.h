/* sivf.h — C ABI of libsivf.so: a GPU-resident, slab-allocated IVF-Flat index
 * with batched in-place insert / delete / search (SIVF, arXiv 2601.11808),
 * written for NVIDIA B200 (sm_100a).
 *
 * Citations: P:n = PAPER.md line n (the paper), S:n = SPEC.md line n, and
 * "reading Cnn" = the ambiguity ledger in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Pointers named d_* are DEVICE pointers on the index's device; h_* are host
 *    pointers.  The caller owns every buffer, including the arena; the library
 *    never allocates device memory after sivf_create (all scratch lives in the
 *    arena, sized by the max_* fields of sivf_config).
 *  - Every call except sivf_arena_bytes/sivf_stats/sivf_rc_string is
 *    asynchronous: it validates its arguments on the host, enqueues kernels on
 *    `stream` and returns.  No call synchronises the stream except
 *    sivf_stats.  Variable sizes are read on the device, so a sequence of
 *    calls with fixed host-side sizes is CUDA-graph capturable.
 *  - A handle is stream-serialised: calls on one handle must be ordered on one
 *    stream (or externally ordered) and made by one host thread at a time.
 *  - Host-detectable errors (null pointers, sizes beyond the max_* limits,
 *    k/nprobe out of range, index not trained) return SIVF_E_* and enqueue
 *    nothing.  Launch failures return SIVF_E_CUDA.  Device-side conditions are
 *    reported per item (sivf_item_status) and in sticky counters (sivf_stats).
 *  - Ids are int64 at the ABI; the id space is dense [0, id_capacity)
 *    (S:151-152), with id_capacity < 2^32 - 1 (ids are stored as u32 inside
 *    slabs).  With sharding, rank r owns ids with id % shard_count == r and its
 *    address table is indexed by id / shard_count (reading C13, §8(e)).
 *  - Distances are squared L2 in fp32 (Eq. l2).  Results are sorted
 *    ascending by (distance, id) and padded with (+inf, -1) (readings C4, C5).
 */
#ifndef SIVF_H
#define SIVF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* sivf_stream_t; /* == cudaStream_t; NULL = legacy default stream */
typedef struct sivf_index_s* sivf_index;

typedef enum {
  SIVF_OK = 0,
  SIVF_E_INVALID_ARG = -1,
  SIVF_E_CUDA = -2,
  SIVF_E_ARENA_TOO_SMALL = -3,
  SIVF_E_NOT_TRAINED = -4,
  SIVF_E_UNSUPPORTED = -5
} sivf_rc;

/* Per-item insert outcome (readings C9, C12, C13). */
typedef enum {
  SIVF_ST_OK = 0,
  SIVF_ST_POOL_EXHAUSTED = 1,  /* no free slab (Alg. 2 "If the pool is exhausted") */
  SIVF_ST_DUPLICATE = 2,       /* id live, or repeated earlier in the same batch */
  SIVF_ST_ID_OUT_OF_RANGE = 3, /* id outside [0, id_capacity) */
  SIVF_ST_WRONG_SHARD = 4,     /* id % shard_count != shard_rank */
  SIVF_ST_DIR_FULL = 5,        /* sivf_insert_concurrent: the list has no spare directory entry
                                  (sivf_reserve_directories before the concurrent phase) */
  SIVF_ST_RETRY_LIMIT = 6      /* sivf_insert_concurrent: 1000 attempts without a slot (C10) */
} sivf_item_status;

/* sivf_config.flags */
enum {
  /* No fp16 copy of the slab payload: the arena is the paper's footprint (fp32
   * payload + ids + metadata) and search scans on CUDA cores.  By default
   * (dim <= 128) the arena also holds an fp16 (RN) copy of every slab that the
   * tensor-core scan reads (+50 % of the payload bytes at dim 128; reading C35). */
  SIVF_CFG_NO_SCAN_COPY = 1,
  /* Room for concurrent phases (NEXT-2): the directory arena gets 256 extra
   * entries per list so that sivf_reserve_directories can give every list up to
   * 256 spare entries (1 MB per 1024 lists). */
  SIVF_CFG_CONCURRENT = 2,
  /* Float-valued data at dim <= 128: keep the split-fp16 (hi + lo, per-vector
   * power-of-2 scale) scan copy instead of the single fp16 copy, and search with
   * the K-chunked GEMM scan (three kind::f16 MMAs per K step, distances within
   * ~2^-20 relative: no exact re-rank of filter survivors).  The fp16 filter of
   * the default copy is exact on small-integer data (SIFT-shaped) but re-ranks
   * every survivor from the fp32 payload on float data.  +100 % of the payload
   * bytes; dim > 128 always uses this copy.  Ignored with SIVF_CFG_NO_SCAN_COPY. */
  SIVF_CFG_SPLIT_COPY = 4
};

typedef struct {
  int32_t dim;          /* D >= 1 */
  int32_t nlist;        /* number of inverted lists, 1..65536 */
  int64_t id_capacity;  /* global id space [0, id_capacity), < 2^32 - 1 */
  int64_t num_slabs;    /* slab pool size; each slab = 32 slots */
  int32_t max_batch;    /* max items per insert/delete call */
  int32_t max_queries;  /* max queries per search call */
  int32_t max_k;        /* 1..128 */
  int32_t max_nprobe;   /* 1..min(nlist, 1024) */
  int32_t max_train;    /* max training points for sivf_train_centroids (0 = none) */
  int32_t shard_rank;   /* 0..shard_count-1 */
  int32_t shard_count;  /* >= 1; owner(id) = id % shard_count */
  int32_t flags;        /* SIVF_CFG_* bits (0 = defaults) */
  uint64_t seed;        /* k-means initialisation seed */
} sivf_config;

typedef struct {
  int64_t live;                 /* slots whose validity bit is set */
  int64_t inserted;             /* successful inserts since create */
  int64_t deleted;              /* 1->0 bit transitions since create (Alg. 4 deleted_count) */
  int64_t slabs_in_use;         /* num_slabs - slabs_free */
  int64_t slabs_free;           /* free-stack height P_top (Eq. 2) */
  int64_t pool_exhausted_items; /* sticky count of SIVF_ST_POOL_EXHAUSTED items */
  int64_t reclaimed_slabs;      /* total slabs recycled by sivf_reclaim / sliding steps */
  int64_t device_errors;        /* sticky internal errors (unreachable directory-arena overflow); must stay 0 */
  double overhead_paper;        /* 128/(32*(4d+8)): the paper's per-slab header accounting (reading C17) */
  double overhead_actual;       /* this build: (16 B metadata/slab * slabs_in_use + 8 B * id slots) / (live payload+id bytes) */
  double overhead_scan_copy;    /* the scan copy of slabs_in_use / (live payload+id bytes): D <= 128 the fp16 records (2 Dh B + norm and id 8 B per slot), D > 128 the split-fp16 copy (4 Dg B + scale 4 B per slot); 0 without */
  int64_t dir_compactions;      /* times the list directories were repacked into the idle arena half (k_reserve) */
  int64_t leaked_slabs;         /* slabs leaked by lost publication CASes of sivf_insert_concurrent */
  int64_t leaked_recycled;      /* of those, returned to the pool by sivf_reclaim */
} sivf_stats_t;

/* Bytes of device memory the index needs for `cfg` (host-only, pure). */
sivf_rc sivf_arena_bytes(const sivf_config* cfg, size_t* bytes);

/* Carve the arena (>= sivf_arena_bytes, 256-B aligned device memory owned by
 * the caller, which must outlive the handle) and initialise it on `stream`:
 * free-slab stack = all slabs ("constructs a free-list array and sets
 * a global stack pointer"), address table = INVALID sentinel, empty
 * lists.  The index is untrained until centroids are set. */
sivf_rc sivf_create(const sivf_config* cfg, void* d_arena, size_t arena_bytes, sivf_stream_t stream,
                    sivf_index* out);
/* Releases host-side state only; does not free the arena. */
sivf_rc sivf_destroy(sivf_index ix);

/* Centroids [nlist][dim] fp32 row-major (the coarse quantizer). */
sivf_rc sivf_set_centroids(sivf_index ix, const float* d_centroids, sivf_stream_t stream);
sivf_rc sivf_get_centroids(sivf_index ix, float* d_centroids, sivf_stream_t stream);

/* Lloyd k-means on d_x[n][dim] (n <= max_train, n >= nlist), niter iterations,
 * initialised from cfg.seed; sets the centroids.  Bit-exact with the oracle's
 * kmeans (reading C31).  Setup only. */
sivf_rc sivf_train_centroids(sivf_index ix, const float* d_x, int64_t n, int32_t niter, sivf_stream_t stream);

/* Batched insert (Alg. 1/2): per item, claim the id,
 * assign it to its nearest centroid (ties -> lowest list, reading C2), reserve
 * a slot at the end of that list (tail slab first, then fresh slabs from the
 * free pool; lists served in ascending order when the pool runs short), write
 * payload + id + address-table entry, then publish the validity bit
 * (P:247).  d_ids[n] int64, d_x[n][dim] fp32 row-major, 0 <= n <=
 * max_batch.  d_status[n] (nullable) receives sivf_item_status; d_list[n]
 * (nullable) receives the assigned list for OK items, -1 otherwise. */
sivf_rc sivf_insert(sivf_index ix, const int64_t* d_ids, const float* d_x, int64_t n, int32_t* d_status,
                    int32_t* d_list, sivf_stream_t stream);

/* Batched lazy eviction (Alg. 4): address-table lookup, atomic
 * bit clear; on a 1->0 transition the table entry becomes INVALID and the
 * counters move.  Absent, repeated, out-of-range and non-owned ids are no-ops.
 * *d_ndeleted (nullable, device int64) receives the number of transitions. */
sivf_rc sivf_delete(sivf_index ix, const int64_t* d_ids, int64_t n, int64_t* d_ndeleted, sivf_stream_t stream);

/* Batched search (Alg. 3): the nprobe nearest lists by
 * (dist32, list) (reading C3), scan of valid slots only (Eq. slot_valid),
 * per-query top-k by (distance, id).  d_q[nq][dim]; d_dist[nq][k] fp32;
 * d_ids[nq][k] int64; d_probes[nq][nprobe] (nullable) receives the probe SET of
 * each query (reading C3): its members are exact, their order within a row is
 * unspecified (nearest-first when the exact distances were needed to decide the
 * set, otherwise by the tensor-core approximation).  A configuration no scan
 * kernel supports (e.g. shared memory for dim) returns SIVF_E_UNSUPPORTED. */
sivf_rc sivf_search(sivf_index ix, const float* d_q, int64_t nq, int32_t k, int32_t nprobe, float* d_dist,
                    int64_t* d_ids, int32_t* d_probes, sivf_stream_t stream);

/* NEXT-3 (query-sharded coarse step): the coarse step alone
 * and the scan + merge given the probe sets.
 * sivf_probe: d_probes[nq][nprobe] (device, caller-owned) receives the exact probe
 * SET of each query row (reading C3), as sivf_search's d_probes.
 * Reads only the centroids: a rank may compute it for its slice of a batch.
 * sivf_search_probed: as sivf_search, with the probe sets taken from
 * d_probes_in[nq][nprobe] (device, read only; every entry in [0, nlist),
 * nearest-first order preferred: it steers the scan's work order, not its
 * results).  Given the probe sets sivf_probe returns (on any shard of the same
 * centroids), its output equals sivf_search's bit for bit.  Entries outside
 * [0, nlist) are undefined behaviour (not validated on the device). */
sivf_rc sivf_probe(sivf_index ix, const float* d_q, int64_t nq, int32_t nprobe, int32_t* d_probes,
                   sivf_stream_t stream);
sivf_rc sivf_search_probed(sivf_index ix, const float* d_q, int64_t nq, int32_t k, int32_t nprobe,
                           const int32_t* d_probes_in, float* d_dist, int64_t* d_ids, sivf_stream_t stream);

/* One sliding-window step (reading C22): insert(new) -> delete(old) ->
 * search(queries) -> reclaim of full, fully-dead slabs.  Arguments as in the
 * individual calls; nq may be 0 (no search). */
sivf_rc sivf_sliding_window_step(sivf_index ix, const int64_t* d_new_ids, const float* d_new_x, int64_t n_new,
                                 const int64_t* d_old_ids, int64_t n_old, const float* d_q, int64_t nq, int32_t k,
                                 int32_t nprobe, float* d_dist, int64_t* d_ids, int32_t* d_status,
                                 int64_t* d_ndeleted, sivf_stream_t stream);

/* Multi-GPU merge (§8(e)): per query, the k smallest (distance, id) of G
 * per-shard lists d_dist_g/d_ids_g [G][nq][k]; entries with id < 0 are padding.
 * Stateless; uses no arena (nq*k*G <= 2^31).  Outputs [nq][k]. */
sivf_rc sivf_merge_topk(const float* d_dist_g, const int64_t* d_ids_g, int32_t G, int64_t nq, int32_t k,
                        float* d_dist, int64_t* d_ids, sivf_stream_t stream);

/* Quiescent reclamation (reading C16): every slab that is full (32 slots
 * reserved) and has no valid slot leaves its list and returns to the free
 * pool; list order is preserved.  *d_nreclaimed (nullable) = slabs freed. */
sivf_rc sivf_reclaim(sivf_index ix, int64_t* d_nreclaimed, sivf_stream_t stream);

/* State export for parity checks.  d_list_of_id[local_capacity]: list of each
 * live local id (index id / shard_count), -1 if not live.  d_live_per_list
 * [nlist].  d_violations (nullable, device int64): number of broken
 * invariants (ATT <-> bitmap <-> slab ids <-> directories <-> free pool). */
sivf_rc sivf_dump_state(sivf_index ix, int32_t* d_list_of_id, int64_t* d_live_per_list, int64_t* d_violations,
                        sivf_stream_t stream);

/* Raw address-table entries (Eq. att_encoding: (slab << 32) | slot,
 * INVALID = all ones) for local ids [0, local_capacity) into d_att. */
sivf_rc sivf_dump_att(sivf_index ix, uint64_t* d_att, sivf_stream_t stream);

/* Counters; synchronises `stream`.  h_out is a host pointer. */
sivf_rc sivf_stats(sivf_index ix, sivf_stats_t* h_out, sivf_stream_t stream);

/* Local address-table size for this shard: ceil((id_capacity - rank) / shard_count). */
int64_t sivf_local_capacity(sivf_index ix);

/* Number of kernel launches this handle has enqueued so far (bench bookkeeping). */
int64_t sivf_launch_count(sivf_index ix);

/* ---- NEXT-2: concurrent mutation + search across streams (Alg. 2) ----
 *
 * A handle is stream-serialised.  For concurrency, VIEWS of an index share its
 * state (payload, bitmaps, ATT, directories, free stack, counters) and own
 * their scratch, so several views can run on several streams at once:
 *   sivf_search, sivf_delete and sivf_insert_concurrent on views (and on the
 *   owner) may overlap one another in any combination;
 *   everything else (sivf_insert, sivf_reclaim, sivf_sliding_window_step,
 *   sivf_train_centroids, sivf_set_centroids, sivf_reserve_directories,
 *   sivf_dump_*) is quiescent: owner only, with no view call in flight.
 * Contract (the paper's publish protocol): an insert becomes visible when its
 * validity bit is set, after its payload, id and ATT entry (__threadfence before
 * the atomicOr); a search returns a hit only for a slot whose bit it observed as
 * set (so never a torn payload), and a concurrent delete makes an id disappear
 * as soon as its bit is cleared (lazy eviction: a hit implies the bit was set at
 * some instant during the search).  Searches on a view use acquire loads of the
 * directory lengths and bitmaps (sivf_set_option SIVF_OPT_CONCURRENT, on by
 * default for views).
 *
 * sivf_view_arena_bytes: bytes of a view's arena for an owner created with cfg.
 * sivf_create_view: a view of `owner` in the caller's arena (256-B aligned,
 *   >= sivf_view_arena_bytes); it reads the owner's centroids on `stream` (create
 *   views after training; views must be destroyed before the owner and recreated
 *   after the centroids change).  SIVF_E_ARENA_TOO_SMALL / SIVF_E_INVALID_ARG.
 * sivf_insert_concurrent: sivf_insert's contract with the paper's lock-free
 *   protocol per vector: CAS slot reservation on the list's tail slab (Eq.
 *   cas_count), speculative slab expansion published by CAS on the list's next
 *   directory entry (Eq. cas_head), leak-on-failure (leaked slabs are counted
 *   and recycled by the next sivf_reclaim), fence + atomicOr publish.  In-flight
 *   ids are claimed by CAS on the ATT (a live or in-flight id: SIVF_ST_DUPLICATE).
 *   Extra statuses: SIVF_ST_DIR_FULL (no spare directory entry), SIVF_ST_RETRY_LIMIT.
 *   The owner must have called sivf_reserve_directories since its last quiescent
 *   mutation (else SIVF_E_UNSUPPORTED).  Order of slots within a list is
 *   nondeterministic; the resulting (list, live) state is not.
 * sivf_reserve_directories (quiescent, owner): every list gets >= `spare` free
 *   directory entries (one per slab a concurrent phase may add to that list;
 *   0 <= spare <= 256, else SIVF_E_INVALID_ARG).  Synchronises `stream`;
 *   SIVF_E_UNSUPPORTED when the directory arena cannot hold them (nothing
 *   changed; unreachable with SIVF_CFG_CONCURRENT). */
sivf_rc sivf_view_arena_bytes(const sivf_config* cfg, size_t* bytes);
sivf_rc sivf_create_view(sivf_index owner, void* d_arena, size_t arena_bytes, sivf_stream_t stream,
                         sivf_index* out);
sivf_rc sivf_insert_concurrent(sivf_index ix, const int64_t* d_ids, const float* d_x, int64_t n, int32_t* d_status,
                               int32_t* d_list, sivf_stream_t stream);
sivf_rc sivf_reserve_directories(sivf_index owner, int32_t spare, sivf_stream_t stream);

/* Latency floors for measurement (bench.py roofline.latency; SURVEY §8(d)
 * "Latency roofline for small batches"); neither touches an index.
 *   sivf_probe_launch: enqueues n (>= 1) launches of an empty kernel on stream
 *     (the per-launch floor of a stream of dependent kernels).
 *   sivf_probe_chase: one thread follows `hops` dependent 4-byte loads through
 *     the caller's int32 array d_next[0..n) (device memory; a single cycle that
 *     the caller lays out, larger than L2 for DRAM latency) starting at index 0,
 *     and stores the final index to *d_out (device pointer): hops x the
 *     dependent-load latency, the floor of an op whose work is a chain of
 *     dependent reads (delete: ATT -> bitmap).
 * Both return SIVF_E_INVALID_ARG on bad arguments (nothing enqueued). */
sivf_rc sivf_probe_launch(int32_t n, sivf_stream_t stream);
sivf_rc sivf_probe_chase(const int32_t* d_next, int64_t n, int32_t hops, int32_t* d_out, sivf_stream_t stream);

/* Phase timing for measurement (bench.py roofline): when enabled, every
 * phase below is bracketed by CUDA events recorded on the call's stream.
 * sivf_profile_read synchronises on the recorded events, adds their elapsed
 * milliseconds into h_ms[SIVF_NPHASE] and the number of intervals into
 * h_count[SIVF_NPHASE] (host arrays), and forgets them.  Not for use inside
 * CUDA-graph capture. */
enum {
  SIVF_PH_ASSIGN = 0,   /* insert: exact coarse assignment */
  SIVF_PH_APPEND = 1,   /* insert: claim + ranks + reserve + append */
  SIVF_PH_DELETE = 2,
  SIVF_PH_COARSE = 3,   /* search: coarse distances + top-nprobe */
  SIVF_PH_INVMAP = 4,   /* search: list -> query inverse map */
  SIVF_PH_SCAN = 5,     /* search: slab scan (k_scan) */
  SIVF_PH_MERGE = 6,    /* search: per-query merge of partial top-k */
  SIVF_PH_RECLAIM = 7,
  SIVF_NPHASE = 8
};
sivf_rc sivf_profile_enable(sivf_index ix, int32_t on);

/* Kernel-path switches (tests compare every path against the oracle).
 *   SIVF_OPT_CONCURRENT (default 0 on an owner, 1 on a view): searches use
 *                      acquire loads of directory lengths and bitmaps and order
 *                      them before the bulk copies of the slab records (needed
 *                      when sivf_insert_concurrent may run at the same time).
 *   SIVF_OPT_TC_SCAN   (default 1): slab scan on tcgen05 tensor cores (kind::f16
 *                      over the fp16 slab copy) when dim <= 128 and k <= 32;
 *                      0 = CUDA-core scan.
 *   SIVF_OPT_TC_TWO_PHASE (default 0): value r0 >= 1 scans every query's r0 nearest
 *                      lists in a first launch and the rest in a second (bounds
 *                      complete before the second phase); 0 = one launch.
 *   SIVF_OPT_TC_COARSE (default 1): assignment and probe selection (nprobe <= 32)
 *                      on tcgen05 tensor cores with a certified band and exact
 *                      dist32 re-rank (bit-identical result); 0 = exact CUDA-core
 *                      distance matrix.
 *   SIVF_OPT_SEED_SLABS (default 0): before the tensor-core scan, each query's
 *                      bound on its k-th distance is seeded with exact distances
 *                      to the first `value` live slabs of its nearest probed list
 *                      (any k real candidates bound the final k-th distance from
 *                      above); 0 = no seeding.  Changes speed only, never results.
 *   SIVF_OPT_RANK_SPLIT (default 1): tensor-core scan work items ordered so that
 *                      every query's nprobe/4 nearest lists are scanned before
 *                      its other lists (when that adds no work items on
 *                      average); the bounds on the k-th distances are then
 *                      tight early.  A value r0 > 1 forces the split at the r0
 *                      nearest lists; 0 = one bucket.  Changes speed only, never
 *                      results.
 *   SIVF_OPT_STEP_GRAPH (default 1): sivf_sliding_window_step and sivf_search
 *                      capture the call as a CUDA graph the second time they see a call
 *                      signature (device pointers, sizes, k, nprobe, stream,
 *                      options) and replays it on later calls (up to 4 graphs,
 *                      LRU); the data are read on the device at replay time.
 *                      Direct launches while phase profiling is on or when the
 *                      caller's stream is being captured; 0 = always direct.
 *   SIVF_OPT_COARSE_SELECT (default 1): tensor-core coarse quantisation stores
 *                      the approximate distance matrix and selects per row (exact
 *                      m-th upper bound by bisection, candidates, exact dist32
 *                      re-rank); 0 = the fused two-pass epilogue.  Same results.
 *   SIVF_OPT_SEED_LIST (default 0): before the tensor-core scan, every query's bound
 *                      on its k-th distance is seeded with the k-th smallest exact
 *                      distance to the first live slab (>= k valid slots) of its
 *                      nearest probed list, one staged slab per list (batches of
 *                      >= 4 queries per list on average; not in concurrent mode).
 *                      Changes speed only, never results (measured neutral on the
 *                      SIFT1M-shaped step: the kernel costs about what it saves). */
enum { SIVF_OPT_TC_SCAN = 1, SIVF_OPT_TC_TWO_PHASE = 2, SIVF_OPT_TC_COARSE = 3, SIVF_OPT_SEED_SLABS = 4,
       SIVF_OPT_RANK_SPLIT = 5, SIVF_OPT_COARSE_SELECT = 6, SIVF_OPT_STEP_GRAPH = 7, SIVF_OPT_CONCURRENT = 8,
       SIVF_OPT_SEED_LIST = 9 };
sivf_rc sivf_set_option(sivf_index ix, int32_t option, int64_t value);
sivf_rc sivf_profile_read(sivf_index ix, double* h_ms, int64_t* h_count);

const char* sivf_rc_string(sivf_rc rc);

#ifdef __cplusplus
}
#endif
#endif /* SIVF_H */
