/* sivf_oracle.h — CPU oracle for the SIVF hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product (paper_2601_11808_b200/, libsivf.so) never links, loads or
 * calls it, and the two share no code, headers or constants.
 *
 * What it computes (PAPER.md = P, SPEC.md = S):
 *   dist32      Eq. l2 as a sequential fp32 sum, no FMA (reading C1)
 *   assign      nearest centroid, ties -> lowest list index (C2)
 *   probe       the nprobe nearest centroids by (dist32, list) (C3)
 *   insert      Alg. 1/2 semantics on plain per-list
 *               arrays; statuses per S:250/S:304 (C9, C12, C13)
 *   delete      Alg. 4: idempotent lazy eviction (C15)
 *   search      Alg. 3 result: top-k over live entries of the
 *               probed lists by (dist32, id), padded (+inf,-1) (C4, C5)
 *   bruteforce  exact top-k over all live entries (recall ground truth)
 *   reclaim     quiescent recycling of full, fully-dead slabs (C16)
 *   kmeans      Lloyd (C31)
 *   stats       counters + P:681 overhead 128/(32(4d+8)) (C17)
 * The slab pool is modelled only as counts: list l's entries, in insertion
 * order, occupy ceil(len_l/32) slabs (entries [32j,32j+32) = slab j).
 */
#ifndef SIVF_ORACLE_H
#define SIVF_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct or_index or_index;

enum { OR_ST_OK = 0, OR_ST_POOL_EXHAUSTED = 1, OR_ST_DUPLICATE = 2, OR_ST_ID_OUT_OF_RANGE = 3,
       OR_ST_WRONG_SHARD = 4 };

typedef struct {
  int64_t live, inserted, deleted, slabs_in_use, slabs_free, pool_exhausted_items;
  double overhead_paper;
} or_stats_t;

/* num_slabs <= 0 : pool not modelled (never exhausts). */
or_index* or_create(int32_t dim, int32_t nlist, int64_t id_capacity, int64_t num_slabs,
                    int32_t shard_rank, int32_t shard_count);
void or_destroy(or_index*);
void or_set_centroids(or_index*, const float* c /*[nlist][dim]*/);
void or_set_threads(int32_t n); /* fan-out for pure per-item loops (results identical) */

float or_dist32(const float* a, const float* b, int32_t d);
double or_dist64(const float* a, const float* b, int32_t d);
int32_t or_assign(const float* C, int32_t nlist, int32_t d, const float* x);
void or_assign_batch(const float* C, int32_t nlist, int32_t d, const float* X, int64_t n, int32_t* out);
void or_probe(const float* C, int32_t nlist, int32_t d, const float* q, int32_t m, int32_t* out);

void or_insert(or_index*, const int64_t* ids, const float* X, int64_t n, int32_t* status, int32_t* list);
int64_t or_delete(or_index*, const int64_t* ids, int64_t n);
void or_search(or_index*, const float* Q, int64_t nq, int32_t k, int32_t nprobe, float* dist, int64_t* ids,
               int32_t* probes /*nullable [nq][nprobe]*/);
/* top-k by (dist32, id) of one query over n given candidates X[n][d] with ids[n] (search restricted to them) */
void or_topk_candidates(const float* q, int32_t d, const float* X, const int64_t* ids, int64_t n, int32_t k,
                        float* dist, int64_t* out_ids);
void or_bruteforce(or_index*, const float* Q, int64_t nq, int32_t k, float* dist, int64_t* ids);
int64_t or_reclaim(or_index*);
void or_dump_state(or_index*, int32_t* list_of_id /*[local capacity]*/, int64_t* live_per_list /*[nlist]*/);
void or_stats(or_index*, or_stats_t*);
int64_t or_local_capacity(or_index*);
/* Adopt another (tie-equivalent) list for a live id: used only by checkers
   when an assignment differs within the BASELINE tie tolerance. */
int32_t or_adopt_list(or_index*, int64_t id, int32_t list);
/* Vector of a live id (copy); returns 0 if not live. */
int32_t or_get_vector(or_index*, int64_t id, float* out);

void or_merge_topk(const float* dist_g, const int64_t* ids_g /*[G][nq][k]*/, int32_t G, int64_t nq, int32_t k,
                   float* dist, int64_t* ids);
void or_kmeans(const float* X, int64_t n, int32_t d, int32_t nlist, int32_t niter, uint64_t seed, float* out,
               double* objective /*nullable [niter]*/);
uint64_t or_kmeans_hash(uint64_t seed, uint64_t i);

#ifdef __cplusplus
}
#endif
#endif
