// sivf_oracle.cpp — plain, slow, obviously-correct CPU oracle for the SIVF hot path.
//
// TEST INFRASTRUCTURE (see sivf_oracle.h).  Compiled with -O2 -ffp-contract=off
// and no fast-math: every fp32 operation below is a single IEEE-754 round-to-
// nearest-even operation, so dist32 is the canonical distance of reading C1.
// Shares no code with the CUDA path.
#include "sivf_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <thread>
#include <utility>
#include <vector>

namespace {

int g_threads = 1;

// Run body(i) for i in [0,n) on g_threads threads.  Every body is a pure
// function of its own item, so results are identical to a sequential loop.
void parallel_for(int64_t n, const std::function<void(int64_t)>& body) {
  int T = g_threads;
  if (T <= 1 || n < 64) {
    for (int64_t i = 0; i < n; ++i) body(i);
    return;
  }
  if (T > n) T = (int)n;
  std::vector<std::thread> th;
  int64_t chunk = (n + T - 1) / T;
  for (int t = 0; t < T; ++t) {
    int64_t b = t * chunk, e = std::min<int64_t>(n, b + chunk);
    th.emplace_back([&, b, e] {
      for (int64_t i = b; i < e; ++i) body(i);
    });
  }
  for (auto& x : th) x.join();
}

// Eq. l2: d(q,x) = sum_k (q_k - x_k)^2, evaluated in fp32 in
// ascending k with each subtraction, product and sum rounded separately (C1).
float dist32(const float* a, const float* b, int d) {
  float s = 0.0f;
  for (int k = 0; k < d; ++k) {
    float t = a[k] - b[k];
    float t2 = t * t;
    s = s + t2;
  }
  return s;
}

double dist64(const float* a, const float* b, int d) {
  double s = 0.0;
  for (int k = 0; k < d; ++k) {
    double t = (double)a[k] - (double)b[k];
    s += t * t;
  }
  return s;
}

// Lexicographic (distance, id) order of S:20/S:243 (reading C4).
struct Hit {
  float d;
  int64_t id;
};
bool hit_less(const Hit& a, const Hit& b) { return a.d < b.d || (a.d == b.d && a.id < b.id); }

// Assignment: argmin over l of (dist32(x, c_l), l) — ties to the lowest list
// index ("assigning each vector to a list"; reading C2).
int32_t assign_one(const float* C, int nlist, int d, const float* x) {
  int32_t best = 0;
  float bd = dist32(x, C, d);
  for (int l = 1; l < nlist; ++l) {
    float dl = dist32(x, C + (size_t)l * d, d);
    if (dl < bd) {  // strict: equal distance keeps the lower index
      bd = dl;
      best = l;
    }
  }
  return best;
}

// Probe set: the first m lists of a sort by (dist32(q,c_l), l) (C3).
void probe_one(const float* C, int nlist, int d, const float* q, int m, int32_t* out) {
  std::vector<std::pair<float, int32_t>> v(nlist);
  for (int l = 0; l < nlist; ++l) v[l] = {dist32(q, C + (size_t)l * d, d), l};
  std::partial_sort(v.begin(), v.begin() + m, v.end());  // pair order = (dist, l)
  for (int i = 0; i < m; ++i) out[i] = v[i].second;
}

uint64_t mix64(uint64_t z) {  // splitmix64 finaliser (oracle's own copy)
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace

struct List {
  std::vector<int64_t> ids;  // insertion order; slab j of the list = entries [32j, 32j+32)
  std::vector<float> x;      // [len][d]
  std::vector<uint8_t> dead;
};

struct or_index {
  int d = 0, nlist = 0;
  int64_t cap = 0, cap_local = 0, num_slabs = 0;
  int rank = 0, G = 1;
  std::vector<float> C;
  bool trained = false;
  std::vector<List> lists;
  std::vector<int32_t> list_of_id;  // local id -> list (live) or -1
  std::vector<int64_t> pos_of_id;   // local id -> position in its list (live only)
  int64_t inserted = 0, deleted = 0, live = 0, exhausted = 0;

  int64_t slabs_in_use() const {
    int64_t s = 0;
    for (const auto& L : lists) s += ((int64_t)L.ids.size() + 31) / 32;
    return s;
  }
  // id -> local ATT index, or -1 when out of range / not owned (C13; sharding §8(e))
  int64_t local(int64_t id, int* why) const {
    if (id < 0 || id >= cap) {
      *why = OR_ST_ID_OUT_OF_RANGE;
      return -1;
    }
    if (id % G != rank) {
      *why = OR_ST_WRONG_SHARD;
      return -1;
    }
    *why = OR_ST_OK;
    return id / G;
  }
};

extern "C" {

void or_set_threads(int32_t n) { g_threads = n < 1 ? 1 : n; }

or_index* or_create(int32_t dim, int32_t nlist, int64_t id_capacity, int64_t num_slabs, int32_t shard_rank,
                    int32_t shard_count) {
  if (dim < 1 || nlist < 1 || id_capacity < 0 || shard_count < 1 || shard_rank < 0 || shard_rank >= shard_count)
    return nullptr;
  or_index* ix = new or_index();
  ix->d = dim;
  ix->nlist = nlist;
  ix->cap = id_capacity;
  ix->G = shard_count;
  ix->rank = shard_rank;
  ix->cap_local = id_capacity > shard_rank ? (id_capacity - shard_rank + shard_count - 1) / shard_count : 0;
  ix->num_slabs = num_slabs;
  ix->C.assign((size_t)nlist * dim, 0.f);
  ix->lists.resize(nlist);
  ix->list_of_id.assign(ix->cap_local, -1);
  ix->pos_of_id.assign(ix->cap_local, -1);
  return ix;
}

void or_destroy(or_index* ix) { delete ix; }

void or_set_centroids(or_index* ix, const float* c) {
  std::memcpy(ix->C.data(), c, sizeof(float) * ix->C.size());
  ix->trained = true;
}

int64_t or_local_capacity(or_index* ix) { return ix->cap_local; }

float or_dist32(const float* a, const float* b, int32_t d) { return dist32(a, b, d); }
double or_dist64(const float* a, const float* b, int32_t d) { return dist64(a, b, d); }

int32_t or_assign(const float* C, int32_t nlist, int32_t d, const float* x) { return assign_one(C, nlist, d, x); }

void or_assign_batch(const float* C, int32_t nlist, int32_t d, const float* X, int64_t n, int32_t* out) {
  parallel_for(n, [&](int64_t i) { out[i] = assign_one(C, nlist, d, X + (size_t)i * d); });
}

void or_probe(const float* C, int32_t nlist, int32_t d, const float* q, int32_t m, int32_t* out) {
  probe_one(C, nlist, d, q, m, out);
}

// Batched insert, items processed in batch order (Alg. 1 Insert, P:205-217;
// Alg. 2) with the statuses of readings C9/C12/C13:
//   id outside [0,cap) -> ID_OUT_OF_RANGE; id not owned by this shard -> WRONG_SHARD;
//   id live, or seen earlier in this batch -> DUPLICATE;
//   else assigned list l = assign(x) and appended, unless the slab pool runs out.
// Pool model (reading C33 / SURVEY a4 deterministic policy): within a list the
// batch's items take ranks 0,1,2,... in batch order; the list's partially
// filled last slab offers 32 - len%32 slots (0 if len%32==0); each further 32
// items need one free slab; lists are served in ascending l from the free
// count; an item whose rank falls beyond the granted slots is POOL_EXHAUSTED.
void or_insert(or_index* ix, const int64_t* ids, const float* X, int64_t n, int32_t* status, int32_t* list) {
  const int d = ix->d;
  std::vector<int32_t> st(n, OR_ST_OK), ls(n, -1);
  std::vector<int64_t> lid(n, -1);
  std::vector<uint8_t> seen(ix->cap_local, 0);
  for (int64_t i = 0; i < n; ++i) {
    int why;
    int64_t u = ix->local(ids[i], &why);
    if (u < 0) {
      st[i] = why;
      continue;
    }
    if (ix->list_of_id[u] >= 0 || seen[u]) {
      st[i] = OR_ST_DUPLICATE;
      continue;
    }
    seen[u] = 1;
    lid[i] = u;
  }
  parallel_for(n, [&](int64_t i) {
    if (st[i] == OR_ST_OK) ls[i] = assign_one(ix->C.data(), ix->nlist, d, X + (size_t)i * d);
  });
  // ranks within list, in batch order
  std::vector<int64_t> cnt(ix->nlist, 0), rank(n, -1);
  for (int64_t i = 0; i < n; ++i)
    if (st[i] == OR_ST_OK) rank[i] = cnt[ls[i]]++;
  std::vector<int64_t> avail(ix->nlist, 0);  // slots granted per list
  if (ix->num_slabs > 0) {
    int64_t free_slabs = ix->num_slabs - ix->slabs_in_use();
    for (int l = 0; l < ix->nlist; ++l) {
      if (cnt[l] == 0) continue;
      int64_t len = (int64_t)ix->lists[l].ids.size();
      int64_t tail_free = (len % 32) ? 32 - len % 32 : 0;
      int64_t rest = cnt[l] > tail_free ? cnt[l] - tail_free : 0;
      int64_t need = (rest + 31) / 32;
      int64_t granted = std::min(need, std::max<int64_t>(free_slabs, 0));
      free_slabs -= granted;
      avail[l] = tail_free + 32 * granted;
    }
  } else {
    for (int l = 0; l < ix->nlist; ++l) avail[l] = cnt[l];
  }
  for (int64_t i = 0; i < n; ++i) {
    if (st[i] != OR_ST_OK) continue;
    int l = ls[i];
    if (rank[i] >= avail[l]) {
      st[i] = OR_ST_POOL_EXHAUSTED;
      ix->exhausted++;
      continue;
    }
    List& L = ix->lists[l];
    ix->pos_of_id[lid[i]] = (int64_t)L.ids.size();
    ix->list_of_id[lid[i]] = l;
    L.ids.push_back(ids[i]);
    L.x.insert(L.x.end(), X + (size_t)i * d, X + (size_t)(i + 1) * d);
    L.dead.push_back(0);
    ix->inserted++;
    ix->live++;
  }
  for (int64_t i = 0; i < n; ++i) {
    if (status) status[i] = st[i];
    if (list) list[i] = (st[i] == OR_ST_OK) ? ls[i] : -1;
  }
}

// Alg. 4: per id, look up its location; if present and live,
// clear it (dead flag = the validity bit), count it; absent/out-of-range ids
// and repeated ids are no-ops (idempotence).
int64_t or_delete(or_index* ix, const int64_t* ids, int64_t n) {
  int64_t c = 0;
  for (int64_t i = 0; i < n; ++i) {
    int why;
    int64_t u = ix->local(ids[i], &why);
    if (u < 0) continue;
    int32_t l = ix->list_of_id[u];
    if (l < 0) continue;
    List& L = ix->lists[l];
    L.dead[ix->pos_of_id[u]] = 1;
    ix->list_of_id[u] = -1;
    ix->pos_of_id[u] = -1;
    ix->deleted++;
    ix->live--;
    c++;
  }
  return c;
}

static void topk_fill(std::vector<Hit>& cand, int k, float* dist, int64_t* ids) {
  int m = std::min<int64_t>(k, (int64_t)cand.size());
  std::partial_sort(cand.begin(), cand.begin() + m, cand.end(), hit_less);
  for (int i = 0; i < k; ++i) {
    if (i < m) {
      dist[i] = cand[i].d;
      ids[i] = cand[i].id;
    } else {  // padding (reading C5)
      dist[i] = std::numeric_limits<float>::infinity();
      ids[i] = -1;
    }
  }
}

// Alg. 3 result: for each query, probe nprobe lists, evaluate Eq. l2
// on every entry whose validity bit is set (Eq. slot_valid), return the k
// smallest by (dist32, id).
void or_search(or_index* ix, const float* Q, int64_t nq, int32_t k, int32_t nprobe, float* dist, int64_t* ids,
               int32_t* probes) {
  const int d = ix->d;
  parallel_for(nq, [&](int64_t qi) {
    const float* q = Q + (size_t)qi * d;
    std::vector<int32_t> P(nprobe);
    probe_one(ix->C.data(), ix->nlist, d, q, nprobe, P.data());
    if (probes) std::copy(P.begin(), P.end(), probes + (size_t)qi * nprobe);
    std::vector<Hit> cand;
    for (int p = 0; p < nprobe; ++p) {
      const List& L = ix->lists[P[p]];
      for (size_t e = 0; e < L.ids.size(); ++e)
        if (!L.dead[e]) cand.push_back({dist32(q, L.x.data() + e * d, d), L.ids[e]});
    }
    topk_fill(cand, k, dist + (size_t)qi * k, ids + (size_t)qi * k);
  });
}

// Alg. 3's result restricted to a given candidate set (readings C4, C5): the
// top-k of (dist32(q, x_i), id_i) over the n candidates, ascending, padded (+inf, -1).
// Used by the sampled checks of configurations too large for an oracle index (config H:
// the candidates are the members of a query's probed lists).
void or_topk_candidates(const float* q, int32_t d, const float* X, const int64_t* ids, int64_t n, int32_t k,
                        float* dist, int64_t* out_ids) {
  std::vector<Hit> cand;
  cand.reserve((size_t)n);
  for (int64_t i = 0; i < n; ++i) cand.push_back({dist32(q, X + (size_t)i * d, d), ids[i]});
  topk_fill(cand, k, dist, out_ids);
}

void or_bruteforce(or_index* ix, const float* Q, int64_t nq, int32_t k, float* dist, int64_t* ids) {
  const int d = ix->d;
  parallel_for(nq, [&](int64_t qi) {
    const float* q = Q + (size_t)qi * d;
    std::vector<Hit> cand;
    for (const List& L : ix->lists)
      for (size_t e = 0; e < L.ids.size(); ++e)
        if (!L.dead[e]) cand.push_back({dist32(q, L.x.data() + e * d, d), L.ids[e]});
    topk_fill(cand, k, dist + (size_t)qi * k, ids + (size_t)qi * k);
  });
}

// Quiescent reclamation (reading C16): a slab that is full (32
// reserved slots) and has no live slot is recycled; surviving slabs keep
// their order.  In the count model: remove each full, all-dead 32-entry chunk.
int64_t or_reclaim(or_index* ix) {
  int64_t freed = 0;
  const int d = ix->d;
  for (int l = 0; l < ix->nlist; ++l) {
    List& L = ix->lists[l];
    size_t nch = L.ids.size() / 32;  // full chunks only
    List K;
    bool changed = false;
    for (size_t c = 0; c * 32 < L.ids.size(); ++c) {
      size_t b = c * 32, e = std::min(L.ids.size(), b + 32);
      bool full = c < nch;
      bool all_dead = true;
      for (size_t i = b; i < e; ++i) all_dead = all_dead && L.dead[i];
      if (full && all_dead) {
        freed++;
        changed = true;
        continue;
      }
      K.ids.insert(K.ids.end(), L.ids.begin() + b, L.ids.begin() + e);
      K.dead.insert(K.dead.end(), L.dead.begin() + b, L.dead.begin() + e);
      K.x.insert(K.x.end(), L.x.begin() + b * d, L.x.begin() + e * d);
    }
    if (!changed) continue;
    L = std::move(K);
    for (size_t i = 0; i < L.ids.size(); ++i)
      if (!L.dead[i]) ix->pos_of_id[L.ids[i] / ix->G] = (int64_t)i;
  }
  return freed;
}

void or_dump_state(or_index* ix, int32_t* list_of_id, int64_t* live_per_list) {
  if (list_of_id) std::copy(ix->list_of_id.begin(), ix->list_of_id.end(), list_of_id);
  if (live_per_list) {
    for (int l = 0; l < ix->nlist; ++l) {
      int64_t c = 0;
      for (uint8_t dd : ix->lists[l].dead) c += dd ? 0 : 1;
      live_per_list[l] = c;
    }
  }
}

void or_stats(or_index* ix, or_stats_t* s) {
  s->live = ix->live;
  s->inserted = ix->inserted;
  s->deleted = ix->deleted;
  s->slabs_in_use = ix->slabs_in_use();
  s->slabs_free = ix->num_slabs > 0 ? ix->num_slabs - s->slabs_in_use : -1;
  s->pool_exhausted_items = ix->exhausted;
  // "128-byte header ... amortized over a batch of 32 vectors";
  // 0.77% / 0.10% = 128 / (32 * (4d + 8)) (reading C17)
  s->overhead_paper = 128.0 / (32.0 * (4.0 * ix->d + 8.0));
}

int32_t or_adopt_list(or_index* ix, int64_t id, int32_t list) {
  int why;
  int64_t u = ix->local(id, &why);
  if (u < 0 || ix->list_of_id[u] < 0 || list < 0 || list >= ix->nlist) return 0;
  int32_t old = ix->list_of_id[u];
  if (old == list) return 1;
  const int d = ix->d;
  List& A = ix->lists[old];
  List& B = ix->lists[list];
  int64_t p = ix->pos_of_id[u];
  // The entry moves to the end of the other list (used right after the insert
  // batch that placed it, so "end" is where the other placement put it).
  B.ids.push_back(id);
  B.x.insert(B.x.end(), A.x.begin() + p * d, A.x.begin() + (p + 1) * d);
  B.dead.push_back(0);
  A.ids.erase(A.ids.begin() + p);
  A.x.erase(A.x.begin() + p * d, A.x.begin() + (p + 1) * d);
  A.dead.erase(A.dead.begin() + p);
  for (size_t i = p; i < A.ids.size(); ++i)
    if (!A.dead[i]) ix->pos_of_id[A.ids[i] / ix->G] = (int64_t)i;
  ix->list_of_id[u] = list;
  ix->pos_of_id[u] = (int64_t)B.ids.size() - 1;
  return 1;
}

int32_t or_get_vector(or_index* ix, int64_t id, float* out) {
  int why;
  int64_t u = ix->local(id, &why);
  if (u < 0 || ix->list_of_id[u] < 0) return 0;
  const List& L = ix->lists[ix->list_of_id[u]];
  std::copy(L.x.begin() + ix->pos_of_id[u] * ix->d, L.x.begin() + (ix->pos_of_id[u] + 1) * ix->d, out);
  return 1;
}

// Multi-GPU merge (§8(e)): the k smallest by (dist, id) of the union of the
// per-shard top-k lists; padding entries (id -1) are not candidates.
void or_merge_topk(const float* dist_g, const int64_t* ids_g, int32_t G, int64_t nq, int32_t k, float* dist,
                   int64_t* ids) {
  for (int64_t q = 0; q < nq; ++q) {
    std::vector<Hit> cand;
    for (int g = 0; g < G; ++g)
      for (int i = 0; i < k; ++i) {
        size_t o = ((size_t)g * nq + q) * k + i;
        if (ids_g[o] >= 0) cand.push_back({dist_g[o], ids_g[o]});
      }
    topk_fill(cand, k, dist + q * k, ids + q * k);
  }
}

uint64_t or_kmeans_hash(uint64_t seed, uint64_t i) { return mix64(seed ^ mix64(i)); }

// Lloyd's k-means (reading C31):
//  init: partial Fisher-Yates over [0,n): for i < nlist, j = i + H(seed,i) mod (n-i),
//        swap(perm[i], perm[j]); centroid l = X[perm[l]].
//  iteration: (1) assign every point by (dist32, l) ties lowest l;
//             (2) each empty cluster e, ascending: take the largest cluster L
//                 (ties: lowest l), move its point farthest from c_L (dist32
//                 from step 1; ties: lowest point index) into e;
//             (3) c_l = fp32( (sum over members, ascending point index, in
//                 fp64) / count ), each coordinate rounded once.
void or_kmeans(const float* X, int64_t n, int32_t d, int32_t nlist, int32_t niter, uint64_t seed, float* out,
               double* objective) {
  if (n < nlist) return;
  std::vector<int64_t> perm(n);
  for (int64_t i = 0; i < n; ++i) perm[i] = i;
  for (int64_t i = 0; i < nlist; ++i) {
    int64_t j = i + (int64_t)(or_kmeans_hash(seed, (uint64_t)i) % (uint64_t)(n - i));
    std::swap(perm[i], perm[j]);
  }
  std::vector<float> C((size_t)nlist * d);
  for (int l = 0; l < nlist; ++l) std::copy(X + perm[l] * d, X + (perm[l] + 1) * d, C.begin() + (size_t)l * d);
  std::vector<int32_t> a(n);
  std::vector<float> dd(n);
  for (int it = 0; it < niter; ++it) {
    parallel_for(n, [&](int64_t i) {
      a[i] = assign_one(C.data(), nlist, d, X + i * d);
      dd[i] = dist32(X + i * d, C.data() + (size_t)a[i] * d, d);
    });
    if (objective) {
      double J = 0;
      for (int64_t i = 0; i < n; ++i) J += dist64(X + i * d, C.data() + (size_t)a[i] * d, d);
      objective[it] = J;
    }
    std::vector<int64_t> cnt(nlist, 0);
    for (int64_t i = 0; i < n; ++i) cnt[a[i]]++;
    for (int e = 0; e < nlist; ++e) {
      if (cnt[e] != 0) continue;
      int L = 0;
      for (int l = 1; l < nlist; ++l)
        if (cnt[l] > cnt[L]) L = l;
      int64_t p = -1;
      for (int64_t i = 0; i < n; ++i)
        if (a[i] == L && (p < 0 || dd[i] > dd[p])) p = i;
      a[p] = e;
      dd[p] = 0.f;
      cnt[L]--;
      cnt[e]++;
    }
    std::vector<double> S((size_t)nlist * d, 0.0);
    for (int64_t i = 0; i < n; ++i)
      for (int k = 0; k < d; ++k) S[(size_t)a[i] * d + k] += (double)X[i * d + k];
    for (int l = 0; l < nlist; ++l)
      for (int k = 0; k < d; ++k) C[(size_t)l * d + k] = (float)(S[(size_t)l * d + k] / (double)cnt[l]);
  }
  std::copy(C.begin(), C.end(), out);
}

}  // extern "C"
