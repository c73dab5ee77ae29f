// sivf_host.h — host-side handle and the internal launcher interface shared by
// the .cu translation units of libsivf.so.
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "sivf_internal.cuh"

namespace sivf {

// Scan tiling (k_scan.cu): QPW queries per compute warp.
constexpr int kQPW = 4;

struct Scratch {
  // insert / train (max_rows = max(max_batch, max_train))
  int64_t max_rows = 0;
  int32_t* row_list = nullptr;      // [max_rows] assigned list
  int32_t* row_rank = nullptr;      // [max_rows] within-chunk rank
  int32_t* row_status = nullptr;    // [max_rows]
  int64_t* row_lid = nullptr;       // [max_rows] local id or -1
  unsigned long long* row_best = nullptr; // [max_rows] argmin key (dist32 bits << 32 | list)
  int32_t* chunk_hist = nullptr;    // [max_chunks][nlist] -> exclusive prefix over chunks
  int64_t max_chunks = 0;
  int32_t* list_cnt = nullptr;      // [nlist]
  int32_t* list_tail_free = nullptr;// [nlist]
  int32_t* list_tail_slab = nullptr;// [nlist]
  int32_t* list_granted = nullptr;  // [nlist]
  int32_t* list_newbase = nullptr;  // [nlist] index into free_stack of the list's first new slab
  int64_t* list_newoff = nullptr;   // [nlist] directory offsets after a compaction (k_reserve)
  // search (max_queries x max_nprobe)
  float* coarse = nullptr;          // [coarse_rows][nlist] distance matrix (exact SIMT path) or the
                                    // tensor-core approximation A (k_coarse_select path)
  int64_t coarse_rows = 0;
  int32_t* probes = nullptr;        // [max_queries][max_nprobe]
  int32_t* inv_cnt = nullptr;       // [2 nlist]   (probe-rank bucket, list)
  int32_t* inv_off = nullptr;       // [2 nlist + 1]
  int32_t* inv_cursor = nullptr;    // [2 nlist]
  int32_t* inv_pairs = nullptr;     // [max_queries * max_nprobe] pair = q * nprobe + p
  int32_t* tile_off = nullptr;      // [2 nlist + 1]
  int32_t* work_l = nullptr;        // [max_work] list of each work item
  int32_t* work_p0 = nullptr;       // [max_work] first pair (index into inv_pairs)
  int32_t* work_n = nullptr;        // [max_work] number of pairs (queries) in the item
  int64_t max_work = 0;
  unsigned long long* partial = nullptr; // [max_queries][max_nprobe][kp]
  int32_t kp = 0;                   // padded k for partials
  // train
  float* train_sums = nullptr;      // unused (sums written straight to centroids)
  int32_t* train_perm = nullptr;    // [max_train]
  int32_t* train_members = nullptr; // [max_train]
  int32_t* train_cnt = nullptr;     // [nlist]
  int32_t* train_off = nullptr;     // [nlist + 1]
  // validation
  uint32_t* slab_mark = nullptr;    // [num_slabs]
  uint32_t* gthr = nullptr;         // [max_queries] per-query global k-th distance bound (fp32 bits)
  // GEMM scan (D > 128, k_scan_gs.cu)
  int64_t gs_items = 0;             // work items of <= 128 queries the query tiles are sized for
  uint16_t* gs_a = nullptr;         // [gs_items][Dg/64][hi 16 KB | lo 16 KB] split-fp16 query tiles
  float* gs_qn = nullptr;           // [gs_items][128] ||q||^2
  float* gs_qs = nullptr;           // [gs_items][128] 2^-e_q
  uint16_t* gs_qh = nullptr;        // [max_queries][Dg] split-fp16 hi half of each query (k_gs_qsplit)
  uint16_t* gs_ql = nullptr;        // [max_queries][Dg] lo half
  float* gs_qqn = nullptr;          // [max_queries] ||q||^2
  float* gs_qqs = nullptr;          // [max_queries] 2^-e_q
  int64_t* item_doff = nullptr;     // [max_work + 1] item's region in dense (-1: SIMT fallback)
  int32_t* item_dlen = nullptr;     // [max_work] directory length at planning (row stride = 32 dlen)
  int32_t* item_nlive = nullptr;    // [max_work] live slabs scanned
  int32_t* item_of = nullptr;       // [npairs] inverse-map position -> work item
  int32_t* pair_pos = nullptr;      // [npairs] pair -> inverse-map position
  float* dense = nullptr;           // [dense_cap] per item: slab ids (pad 4) + [rows][32 dlen] distances
  int64_t dense_cap = 0;
  long long* tmp64 = nullptr;       // [16] small device scalars
  // tensor-core coarse quantisation (k_coarse_tc.cu)
  int64_t tc_rows = 0;              // rows per k_coarse_gemm pass
  float* x_tiles = nullptr;         // [tc_rows/128][Dp/4][128][4]
  float* x_norm = nullptr;          // [tc_rows]
  float* c_tiles = nullptr;         // [nlist/256][Dp/4][256][4]
  float* c_norm = nullptr;          // [nlist/256 * 256] ||c||^2
  float* c_csa = nullptr;           // [nlist/256 * 256] ka ||c||
  float* c_cnb = nullptr;           // [nlist/256 * 256] kb ||c||^2
  unsigned long long* cand = nullptr; // [rows][cap] candidate lower-bound keys
  float* cand_ubv = nullptr;        // [rows][cap] candidate upper bounds
  int32_t* cand_cnt = nullptr;      // [tc_rows]
  int32_t cand_cap_assign = 0, cand_cap_probe = 0;
  // the search front's own coarse scratch (overlaps insert's assignment in the sliding step)
  int64_t q_rows = 0;               // max_queries rounded up to 128
  float* qx_tiles = nullptr;        // [q_rows/128][hi, lo][Dp/4][128][4]
  float* qx_norm = nullptr;         // [q_rows]
  float* qcoarse = nullptr;         // [q_rows][nlist]
};

struct PhaseRec {
  int phase;
  cudaEvent_t a, b;
};

struct Index {
  sivf_config cfg{};
  DevState st{};
  Scratch sc{};
  // NEXT-2: a view (sivf_create_view) shares its owner's index state and owns its scratch
  bool view = false;
  Index* owner = nullptr;       // a view's owner (nullptr on an owner)
  bool dirs_prepared = false;   // owner: sivf_reserve_directories ran since the last quiescent mutation
  bool conc_used = false;       // owner: sivf_insert_concurrent ran (reclaim then also recycles leaked slabs)
  bool trained = false;
  bool use_tc_scan = true;
  bool use_tc_coarse = true;  // tcgen05 coarse quantisation (k_coarse_tc.cu); false = exact SIMT k_dist_exact
  int tc_two_phase = 0;    // nearest-list-first scan phase (SIVF_OPT_TC_TWO_PHASE)  // tensor-core scan when Dp <= 256 and k <= 32 (k_scan_tc.cu)
  // search -> coarse hand-off: when set, k_coarse_select also counts the inverse probe map
  // (k_inv_count fused) into fuse_inv_cnt and sets fuse_inv_done
  int32_t* fuse_inv_cnt = nullptr;
  int fuse_nb = 1, fuse_r0 = 0;
  bool fuse_inv_done = false;
  bool coarse_select = true;  // A-matrix + per-row selection coarse path (SIVF_OPT_COARSE_SELECT)
  bool coarse_select_ok = true;  // the selection kernels' shared memory fits (setup_coarse_tc)
  int rank_split = 1;         // nearest-probes-first work order (SIVF_OPT_RANK_SPLIT; > 1: r0)
  int dbg = 0;                // experiment switches (SIVF_OPT_DEBUG)
  int tc_max_stages = 0;      // experiments: cap on the tensor-core scan's stage ring (option 98; 0 = as many as fit)
  int seed_list = 0;          // per-list seed of the k-th distance bounds before the tensor-core scan (SIVF_OPT_SEED_LIST; off: measured neutral)
  int seed_slabs = 0;         // k-th distance seeding before the tensor-core scan (SIVF_OPT_SEED_SLABS; off: it costs more than it saves)
  int64_t launches = 0;
  alignas(64) unsigned char coarse_tmap[128] = {};  // TMA store descriptor of sc.coarse (k_coarse_tc.cu)
  bool coarse_tmap_ok = false;
  alignas(64) unsigned char qcoarse_tmap[128] = {};  // TMA store descriptor of sc.qcoarse
  bool qcoarse_tmap_ok = false;
  bool coarse_alt = false;    // launch_coarse_tc: use the search-front scratch set
  cudaStream_t side = nullptr;  // second stream for the sliding step's search front
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // sliding-step graph cache (SIVF_OPT_STEP_GRAPH): one instantiated CUDA graph per
  // distinct call signature (pointers, sizes, stream, options epoch), replayed on
  // repeat calls; captured on cap_stream, launched on the caller's stream
  struct StepGraph {
    const void* p[8] = {};
    int64_t n[3] = {};
    int32_t k = 0, nprobe = 0, kind = 0;  // kind: 0 sliding step, 1 search
    cudaStream_t s = nullptr;
    uint64_t epoch = 0, used = 0;
    int64_t launches = 0;
    bool bad = false;  // step_seen: this signature failed to capture; always launched directly
    cudaGraphExec_t exec = nullptr;
  };
  static constexpr int kStepGraphs = 4;
  StepGraph step_graphs[kStepGraphs];
  StepGraph step_seen[kStepGraphs];  // signatures seen once (captured on their second call)
  bool step_graph = true;
  uint64_t opt_epoch = 1, step_tick = 0;
  cudaStream_t cap_stream = nullptr;
  int num_sms = 148;
  size_t smem_optin = 227 * 1024;
  // phase profiling (sivf_profile_*)
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<PhaseRec> recs;
  cudaEvent_t get_event() {
    if (ev_pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = ev_pool.back();
    ev_pool.pop_back();
    return e;
  }
  ~Index() {
    if (side) cudaStreamDestroy(side);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    for (auto& g : step_graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    for (auto& r : recs) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    for (auto e : ev_pool) cudaEventDestroy(e);
  }
};

// RAII phase bracket: records an event pair on `s` when profiling is on.
struct PhaseTimer {
  Index& ix;
  int phase;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  PhaseTimer(Index& ix_, int ph, cudaStream_t s_) : ix(ix_), phase(ph), s(s_) {
    if (ix.prof) {
      a = ix.get_event();
      cudaEventRecord(a, s);
    }
  }
  ~PhaseTimer() {
    if (ix.prof) {
      cudaEvent_t b = ix.get_event();
      cudaEventRecord(b, s);
      ix.recs.push_back(PhaseRec{phase, a, b});
    }
  }
};

// ---- launchers (each returns cudaGetLastError after enqueueing) ----
// k_insert.cu
cudaError_t launch_insert(Index& ix, const int64_t* d_ids, const float* d_x, int64_t n, int32_t* d_status,
                          int32_t* d_list, cudaStream_t s);
cudaError_t launch_insert_concurrent(Index& ix, const int64_t* d_ids, const float* d_x, int64_t n, int32_t* d_status,
                                     int32_t* d_list, cudaStream_t s);
cudaError_t launch_reserve_dirs(Index& ix, int spare, int32_t* d_fail, cudaStream_t s);
// k_delete.cu
cudaError_t launch_delete(Index& ix, const int64_t* d_ids, int64_t n, int64_t* d_ndeleted, cudaStream_t s);
cudaError_t launch_reclaim(Index& ix, int64_t* d_nreclaimed, cudaStream_t s);
cudaError_t launch_dump(Index& ix, int32_t* d_list_of_id, int64_t* d_live_per_list, int64_t* d_viol, cudaStream_t s);
// k_coarse.cu (dispatch: tensor cores when supported, else exact SIMT)
// -> sc.row_best (list in the low word; the dist32 in the high word only when need_dist)
cudaError_t launch_assign_exact(Index& ix, const float* d_x, int64_t n, cudaStream_t s, bool need_dist = true);
cudaError_t launch_probe_exact(Index& ix, const float* d_q, int64_t nq, int32_t nprobe, cudaStream_t s); // -> sc.probes
cudaError_t setup_coarse_exact(Index& ix);
// k_coarse_tc.cu
bool coarse_tc_supported(const Index& ix, int m);
cudaError_t setup_coarse_tc(Index& ix);
cudaError_t refresh_centroid_tiles(Index& ix, cudaStream_t s);
int coarse_tc_tile_rows();
int coarse_tc_tile_cols();
cudaError_t launch_coarse_tc(Index& ix, const float* d_x, int64_t n, int m, unsigned long long* best,
                             int32_t* probes, cudaStream_t s, bool need_dist = true);
// k_search.cu
struct SearchPlan {
  bool tc, ok;
  bool gs;  // D > 128: the split-fp16 GEMM scan + per-query selection (k_scan_gs.cu)
  int nw, QT, nb, r0;
  size_t smem;
};
SearchPlan plan_search(const Index& ix, int64_t nq, int32_t k, int32_t nprobe);
cudaError_t launch_search_front(Index& ix, const SearchPlan& p, const float* d_q, int64_t nq, int32_t nprobe,
                                int32_t* d_probes, cudaStream_t s, const int32_t* probes_in = nullptr);
cudaError_t launch_search_back(Index& ix, const SearchPlan& p, const float* d_q, int64_t nq, int32_t k,
                               int32_t nprobe, float* d_dist, int64_t* d_ids, cudaStream_t s,
                               cudaEvent_t after_scan = nullptr);
bool coarse_front_concurrent_ok(const Index& ix, int32_t nprobe);
cudaError_t launch_search(Index& ix, const float* d_q, int64_t nq, int32_t k, int32_t nprobe, float* d_dist,
                          int64_t* d_ids, int32_t* d_probes, cudaStream_t s, const int32_t* probes_in = nullptr);
cudaError_t launch_seed_bound(Index& ix, const float* d_q, int64_t nq, int k, int nprobe, cudaStream_t s);
cudaError_t launch_merge_topk(const float* d_dist_g, const int64_t* d_ids_g, int32_t G, int64_t nq, int32_t k,
                              float* d_dist, int64_t* d_ids, cudaStream_t s, int64_t* launches);
// k_train.cu
cudaError_t launch_train(Index& ix, const float* d_x, int64_t n, int32_t niter, cudaStream_t s);
// shared by insert and train: stable per-list ranks of rows with row_status==OK
cudaError_t launch_stable_ranks(Index& ix, int64_t n, int check_claim, cudaStream_t s);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace sivf
