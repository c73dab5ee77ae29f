// sivf_api.cu — the C ABI (include/sivf.h): argument validation, arena
// carving, and stream-ordered sequencing of the kernels.
#include <cstring>
#include <new>

#include "sivf_host.h"

namespace sivf {
size_t scan_smem_for(const Index& ix, int k, int* nw_out);
cudaError_t setup_search_kernels(Index& ix);

namespace {

constexpr size_t kAlign = 256;

struct Layout {
  size_t total = 0;
  size_t payload, payload16, payload_g, slab_xs, slab_ids, slab_norm, slab_flag, bitmap, cursor, slab_list, free_stack, slab_mark, att, claim,
      dir_off, dir_len, dir_cap, dir_arena, centroids, ctr, ictr, sctr, tmp64, gthr;
  size_t row_list, row_rank, row_status, row_lid, row_best, chunk_hist, list_cnt, list_tail_free, list_tail_slab,
      list_granted, list_newbase, list_newoff;
  size_t coarse, probes, inv_cnt, inv_off, inv_cursor, inv_pairs, tile_off, work_l, work_p0, work_n, partial;
  size_t train_perm, train_members, train_off;
  size_t qx_tiles, qx_norm, qcoarse;
  int64_t q_rows;
  size_t x_tiles, x_norm, c_tiles, c_norm, c_csa, c_cnb, cand, cand_ubv, cand_cnt;
  int64_t tc_rows, cap_assign, cap_probe;
  size_t gs_a, gs_qn, gs_qs, gs_qh, gs_ql, gs_qqn, gs_qqs, item_doff, item_dlen, item_nlive, item_of, pair_pos, dense;
  int64_t gs_items, dense_cap;
  int64_t Dp, Dh, Dg, cap_local, dir_half, max_rows, max_chunks, coarse_rows, max_work;
};

size_t take(Layout& L, size_t bytes) {
  size_t off = L.total;
  L.total += (bytes + kAlign - 1) / kAlign * kAlign;
  return off;
}

bool valid_config(const sivf_config* c) {
  if (!c) return false;
  if (c->dim < 1 || c->nlist < 1 || c->nlist > 65536) return false;
  if (c->id_capacity < 0 || c->id_capacity > 0xFFFFFFFEll) return false;
  if (c->num_slabs < 1 || c->num_slabs > 0x7FFFFFFFll) return false;
  if (c->max_batch < 0 || c->max_queries < 0 || c->max_train < 0) return false;
  if (c->max_k < 1 || c->max_k > 128) return false;
  if (c->max_nprobe < 1 || c->max_nprobe > c->nlist || c->max_nprobe > 1024) return false;
  if (c->shard_count < 1 || c->shard_rank < 0 || c->shard_rank >= c->shard_count) return false;
  if (c->max_train > 0 && c->max_train < c->nlist) return false;
  if ((int64_t)c->max_queries * c->max_nprobe > 0x7FFFFFFFll) return false;
  if (c->flags & ~(int32_t)(SIVF_CFG_NO_SCAN_COPY | SIVF_CFG_CONCURRENT | SIVF_CFG_SPLIT_COPY))
    return false;  // unknown flag bits
  return true;
}

// view == true: a view's arena (sivf_create_view): the index state arrays are the
// owner's (zero bytes here), every scratch array is the view's own.
Layout make_layout(const sivf_config* c, bool view = false) {
  Layout L;
  const int64_t D = c->dim, nl = c->nlist, S = c->num_slabs;
  L.Dp = (D + 7) / 8 * 8;  // tf32 MMA K-step = 8 dims
  // fp16 scan copy (kind::f16 K-step = 16 dims); none for D > 128 or SIVF_CFG_NO_SCAN_COPY
  const bool nocopy = (c->flags & SIVF_CFG_NO_SCAN_COPY) != 0;
  const bool split = D > 128 || (c->flags & SIVF_CFG_SPLIT_COPY) != 0;
  L.Dh = (!split && !nocopy) ? (D + 15) / 16 * 16 : 0;
  // split-fp16 scan copy for D > 128 or SIVF_CFG_SPLIT_COPY (k_scan_gs.cu, 64-dim K chunks)
  L.Dg = (split && !nocopy) ? (D + 63) / 64 * 64 : 0;
  const int64_t cap = c->id_capacity, G = c->shard_count, r = c->shard_rank;
  L.cap_local = cap > r ? (cap - r + G - 1) / G : 0;
  // directory arena: two halves; a compaction into the idle half needs at most
  // sum over lists of max(8, 2 len) <= 2 S + 8 nl entries (k_reserve), or of
  // max(8, 2 len, len + spare) <= 2 S + 264 nl with spare <= 256 (k_reserve_dirs,
  // SIVF_CFG_CONCURRENT)
  L.dir_half = 2 * S + ((c->flags & SIVF_CFG_CONCURRENT) ? 264 : 8) * nl + 64;
  L.max_rows = c->max_batch > c->max_train ? c->max_batch : c->max_train;
  if (L.max_rows < 1) L.max_rows = 1;
  L.max_chunks = (L.max_rows + 1023) / 1024;
  int64_t cr = ((int64_t)1 << 26) / nl;
  if (cr < 64) cr = 64;
  {
    // rows per coarse pass: a whole search batch or insert batch when it fits (whole 128-row tiles)
    const int64_t want = c->max_queries > c->max_batch ? c->max_queries : c->max_batch;
    L.coarse_rows = want < cr ? want : cr;
    if (L.coarse_rows < 1) L.coarse_rows = 1;
    L.coarse_rows = (L.coarse_rows + 127) / 128 * 128;
  }
  const int64_t npairs = (int64_t)c->max_queries * c->max_nprobe;
  L.max_work = (npairs + 7) / 8 + 2 * nl + 1;

  const size_t sv = view ? 0 : 1;  // state arrays: the owner's in a view
  L.payload = take(L, sv * (size_t)S * kSlot * L.Dp * 4);
  L.payload16 = take(L, L.Dh ? sv * (size_t)S * rec16_bytes((int)L.Dh) : 0);
  L.payload_g = take(L, L.Dg ? sv * (size_t)S * recg_bytes((int)L.Dg) : 0);
  L.slab_xs = take(L, L.Dg ? sv * (size_t)S * kSlot * 4 : 0);
  L.slab_ids = take(L, sv * (size_t)S * kSlot * 4);
  L.slab_norm = take(L, sv * (size_t)S * kSlot * 4);
  L.slab_flag = take(L, sv * (size_t)S * 4);
  L.bitmap = take(L, sv * (size_t)S * 4);
  L.cursor = take(L, sv * (size_t)S * 4);
  L.slab_list = take(L, sv * (size_t)S * 4);
  L.free_stack = take(L, sv * (size_t)S * 4);
  L.slab_mark = take(L, sv * (size_t)S * 4);
  L.att = take(L, sv * (size_t)L.cap_local * 8);
  L.claim = take(L, sv * (size_t)L.cap_local * 4);
  L.dir_off = take(L, sv * (size_t)nl * 8);
  L.dir_len = take(L, sv * (size_t)nl * 4);
  L.dir_cap = take(L, sv * (size_t)nl * 4);
  L.dir_arena = take(L, sv * (size_t)2 * L.dir_half * 4);
  L.centroids = take(L, sv * (size_t)nl * L.Dp * 4);
  L.ctr = take(L, sv * C_NCTR * 8);
  L.ictr = take(L, sv * I_NICTR * 4);
  L.sctr = take(L, I_NICTR * 4);
  L.tmp64 = take(L, 16 * 8);
  L.gthr = take(L, (size_t)(c->max_queries > 0 ? c->max_queries : 1) * 4);
  L.row_list = take(L, (size_t)L.max_rows * 4);
  L.row_rank = take(L, (size_t)L.max_rows * 4);
  L.row_status = take(L, (size_t)L.max_rows * 4);
  L.row_lid = take(L, (size_t)L.max_rows * 8);
  L.row_best = take(L, (size_t)L.max_rows * 8);
  L.chunk_hist = take(L, (size_t)L.max_chunks * nl * 4);
  L.list_cnt = take(L, (size_t)nl * 4);
  L.list_tail_free = take(L, (size_t)nl * 4);
  L.list_tail_slab = take(L, (size_t)nl * 4);
  L.list_granted = take(L, (size_t)nl * 4);
  L.list_newbase = take(L, (size_t)nl * 4);
  L.list_newoff = take(L, (size_t)nl * 8);
  L.coarse = take(L, (size_t)L.coarse_rows * nl * 4);
  L.probes = take(L, (size_t)npairs * 4 + 4);
  L.inv_cnt = take(L, (size_t)2 * nl * 4);
  L.inv_off = take(L, (size_t)(2 * nl + 1) * 4);
  L.inv_cursor = take(L, (size_t)2 * nl * 4);
  L.inv_pairs = take(L, (size_t)npairs * 4 + 4);
  L.tile_off = take(L, (size_t)(2 * nl + 1) * 4);
  L.work_l = take(L, (size_t)L.max_work * 4);
  L.work_p0 = take(L, (size_t)L.max_work * 4);
  L.work_n = take(L, (size_t)L.max_work * 4);
  L.partial = take(L, (size_t)npairs * c->max_k * 8 + 8);
  L.train_perm = take(L, (size_t)(c->max_train > 0 ? c->max_train : 1) * 4);
  L.train_members = take(L, (size_t)(c->max_train > 0 ? c->max_train : 1) * 4);
  L.train_off = take(L, (size_t)(nl + 1) * 4);
  // tensor-core coarse quantisation: rows per pass = max(batch, queries), 128-row tiles
  int64_t tr = c->max_batch > c->max_queries ? c->max_batch : c->max_queries;
  if (tr < 128) tr = 128;
  L.tc_rows = (tr + 127) / 128 * 128;
  const int64_t nct = (nl + 255) / 256;
  L.cap_assign = nl < 32 ? nl : 32;
  L.cap_probe = nl < 512 ? nl : 512;
  const int64_t cap_rows = L.tc_rows * L.cap_assign > (int64_t)c->max_queries * L.cap_probe
                               ? L.tc_rows * L.cap_assign
                               : (int64_t)c->max_queries * L.cap_probe;
  L.x_tiles = take(L, (size_t)2 * L.tc_rows * L.Dp * 4);  // hi and lo tf32 parts
  L.x_norm = take(L, (size_t)L.tc_rows * 4);
  L.c_tiles = take(L, (size_t)2 * nct * 256 * L.Dp * 4);
  L.c_norm = take(L, (size_t)nct * 256 * 4);
  L.c_csa = take(L, (size_t)nct * 256 * 4);
  L.c_cnb = take(L, (size_t)nct * 256 * 4);
  L.cand = take(L, (size_t)cap_rows * 8);
  L.cand_ubv = take(L, (size_t)cap_rows * 4);
  L.cand_cnt = take(L, (size_t)L.tc_rows * 4);
  L.q_rows = (c->max_queries + 127) / 128 * 128;
  if (nl > 1024) L.q_rows = 0;  // the concurrent search front needs the k_coarse_select path
  L.qx_tiles = take(L, (size_t)2 * L.q_rows * L.Dp * 4);
  L.qx_norm = take(L, (size_t)L.q_rows * 4);
  L.qcoarse = take(L, (size_t)L.q_rows * nl * 4);
  // GEMM scan (D > 128, k_scan_gs.cu): per work item of <= 128 queries its split-fp16
  // query tile, per pair its row of list distances in the dense buffer, sized for lists
  // up to twice the average length (items beyond it take the SIMT fallback)
  L.gs_items = L.Dg ? npairs / 128 + nl + 1 : 0;
  L.gs_a = take(L, (size_t)L.gs_items * L.Dg * 512);
  L.gs_qn = take(L, (size_t)L.gs_items * 128 * 4);
  L.gs_qs = take(L, (size_t)L.gs_items * 128 * 4);
  {
    const size_t mq = (size_t)(c->max_queries > 0 ? c->max_queries : 1);
    L.gs_qh = take(L, L.Dg ? mq * L.Dg * 2 : 0);
    L.gs_ql = take(L, L.Dg ? mq * L.Dg * 2 : 0);
    L.gs_qqn = take(L, L.Dg ? mq * 4 : 0);
    L.gs_qqs = take(L, L.Dg ? mq * 4 : 0);
  }
  L.item_doff = take(L, L.Dg ? (size_t)(L.max_work + 1) * 8 : 0);
  L.item_dlen = take(L, L.Dg ? (size_t)L.max_work * 4 : 0);
  L.item_nlive = take(L, L.Dg ? (size_t)L.max_work * 4 : 0);
  L.item_of = take(L, L.Dg ? (size_t)npairs * 4 + 4 : 0);
  L.pair_pos = take(L, L.Dg ? (size_t)npairs * 4 + 4 : 0);
  {
    int64_t lavg = (2 * S + nl - 1) / nl;
    if (lavg < 8) lavg = 8;
    int64_t cap = L.Dg ? npairs * 33 * lavg + 4 * L.max_work : 0;
    if (cap > ((int64_t)3 << 29)) cap = (int64_t)3 << 29;  // 6 GB
    L.dense_cap = cap;
    L.dense = take(L, (size_t)cap * 4);
  }
  return L;
}

__global__ void k_init(DevState st) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < st.num_slabs) {
    st.free_stack[i] = (int32_t)i;  // free list [0..num_slabs), P_top = pool size
    st.slab_list[i] = -1;
    st.bitmap[i] = 0u;
    st.cursor[i] = 0u;
  }
  if (i < st.nlist) {
    st.dir_off[i] = 0;
    st.dir_len[i] = 0;  // P:194 list heads "initialized to an invalid value"
    st.dir_cap[i] = 0;
  }
  if (i < C_NCTR) st.ctr[i] = 0ull;
  if (i < I_NICTR) {
    st.ictr[i] = 0;
    st.sctr[i] = 0;
  }
  if (i == 0) st.ictr[I_FREE_TOP] = (int32_t)st.num_slabs;
}

template <typename T>
T* at(void* base, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(base) + off);
}

sivf_rc cuda_rc(cudaError_t e) { return e == cudaSuccess ? SIVF_OK : SIVF_E_CUDA; }

// Scratch carving of an arena (an owner's or a view's; the layout puts every
// scratch array after the state arrays).
void carve_scratch(Scratch& sc, void* d_arena, const Layout& L) {
  sc.max_rows = L.max_rows;
  sc.row_list = at<int32_t>(d_arena, L.row_list);
  sc.row_rank = at<int32_t>(d_arena, L.row_rank);
  sc.row_status = at<int32_t>(d_arena, L.row_status);
  sc.row_lid = at<int64_t>(d_arena, L.row_lid);
  sc.row_best = at<unsigned long long>(d_arena, L.row_best);
  sc.chunk_hist = at<int32_t>(d_arena, L.chunk_hist);
  sc.max_chunks = L.max_chunks;
  sc.list_cnt = at<int32_t>(d_arena, L.list_cnt);
  sc.list_tail_free = at<int32_t>(d_arena, L.list_tail_free);
  sc.list_tail_slab = at<int32_t>(d_arena, L.list_tail_slab);
  sc.list_granted = at<int32_t>(d_arena, L.list_granted);
  sc.list_newbase = at<int32_t>(d_arena, L.list_newbase);
  sc.list_newoff = at<int64_t>(d_arena, L.list_newoff);
  sc.coarse = at<float>(d_arena, L.coarse);
  sc.q_rows = L.q_rows;
  sc.qx_tiles = at<float>(d_arena, L.qx_tiles);
  sc.qx_norm = at<float>(d_arena, L.qx_norm);
  sc.qcoarse = at<float>(d_arena, L.qcoarse);
  sc.coarse_rows = L.coarse_rows;
  sc.probes = at<int32_t>(d_arena, L.probes);
  sc.inv_cnt = at<int32_t>(d_arena, L.inv_cnt);
  sc.inv_off = at<int32_t>(d_arena, L.inv_off);
  sc.inv_cursor = at<int32_t>(d_arena, L.inv_cursor);
  sc.inv_pairs = at<int32_t>(d_arena, L.inv_pairs);
  sc.tile_off = at<int32_t>(d_arena, L.tile_off);
  sc.work_l = at<int32_t>(d_arena, L.work_l);
  sc.work_p0 = at<int32_t>(d_arena, L.work_p0);
  sc.work_n = at<int32_t>(d_arena, L.work_n);
  sc.max_work = L.max_work;
  sc.partial = at<unsigned long long>(d_arena, L.partial);
  sc.train_perm = at<int32_t>(d_arena, L.train_perm);
  sc.train_members = at<int32_t>(d_arena, L.train_members);
  sc.train_off = at<int32_t>(d_arena, L.train_off);
  sc.slab_mark = at<uint32_t>(d_arena, L.slab_mark);
  sc.tmp64 = at<long long>(d_arena, L.tmp64);
  sc.gthr = at<uint32_t>(d_arena, L.gthr);
  sc.tc_rows = L.tc_rows;
  sc.x_tiles = at<float>(d_arena, L.x_tiles);
  sc.x_norm = at<float>(d_arena, L.x_norm);
  sc.c_tiles = at<float>(d_arena, L.c_tiles);
  sc.c_norm = at<float>(d_arena, L.c_norm);
  sc.c_csa = at<float>(d_arena, L.c_csa);
  sc.c_cnb = at<float>(d_arena, L.c_cnb);
  sc.cand = at<unsigned long long>(d_arena, L.cand);
  sc.cand_ubv = at<float>(d_arena, L.cand_ubv);
  sc.cand_cnt = at<int32_t>(d_arena, L.cand_cnt);
  sc.cand_cap_assign = (int32_t)L.cap_assign;
  sc.cand_cap_probe = (int32_t)L.cap_probe;
  sc.gs_items = L.gs_items;
  sc.gs_a = at<uint16_t>(d_arena, L.gs_a);
  sc.gs_qn = at<float>(d_arena, L.gs_qn);
  sc.gs_qs = at<float>(d_arena, L.gs_qs);
  sc.gs_qh = at<uint16_t>(d_arena, L.gs_qh);
  sc.gs_ql = at<uint16_t>(d_arena, L.gs_ql);
  sc.gs_qqn = at<float>(d_arena, L.gs_qqn);
  sc.gs_qqs = at<float>(d_arena, L.gs_qqs);
  sc.item_doff = at<int64_t>(d_arena, L.item_doff);
  sc.item_dlen = at<int32_t>(d_arena, L.item_dlen);
  sc.item_nlive = at<int32_t>(d_arena, L.item_nlive);
  sc.item_of = at<int32_t>(d_arena, L.item_of);
  sc.pair_pos = at<int32_t>(d_arena, L.pair_pos);
  sc.dense = at<float>(d_arena, L.dense);
  sc.dense_cap = L.dense_cap;
}

}  // namespace
}  // namespace sivf

using namespace sivf;

namespace sivf {
// measurement probes (sivf_probe_*): an empty kernel, and a dependent-load chain
__global__ void k_probe_empty() {}
__global__ void k_probe_chase(const int32_t* __restrict__ next, int64_t n, int32_t hops, int32_t* __restrict__ out) {
  int32_t i = 0;
  for (int32_t h = 0; h < hops; ++h) i = __ldcg(next + (i < n && i >= 0 ? i : 0));
  *out = i;
}
}  // namespace sivf

extern "C" {

const char* sivf_rc_string(sivf_rc rc) {
  switch (rc) {
    case SIVF_OK: return "ok";
    case SIVF_E_INVALID_ARG: return "invalid argument";
    case SIVF_E_CUDA: return "CUDA error";
    case SIVF_E_ARENA_TOO_SMALL: return "arena too small or misaligned";
    case SIVF_E_NOT_TRAINED: return "index has no centroids";
    case SIVF_E_UNSUPPORTED: return "unsupported configuration";
  }
  return "unknown";
}

sivf_rc sivf_arena_bytes(const sivf_config* cfg, size_t* bytes) {
  if (!valid_config(cfg) || !bytes) return SIVF_E_INVALID_ARG;
  *bytes = make_layout(cfg).total;
  return SIVF_OK;
}

sivf_rc sivf_create(const sivf_config* cfg, void* d_arena, size_t arena_bytes, sivf_stream_t stream,
                    sivf_index* out) {
  if (!valid_config(cfg) || !out) return SIVF_E_INVALID_ARG;
  const Layout L = make_layout(cfg);
  if (!d_arena || arena_bytes < L.total || (reinterpret_cast<uintptr_t>(d_arena) % kAlign) != 0)
    return SIVF_E_ARENA_TOO_SMALL;
  Index* ix = new (std::nothrow) Index();
  if (!ix) return SIVF_E_INVALID_ARG;
  ix->cfg = *cfg;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&ix->num_sms, cudaDevAttrMultiProcessorCount, dev);
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (optin > 0) ix->smem_optin = (size_t)optin;
  DevState& st = ix->st;
  st.D = cfg->dim;
  st.Dp = (int32_t)L.Dp;
  st.Dh = (int32_t)L.Dh;
  st.nlist = cfg->nlist;
  st.G = cfg->shard_count;
  st.rank = cfg->shard_rank;
  st.cap = cfg->id_capacity;
  st.cap_local = L.cap_local;
  st.num_slabs = cfg->num_slabs;
  st.payload = at<float>(d_arena, L.payload);
  st.payload16 = L.Dh ? at<uint16_t>(d_arena, L.payload16) : nullptr;
  st.Dg = (int32_t)L.Dg;
  st.payload_g = L.Dg ? at<uint16_t>(d_arena, L.payload_g) : nullptr;
  st.slab_xs = L.Dg ? at<float>(d_arena, L.slab_xs) : nullptr;
  st.slab_ids = at<uint32_t>(d_arena, L.slab_ids);
  st.slab_norm = at<float>(d_arena, L.slab_norm);
  st.slab_flag = at<uint32_t>(d_arena, L.slab_flag);
  st.bitmap = at<uint32_t>(d_arena, L.bitmap);
  st.cursor = at<uint32_t>(d_arena, L.cursor);
  st.slab_list = at<int32_t>(d_arena, L.slab_list);
  st.free_stack = at<int32_t>(d_arena, L.free_stack);
  st.att = at<uint64_t>(d_arena, L.att);
  st.claim = at<int32_t>(d_arena, L.claim);
  st.dir_off = at<int64_t>(d_arena, L.dir_off);
  st.dir_len = at<int32_t>(d_arena, L.dir_len);
  st.dir_cap = at<int32_t>(d_arena, L.dir_cap);
  st.dir_arena = at<int32_t>(d_arena, L.dir_arena);
  st.dir_half = L.dir_half;
  st.centroids = at<float>(d_arena, L.centroids);
  st.ctr = at<unsigned long long>(d_arena, L.ctr);
  st.ictr = at<int32_t>(d_arena, L.ictr);
  st.sctr = at<int32_t>(d_arena, L.sctr);
  st.conc = 0;
  carve_scratch(ix->sc, d_arena, L);

  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaMemsetAsync(st.att, 0xff, (size_t)L.cap_local * 8, s);          // ATT <- INVALID
  cudaMemsetAsync(st.claim, 0x7f, (size_t)L.cap_local * 4, s);        // kClaimEmpty
  cudaMemsetAsync(st.centroids, 0, (size_t)cfg->nlist * L.Dp * 4, s);
  int64_t m = st.num_slabs > st.nlist ? st.num_slabs : st.nlist;
  if (m < 64) m = 64;
  k_init<<<ceil_div(m, 256), 256, 0, s>>>(st);
  ix->launches += 1;
  cudaStreamCreateWithFlags(&ix->side, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&ix->cap_stream, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&ix->ev_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ix->ev_join, cudaEventDisableTiming);
  cudaError_t e = setup_search_kernels(*ix);
  if (e == cudaSuccess) e = setup_coarse_tc(*ix);
  if (e == cudaSuccess) e = setup_coarse_exact(*ix);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    delete ix;
    return SIVF_E_CUDA;
  }
  *out = reinterpret_cast<sivf_index>(ix);
  return SIVF_OK;
}

sivf_rc sivf_view_arena_bytes(const sivf_config* cfg, size_t* bytes) {
  if (!valid_config(cfg) || !bytes) return SIVF_E_INVALID_ARG;
  *bytes = make_layout(cfg, true).total;
  return SIVF_OK;
}

sivf_rc sivf_create_view(sivf_index owner_h, void* d_arena, size_t arena_bytes, sivf_stream_t stream,
                         sivf_index* out) {
  if (!owner_h || !out) return SIVF_E_INVALID_ARG;
  Index* own = reinterpret_cast<Index*>(owner_h);
  if (own->view) return SIVF_E_INVALID_ARG;  // views of views are not needed
  const Layout L = make_layout(&own->cfg, true);
  if (!d_arena || arena_bytes < L.total || (reinterpret_cast<uintptr_t>(d_arena) % kAlign) != 0)
    return SIVF_E_ARENA_TOO_SMALL;
  Index* ix = new (std::nothrow) Index();
  if (!ix) return SIVF_E_INVALID_ARG;
  ix->cfg = own->cfg;
  ix->view = true;
  ix->owner = own;
  ix->num_sms = own->num_sms;
  ix->smem_optin = own->smem_optin;
  ix->trained = own->trained;
  ix->st = own->st;  // shared index state
  ix->st.sctr = at<int32_t>(d_arena, L.sctr);
  ix->st.conc = 1;
  carve_scratch(ix->sc, d_arena, L);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaMemsetAsync(ix->st.sctr, 0, I_NICTR * 4, s);
  cudaStreamCreateWithFlags(&ix->side, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&ix->cap_stream, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&ix->ev_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ix->ev_join, cudaEventDisableTiming);
  cudaError_t e = setup_search_kernels(*ix);
  if (e == cudaSuccess) e = setup_coarse_tc(*ix);
  if (e == cudaSuccess) e = setup_coarse_exact(*ix);
  if (e == cudaSuccess && ix->trained) e = refresh_centroid_tiles(*ix, s);  // the view's own centroid tiles
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    delete ix;
    return SIVF_E_CUDA;
  }
  *out = reinterpret_cast<sivf_index>(ix);
  return SIVF_OK;
}

sivf_rc sivf_insert_concurrent(sivf_index h, const int64_t* d_ids, const float* d_x, int64_t n, int32_t* d_status,
                               int32_t* d_list, sivf_stream_t stream) {
  if (!h) return SIVF_E_INVALID_ARG;
  Index* ix = reinterpret_cast<Index*>(h);
  if (n < 0 || n > ix->cfg.max_batch) return SIVF_E_INVALID_ARG;
  if (n > 0 && (!d_ids || !d_x)) return SIVF_E_INVALID_ARG;
  if (!ix->trained) return SIVF_E_NOT_TRAINED;
  Index* own = ix->view ? ix->owner : ix;
  if (!own->dirs_prepared) return SIVF_E_UNSUPPORTED;
  own->conc_used = true;
  return cuda_rc(launch_insert_concurrent(*ix, d_ids, d_x, n, d_status, d_list, reinterpret_cast<cudaStream_t>(stream)));
}

sivf_rc sivf_reserve_directories(sivf_index h, int32_t spare, sivf_stream_t stream) {
  if (!h || spare < 0 || spare > 256) return SIVF_E_INVALID_ARG;
  Index* ix = reinterpret_cast<Index*>(h);
  if (ix->view) return SIVF_E_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int32_t* d_fail = reinterpret_cast<int32_t*>(ix->sc.tmp64 + 15);
  cudaMemsetAsync(d_fail, 0, 4, s);
  cudaError_t e = launch_reserve_dirs(*ix, spare, d_fail, s);
  int32_t fail = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&fail, d_fail, 4, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return SIVF_E_CUDA;
  if (fail) return SIVF_E_UNSUPPORTED;
  ix->dirs_prepared = true;
  return SIVF_OK;
}

sivf_rc sivf_destroy(sivf_index h) {
  if (!h) return SIVF_E_INVALID_ARG;
  delete reinterpret_cast<Index*>(h);
  return SIVF_OK;
}

sivf_rc sivf_set_centroids(sivf_index h, const float* d_c, sivf_stream_t stream) {
  if (!h || !d_c) return SIVF_E_INVALID_ARG;
  Index* ix = reinterpret_cast<Index*>(h);
  if (ix->view) return SIVF_E_INVALID_ARG;  // quiescent, owner only
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int D = ix->st.D, Dp = ix->st.Dp;
  cudaError_t e = cudaMemcpy2DAsync(ix->st.centroids, (size_t)Dp * 4, d_c, (size_t)D * 4, (size_t)D * 4,
                                    ix->st.nlist, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess) e = refresh_centroid_tiles(*ix, s);
  if (e != cudaSuccess) return SIVF_E_CUDA;
  ix->trained = true;
  return SIVF_OK;
}

sivf_rc sivf_get_centroids(sivf_index h, float* d_c, sivf_stream_t stream) {
  if (!h || !d_c) return SIVF_E_INVALID_ARG;
  Index* ix = reinterpret_cast<Index*>(h);
  if (!ix->trained) return SIVF_E_NOT_TRAINED;
  const int D = ix->st.D, Dp = ix->st.Dp;
  return cuda_rc(cudaMemcpy2DAsync(d_c, (size_t)D * 4, ix->st.centroids, (size_t)Dp * 4, (size_t)D * 4,
                                   ix->st.nlist, cudaMemcpyDeviceToDevice, reinterpret_cast<cudaStream_t>(stream)));
}

sivf_rc sivf_train_centroids(sivf_index h, const float* d_x, int64_t n, int32_t niter, sivf_stream_t stream) {
  if (!h || !d_x) return SIVF_E_INVALID_ARG;
  Index* ix = reinterpret_cast<Index*>(h);
  if (ix->view) return SIVF_E_INVALID_ARG;  // quiescent, owner only
  if (n < ix->st.nlist || n > ix->cfg.max_train || niter < 0) return SIVF_E_INVALID_ARG;
  cudaError_t e = launch_train(*ix, d_x, n, niter, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return SIVF_E_CUDA;
  ix->trained = true;
  return SIVF_OK;
}

sivf_rc sivf_insert(sivf_index h, const int64_t* d_ids, const float* d_x, int64_t n, int32_t* d_status,
                    int32_t* d_list, sivf_stream_t stream) {
  if (!h) return SIVF_E_INVALID_ARG;
  Index* ix = reinterpret_cast<Index*>(h);
  if (ix->view) return SIVF_E_INVALID_ARG;  // quiescent, owner only (views: sivf_insert_concurrent)
  if (n < 0 || n > ix->cfg.max_batch) return SIVF_E_INVALID_ARG;
  if (n > 0 && (!d_ids || !d_x)) return SIVF_E_INVALID_ARG;
  if (!ix->trained) return SIVF_E_NOT_TRAINED;
  ix->dirs_prepared = false;  // directories may grow without spare entries
  return cuda_rc(launch_insert(*ix, d_ids, d_x, n, d_status, d_list, reinterpret_cast<cudaStream_t>(stream)));
}

sivf_rc sivf_delete(sivf_index h, const int64_t* d_ids, int64_t n, int64_t* d_ndeleted, sivf_stream_t stream) {
  if (!h || n < 0 || (n > 0 && !d_ids)) return SIVF_E_INVALID_ARG;
  Index* ix = reinterpret_cast<Index*>(h);
  return cuda_rc(launch_delete(*ix, d_ids, n, d_ndeleted, reinterpret_cast<cudaStream_t>(stream)));
}

}  // extern "C" (a template helper follows)

// Graph cache of repeated API calls (SIVF_OPT_STEP_GRAPH): `body(stream)` enqueues
// the call's launches; a call signature (key) is captured as a CUDA graph on its
// second sighting and replayed afterwards.  Direct launches while profiling or when
// the caller's stream is itself being captured.
template <class Body>
static sivf_rc graph_cached(Index* ix, Index::StepGraph key, cudaStream_t s, Body&& body) {
  cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cst) != cudaSuccess) {
    cudaGetLastError();
    cst = cudaStreamCaptureStatusActive;  // unknown: stay with direct launches
  }
  // a caller that is itself capturing s gets the launches recorded into its graph
  if (ix->step_graph && !ix->prof && ix->cap_stream && cst == cudaStreamCaptureStatusNone) {
    // repeat calls with the same signature replay one CUDA graph of the whole step
    // (every launch parameter is a function of the signature and the options; the
    // data are read on the device at replay time)
    key.s = s, key.epoch = ix->opt_epoch;
    auto same_sig = [&](const Index::StepGraph& g) {
      if (g.used == 0 || g.kind != key.kind || g.s != key.s || g.epoch != key.epoch || g.k != key.k ||
          g.nprobe != key.nprobe)
        return false;
      for (int i = 0; i < 8; ++i)
        if (g.p[i] != key.p[i]) return false;
      return g.n[0] == key.n[0] && g.n[1] == key.n[1] && g.n[2] == key.n[2];
    };
    auto same = [&](const Index::StepGraph& g) { return g.exec && same_sig(g); };
    Index::StepGraph* hit = nullptr;
    Index::StepGraph* victim = &ix->step_graphs[0];
    for (auto& g : ix->step_graphs) {
      if (same(g)) hit = &g;
      if (g.used < victim->used) victim = &g;
    }
    if (!hit) {
      // a signature is captured on its second call: callers that pass fresh buffers
      // every step never pay for a capture
      Index::StepGraph* seen = nullptr;
      Index::StepGraph* oldest = &ix->step_seen[0];
      for (auto& g : ix->step_seen) {
        if (same_sig(g)) seen = &g;
        if (g.used < oldest->used) oldest = &g;
      }
      if (!seen) {
        *oldest = key;
        oldest->used = ++ix->step_tick;
        return body(s);
      }
      if (seen->bad) {  // not capturable (remembered per signature)
        seen->used = ++ix->step_tick;
        return body(s);
      }
      seen->used = 0;  // promoted to a captured graph below
      // capture on cap_stream (the caller's stream may be the legacy default stream)
      cudaGraph_t graph = nullptr;
      const int64_t l0 = ix->launches;
      cudaError_t e = cudaStreamBeginCapture(ix->cap_stream, cudaStreamCaptureModeThreadLocal);
      if (e == cudaSuccess) {
        const sivf_rc rc = body(ix->cap_stream);
        e = cudaStreamEndCapture(ix->cap_stream, &graph);
        if (rc != SIVF_OK && e == cudaSuccess) e = cudaErrorUnknown;
      }
      cudaGraphExec_t exec = nullptr;
      if (e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
      if (graph) cudaGraphDestroy(graph);
      if (e != cudaSuccess) {
        cudaGetLastError();
        ix->launches = l0;
        // this signature is not capturable: direct launches for it from now on
        // (other signatures keep their graphs)
        seen->bad = true;
        seen->used = ++ix->step_tick;
        return body(s);
      }
      if (victim->exec) cudaGraphExecDestroy(victim->exec);
      *victim = key;
      victim->exec = exec;
      victim->launches = ix->launches - l0;
      ix->launches = l0;
      hit = victim;
    }
    hit->used = ++ix->step_tick;
    ix->launches += hit->launches;
    return cuda_rc(cudaGraphLaunch(hit->exec, s));
  }
  return body(s);
}

extern "C" {

sivf_rc sivf_search(sivf_index h, const float* d_q, int64_t nq, int32_t k, int32_t nprobe, float* d_dist,
                    int64_t* d_ids, int32_t* d_probes, sivf_stream_t stream) {
  if (!h) return SIVF_E_INVALID_ARG;
  Index* ix = reinterpret_cast<Index*>(h);
  if (nq < 0 || nq > ix->cfg.max_queries) return SIVF_E_INVALID_ARG;
  if (k < 1 || k > ix->cfg.max_k) return SIVF_E_INVALID_ARG;
  if (nprobe < 1 || nprobe > ix->cfg.max_nprobe || nprobe > ix->st.nlist) return SIVF_E_INVALID_ARG;
  if (nq > 0 && (!d_q || !d_dist || !d_ids)) return SIVF_E_INVALID_ARG;
  if (!ix->trained) return SIVF_E_NOT_TRAINED;
  if (nq > 0 && !plan_search(*ix, nq, k, nprobe).ok) return SIVF_E_UNSUPPORTED;  // before any capture
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  Index::StepGraph key;
  const void* p[8] = {d_q, d_dist, d_ids, d_probes, nullptr, nullptr, nullptr, nullptr};
  for (int i = 0; i < 8; ++i) key.p[i] = p[i];
  key.n[2] = nq, key.k = k, key.nprobe = nprobe, key.kind = 1;
  return graph_cached(ix, key, s, [&](cudaStream_t cs) {
    return cuda_rc(launch_search(*ix, d_q, nq, k, nprobe, d_dist, d_ids, d_probes, cs));
  });
}

// Coarse step alone (a7): the exact probe set of each query row (NEXT-3: ranks
// compute the probe sets of their slice of the queries, then all-gather them).
sivf_rc sivf_probe(sivf_index h, const float* d_q, int64_t nq, int32_t nprobe, int32_t* d_probes,
                   sivf_stream_t stream) {
  if (!h) return SIVF_E_INVALID_ARG;
  Index* ix = reinterpret_cast<Index*>(h);
  if (nq < 0 || nq > ix->cfg.max_queries) return SIVF_E_INVALID_ARG;
  if (nprobe < 1 || nprobe > ix->cfg.max_nprobe || nprobe > ix->st.nlist) return SIVF_E_INVALID_ARG;
  if (nq > 0 && (!d_q || !d_probes)) return SIVF_E_INVALID_ARG;
  if (!ix->trained) return SIVF_E_NOT_TRAINED;
  if (nq == 0) return SIVF_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  Index::StepGraph key;
  const void* p[8] = {d_q, d_probes, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  for (int i = 0; i < 8; ++i) key.p[i] = p[i];
  key.n[2] = nq, key.nprobe = nprobe, key.kind = 2;
  return graph_cached(ix, key, s, [&](cudaStream_t cs) {
    cudaError_t e = launch_probe_exact(*ix, d_q, nq, nprobe, cs);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(d_probes, ix->sc.probes, sizeof(int32_t) * nq * nprobe, cudaMemcpyDeviceToDevice, cs);
    return cuda_rc(e);
  });
}

// Scan + merge with caller-supplied probe sets (d_probes_in[nq][nprobe], e.g. the
// all-gathered output of sivf_probe): the same results as sivf_search when they
// are the probe sets sivf_search would compute.
sivf_rc sivf_search_probed(sivf_index h, const float* d_q, int64_t nq, int32_t k, int32_t nprobe,
                           const int32_t* d_probes_in, float* d_dist, int64_t* d_ids, sivf_stream_t stream) {
  if (!h) return SIVF_E_INVALID_ARG;
  Index* ix = reinterpret_cast<Index*>(h);
  if (nq < 0 || nq > ix->cfg.max_queries) return SIVF_E_INVALID_ARG;
  if (k < 1 || k > ix->cfg.max_k) return SIVF_E_INVALID_ARG;
  if (nprobe < 1 || nprobe > ix->cfg.max_nprobe || nprobe > ix->st.nlist) return SIVF_E_INVALID_ARG;
  if (nq > 0 && (!d_q || !d_probes_in || !d_dist || !d_ids)) return SIVF_E_INVALID_ARG;
  if (nq > 0 && !plan_search(*ix, nq, k, nprobe).ok) return SIVF_E_UNSUPPORTED;
  if (nq == 0) return SIVF_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  Index::StepGraph key;
  const void* p[8] = {d_q, d_dist, d_ids, d_probes_in, nullptr, nullptr, nullptr, nullptr};
  for (int i = 0; i < 8; ++i) key.p[i] = p[i];
  key.n[2] = nq, key.k = k, key.nprobe = nprobe, key.kind = 3;
  return graph_cached(ix, key, s, [&](cudaStream_t cs) {
    return cuda_rc(launch_search(*ix, d_q, nq, k, nprobe, d_dist, d_ids, nullptr, cs, d_probes_in));
  });
}

sivf_rc sivf_reclaim(sivf_index h, int64_t* d_nreclaimed, sivf_stream_t stream) {
  if (!h) return SIVF_E_INVALID_ARG;
  if (reinterpret_cast<Index*>(h)->view) return SIVF_E_INVALID_ARG;  // quiescent, owner only
  reinterpret_cast<Index*>(h)->dirs_prepared = false;
  return cuda_rc(launch_reclaim(*reinterpret_cast<Index*>(h), d_nreclaimed, reinterpret_cast<cudaStream_t>(stream)));
}

// One sliding-window step enqueued on s (direct launches; also the body captured by
// the step graph cache).
static sivf_rc sliding_step_body(Index* ix, const int64_t* d_new_ids, const float* d_new_x, int64_t n_new,
                          const int64_t* d_old_ids, int64_t n_old, const float* d_q, int64_t nq, int32_t k,
                          int32_t nprobe, float* d_dist, int64_t* d_ids, int32_t* d_status, int64_t* d_ndeleted,
                          cudaStream_t s) {
  // The search's coarse quantisation and inverse probe map read only centroids and
  // queries, so they run on a side stream concurrently with insert + delete; the
  // scan joins after the mutations (C22: the search sees the post-step window).
  const SearchPlan sp = plan_search(*ix, nq, k, nprobe);
  if (nq > 0 && !sp.ok) return SIVF_E_UNSUPPORTED;
  const bool fork = nq > 0 && coarse_front_concurrent_ok(*ix, nprobe) && ix->side;
  cudaError_t e = cudaSuccess;
  if (fork) {
    cudaEventRecord(ix->ev_fork, s);
    cudaStreamWaitEvent(ix->side, ix->ev_fork, 0);
    ix->coarse_alt = true;
    e = launch_search_front(*ix, sp, d_q, nq, nprobe, nullptr, ix->side);
    ix->coarse_alt = false;
    cudaEventRecord(ix->ev_join, ix->side);
  }
  if (e == cudaSuccess) e = launch_insert(*ix, d_new_ids, d_new_x, n_new, d_status, nullptr, s);
  if (e == cudaSuccess) e = launch_delete(*ix, d_old_ids, n_old, d_ndeleted, s);
  if (fork) cudaStreamWaitEvent(s, ix->ev_join, 0);  // always join, even after an error
  if (e == cudaSuccess && nq > 0 && !fork) e = launch_search_front(*ix, sp, d_q, nq, nprobe, nullptr, s);
  if (e == cudaSuccess && nq > 0 && ix->side && !ix->prof) {
    // the merge reads only the per-(query, probe) partial lists: the reclaim (which
    // rewrites directories) runs beside it on the side stream once the scan is done
    e = launch_search_back(*ix, sp, d_q, nq, k, nprobe, d_dist, d_ids, s, ix->ev_fork);
    if (e == cudaSuccess) {
      cudaStreamWaitEvent(ix->side, ix->ev_fork, 0);
      e = launch_reclaim(*ix, nullptr, ix->side);
      cudaEventRecord(ix->ev_join, ix->side);
      cudaStreamWaitEvent(s, ix->ev_join, 0);
    }
    return cuda_rc(e);
  }
  if (e == cudaSuccess && nq > 0) e = launch_search_back(*ix, sp, d_q, nq, k, nprobe, d_dist, d_ids, s);
  if (e == cudaSuccess) e = launch_reclaim(*ix, nullptr, s);
  return cuda_rc(e);
}


sivf_rc sivf_sliding_window_step(sivf_index h, const int64_t* d_new_ids, const float* d_new_x, int64_t n_new,
                                 const int64_t* d_old_ids, int64_t n_old, const float* d_q, int64_t nq, int32_t k,
                                 int32_t nprobe, float* d_dist, int64_t* d_ids, int32_t* d_status,
                                 int64_t* d_ndeleted, sivf_stream_t stream) {
  if (!h) return SIVF_E_INVALID_ARG;
  if (reinterpret_cast<Index*>(h)->view) return SIVF_E_INVALID_ARG;  // quiescent, owner only
  reinterpret_cast<Index*>(h)->dirs_prepared = false;
  Index* ix = reinterpret_cast<Index*>(h);
  if (n_new < 0 || n_new > ix->cfg.max_batch || n_old < 0 || nq < 0 || nq > ix->cfg.max_queries)
    return SIVF_E_INVALID_ARG;
  if ((n_new > 0 && (!d_new_ids || !d_new_x)) || (n_old > 0 && !d_old_ids)) return SIVF_E_INVALID_ARG;
  if (nq > 0) {
    if (k < 1 || k > ix->cfg.max_k || nprobe < 1 || nprobe > ix->cfg.max_nprobe || nprobe > ix->st.nlist)
      return SIVF_E_INVALID_ARG;
    if (!d_q || !d_dist || !d_ids) return SIVF_E_INVALID_ARG;
  }
  if (!ix->trained) return SIVF_E_NOT_TRAINED;
  if (nq > 0 && !plan_search(*ix, nq, k, nprobe).ok) return SIVF_E_UNSUPPORTED;  // before any capture
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  Index::StepGraph key;
  const void* p[8] = {d_new_ids, d_new_x, d_old_ids, d_q, d_dist, d_ids, d_status, d_ndeleted};
  for (int i = 0; i < 8; ++i) key.p[i] = p[i];
  key.n[0] = n_new, key.n[1] = n_old, key.n[2] = nq;
  key.k = nq > 0 ? k : 0, key.nprobe = nq > 0 ? nprobe : 0, key.kind = 0;
  return graph_cached(ix, key, s, [&](cudaStream_t cs) {
    return sliding_step_body(ix, d_new_ids, d_new_x, n_new, d_old_ids, n_old, d_q, nq, k, nprobe, d_dist, d_ids,
                             d_status, d_ndeleted, cs);
  });
}


sivf_rc sivf_merge_topk(const float* d_dist_g, const int64_t* d_ids_g, int32_t G, int64_t nq, int32_t k,
                        float* d_dist, int64_t* d_ids, sivf_stream_t stream) {
  if (G < 1 || nq < 0 || k < 1 || k > 1024) return SIVF_E_INVALID_ARG;
  if (nq > 0 && (!d_dist_g || !d_ids_g || !d_dist || !d_ids)) return SIVF_E_INVALID_ARG;
  if ((int64_t)G * nq * k > 0x7FFFFFFFll) return SIVF_E_INVALID_ARG;
  return cuda_rc(launch_merge_topk(d_dist_g, d_ids_g, G, nq, k, d_dist, d_ids, reinterpret_cast<cudaStream_t>(stream),
                                   nullptr));
}

sivf_rc sivf_dump_state(sivf_index h, int32_t* d_list_of_id, int64_t* d_live_per_list, int64_t* d_violations,
                        sivf_stream_t stream) {
  if (!h) return SIVF_E_INVALID_ARG;
  if (reinterpret_cast<Index*>(h)->view) return SIVF_E_INVALID_ARG;  // quiescent, owner only
  return cuda_rc(launch_dump(*reinterpret_cast<Index*>(h), d_list_of_id, d_live_per_list, d_violations,
                             reinterpret_cast<cudaStream_t>(stream)));
}

// debug (not in sivf.h): the last sivf_dump_state's violations by type: [ATT entry ->
// slot, slab_list, bits above the cursor, partial non-tail slab, slot -> ATT, live sum,
// slab marks]; synchronises the device
extern "C" int sivf_debug_violations(sivf_index h, int64_t* host7) {
  if (!h || !host7) return SIVF_E_INVALID_ARG;
  return cudaMemcpy(host7, reinterpret_cast<Index*>(h)->sc.tmp64 + 2, 7 * 8, cudaMemcpyDeviceToHost) == cudaSuccess
             ? SIVF_OK : SIVF_E_CUDA;
}

sivf_rc sivf_dump_att(sivf_index h, uint64_t* d_att, sivf_stream_t stream) {
  if (!h || !d_att) return SIVF_E_INVALID_ARG;
  Index* ix = reinterpret_cast<Index*>(h);
  return cuda_rc(cudaMemcpyAsync(d_att, ix->st.att, (size_t)ix->st.cap_local * 8, cudaMemcpyDeviceToDevice,
                                 reinterpret_cast<cudaStream_t>(stream)));
}

sivf_rc sivf_stats(sivf_index h, sivf_stats_t* out, sivf_stream_t stream) {
  if (!h || !out) return SIVF_E_INVALID_ARG;
  Index* ix = reinterpret_cast<Index*>(h);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  unsigned long long c[C_NCTR];
  int32_t ic[I_NICTR];
  cudaError_t e = cudaMemcpyAsync(c, ix->st.ctr, sizeof(c), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(ic, ix->st.ictr, sizeof(ic), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return SIVF_E_CUDA;
  std::memset(out, 0, sizeof(*out));
  out->live = (int64_t)c[C_LIVE];
  out->inserted = (int64_t)c[C_INSERTED];
  out->deleted = (int64_t)c[C_DELETED];
  out->pool_exhausted_items = (int64_t)c[C_EXHAUSTED];
  out->reclaimed_slabs = (int64_t)c[C_RECLAIMED];
  out->device_errors = (int64_t)c[C_DEVERR];
  out->leaked_slabs = (int64_t)c[C_LEAKED];
  out->leaked_recycled = (int64_t)c[C_LEAKRECL];
  out->dir_compactions = (int64_t)c[C_DIRCOMPACT];
  out->slabs_free = ic[I_FREE_TOP];
  out->slabs_in_use = ix->st.num_slabs - ic[I_FREE_TOP];
  const double d = ix->st.D;
  out->overhead_paper = 128.0 / (32.0 * (4.0 * d + 8.0));
  const double live_bytes = (double)out->live * (4.0 * d + 4.0);
  out->overhead_actual =
      live_bytes > 0 ? (16.0 * out->slabs_in_use + 8.0 * (double)ix->st.cap_local) / live_bytes : 0.0;
  const double copy_bytes = ix->st.Dh ? (double)rec16_bytes(ix->st.Dh)
                          : ix->st.Dg ? (double)recg_bytes(ix->st.Dg) + 4.0 * kSlot  // + the slots' scales
                                      : 0.0;
  out->overhead_scan_copy = live_bytes > 0 ? copy_bytes * (double)out->slabs_in_use / live_bytes : 0.0;
  return SIVF_OK;
}

int64_t sivf_local_capacity(sivf_index h) { return h ? reinterpret_cast<Index*>(h)->st.cap_local : -1; }

int64_t sivf_launch_count(sivf_index h) { return h ? reinterpret_cast<Index*>(h)->launches : -1; }

sivf_rc sivf_probe_launch(int32_t n, sivf_stream_t stream) {
  if (n < 1) return SIVF_E_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i) sivf::k_probe_empty<<<1, 32, 0, (cudaStream_t)stream>>>();
  return cudaGetLastError() == cudaSuccess ? SIVF_OK : SIVF_E_CUDA;
}

sivf_rc sivf_probe_chase(const int32_t* d_next, int64_t n, int32_t hops, int32_t* d_out, sivf_stream_t stream) {
  if (!d_next || !d_out || n < 1 || hops < 0) return SIVF_E_INVALID_ARG;
  sivf::k_probe_chase<<<1, 1, 0, (cudaStream_t)stream>>>(d_next, n, hops, d_out);
  return cudaGetLastError() == cudaSuccess ? SIVF_OK : SIVF_E_CUDA;
}

sivf_rc sivf_set_option(sivf_index h, int32_t option, int64_t value) {
  if (!h) return SIVF_E_INVALID_ARG;
  Index* ix = reinterpret_cast<Index*>(h);
  ++ix->opt_epoch;  // cached step graphs captured under other options never match again
  switch (option) {
    case SIVF_OPT_STEP_GRAPH: ix->step_graph = value != 0; return SIVF_OK;
    case SIVF_OPT_TC_SCAN: ix->use_tc_scan = value != 0; return SIVF_OK;
    case SIVF_OPT_TC_TWO_PHASE: ix->tc_two_phase = value < 0 ? 0 : (int)value; return SIVF_OK;
    case SIVF_OPT_TC_COARSE: ix->use_tc_coarse = value != 0; return SIVF_OK;
    case SIVF_OPT_COARSE_SELECT: ix->coarse_select = value != 0 && ix->coarse_select_ok; return SIVF_OK;
    case SIVF_OPT_RANK_SPLIT: ix->rank_split = value < 0 ? 0 : (int)value; return SIVF_OK;
    case 99: ix->dbg = (int)value; return SIVF_OK;  // SIVF_OPT_DEBUG: experiments only
    case 98: ix->tc_max_stages = (int)value; return SIVF_OK;  // experiments only: scan stage-ring cap
    case SIVF_OPT_CONCURRENT: ix->st.conc = value != 0; return SIVF_OK;
    case SIVF_OPT_SEED_LIST: ix->seed_list = value != 0; return SIVF_OK;
    case SIVF_OPT_SEED_SLABS:
      if (value < 0 || value > (1 << 20)) return SIVF_E_INVALID_ARG;
      ix->seed_slabs = (int)value;
      return SIVF_OK;
  }
  return SIVF_E_INVALID_ARG;
}

sivf_rc sivf_profile_enable(sivf_index h, int32_t on) {
  if (!h) return SIVF_E_INVALID_ARG;
  reinterpret_cast<Index*>(h)->prof = on != 0;
  return SIVF_OK;
}

sivf_rc sivf_profile_read(sivf_index h, double* ms, int64_t* count) {
  if (!h || !ms || !count) return SIVF_E_INVALID_ARG;
  Index* ix = reinterpret_cast<Index*>(h);
  for (auto& r : ix->recs) {
    if (cudaEventSynchronize(r.b) != cudaSuccess) return SIVF_E_CUDA;
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) return SIVF_E_CUDA;
    if (r.phase >= 0 && r.phase < SIVF_NPHASE) {
      ms[r.phase] += t;
      count[r.phase] += 1;
    }
    ix->ev_pool.push_back(r.a);
    ix->ev_pool.push_back(r.b);
  }
  ix->recs.clear();
  return SIVF_OK;
}

}  // extern "C"
