// k_search.cu — batched search: coarse probe -> inverse map -> slab scan -> merge.
//
// Paper: Alg. 3 scans, per query, the slab chains of its nprobe
// lists with one warp (lane j = slot j), gated by the validity bitmap
// (Eq. slot_valid), computing Eq. l2, keeping a
// per-lane top-k and merging.
//
// B200 design: the work is inverted to list-major.  A work
// item is (list l, tile of <= QT queries that probe l).  A persistent CTA
// stages each live slab of l (skipping bitmap == 0 slabs, Eq. slot_valid at
// slab granularity) into shared memory with cp.async.bulk + mbarrier (one
// producer warp, NS-deep ring) and every compute warp reuses it for its 4
// queries: HBM bytes per list are read once per tile instead of once per
// query.  In the slab layout [4 row groups][Dp/4][8][4] (pay_off()) a 128-dim
// chunk of a slab is 4 contiguous pieces, one bulk copy each, staged as
// [4][kCH/4][8][4] so that lane = slot float4 reads are conflict-free.
// Lane (lq, ls) of a compute warp owns query lq and slots ls, ls+8, ls+16,
// ls+24; distances use the difference form t = q - x, acc = fma(t, t, acc)
// in ascending dimension order (|err| <= (D+2) u relative; exact on
// integer-valued data).  Invalid slots (bit clear) become padding keys.
// Per-(query, probe) partial top-k keys go to scratch; k_merge reduces the
// nprobe partials of each query to the final (distance, id) top-k.
#include "sivf_host.h"

namespace sivf {

namespace {

constexpr int kNS = 4;     // stage ring depth
constexpr int kCH = 128;   // dims per stage (16 KB of payload per stage)

struct StageMeta {
  int32_t slab;    // -1 = end of work item
  uint32_t bitmap;
  int32_t chunk;
  int32_t last;    // 1 if this is the slab's last dim-chunk
};

struct ScanArgs {
  DevState st;
  const float* Q;
  int nprobe, k;
  const int32_t* inv_pairs;
  const int32_t* work_l;
  const int32_t* work_p0;
  const int32_t* work_n;
  unsigned long long* partial;
};

__host__ __device__ inline size_t scan_smem_bytes(int NW, int Dp, int k) {
  const int QT = kQPW * NW;
  size_t b = 0;
  b += (size_t)kNS * (kCH * kSlot * 4 + kSlot * 4);  // stage payload + ids
  b += (size_t)QT * (Dp + 4) * 4;                   // query tile
  b += (size_t)QT * k * 8;                          // top-k per query
  b += (size_t)NW * k * 8;                          // merge tmp per warp
  b += (size_t)NW * kQPW * kSlot * 8;               // candidate transposition
  b += (size_t)kNS * sizeof(StageMeta) + 2 * kNS * 8 + 64;
  return b;
}

template <int NW>
__global__ void __launch_bounds__(32 * (NW + 1), 1) k_scan(ScanArgs a) {
  constexpr int QT = kQPW * NW;
  extern __shared__ __align__(128) unsigned char smem[];
  const DevState& st = a.st;
  const int Dp = st.Dp, Dq = Dp + 4, k = a.k;
  float* stage_x = reinterpret_cast<float*>(smem);                        // [NS][CH*32]
  uint32_t* stage_id = reinterpret_cast<uint32_t*>(stage_x + kNS * kCH * kSlot);  // [NS][32]
  float* qs = reinterpret_cast<float*>(stage_id + kNS * kSlot);           // [QT][Dq]
  unsigned long long* top = reinterpret_cast<unsigned long long*>(qs + (size_t)QT * Dq);  // [QT][k]
  unsigned long long* tmp = top + (size_t)QT * k;                          // [NW][k]
  unsigned long long* cand = tmp + (size_t)NW * k;                         // [NW][4][32]
  StageMeta* meta = reinterpret_cast<StageMeta*>(cand + NW * kQPW * kSlot);
  uint64_t* full = reinterpret_cast<uint64_t*>(meta + kNS);
  uint64_t* empty = full + kNS;
  int* ctrl = reinterpret_cast<int*>(empty + kNS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = (Dp + kCH - 1) / kCH;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kNS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int ntiles = st.sctr[I_NTILES];
  uint32_t it = 0;  // stage sequence number (same sequence in producer and consumers)

  for (;;) {
    if (threadIdx.x == 0) ctrl[0] = atomicAdd(&st.sctr[I_WORK], 1);
    __syncthreads();
    const int w_item = ctrl[0];
    if (w_item >= ntiles) break;
    const int l = a.work_l[w_item];
    const int p0 = a.work_p0[w_item];
    const int nqt = a.work_n[w_item];
    // stage the query tile (zero padded) and reset the top-k lists
    for (int e = threadIdx.x; e < QT * (Dp >> 2); e += blockDim.x) {
      const int r = e / (Dp >> 2), c4 = e % (Dp >> 2);
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < nqt) {
        const int q = a.inv_pairs[p0 + r] / a.nprobe;
        const float* qr = a.Q + (int64_t)q * st.D;
        float t[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) t[j] = (4 * c4 + j < st.D) ? qr[4 * c4 + j] : 0.f;
        v = make_float4(t[0], t[1], t[2], t[3]);
      }
      *reinterpret_cast<float4*>(&qs[r * Dq + 4 * c4]) = v;
    }
    for (int e = threadIdx.x; e < QT * k; e += blockDim.x) top[e] = kPadKey;
    __syncthreads();

    if (warp == NW) {
      // ---------------- producer: one elected lane issues bulk copies
      if (lane == 0) {
        const int len = ld_state_s32(&st.dir_len[l], st.conc);
        const int32_t* dir = st.dir_arena + st.dir_off[l];
        for (int j = 0; j < len; ++j) {
          const int s = ld_state_s32(&dir[j], st.conc);
          const uint32_t bm = ld_state_u32(&st.bitmap[s], st.conc);
          if (bm == 0u) continue;  // nothing valid in this slab
          if (st.conc) fence_proxy_async_global();  // the bitmap acquire orders the copies (NEXT-2)
          const float* src = st.payload + (size_t)s * kSlot * Dp;
          for (int c = 0; c < nch; ++c, ++it) {
            const int stg = it % kNS;
            mbar_wait(&empty[stg], ((it / kNS) & 1u) ^ 1u);
            const int cw = min(kCH, Dp - c * kCH);
            const bool last = c == nch - 1;
            meta[stg] = StageMeta{s, bm, c, last ? 1 : 0};
            mbar_arrive_expect_tx(&full[stg], cw * kSlot * 4 + (last ? kSlot * 4 : 0));
            // dims [c kCH, c kCH + cw) of the slab: one piece per 8-slot row group
            // (pay_off layout), staged as [4][kCH/4][8][4]
            for (int r = 0; r < kSlot / 8; ++r)
              bulk_g2s(stage_x + stg * kCH * kSlot + r * (kCH / 4) * 32, src + pay_off(Dp, 8 * r, c * (kCH / 4)),
                       cw * 32, &full[stg]);
            if (last) bulk_g2s(stage_id + stg * kSlot, st.slab_ids + (size_t)s * kSlot, kSlot * 4, &full[stg]);
          }
        }
        const int stg = it % kNS;
        mbar_wait(&empty[stg], ((it / kNS) & 1u) ^ 1u);
        meta[stg].slab = -1;
        mbar_arrive(&full[stg]);
        ++it;
      }
    } else {
      // ---------------- compute warps: lane = slot, kQPW = 4 queries per lane (the query
      // loads are warp-wide broadcasts, each slab float4 feeds 4 queries: shared-memory
      // traffic per distance term ~4x lower than one query x 4 slots per lane)
      const int sj = lane >> 3, ls = lane & 7;  // the slot's row group and position in it
      const bool warp_active = warp * kQPW < nqt;
      const float* qp = qs + (warp * kQPW) * Dq;
      // packed fp32x2 arithmetic (FFMA2/FADD2): two partial sums per query (even and odd
      // dimensions), t = q - x and t*t + acc per pair of dimensions in one instruction each
      float2 acc[kQPW];
#pragma unroll
      for (int j = 0; j < kQPW; ++j) acc[j] = make_float2(0.f, 0.f);
      unsigned long long* mycand = cand + warp * kQPW * kSlot;
      for (;; ++it) {
        const int stg = it % kNS;
        mbar_wait(&full[stg], (it / kNS) & 1u);
        const StageMeta m = meta[stg];
        if (m.slab < 0) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[stg]);
          ++it;
          break;
        }
        if (warp_active) {
          const float* xs = stage_x + stg * kCH * kSlot + (sj * (kCH / 4) * 8 + ls) * 4;
          const int cw = min(kCH, Dp - m.chunk * kCH);
          const float* qc = qp + m.chunk * kCH;
#pragma unroll 4
          for (int i4 = 0; i4 < (cw >> 2); ++i4) {
            const float4 xv = *reinterpret_cast<const float4*>(xs + i4 * 32);
            const float2 nx01 = make_float2(-xv.x, -xv.y), nx23 = make_float2(-xv.z, -xv.w);
#pragma unroll
            for (int j = 0; j < kQPW; ++j) {
              const float4 qv = *reinterpret_cast<const float4*>(qc + j * Dq + 4 * i4);
              const float2 t01 = __fadd2_rn(make_float2(qv.x, qv.y), nx01);
              const float2 t23 = __fadd2_rn(make_float2(qv.z, qv.w), nx23);
              acc[j] = __ffma2_rn(t01, t01, acc[j]);
              acc[j] = __ffma2_rn(t23, t23, acc[j]);
            }
          }
          if (m.last) {
            const uint32_t* ids = stage_id + stg * kSlot;
            const bool valid = ((m.bitmap >> lane) & 1u) != 0u;  // Eq. slot_valid
#pragma unroll
            for (int j = 0; j < kQPW; ++j) {
              const bool qvalid = warp * kQPW + j < nqt;
              mycand[j * kSlot + lane] = (valid && qvalid) ? make_key(acc[j].x + acc[j].y, ids[lane]) : kPadKey;
              acc[j] = make_float2(0.f, 0.f);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stg]);  // stage buffer free
        if (warp_active && m.last) {
#pragma unroll 1
          for (int qq = 0; qq < kQPW; ++qq) {
            if (warp * kQPW + qq >= nqt) break;
            warp_topk_insert(top + (size_t)(warp * kQPW + qq) * k, tmp + (size_t)warp * k, k,
                             mycand[qq * kSlot + lane]);
          }
        }
      }
    }
    __syncthreads();
    // write the partial top-k of every (query, probe) pair of the tile
    for (int e = threadIdx.x; e < nqt * k; e += blockDim.x) {
      const int r = e / k, j = e % k;
      const int pair = a.inv_pairs[p0 + r];
      a.partial[(size_t)pair * k + j] = top[r * k + j];
    }
  }
}

// ---- inverse probe map (list -> pairs), bucketed by probe rank ----
// Entry idx = b * nlist + l.  With nb = 2, bucket 0 holds every query's nearest
// probed list (rank 0) and bucket 1 the rest; work items are laid out bucket-
// major, so each query's nearest list is scanned first and the per-query bound
// on its k-th distance is already in place for its other lists.
__global__ void k_inv_count(const int32_t* __restrict__ probes, int64_t npairs, int nprobe, int nb, int r0,
                            int nlist, int32_t* __restrict__ cnt, uint32_t* __restrict__ gthr, int keep) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npairs) return;
  const int p = (int)(i % nprobe);
  if (p == 0 && !keep) gthr[i / nprobe] = 0x7F800000u;  // per-query bound = +inf
  const int b = (nb == 2 && p >= r0) ? 1 : 0;
  atomicAdd(&cnt[b * nlist + probes[i]], 1);
}

__global__ void __launch_bounds__(1024) k_inv_scan(const int32_t* __restrict__ cnt, int nent, int QT,
                                                   int32_t* __restrict__ off, int32_t* __restrict__ cursor,
                                                   int32_t* __restrict__ tile_off, int32_t* __restrict__ ictr,
                                                   int nlist, int32_t* __restrict__ work_l,
                                                   int32_t* __restrict__ work_p0, int32_t* __restrict__ work_n,
                                                   int32_t* __restrict__ item_of) {
  __shared__ int32_t ws[2][32];
  __shared__ int32_t carry[2];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t == 0) carry[0] = carry[1] = 0;
  __syncthreads();
  // prefix order: bucket 0 by list, then bucket 1 by list in REVERSE, so the lists the
  // first bucket scanned last (still in L2) are the first the second bucket reads
  auto ent = [&](int r) { return r < nlist ? r : nlist + (nent - 1 - r); };
  for (int l0 = 0; l0 < nent; l0 += 1024) {
    const int l = l0 + t < nent ? ent(l0 + t) : nent;  // entry at prefix rank l0 + t
    const int c = l < nent ? cnt[l] : 0;
    const int tl = (c + QT - 1) / QT;
    int v0 = c, v1 = tl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int a0 = __shfl_up_sync(kFull, v0, o), a1 = __shfl_up_sync(kFull, v1, o);
      if (lane >= o) {
        v0 += a0;
        v1 += a1;
      }
    }
    if (lane == 31) {
      ws[0][w] = v0;
      ws[1][w] = v1;
    }
    __syncthreads();
    if (w == 0) {
      int x0 = ws[0][lane], x1 = ws[1][lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int a0 = __shfl_up_sync(kFull, x0, o), a1 = __shfl_up_sync(kFull, x1, o);
        if (lane >= o) {
          x0 += a0;
          x1 += a1;
        }
      }
      ws[0][lane] = x0;
      ws[1][lane] = x1;
    }
    __syncthreads();
    if (l < nent) {
      const int e0 = carry[0] + (w ? ws[0][w - 1] : 0) + v0 - c;
      const int e1 = carry[1] + (w ? ws[1][w - 1] : 0) + v1 - tl;
      off[l] = e0;
      cursor[l] = e0;
      tile_off[l] = e1;
    }
    __syncthreads();
    if (t == 0) {
      carry[0] += ws[0][31];
      carry[1] += ws[1][31];
    }
    __syncthreads();
  }
  if (t == 0) {
    off[nent] = carry[0];
    tile_off[nent] = carry[1];
    ictr[I_NTILES] = carry[1];
    ictr[I_WORK] = 0;
    // bucket 0 (each query's r0 nearest lists) = tiles [0, t0), t0 = the offset of the
    // first entry of bucket 1 in prefix order (its last list): the phased
    // tensor-core scan runs bucket 0 to completion before bucket 1
    const int t0 = nent > nlist ? tile_off[nent - 1] : carry[1];
    ictr[I_NTILES0] = t0;
    ictr[I_WORK2] = t0;
  }
  __syncthreads();  // the block's offsets are visible to all of its threads
  // work items (list, first pair, number of pairs), bucket-major (k_work_fill fused)
  for (int e = t; e < nent; e += blockDim.x) {
    const int c = cnt[e];  // (entries are not contiguous in prefix order: no off[e + 1] - off[e])
    for (int tt = tile_off[e], j = 0; j * QT < c; ++tt, ++j) {
      work_l[tt] = e % nlist;
      work_p0[tt] = off[e] + j * QT;
      work_n[tt] = min(QT, c - j * QT);
    }
  }
}

// Inverse-map position -> work item (k_gs_select), warp per work item, grid-stride
// over the device-side item count (was a sequential loop per list entry inside the
// single-CTA k_inv_scan: 0.17 ms per 10k x 32 pairs).
__global__ void __launch_bounds__(256) k_item_of(const int32_t* __restrict__ ictr, const int32_t* __restrict__ work_p0,
                                                 const int32_t* __restrict__ work_n, int32_t* __restrict__ item_of) {
  const int lane = threadIdx.x & 31;
  const int ntiles = ictr[I_NTILES];
  for (int w = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); w < ntiles;
       w += (int)(((int64_t)gridDim.x * blockDim.x) >> 5)) {
    const int p0 = work_p0[w], n = work_n[w];
    for (int u = lane; u < n; u += 32) item_of[p0 + u] = w;
  }
}

__global__ void k_inv_scatter(const int32_t* __restrict__ probes, int64_t npairs, int nprobe, int nb, int r0,
                              int nlist, int32_t* __restrict__ cursor, int32_t* __restrict__ pairs,
                              int32_t* __restrict__ pair_pos) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npairs) return;
  const int p = (int)(i % nprobe);
  const int b = (nb == 2 && p >= r0) ? 1 : 0;
  const int pos = atomicAdd(&cursor[b * nlist + probes[i]], 1);
  pairs[pos] = (int32_t)i;
  if (pair_pos) pair_pos[i] = pos;
}

// Block-aggregated scatter (nb * nlist <= kScatterEnt): a block of 1024 threads x 4
// pairs ranks its pairs per entry with shared-memory atomics, reserves each entry's
// range with ONE global atomicAdd per (block, entry) and writes the pairs: ~50x fewer
// contended global atomics than one per pair (every list receives ~nq nprobe / nlist).
constexpr int kScatterEnt = 12288, kScatterPPT = 4;  // 48 KB of static shared memory
__global__ void __launch_bounds__(1024) k_inv_scatter_blk(const int32_t* __restrict__ probes, int64_t npairs,
                                                         int nprobe, int nb, int r0, int nlist,
                                                         int32_t* __restrict__ cursor, int32_t* __restrict__ pairs,
                                                         int32_t* __restrict__ pair_pos) {
  __shared__ int32_t hist[kScatterEnt];
  const int nent = nb * nlist;
  for (int e = threadIdx.x; e < nent; e += blockDim.x) hist[e] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * blockDim.x * kScatterPPT;
  int ent[kScatterPPT], loc[kScatterPPT];
#pragma unroll
  for (int u = 0; u < kScatterPPT; ++u) {
    const int64_t i = base + (int64_t)u * blockDim.x + threadIdx.x;
    ent[u] = -1;
    if (i < npairs) {
      const int p = (int)(i % nprobe);
      ent[u] = ((nb == 2 && p >= r0) ? nlist : 0) + probes[i];
      loc[u] = atomicAdd(&hist[ent[u]], 1);
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nent; e += blockDim.x) {
    const int c = hist[e];
    if (c) hist[e] = atomicAdd(&cursor[e], c);  // the entry's range for this block
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kScatterPPT; ++u) {
    const int64_t i = base + (int64_t)u * blockDim.x + threadIdx.x;
    if (ent[u] >= 0) {
      pairs[hist[ent[u]] + loc[u]] = (int32_t)i;
      if (pair_pos) pair_pos[i] = hist[ent[u]] + loc[u];
    }
  }
}

// Warp per query, nprobe <= 32, k <= KM: lane p holds probe p's sorted partial list in
// registers; k rounds of a warp-wide minimum over the list heads, the winning lane
// shifts its list (static register moves, no local memory).  Same result as k_merge.
template <int KM>
__global__ void __launch_bounds__(128) k_merge_regs(const unsigned long long* __restrict__ partial, int64_t nq,
                                                    int nprobe, int k, float* __restrict__ dist,
                                                    int64_t* __restrict__ ids) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t q = (int64_t)blockIdx.x * 4 + w;
  if (q >= nq) return;  // warp-uniform
  unsigned long long h[KM];
  const unsigned long long* src = partial + ((size_t)q * nprobe + lane) * k;
#pragma unroll
  for (int j = 0; j < KM; ++j) h[j] = (lane < nprobe && j < k) ? src[j] : kPadKey;
  unsigned long long out = kPadKey;
  for (int r = 0; r < k; ++r) {
    unsigned long long m = h[0];
#pragma unroll
    for (int off = 16; off; off >>= 1) m = umin64(m, __shfl_xor_sync(kFull, m, off));
    if (lane == r) out = m;
    if (h[0] == m) {  // keys are unique (ids), so exactly one lane advances
#pragma unroll
      for (int j = 0; j < KM - 1; ++j) h[j] = h[j + 1];
      h[KM - 1] = kPadKey;
    }
  }
  if (lane < k) {
    const bool pad = out == kPadKey;
    dist[q * k + lane] = pad ? __int_as_float(0x7f800000) : key_dist(out);
    ids[q * k + lane] = pad ? -1 : (int64_t)key_id(out);
  }
}

// Warp per query: k smallest of its nprobe partial lists (P:355 merge; C4, C5).
__global__ void k_merge(const unsigned long long* __restrict__ partial, int64_t nq, int nprobe, int k,
                        float* __restrict__ dist, int64_t* __restrict__ ids) {
  extern __shared__ __align__(16) unsigned long long sm_merge[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + w;
  if (q >= nq) return;
  unsigned long long* top = sm_merge + (size_t)w * 2 * k;
  unsigned long long* tmp = top + k;
  warp_topk_init(top, k);
  const unsigned long long* src = partial + (size_t)q * nprobe * k;
  const int total = nprobe * k;
  for (int i0 = 0; i0 < total; i0 += 32) {
    const int i = i0 + lane;
    warp_topk_insert(top, tmp, k, i < total ? src[i] : kPadKey);
  }
  for (int j = lane; j < k; j += 32) {
    const uint64_t key = top[j];
    const bool pad = key == kPadKey;
    dist[q * k + j] = pad ? __int_as_float(0x7f800000) : key_dist(key);
    ids[q * k + j] = pad ? -1 : (int64_t)key_id(key);
  }
}

__global__ void k_merge_shards(const float* __restrict__ dg, const int64_t* __restrict__ ig, int G, int64_t nq, int k,
                               float* __restrict__ dist, int64_t* __restrict__ ids) {
  extern __shared__ __align__(16) unsigned long long sm_mg[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + w;
  if (q >= nq) return;
  unsigned long long* top = sm_mg + (size_t)w * 2 * k;
  unsigned long long* tmp = top + k;
  warp_topk_init(top, k);
  const int total = G * k;
  for (int i0 = 0; i0 < total; i0 += 32) {
    const int i = i0 + lane;
    uint64_t key = kPadKey;
    if (i < total) {
      const int g = i / k, j = i % k;
      const size_t o = ((size_t)g * nq + q) * k + j;
      const int64_t id = ig[o];
      if (id >= 0) key = make_key(dg[o], (uint32_t)id);
    }
    warp_topk_insert(top, tmp, k, key);
  }
  for (int j = lane; j < k; j += 32) {
    const uint64_t key = top[j];
    const bool pad = key == kPadKey;
    dist[q * k + j] = pad ? __int_as_float(0x7f800000) : key_dist(key);
    ids[q * k + j] = pad ? -1 : (int64_t)key_id(key);
  }
}

int pick_nw(const Index& ix, int k) {
  for (int nw : {8, 4, 2})
    if (scan_smem_bytes(nw, ix.st.Dp, k) <= ix.smem_optin) return nw;
  return 0;
}

}  // namespace

size_t scan_smem_for(const Index& ix, int k, int* nw_out) {
  int nw = pick_nw(ix, k);
  if (nw_out) *nw_out = nw;
  return nw ? scan_smem_bytes(nw, ix.st.Dp, k) : 0;
}

bool scan_tc_supported(const Index& ix, int k);
cudaError_t setup_scan_tc(Index& ix);
cudaError_t launch_scan_tc(Index& ix, const float* d_q, int k, int nprobe, cudaStream_t s, int phase);
int scan_tc_tile();
bool scan_gs_supported(const Index& ix);
cudaError_t setup_scan_gs(Index& ix);
cudaError_t launch_scan_gs(Index& ix, const float* d_q, int64_t nq, int k, int nprobe, cudaStream_t s);
cudaError_t launch_select_gs(Index& ix, const float* d_q, int64_t nq, int k, int nprobe, float* d_dist,
                             int64_t* d_ids, cudaStream_t s);

cudaError_t setup_search_kernels(Index& ix) {
  cudaError_t e = setup_scan_tc(ix);
  if (e == cudaSuccess) e = setup_scan_gs(ix);
  if (e != cudaSuccess) return e;
  for (int nw : {8, 4, 2}) {
    size_t need = scan_smem_bytes(nw, ix.st.Dp, ix.cfg.max_k);
    size_t want = need < ix.smem_optin ? need : ix.smem_optin;
    if (nw == 8) e = cudaFuncSetAttribute(k_scan<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want);
    if (nw == 4) e = cudaFuncSetAttribute(k_scan<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want);
    if (nw == 2) e = cudaFuncSetAttribute(k_scan<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

SearchPlan plan_search(const Index& ix, int64_t nq, int32_t k, int32_t nprobe) {
  SearchPlan p{};
  const int nlist = ix.st.nlist;
  p.tc = ix.use_tc_scan && scan_tc_supported(ix, k);
  p.gs = !p.tc && ix.use_tc_scan && scan_gs_supported(ix);
  p.smem = p.tc || p.gs ? 0 : scan_smem_for(ix, k, &p.nw);
  p.ok = p.tc || p.gs || p.nw != 0;
  p.QT = p.tc ? scan_tc_tile() : p.gs ? 128 : kQPW * p.nw;
  // Tensor-core path: probe-rank buckets, one scan launch.  Work items are laid
  // out bucket-major, so with nb = 2 every query's r0 nearest lists are scanned
  // first and its k-th distance bound is tight before the other lists are
  // reached (far fewer survivors of the tensor-core filter).  Split only when
  // the lists are long enough in queries that it adds no tiles on average.
  p.nb = 1;
  p.r0 = nprobe;
  if (p.tc && nprobe >= 8) {
    const int64_t per_list = nq * nprobe / nlist;
    const int rr = ix.tc_two_phase ? (ix.tc_two_phase < nprobe ? ix.tc_two_phase : nprobe - 1)
                 : ix.rank_split > 1 ? (ix.rank_split < nprobe ? ix.rank_split : nprobe - 1) : nprobe / 4;
    const int64_t ta = ceil_div(per_list * rr / nprobe, p.QT),
                  tb = ceil_div(per_list - per_list * rr / nprobe, p.QT);
    if (ix.tc_two_phase || ix.rank_split > 1 || (ix.rank_split && ta + tb <= ceil_div(per_list, p.QT))) {
      p.nb = 2;
      p.r0 = rr;
    }
  }
  return p;
}

// Coarse quantisation + inverse probe map: reads only the centroids and the
// queries (never the index state), so it may run concurrently with mutations.
cudaError_t launch_search_front(Index& ix, const SearchPlan& p, const float* d_q, int64_t nq, int32_t nprobe,
                                int32_t* d_probes, cudaStream_t s, const int32_t* probes_in) {
  Scratch& sc = ix.sc;
  const int nlist = ix.st.nlist;
  const int64_t npairs = nq * nprobe;
  // the coarse selection may count the inverse map on the fly (k_inv_count fused)
  cudaMemsetAsync(sc.inv_cnt, 0, sizeof(int32_t) * p.nb * nlist, s);
  bool counted = false;
  if (probes_in) {
    // probe sets computed elsewhere (the query-sharded coarse step, NEXT-3): only the
    // inverse map is built here
    cudaMemcpyAsync(sc.probes, probes_in, sizeof(int32_t) * npairs, cudaMemcpyDeviceToDevice, s);
  } else {
    ix.fuse_inv_cnt = sc.inv_cnt;
    ix.fuse_nb = p.nb;
    ix.fuse_r0 = p.r0;
    ix.fuse_inv_done = false;
    cudaError_t e = launch_probe_exact(ix, d_q, nq, nprobe, s);
    counted = ix.fuse_inv_done;
    ix.fuse_inv_cnt = nullptr;
    ix.fuse_inv_done = false;
    if (e != cudaSuccess) return e;
  }
  if (d_probes) cudaMemcpyAsync(d_probes, sc.probes, sizeof(int32_t) * npairs, cudaMemcpyDeviceToDevice, s);
  const int nent = p.nb * nlist;
  PhaseTimer pt(ix, SIVF_PH_INVMAP, s);
  if (!counted) {
    k_inv_count<<<ceil_div(npairs, 256), 256, 0, s>>>(sc.probes, npairs, nprobe, p.nb, p.r0, nlist, sc.inv_cnt,
                                                       sc.gthr, (ix.dbg >> 6) & 1);
    ix.launches += 1;
  }
  k_inv_scan<<<1, 1024, 0, s>>>(sc.inv_cnt, nent, p.QT, sc.inv_off, sc.inv_cursor, sc.tile_off, ix.st.sctr, nlist,
                                sc.work_l, sc.work_p0, sc.work_n, nullptr);
  if (p.gs) {
    k_item_of<<<4 * ix.num_sms, 256, 0, s>>>(ix.st.sctr, sc.work_p0, sc.work_n, sc.item_of);
    ix.launches += 1;
  }
  int32_t* pair_pos = p.gs ? sc.pair_pos : nullptr;
  if (nent <= kScatterEnt && !(ix.dbg & 4096)) {  // dbg 4096 (experiments): the per-pair scatter
    k_inv_scatter_blk<<<ceil_div(npairs, 1024 * kScatterPPT), 1024, 0, s>>>(sc.probes, npairs, nprobe, p.nb, p.r0,
                                                                            nlist, sc.inv_cursor, sc.inv_pairs, pair_pos);
  } else
  k_inv_scatter<<<ceil_div(npairs, 256), 256, 0, s>>>(sc.probes, npairs, nprobe, p.nb, p.r0, nlist, sc.inv_cursor,
                                                       sc.inv_pairs, pair_pos);
  ix.launches += 2;
  return cudaGetLastError();
}

// Slab scan + per-query merge (reads the index state).
cudaError_t launch_search_back(Index& ix, const SearchPlan& p, const float* d_q, int64_t nq, int32_t k,
                               int32_t nprobe, float* d_dist, int64_t* d_ids, cudaStream_t s, cudaEvent_t after_scan) {
  Scratch& sc = ix.sc;
  cudaError_t e = cudaSuccess;
  ScanArgs a{ix.st, d_q, nprobe, k, sc.inv_pairs, sc.work_l, sc.work_p0, sc.work_n, sc.partial};
  const int grid = ix.num_sms;  // persistent: one CTA per SM
  {
    PhaseTimer pt(ix, SIVF_PH_SCAN, s);
    if (p.gs) {
      e = launch_scan_gs(ix, d_q, nq, k, nprobe, s);
    } else if (p.tc) {
      e = launch_seed_bound(ix, d_q, nq, k, nprobe, s);  // after the front reset gthr to +inf
      if (e == cudaSuccess && p.nb == 2 && ix.tc_two_phase) {
        // two launches: every query's r0 nearest lists complete (and its k-th
        // distance bound is published) before any of its other lists starts
        e = launch_scan_tc(ix, d_q, k, nprobe, s, 1);
        if (e == cudaSuccess) e = launch_scan_tc(ix, d_q, k, nprobe, s, 2);
      } else if (e == cudaSuccess) {
        e = launch_scan_tc(ix, d_q, k, nprobe, s, 0);
      }
    } else if (p.nw == 8) {
      k_scan<8><<<grid, 32 * 9, p.smem, s>>>(a);
    } else if (p.nw == 4) {
      k_scan<4><<<grid, 32 * 5, p.smem, s>>>(a);
    } else {
      k_scan<2><<<grid, 32 * 3, p.smem, s>>>(a);
    }
    if (!p.tc && !p.gs) ix.launches += 1;
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return e;  // a failed scan launch must not be masked by the merge below
  }
  if (after_scan) cudaEventRecord(after_scan, s);  // the index is no longer read by this search
  PhaseTimer pt(ix, SIVF_PH_MERGE, s);
  if (p.gs) return launch_select_gs(ix, d_q, nq, k, nprobe, d_dist, d_ids, s);
  const int wpb = 4;
  if (nprobe <= 32 && k <= 16) {
    if (k <= 10) k_merge_regs<10><<<ceil_div(nq, 4), 128, 0, s>>>(sc.partial, nq, nprobe, k, d_dist, d_ids);
    else k_merge_regs<16><<<ceil_div(nq, 4), 128, 0, s>>>(sc.partial, nq, nprobe, k, d_dist, d_ids);
  } else {
    k_merge<<<ceil_div(nq, wpb), 32 * wpb, sizeof(unsigned long long) * 2 * k * wpb, s>>>(sc.partial, nq, nprobe, k,
                                                                                          d_dist, d_ids);
  }
  ix.launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_search(Index& ix, const float* d_q, int64_t nq, int32_t k, int32_t nprobe, float* d_dist,
                          int64_t* d_ids, int32_t* d_probes, cudaStream_t s, const int32_t* probes_in) {
  if (nq <= 0) return cudaSuccess;
  const SearchPlan p = plan_search(ix, nq, k, nprobe);
  if (!p.ok) return cudaErrorInvalidConfiguration;
  cudaError_t e = launch_search_front(ix, p, d_q, nq, nprobe, d_probes, s, probes_in);
  if (e != cudaSuccess) return e;
  return launch_search_back(ix, p, d_q, nq, k, nprobe, d_dist, d_ids, s);
}

cudaError_t launch_merge_topk(const float* d_dist_g, const int64_t* d_ids_g, int32_t G, int64_t nq, int32_t k,
                              float* d_dist, int64_t* d_ids, cudaStream_t s, int64_t* launches) {
  if (nq <= 0) return cudaSuccess;
  const int wpb = 4;
  const size_t smem = sizeof(unsigned long long) * 2 * k * wpb;  // 64 k B: beyond 48 KB for k > 768
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_merge_shards, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_merge_shards<<<ceil_div(nq, wpb), 32 * wpb, sizeof(unsigned long long) * 2 * k * wpb, s>>>(d_dist_g, d_ids_g, G,
                                                                                              nq, k, d_dist, d_ids);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

}  // namespace sivf
