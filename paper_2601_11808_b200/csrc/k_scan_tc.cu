// k_scan_tc.cu — slab scan on the 5th-generation tensor cores (tcgen05).
//
// Same work decomposition as k_search.cu's SIMT scan (a work item = list l x
// a tile of <= 128 queries probing l), but the distance evaluation of
// Eq. l2 for a (query tile, slab) pair is a dense contraction:
//   d(q, x) = ||q||^2 + ||x||^2 - 2 q.x
// q.x for 128 queries x 32 slots is one chain of tcgen05.mma kind::tf32
// (M=128, N=32, K=8 per instruction): A = the query tile, resident in TMEM for
// the whole work item; B = the slab, bulk-copied into shared memory, consumed
// straight from the paper's fp32 payload because the dim-interleaved slab
// layout [D/4][32][4] IS the K-major SWIZZLE_NONE UMMA layout (LBO 512 B,
// SBO 128 B).  Accumulators live in TMEM (one 32-column buffer per stage).
//
// Exactness (BASELINE.json tolerances): when the query and the slab are
// integer-valued with |v| <= 2048 (tf32-exact; flag set by k_append) and
// ||q||^2 + ||x||^2 < 2^24, every product and partial sum is an exact
// integer, so the tensor-core distance IS the exact distance (this is the
// SIFT-shaped case).  Otherwise the tensor-core value only filters: a slot
// is re-ranked with the exact fp32 difference form (same order as the SIMT
// scan) iff  d_tc - E <= current k-th distance, with E a certified bound on
// |d_tc - d_exact| (tf32 truncation + fp32 accumulation), so no candidate of
// the exact top-k is ever dropped.
//
// Roles (1 CTA per SM, persistent): warp 0 = bulk-copy producer, warp 1 =
// MMA issuer (one lane) + TMEM owner, warps 2..9 = epilogue (TMEM lane
// quarter = warp % 4 -> 32 query rows; column half -> 16 of the 32 slots).
// Each epilogue thread keeps a sorted register top-k for its (query, half);
// the halves are merged at the end of the work item.  A per-query global
// bound (atomicMin of the k-th distance of any finished half list) prunes
// later work items: a candidate above the k-th distance of ANY k real
// candidates cannot be in the final top-k.
#include "sivf_host.h"

namespace sivf {

namespace {

constexpr int TM = 128;         // queries per tile (TMEM lanes, UMMA M)
constexpr int TNS = 4;          // stage ring depth
constexpr int TEPI = 8;         // epilogue warps
constexpr int TTHREADS = 32 * (2 + TEPI);

struct TcArgs {
  DevState st;
  const float* Q;
  int nprobe, k;
  const int32_t* inv_off;
  const int32_t* inv_pairs;
  const int32_t* tile_off;
  const int32_t* work_list;
  unsigned long long* partial;
  uint32_t* gthr;
  uint32_t tmem_cols;
};

struct TcMeta {
  int32_t slab;
  uint32_t bitmap;
  uint32_t flag;
  int32_t pad;
};

__host__ __device__ inline size_t tc_smem_bytes(int Dp, int KP) {
  size_t b = 0;
  b += (size_t)TNS * kSlot * Dp * 4;        // stage payload
  b += (size_t)TNS * kSlot * 4 * 2;         // stage ids + norms
  size_t qs = (size_t)TM * (Dp + 4) * 4;    // query rows (re-rank) / end-of-item half lists
  size_t mrg = (size_t)TM * 2 * KP * 8;
  b += qs > mrg ? qs : mrg;
  b += (size_t)TM * 4 * 3;                  // norm halves, pair index
  b += (size_t)TNS * sizeof(TcMeta) + 3 * TNS * 8 + 64;
  return b;
}

template <int KP>
__device__ __forceinline__ void topk_reg_insert(u64 (&keys)[KP], u64 c) {
#pragma unroll
  for (int i = KP - 1; i > 0; --i) {
    const u64 prev = keys[i - 1];
    keys[i] = prev > c ? prev : (keys[i] > c ? c : keys[i]);
  }
  keys[0] = keys[0] > c ? c : keys[0];
}


template <int KP>
__global__ void __launch_bounds__(TTHREADS, 1) k_scan_tc(TcArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const DevState& st = a.st;
  const int Dp = st.Dp, Dq = Dp + 4, k = a.k;
  float* stage_x = reinterpret_cast<float*>(smem);                               // [TNS][32*Dp]
  uint32_t* stage_id = reinterpret_cast<uint32_t*>(stage_x + (size_t)TNS * kSlot * Dp);  // [TNS][32]
  float* stage_nrm = reinterpret_cast<float*>(stage_id + TNS * kSlot);           // [TNS][32]
  float* qs = stage_nrm + TNS * kSlot;                                           // [TM][Dq] | merge lists
  u64* mrg = reinterpret_cast<u64*>(qs);
  const size_t qs_bytes = (size_t)TM * Dq * 4, mrg_bytes = (size_t)TM * 2 * KP * 8;
  float* qn_half = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(qs) +
                                            (qs_bytes > mrg_bytes ? qs_bytes : mrg_bytes));  // [2][TM]
  int* qpair = reinterpret_cast<int*>(qn_half + 2 * TM);                          // [TM]
  TcMeta* meta = reinterpret_cast<TcMeta*>(qpair + TM);
  uint64_t* full = reinterpret_cast<uint64_t*>(meta + TNS);
  uint64_t* mmad = full + TNS;
  uint64_t* empty = mmad + TNS;
  int* ctrl = reinterpret_cast<int*>(empty + TNS);
  uint32_t* tmem_base_sm = reinterpret_cast<uint32_t*>(ctrl + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < TNS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&mmad[i], 1);
      mbar_init(&empty[i], TEPI);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_base_sm, a.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_base_sm;
  const uint32_t dcol0 = (uint32_t)Dp;  // A occupies TMEM columns [0, Dp)
  const int ntiles = st.ictr[I_NTILES];
  const uint32_t idesc = umma_idesc_tf32(TM, kSlot);
  uint32_t it = 0;     // stage sequence (producer, MMA and epilogue agree)
  uint32_t mmph = 0;   // epilogue: per-stage parity of the MMA-done barrier

  for (;;) {
    if (threadIdx.x == 0) ctrl[0] = atomicAdd(&st.ictr[I_WORK], 1);
    __syncthreads();
    const int w_item = ctrl[0];
    if (w_item >= ntiles) break;
    const int l = a.work_list[w_item];
    const int p0 = a.inv_off[l] + (w_item - a.tile_off[l]) * TM;
    const int nqt = min(TM, a.inv_off[l + 1] - p0);

    const bool epi = warp >= 2;
    const int g = warp & 3, h = (warp - 2) >> 2;
    const int row = 32 * g + lane;

    if (warp == 0) {
      // ---------------- producer: the warp loads directory entries, bitmaps and
      // flags 32 at a time (independent loads in flight); lane 0 issues the copies
      const int len = st.dir_len[l];
      const int32_t* dir = st.dir_arena + st.dir_off[l];
      const uint32_t bytes = (uint32_t)kSlot * Dp * 4;
      for (int j0 = 0; j0 < len; j0 += 32) {
        const int j = j0 + lane;
        int s = 0;
        uint32_t bm = 0u, fl = 0u;
        if (j < len) {
          s = dir[j];
          bm = st.bitmap[s];
          fl = st.slab_flag[s];
        }
        unsigned live = __ballot_sync(kFull, bm != 0u);  // Eq. slot_valid at slab granularity
        while (live) {
          const int src = __ffs(live) - 1;
          live &= live - 1;
          const int ss = __shfl_sync(kFull, s, src);
          const uint32_t sbm = __shfl_sync(kFull, bm, src), sfl = __shfl_sync(kFull, fl, src);
          if (lane == 0) {
            const int stg = it % TNS;
            mbar_wait(&empty[stg], ((it / TNS) & 1u) ^ 1u);
            meta[stg] = TcMeta{ss, sbm, sfl, 0};
            mbar_arrive_expect_tx(&full[stg], bytes + 2 * kSlot * 4);
            bulk_g2s(stage_x + (size_t)stg * kSlot * Dp, st.payload + (size_t)ss * kSlot * Dp, bytes, &full[stg]);
            bulk_g2s(stage_id + stg * kSlot, st.slab_ids + (size_t)ss * kSlot, kSlot * 4, &full[stg]);
            bulk_g2s(stage_nrm + stg * kSlot, st.slab_norm + (size_t)ss * kSlot, kSlot * 4, &full[stg]);
          }
          ++it;
        }
      }
      if (lane == 0) {
        const int stg = it % TNS;
        mbar_wait(&empty[stg], ((it / TNS) & 1u) ^ 1u);
        meta[stg].slab = -1;
        mbar_arrive(&full[stg]);
      }
      ++it;
    } else if (warp == 1) {
      // ---------------- MMA issuer: D[stg] = Q_tile . slab^T (after the epilogue put A in TMEM)
      asm volatile("bar.sync 2, %0;" ::"r"(32 * (1 + TEPI)));
      tc_fence_after();
      if (lane == 0) {
        for (;;) {
          const int stg = it % TNS;
          mbar_wait(&full[stg], (it / TNS) & 1u);
          const int slab = meta[stg].slab;
          ++it;
          if (slab < 0) break;
          tc_fence_after();
          const uint32_t bsm = smem_u32(stage_x + (size_t)stg * kSlot * Dp);
          const uint32_t dt = tbase + dcol0 + (uint32_t)stg * kSlot;
          for (int kk = 0; kk < (Dp >> 3); ++kk)
            umma_tf32_ts(dt, tbase + (uint32_t)(8 * kk), umma_sdesc(bsm + (uint32_t)kk * 1024u, 512u, 128u), idesc,
                         kk > 0 ? 1u : 0u);
          umma_commit(&mmad[stg]);  // implies tcgen05.fence::before_thread_sync
        }
      }
    } else {
      // ---------------- epilogue: stage the query tile (coalesced global -> smem rows,
      // then each thread moves its row half into TMEM as the UMMA A operand)
      const int te = threadIdx.x - 64;
      if (te < TM) qpair[te] = te < nqt ? a.inv_pairs[p0 + te] : -1;
      asm volatile("bar.sync 3, %0;" ::"r"(32 * TEPI));
      const int nc4 = Dp >> 2;
      for (int e = te; e < TM * nc4; e += 32 * TEPI) {
        const int r = e / nc4, c4 = e % nc4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        const int pr = qpair[r];
        if (pr >= 0) {
          const float* qr = a.Q + (int64_t)(pr / a.nprobe) * st.D;
          if ((st.D & 3) == 0 && 4 * c4 + 3 < st.D) {
            v = *reinterpret_cast<const float4*>(qr + 4 * c4);
          } else {
            float t[4];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) t[jj] = 4 * c4 + jj < st.D ? qr[4 * c4 + jj] : 0.f;
            v = make_float4(t[0], t[1], t[2], t[3]);
          }
        }
        *reinterpret_cast<float4*>(qs + r * Dq + 4 * c4) = v;
      }
      asm volatile("bar.sync 3, %0;" ::"r"(32 * TEPI));
      {
        float nrm = 0.f;
        for (int c8 = h; c8 < (Dp >> 3); c8 += 2) {
          uint32_t v[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float x = qs[row * Dq + 8 * c8 + j];
            v[j] = __float_as_uint(x);
            nrm = fmaf(x, x, nrm);
          }
          tmem_st8(tbase + ((uint32_t)(32 * g) << 16) + (uint32_t)(8 * c8), v);
        }
        qn_half[h * TM + row] = nrm;
        tmem_st_wait();
      }
      tc_fence_before();
      asm volatile("bar.sync 2, %0;" ::"r"(32 * (1 + TEPI)));  // A is in TMEM: release the MMA warp
      const int pair = qpair[row];
      const int qglob = pair >= 0 ? pair / a.nprobe : -1;
      const bool rv = row < nqt;
      const float qn = qn_half[row] + qn_half[TM + row];
      // tf32-exact query: every coordinate an integer with |q| <= 2048
      bool qint = true;
      {
        const float* qrow = qs + row * Dq;
        for (int d = 0; d < Dp; ++d) {
          const float x = qrow[d];
          qint = qint && x == rintf(x) && fabsf(x) <= 2048.f;
        }
      }
      float thr = rv ? __uint_as_float(a.gthr[qglob]) : -1.f;
      // sorted register list; the first KP-k entries are 0 (below every key), so the
      // k smallest always sit in keys[KP-k .. KP) and the k-th is keys[KP-1]
      u64 keys[KP];
#pragma unroll
      for (int i = 0; i < KP; ++i) keys[i] = i < KP - k ? 0ull : kPadKey;
      u64 kth = kPadKey;
      const float eps1 = 0x1p-9f + 0x1p-19f + (float)Dp * 0x1p-23f;
      const float eps2 = (float)(2 * Dp + 8) * 0x1p-24f;
      for (;;) {
        const int stg = it % TNS;
        mbar_wait(&full[stg], (it / TNS) & 1u);
        const TcMeta m = meta[stg];
        if (m.slab < 0) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[stg]);
          ++it;
          break;
        }
        mbar_wait(&mmad[stg], (mmph >> stg) & 1u);
        mmph ^= 1u << stg;
        tc_fence_after();
        uint32_t v[16];
        tmem_ld16(tbase + ((uint32_t)(32 * g) << 16) + dcol0 + (uint32_t)stg * kSlot + (uint32_t)(16 * h), v);
        tmem_ld_wait();
        const bool sint = (m.flag & 1u) != 0u && qint;
        const uint32_t bm = rv ? (m.bitmap >> (16 * h)) & 0xFFFFu : 0u;
        // pass 1 (branch-free, unrolled): slots whose tensor-core distance can still enter the top-k
        const float* nrm = stage_nrm + stg * kSlot + 16 * h;
        uint32_t pm = 0u, exm = 0u;
        float dtc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float xn = nrm[j];
          const float sn = qn + xn;
          dtc[j] = fmaf(-2.f, __uint_as_float(v[j]), sn);
          const bool ex = sint && sn < 16777216.f;  // exact: integer products/partial sums < 2^24
          const float cs = sqrtf(qn * xn);
          const float E = ex ? 0.f : 2.f * (2.f * eps1 * cs + eps2 * (sn + 2.f * cs));
          pm |= (dtc[j] - E <= thr ? 1u : 0u) << j;
          exm |= (ex ? 1u : 0u) << j;
        }
        pm &= bm;
        // pass 2: the (rare) survivors: exact re-rank when needed, then the register top-k
        while (pm) {
          const int j = __ffs(pm) - 1;
          pm &= pm - 1;
          const int slot = 16 * h + j;
          float d = 0.f;
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) d = (jj == j) ? dtc[jj] : d;
          if (!((exm >> j) & 1u)) {
            const float* qrow = qs + row * Dq;
            const float* xs = stage_x + (size_t)stg * kSlot * Dp;
            float acc = 0.f;
            for (int i4 = 0; i4 < (Dp >> 2); ++i4) {
              const float4 qv = *reinterpret_cast<const float4*>(qrow + 4 * i4);
              const float4 xv = *reinterpret_cast<const float4*>(xs + (i4 * kSlot + slot) * 4);
              float t;
              t = qv.x - xv.x; acc = fmaf(t, t, acc);
              t = qv.y - xv.y; acc = fmaf(t, t, acc);
              t = qv.z - xv.z; acc = fmaf(t, t, acc);
              t = qv.w - xv.w; acc = fmaf(t, t, acc);
            }
            d = acc;
          }
          if (!(d <= thr)) continue;
          const u64 key = make_key(d, stage_id[stg * kSlot + slot]);
          if (key >= kth) continue;
          topk_reg_insert<KP>(keys, key);
          kth = keys[KP - 1];
          if (kth != kPadKey) thr = fminf(thr, key_dist(kth));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stg]);
        ++it;
      }
      // hand the half list to the merge buffer (qs is no longer needed)
      asm volatile("bar.sync 1, %0;" ::"r"(32 * TEPI));
#pragma unroll
      for (int i = 0; i < KP; ++i) mrg[((size_t)row * 2 + h) * KP + i] = keys[i];
      asm volatile("bar.sync 1, %0;" ::"r"(32 * TEPI));
      if (h == 0 && rv) {
        const u64* A0 = mrg + (size_t)row * 2 * KP + (KP - k);
        const u64* A1 = A0 + KP;
        int i0 = 0, i1 = 0;
        u64 last = kPadKey;
        for (int j = 0; j < k; ++j) {
          const u64 x0 = A0[i0], x1 = A1[i1];
          const u64 x = x0 < x1 ? x0 : x1;
          if (x0 < x1) ++i0; else ++i1;
          a.partial[(size_t)pair * k + j] = x;
          last = x;
        }
        if (last != kPadKey) atomicMin(&a.gthr[qglob], __float_as_uint(key_dist(last)));
      }
    }
    __syncthreads();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tbase, a.tmem_cols);
}

}  // namespace

bool scan_tc_supported(const Index& ix, int k) {
  if (ix.st.Dp > 256 || k > 32) return false;
  const int KP = k <= 16 ? 16 : 32;
  return tc_smem_bytes(ix.st.Dp, KP) <= ix.smem_optin;
}

cudaError_t setup_scan_tc(Index& ix) {
  if (ix.st.Dp > 256) return cudaSuccess;
  for (int KP : {16, 32}) {
    size_t need = tc_smem_bytes(ix.st.Dp, KP);
    if (need > ix.smem_optin) continue;
    cudaError_t e = KP == 16
                        ? cudaFuncSetAttribute(k_scan_tc<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need)
                        : cudaFuncSetAttribute(k_scan_tc<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_scan_tc(Index& ix, const float* d_q, int k, int nprobe, cudaStream_t s) {
  Scratch& sc = ix.sc;
  TcArgs a{ix.st, d_q, nprobe, k, sc.inv_off, sc.inv_pairs, sc.tile_off, sc.work_list, sc.partial, sc.gthr, 0};
  uint32_t need = (uint32_t)ix.st.Dp + TNS * kSlot;
  uint32_t cols = 32;
  while (cols < need) cols <<= 1;
  a.tmem_cols = cols;
  const int KP = k <= 16 ? 16 : 32;
  const size_t smem = tc_smem_bytes(ix.st.Dp, KP);
  if (KP == 16) k_scan_tc<16><<<ix.num_sms, TTHREADS, smem, s>>>(a);
  else k_scan_tc<32><<<ix.num_sms, TTHREADS, smem, s>>>(a);
  ix.launches += 1;
  return cudaGetLastError();
}

int scan_tc_tile() { return TM; }

}  // namespace sivf
