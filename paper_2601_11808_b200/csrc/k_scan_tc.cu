// k_scan_tc.cu — slab scan on the 5th-generation tensor cores (tcgen05).
//
// Work decomposition as in k_search.cu (a work item = list l x a tile of
// <= 128 queries probing l).  Eq. l2 for (query tile, slabs) is a
// dense contraction:  d(q, x) = ||q||^2 + ||x||^2 - 2 q.x.
// q.x is computed with tcgen05.mma kind::tf32, M = 128 queries (A, resident in
// TMEM for the whole work item), N = 128 slots = a GROUP of 4 slabs (B, in
// shared memory), K = 8 per instruction, fp32 accumulators in TMEM.
//
// Why groups of 4 slabs: one MMA re-reads the whole A tile, so an N=32 (one
// slab) instruction costs as much as N=128 (measured: ~68 cycles each,
// tools/mma_probe.cu); N=128 reaches the tf32 tensor floor.  The B operand must
// be in the K-major SWIZZLE_NONE layout with a uniform 8-row-group stride, so
// the 4 bulk-copied slabs (each [D/4][32][4], itself a valid B layout for N=32)
// are interleaved into [D/4][4 slabs][32][4] by two "transposer" warps: a
// shared-memory pass at full bandwidth (512-B bulk copies of the same layout
// run at ~40% of HBM bandwidth, tools/pipe_probe.cu).
//
// Roles (1 CTA per SM, persistent, 12 warps):
//   warp 0      producer: counts the item's live slabs (bitmap != 0, Eq.
//               slot_valid at slab granularity), then bulk-copies them into a
//               4-stage ring (stage j = slab position j of a group)
//   warp 1      MMA issuer (one lane) and TMEM owner
//   warps 2-3   transposers: stage -> interleaved group buffer (x2), group
//               metadata (ids, norms, bitmaps)
//   warps 4-11  epilogue: TMEM lane quarter (warp % 4) = 32 query rows,
//               column half = 2 of the 4 slabs; filter + register top-k
//
// Exactness (BASELINE.json tolerances): when query and slab values are
// integers with |v| <= 2048 (tf32-exact; slab flag set by k_append) and
// ||q||^2 + ||x||^2 < 2^24, every product and partial sum is an exact integer,
// so the tensor-core distance IS the exact distance (the SIFT-shaped case).
// Otherwise the tensor-core value only filters: a slot is re-ranked with the
// exact fp32 difference form iff d_tc - E <= current k-th distance, E a
// certified bound on |d_tc - d_exact| (tf32 truncation + fp32 accumulation),
// so no member of the exact top-k is ever dropped.  A per-query bound
// (atomicMin of the k-th distance of finished half lists, shared between
// the two halves of a row every group) prunes later candidates: any k real
// candidates bound the final k-th distance from above.
#include <cstdio>

#include "sivf_host.h"

namespace sivf {

namespace {

constexpr int TM = 128;   // queries per tile (TMEM lanes, UMMA M)
constexpr int GS = 4;     // slabs per group (UMMA N = 128)
constexpr int GN = GS * kSlot;
constexpr int NST = 2 * GS;  // stage ring: two groups in flight
constexpr int TEPI = 8;   // epilogue warps
constexpr int NTR = 2;    // transposer warps
constexpr int W_PROD = 0, W_MMA = 1, W_TR0 = 2, W_EPI0 = W_TR0 + NTR;
constexpr int TTHREADS = 32 * (W_EPI0 + TEPI);

struct TcArgs {
  DevState st;
  const float* Q;
  int nprobe, k;
  const int32_t* inv_pairs;
  const int32_t* work_l;
  const int32_t* work_p0;
  const int32_t* work_n;
  unsigned long long* partial;
  uint32_t* gthr;
};

struct StageMeta {
  int32_t slab;   // -1: padding (no slab at this group position)
  uint32_t bitmap;
  uint32_t flag;
  int32_t pad;
};

struct GroupMeta {
  uint32_t id[GN];
  float xn[GN];
  uint32_t bm[GS];
  uint32_t flag[GS];
  int32_t slab[GS];
};

// shared memory plan (bytes)
struct TcSmem {
  size_t stage, ib, gmeta, misc, total;
};
__host__ __device__ inline TcSmem tc_smem_plan(int Dp, int KP) {
  TcSmem p;
  p.stage = (size_t)NST * (kSlot * Dp * 4 + kSlot * 8);  // payload + ids + norms per stage
  p.ib = (size_t)GN * Dp * 4;                           // one interleaved group buffer
  const size_t q = (size_t)TM * (Dp + 4) * 4;           // query staging (aliases the group buffers)
  const size_t m = (size_t)TM * 2 * KP * 8;             // end-of-item half lists (alias too)
  if (q > p.ib) p.ib = q;
  if (m > p.ib) p.ib = m;
  p.gmeta = 2 * sizeof(GroupMeta);
  p.misc = (size_t)TM * 4 * 5 + NST * sizeof(StageMeta) + (2 * NST + 8) * 8 + 64;
  p.total = p.stage + p.ib + p.gmeta + p.misc;
  return p;
}

#ifdef SIVF_TC_PROF
#define PW(slot, stmt)                    \
  do {                                    \
    long long _t0 = clock64();            \
    stmt;                                 \
    pw[slot] += clock64() - _t0;          \
  } while (0)
#else
#define PW(slot, stmt) stmt
#endif

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
  const int Dp = st.Dp, Dq = Dp + 4, k = a.k, nquad = Dp >> 2;
  const TcSmem plan = tc_smem_plan(Dp, KP);
  float* stage_x = reinterpret_cast<float*>(smem);                                  // [NST][32*Dp]
  uint32_t* stage_id = reinterpret_cast<uint32_t*>(stage_x + (size_t)NST * kSlot * Dp);  // [NST][32]
  float* stage_nrm = reinterpret_cast<float*>(stage_id + NST * kSlot);              // [NST][32]
  float* ib = reinterpret_cast<float*>(smem + plan.stage);                          // [Dp/4][128][4]
  float* qs = ib;                                                                   // item start only
  u64* mrg = reinterpret_cast<u64*>(ib);                                            // item end only
  GroupMeta* gm = reinterpret_cast<GroupMeta*>(smem + plan.stage + plan.ib);        // [2]
  float* qn_half = reinterpret_cast<float*>(gm + 2);                                // [2][TM]
  int* qpair = reinterpret_cast<int*>(qn_half + 2 * TM);                           // [TM]
  float* thr_sh = reinterpret_cast<float*>(qpair + TM);                            // [2][TM]
  StageMeta* smeta = reinterpret_cast<StageMeta*>(thr_sh + 2 * TM);                // [NST]
  uint64_t* full = reinterpret_cast<uint64_t*>(smeta + NST);                        // [NST] producer -> transposer
  uint64_t* empty = full + NST;                                                     // [NST] transposer -> producer
  uint64_t* ib_full = empty + NST;                                                  // [1]   transposers -> MMA
  uint64_t* ib_free = ib_full + 1;                                                  // [1]   MMA commit -> transposers
  uint64_t* d_full = ib_free + 1;                                                   // [2]   MMA -> epilogue
  uint64_t* grp_free = d_full + 2;                                                  // [2]   epilogue -> MMA, transposers
  int* ctrl = reinterpret_cast<int*>(grp_free + 2);                                 // [0] item, [1] nlive
  uint32_t* tmem_base_sm = reinterpret_cast<uint32_t*>(ctrl + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef SIVF_TC_PROF
  long long pw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long tstart = clock64();
  long long nitems = 0, ngrp = 0;
#endif
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(ib_full, NTR);
    mbar_init(ib_free, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&d_full[b], 1);
      mbar_init(&grp_free[b], TEPI);
    }
    fence_mbar_init();
  }
  if (warp == W_MMA) tmem_alloc(tmem_base_sm, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_base_sm;
  const uint32_t dcol0 = 128;  // A: columns [0, Dp <= 128); D[b]: columns [128 + 128 b, 256 + 128 b)
  const int ntiles = st.ictr[I_NTILES];
  const uint32_t idesc = umma_idesc_tf32(TM, GN);
  uint32_t gg = 0;  // global group sequence number (all roles agree)

  for (;;) {
    if (threadIdx.x == 0) ctrl[0] = atomicAdd(&st.ictr[I_WORK], 1);
    PW(0, __syncthreads());
    const int w_item = ctrl[0];
    if (w_item >= ntiles) break;
    const int l = a.work_l[w_item];
    const int p0 = a.work_p0[w_item];
    const int nqt = a.work_n[w_item];
    const int len = st.dir_len[l];
    const int32_t* dir = st.dir_arena + st.dir_off[l];
    const int g4 = warp & 3, h = (warp - W_EPI0) >> 2;
    const int row = 32 * g4 + lane;

    // ------------------------------------------------ item setup
    if (warp == W_PROD) {
      int nlive = 0;
      for (int j0 = 0; j0 < len; j0 += 32) {
        const int j = j0 + lane;
        const bool live = j < len && st.bitmap[dir[j]] != 0u;
        nlive += __popc(__ballot_sync(kFull, live));
      }
      if (lane == 0) ctrl[1] = nlive;
    } else if (warp >= W_EPI0) {
#ifdef SIVF_TC_PROF
      long long _tst = clock64();
#endif
      // stage the query tile: coalesced global -> smem rows, then each thread moves
      // its row half into TMEM (the UMMA A operand)
      const int te = threadIdx.x - 32 * W_EPI0;
      if (te < TM) qpair[te] = te < nqt ? a.inv_pairs[p0 + te] : -1;
      asm volatile("bar.sync 3, %0;" ::"r"(32 * TEPI));
      {
        // 2 threads per row, each a contiguous half row: independent loads in flight
        const int r = te >> 1, hq = nquad >> 1, q0 = (te & 1) * hq;
        const int pr = qpair[r];
        const float* qr = a.Q + (int64_t)(pr >= 0 ? pr / a.nprobe : 0) * st.D;
        const bool vec = (st.D & 3) == 0;
#pragma unroll 8
        for (int c4 = q0; c4 < q0 + hq + ((te & 1) ? (nquad & 1) : 0); ++c4) {
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (pr >= 0) {
            if (vec && 4 * c4 + 3 < st.D) {
              v = __ldg(reinterpret_cast<const float4*>(qr + 4 * c4));
            } else {
              float t[4];
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) t[jj] = 4 * c4 + jj < st.D ? qr[4 * c4 + jj] : 0.f;
              v = make_float4(t[0], t[1], t[2], t[3]);
            }
          }
          *reinterpret_cast<float4*>(qs + r * Dq + 4 * c4) = v;
        }
      }
      asm volatile("bar.sync 3, %0;" ::"r"(32 * TEPI));
      float nrm = 0.f;
      bool integral = true;
      for (int c8 = h; c8 < (Dp >> 3); c8 += 2) {
        uint32_t v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float x = qs[row * Dq + 8 * c8 + j];
          v[j] = __float_as_uint(x);
          nrm = fmaf(x, x, nrm);
          integral = integral && x == rintf(x) && fabsf(x) <= 2048.f;
        }
        tmem_st8(tbase + ((uint32_t)(32 * g4) << 16) + (uint32_t)(8 * c8), v);
      }
      qn_half[h * TM + row] = integral ? nrm : -1.f - nrm;  // sign carries this half's integrality
      const int pair = qpair[row];
      thr_sh[h * TM + row] = pair >= 0 ? __uint_as_float(a.gthr[pair / a.nprobe]) : -1.f;
      tmem_st_wait();
#ifdef SIVF_TC_PROF
      pw[0] += clock64() - _tst;
#endif
    }
    tc_fence_before();
    PW(1, __syncthreads());  // A in TMEM, nlive known, query staging area free again
    tc_fence_after();
    const int nlive = ctrl[1];
    const int ngroups = (nlive + GS - 1) / GS;

    // ------------------------------------------------ roles
    if (warp == W_PROD) {
      // bulk copies of the live slabs; group positions beyond nlive get an empty arrival
      const uint32_t bytes = (uint32_t)kSlot * Dp * 4;
      int i = 0;  // live slab counter
      for (int j0 = 0; j0 < len; j0 += 32) {
        const int j = j0 + lane;
        int s = 0;
        uint32_t bm = 0u, fl = 0u;
        if (j < len) {
          s = dir[j];
          bm = st.bitmap[s];
          fl = st.slab_flag[s];
        }
        unsigned live = __ballot_sync(kFull, bm != 0u);
        while (live) {
          const int src = __ffs(live) - 1;
          live &= live - 1;
          const int ss = __shfl_sync(kFull, s, src);
          const uint32_t sbm = __shfl_sync(kFull, bm, src), sfl = __shfl_sync(kFull, fl, src);
          if (lane == 0) {
            const uint32_t seq = gg * GS + (uint32_t)i;
            const int pos = (int)(seq % NST);
            const uint32_t use = seq / NST;
            PW(2, mbar_wait(&empty[pos], (use & 1u) ^ 1u));
            smeta[pos] = StageMeta{ss, sbm, sfl, 0};
            mbar_arrive_expect_tx(&full[pos], bytes + 2 * kSlot * 4);
            bulk_g2s(stage_x + (size_t)pos * kSlot * Dp, st.payload + (size_t)ss * kSlot * Dp, bytes, &full[pos]);
            bulk_g2s(stage_id + pos * kSlot, st.slab_ids + (size_t)ss * kSlot, kSlot * 4, &full[pos]);
            bulk_g2s(stage_nrm + pos * kSlot, st.slab_norm + (size_t)ss * kSlot, kSlot * 4, &full[pos]);
          }
          ++i;
        }
      }
      if (lane == 0) {
        for (; i < ngroups * GS; ++i) {  // pad the last group
          const uint32_t seq = gg * GS + (uint32_t)i;
          const int pos = (int)(seq % NST);
          const uint32_t use = seq / NST;
          mbar_wait(&empty[pos], (use & 1u) ^ 1u);
          smeta[pos].slab = -1;
          mbar_arrive(&full[pos]);
        }
      }
    } else if (warp == W_MMA) {
      if (lane == 0) {
        for (int G = 0; G < ngroups; ++G) {
          const uint32_t u = gg + (uint32_t)G, b = u & 1u;
          PW(2, mbar_wait(ib_full, u & 1u));
          mbar_wait(&grp_free[b], ((u >> 1) & 1u) ^ 1u);  // epilogue done reading D[b] (group u-2)
          tc_fence_after();
          const uint32_t bsm = smem_u32(ib);
          const uint32_t dt = tbase + dcol0 + b * GN;
          for (int kk = 0; kk < (Dp >> 3); ++kk)
            umma_tf32_ts(dt, tbase + (uint32_t)(8 * kk),
                         umma_sdesc(bsm + (uint32_t)kk * 2u * GN * 16u, (uint32_t)GN * 16u, 128u), idesc,
                         kk > 0 ? 1u : 0u);
          umma_commit(ib_free);      // interleave buffer may be refilled
          umma_commit(&d_full[b]);
        }
      }
    } else if (warp < W_EPI0) {
      // transposers: warp t handles group positions 2t, 2t+1
      const int t = warp - W_TR0;
      for (int G = 0; G < ngroups; ++G) {
        const uint32_t u = gg + (uint32_t)G, b = u & 1u;
        PW(2, mbar_wait(ib_free, (u & 1u) ^ 1u));               // MMA of the previous group has read the buffer
        mbar_wait(&grp_free[b], ((u >> 1) & 1u) ^ 1u);           // epilogue done with gm[b] (group u-2)
        float* dst = ib;
        GroupMeta& m = gm[b];
        for (int pp = 0; pp < 2; ++pp) {
          const int gpos = 2 * t + pp;                          // position within the group
          const uint32_t seq = u * GS + (uint32_t)gpos;
          const int pos = (int)(seq % NST);                     // stage
          PW(3, mbar_wait(&full[pos], (seq / NST) & 1u));
          const StageMeta sm = smeta[pos];
          const float* src = stage_x + (size_t)pos * kSlot * Dp;
          if (sm.slab >= 0) {
#pragma unroll 8
            for (int q = 0; q < nquad; ++q)
              *reinterpret_cast<float4*>(dst + ((size_t)q * GN + gpos * kSlot + lane) * 4) =
                  *reinterpret_cast<const float4*>(src + ((size_t)q * kSlot + lane) * 4);
            m.id[gpos * kSlot + lane] = stage_id[pos * kSlot + lane];
            m.xn[gpos * kSlot + lane] = stage_nrm[pos * kSlot + lane];
          }
          if (lane == 0) {
            m.bm[gpos] = sm.slab >= 0 ? sm.bitmap : 0u;
            m.flag[gpos] = sm.slab >= 0 ? sm.flag : 0u;
            m.slab[gpos] = sm.slab;
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[pos]);
        }
        fence_proxy_async_smem();  // generic smem writes -> visible to the tensor core (async proxy)
        __syncwarp();
        if (lane == 0) mbar_arrive(ib_full);
      }
    } else {
      // ------------------------------------------------ epilogue
      const int pair = qpair[row];
      const int qglob = pair >= 0 ? pair / a.nprobe : -1;
      const bool rv = row < nqt;
      const float h0 = qn_half[row], h1 = qn_half[TM + row];
      const bool qint = h0 >= 0.f && h1 >= 0.f;
      const float qn = (h0 >= 0.f ? h0 : -1.f - h0) + (h1 >= 0.f ? h1 : -1.f - h1);
      float thr = fminf(thr_sh[row], thr_sh[TM + row]);
      u64 keys[KP];
#pragma unroll
      for (int i = 0; i < KP; ++i) keys[i] = i < KP - k ? 0ull : kPadKey;  // k-th = keys[KP-1]
      u64 kth = kPadKey;
      const float eps1 = 0x1p-9f + 0x1p-19f + (float)Dp * 0x1p-23f;
      const float eps2 = (float)(2 * Dp + 8) * 0x1p-24f;
      const bool exact_q = qint && qn < 8388608.f;
      for (int G = 0; G < ngroups; ++G) {
        const uint32_t u = gg + (uint32_t)G, b = u & 1u;
        thr = fminf(thr, thr_sh[(1 - h) * TM + row]);  // partner half's bound
        PW(2, mbar_wait(&d_full[b], (u >> 1) & 1u));
        tc_fence_after();
        const GroupMeta& m = gm[b];
#ifdef SIVF_TC_PROF
        ngrp++;
        long long _tg = clock64();
#endif
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          const int col0 = 64 * h + 16 * c;  // group column = pos * 32 + slot
          const int pos = col0 >> 5, sb = col0 & 31;
          uint32_t v[16];
#ifdef SIVF_TC_PROF
          long long _tl = clock64();
#endif
          tmem_ld16(tbase + ((uint32_t)(32 * g4) << 16) + dcol0 + b * GN + (uint32_t)col0, v);
          tmem_ld_wait();
#ifdef SIVF_TC_PROF
          pw[6] += clock64() - _tl;
#endif
          const uint32_t bm = rv ? (m.bm[pos] >> sb) & 0xFFFFu : 0u;
          if (!bm) continue;
          const float4* nrm4 = reinterpret_cast<const float4*>(m.xn + col0);
          const bool sint = exact_q && (m.flag[pos] & 1u) != 0u;
          uint32_t pm = 0u, exm = 0u;
          float dtc[16];
          if (sint) {
#pragma unroll
            for (int j4 = 0; j4 < 4; ++j4) {
              const float4 xn = nrm4[j4];
              const float xa[4] = {xn.x, xn.y, xn.z, xn.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int j = 4 * j4 + e;
                const float sn = qn + xa[e];
                dtc[j] = fmaf(-2.f, __uint_as_float(v[j]), sn);
                const bool ex = sn < 16777216.f;  // every sum an integer < 2^24: exact
                pm |= (dtc[j] <= thr && ex ? 1u : 0u) << j;
                exm |= (ex ? 1u : 0u) << j;
              }
            }
            const uint32_t fb = ~exm & 0xFFFFu;
            if (fb) {
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const float xn = m.xn[col0 + j];
                const float cs = sqrtf(qn * xn), sn = qn + xn;
                const float E = 2.f * (2.f * eps1 * cs + eps2 * (sn + 2.f * cs));
                if ((fb >> j) & 1u) pm |= (dtc[j] - E <= thr ? 1u : 0u) << j;
              }
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float xn = m.xn[col0 + j];
              const float sn = qn + xn;
              dtc[j] = fmaf(-2.f, __uint_as_float(v[j]), sn);
              const float cs = sqrtf(qn * xn);
              const float E = 2.f * (2.f * eps1 * cs + eps2 * (sn + 2.f * cs));
              pm |= (dtc[j] - E <= thr ? 1u : 0u) << j;
            }
          }
          pm &= bm;
#ifdef SIVF_TC_PROF
          long long _ts = clock64();
          pw[3] += __popc(pm);
#endif
          while (pm) {  // survivors: exact re-rank if needed, then the register top-k
            const int j = __ffs(pm) - 1;
            pm &= pm - 1;
            float d = 0.f;
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) d = (jj == j) ? dtc[jj] : d;
            if (!((exm >> j) & 1u)) {
              const float* qr = a.Q + (int64_t)qglob * st.D;
              const float* xs = st.payload + (size_t)m.slab[pos] * kSlot * Dp;
              const int slot = sb + j;
              float acc = 0.f;
              for (int i4 = 0; i4 < nquad; ++i4) {
                const float4 xv = __ldg(reinterpret_cast<const float4*>(xs + (i4 * kSlot + slot) * 4));
                float qv[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) qv[e] = 4 * i4 + e < st.D ? __ldg(qr + 4 * i4 + e) : 0.f;
                float tt;
                tt = qv[0] - xv.x; acc = fmaf(tt, tt, acc);
                tt = qv[1] - xv.y; acc = fmaf(tt, tt, acc);
                tt = qv[2] - xv.z; acc = fmaf(tt, tt, acc);
                tt = qv[3] - xv.w; acc = fmaf(tt, tt, acc);
              }
              d = acc;
            }
            if (!(d <= thr)) continue;
            const u64 key = make_key(d, m.id[col0 + j]);
            if (key >= kth) continue;
            topk_reg_insert<KP>(keys, key);
            kth = keys[KP - 1];
            if (kth != kPadKey) thr = fminf(thr, key_dist(kth));
#ifdef SIVF_TC_PROF
            pw[4]++;
#endif
          }
#ifdef SIVF_TC_PROF
          pw[7] += clock64() - _ts;
#endif
        }
        thr_sh[h * TM + row] = thr;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&grp_free[b]);
#ifdef SIVF_TC_PROF
        pw[5] += clock64() - _tg;
#endif
      }
      // merge the two half lists of each row (the group buffers are idle now)
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
    gg += (uint32_t)ngroups;
#ifdef SIVF_TC_PROF
    nitems++;
#endif
    __syncthreads();
  }
#ifdef SIVF_TC_PROF
  if (blockIdx.x < 2 && lane == 0 && (warp <= W_TR0 || warp == W_EPI0))
    printf("blk %d warp %d total %lld items %lld grp %lld | staging %lld setupsync %lld wait %lld surv %lld ins %lld groupbody %lld tmemld %lld survloop %lld\n",
           blockIdx.x, warp, clock64() - tstart, nitems, ngrp, pw[0], pw[1], pw[2], pw[3], pw[4], pw[5], pw[6], pw[7]);
#endif
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == W_MMA) tmem_dealloc(tbase, 512);
}

}  // namespace

bool scan_tc_supported(const Index& ix, int k) {
  if (ix.st.Dp > 128 || k > 32) return false;
  const int KP = k <= 16 ? 16 : 32;
  return tc_smem_plan(ix.st.Dp, KP).total <= ix.smem_optin;
}

cudaError_t setup_scan_tc(Index& ix) {
  if (ix.st.Dp > 128) return cudaSuccess;
  for (int KP : {16, 32}) {
    const size_t need = tc_smem_plan(ix.st.Dp, KP).total;
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
  TcArgs a{ix.st, d_q, nprobe, k, sc.inv_pairs, sc.work_l, sc.work_p0, sc.work_n, sc.partial, sc.gthr};
  const int KP = k <= 16 ? 16 : 32;
  const size_t smem = tc_smem_plan(ix.st.Dp, KP).total;
  if (KP == 16) k_scan_tc<16><<<ix.num_sms, TTHREADS, smem, s>>>(a);
  else k_scan_tc<32><<<ix.num_sms, TTHREADS, smem, s>>>(a);
  ix.launches += 1;
  return cudaGetLastError();
}

int scan_tc_tile() { return TM; }

}  // namespace sivf
