// k_scan_tc.cu — slab scan on the 5th-generation tensor cores (tcgen05).
//
// Work decomposition as in k_search.cu (a work item = list l x a tile of
// <= 128 queries probing l).  Eq. l2 for (query tile, slabs) is a
// dense contraction:  d(q, x) = ||q||^2 + ||x||^2 - 2 q.x.
// q.x runs on tcgen05.mma kind::f16 (fp16 operands, fp32 accumulation) with
// M = 128 queries (A, resident in TMEM), N = 128 slots = a GROUP of 4 slabs
// (B, shared memory), K = 16 per instruction, accumulators in TMEM.  The B
// operand is the slab's fp16 (RN) copy written by k_append beside the fp32
// payload (reading C35); kind::f16 with A in TMEM issues a 128x128x16 MMA per
// 68 cycles, 4x the kind::tf32 TMEM-A rate (tools/mma_probe.cu).
//
// Why groups of 4 slabs: one MMA re-reads the whole A tile, so an N=32 (one
// slab) instruction costs as much as N=128 (tools/mma_probe.cu).  The B
// operand must be K-major SWIZZLE_NONE with a uniform 8-row-group stride.  The
// fp16 copy is stored as exactly that (pay16_off(): [4 row groups][Dh/8][8
// slots][8 halves], LBO = 128 B, SBO = 16 Dh B), so each slab of a group is
// ONE contiguous cp.async.bulk of 8 KB into consecutive stage slots and the
// four together are the N = 128 operand.  No gather, no shared-memory
// transpose (bulk copies stream 2x faster than TMA tile::gather4 from L2,
// tools/g4_probe.cu).
//
// Roles (1 persistent CTA per SM, 15 warps, no CTA-wide barrier after setup;
// every hand-off is an mbarrier):
//   warp 0      scheduler: claims work items (up to NITEM - 1 ahead, in an
//               item ring) and walks each list's slab directory ahead of
//               the producer, keeping the live slabs (bitmap != 0, Eq.
//               slot_valid at slab granularity) with their flags
//   warp 14     producer: per group of 4 live slabs, bulk copies of the fp16
//               payloads, slot norms and ids into an nst-stage ring; a stage
//               is refilled once the group that used it has completed
//   warp 1      MMA: per group turns the bitmap into a NaN mask on the slot
//               norms (group metadata for the epilogue), then one lane
//               issues Dh/16 tcgen05.mma into one of NB = 3 TMEM accumulators;
//               one tcgen05.commit per group (each costs ~200 cycles of
//               tensor pipe) signals the epilogue and frees the stage
//   warps 2-5   query loaders: the next item's 128 query rows as fp16 into
//               the spare one of two TMEM A buffers (double-buffered across
//               items), with ||q||^2 (fp32), the integrality and fp16-range
//               flags (QInfo ring: up to NQI items ahead of the epilogue)
//   warps 6-13  epilogue: thread = (query row, slab half); per slab,
//               t = ||x||^2 - 2 q.x is one FFMA and the slab's filter one
//               FMNMX per candidate; only chunks whose min passes the row's
//               threshold take the per-lane slow path (exact distance, then
//               a sorted register top-k of (dist, id) keys); the two halves
//               of a row merge at the item's end
// TMEM columns: A[0] [0,64), A[1] [64,128), D[b] = [128 + 128 b, 256 + 128 b), b < 3.
//
// Exactness (BASELINE.json tolerances): when query and slab values are
// integers with |v| <= 2048 (exact in fp16; slab flag set by k_append) and
// (||q|| + ||x||)^2 < 2^24, every product, partial sum, t and ||q||^2 + t is
// an exact integer: the tensor-core distance IS the exact distance (the
// SIFT-shaped case).  Otherwise the value only filters: a slot is re-ranked
// with the exact fp32 difference form iff t <= (thr - ||q||^2) + E, rounded
// up, E a certified bound on |d_tc - d_exact| evaluated at the slab's largest
// ||x||^2 (operand rounding + fp32 accumulation + subnormals + the roundings
// of t and the norms, safety factor 2), so no member of the exact top-k is
// ever dropped; a slab or query without a finite fp16 copy (|v| > 65504)
// re-ranks every valid slot.  thr is the row's current k-th distance, seeded
// from a per-query bound (atomicMin of the k-th distance of the query's
// other items, read every group).
#include <cuda.h>
#include <cuda_fp16.h>

#include <cstdio>

#include "sivf_host.h"

namespace sivf {

namespace {

constexpr int TM = 128;   // queries per tile (TMEM lanes, UMMA M)
constexpr int GS = 4;     // slabs per group (UMMA N = 128)
constexpr int GN = GS * kSlot;
constexpr int NITEM = 8;  // work-item ring
constexpr int NQI = 4;    // QInfo buffers: the loaders may run NQI items ahead of the epilogue
constexpr int NB = 3;     // TMEM accumulator buffers (3 x 128 columns after the two 64-column A buffers)
constexpr int MAXST = NB; // group ring depth cap (stages are freed through the accumulator barriers)
constexpr int NLD = 4, NEPI = 8;
constexpr int W_SCHED = 0, W_MMA = 1, W_LD0 = 2, W_EPI0 = W_LD0 + NLD, W_TMA = W_EPI0 + NEPI;
constexpr int TTHREADS = 32 * (W_TMA + 1);
constexpr int MAXS = 64;  // live slabs per item prefetched by the scheduler (the producer walks the rest)

struct TcArgs {
  DevState st;
  const float* Q;
  int nprobe, k, nst;
  const int32_t* inv_pairs;
  const int32_t* work_l;
  const int32_t* work_p0;
  const int32_t* work_n;
  unsigned long long* partial;
  uint32_t* gthr;
  int phase;  // 0: every work item; 1: bucket 0 only; 2: bucket 1 only (phased scan)
  int dbg;  // experiments only (SIVF_OPT_DEBUG): bit0 skip the slow path, bit1 skip the fast path,
            // bit2 skip the MMAs, bit3 skip the B copies, bit4 skip the A loads
};

struct ItemRec {
  int32_t l, p0, nqt;  // l < 0: no more work
  int32_t npre;        // live slabs prefetched into the slot's record array
  int32_t dir_pos;     // directory position where the prefetch stopped (-1: complete)
  int32_t len, pad[2];
};
struct StageMeta {
  int32_t slab[GS];  // -1: padding position
  uint32_t bm[GS];
  uint32_t flag[GS];
  int32_t last, pad[3];
};
struct GroupMeta {
  float xnm[GN];     // ||x||^2 per slot, NaN where the validity bit is clear
  uint32_t id[GN];
  float xnmax[GS];   // max ||x||^2 over the slab's valid slots
  uint32_t flag[GS];
  int32_t slab[GS];
  int32_t last, pad[3];
};
struct QInfo {
  float qn;
  int32_t pair;
  uint32_t qint;  // every value an integer with |v| <= 2048 (exact in fp16)
  uint32_t qover; // some |v| > 65504: no finite fp16 copy, every candidate is re-ranked
};

struct TcPlan {
  size_t stage_bytes, off_meta, off_gm, off_q, off_items, off_thr, off_mrg, off_bar, total;
};
__host__ __device__ inline TcPlan tc_plan(int Dh, int nst, int KP) {
  TcPlan p;
  p.stage_bytes = ((size_t)GN * Dh * 2 + 2 * GN * 4 + 1023) & ~(size_t)1023;  // fp16 payload + slot norms + ids
  p.off_meta = (size_t)nst * p.stage_bytes;
  p.off_gm = p.off_meta + MAXST * sizeof(StageMeta);
  p.off_q = p.off_gm + NB * sizeof(GroupMeta);
  p.off_items = p.off_q + NQI * TM * sizeof(QInfo);
  p.off_thr = p.off_items + NITEM * (sizeof(ItemRec) + MAXS * sizeof(uint2));
  p.off_mrg = p.off_thr + 2 * TM * 8;
  p.off_bar = p.off_mrg + (size_t)TM * KP * 8;
  p.total = p.off_bar + (2 * MAXST + 2 * NB + 4 + 2 * NQI + 2 * NITEM + 2) * 8 + 1024;  // + alignment slack
  return p;
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

// v[c] for a per-lane dynamic c without local memory: a 31-select tree.
__device__ __forceinline__ uint32_t pick32(const uint32_t (&v)[32], int c) {
  uint32_t a16[16], a8[8], a4[4], a2[2];
#pragma unroll
  for (int i = 0; i < 16; ++i) a16[i] = (c & 1) ? v[2 * i + 1] : v[2 * i];
#pragma unroll
  for (int i = 0; i < 8; ++i) a8[i] = (c & 2) ? a16[2 * i + 1] : a16[2 * i];
#pragma unroll
  for (int i = 0; i < 4; ++i) a4[i] = (c & 4) ? a8[2 * i + 1] : a8[2 * i];
#pragma unroll
  for (int i = 0; i < 2; ++i) a2[i] = (c & 8) ? a4[2 * i + 1] : a4[2 * i];
  return (c & 16) ? a2[1] : a2[0];
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

#ifdef SIVF_TC_PROF
#ifdef SIVF_TC_NOCOUNT  // timing builds: no contended counters on the slow path
#define SCNT_ADD(p, v) ((void)0)
#else
#define SCNT_ADD(p, v) atomicAdd(p, v)
#endif
__device__ long long g_tr[6][1024];
__device__ unsigned long long g_scnt[4];  // slow-path entries, survivors, insertions, warp-level loop iterations
#define TR(r, g, v) \
  do {              \
    if (blockIdx.x == 0 && (g) < 1024u) g_tr[r][g] = (v); \
  } while (0)
#else
#define TR(r, g, v) \
  do {              \
  } while (0)
#endif

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
__global__ void __launch_bounds__(TTHREADS, 1) k_scan_tc(TcArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const DevState& st = a.st;
  const int Dp = st.Dp, nq4 = Dp >> 2, Dh = st.Dh, nst = a.nst, k = a.k;
  const TcPlan p = tc_plan(Dh, nst, KP);
  StageMeta* smeta = reinterpret_cast<StageMeta*>(smem + p.off_meta);
  GroupMeta* gm = reinterpret_cast<GroupMeta*>(smem + p.off_gm);
  QInfo* qinfo = reinterpret_cast<QInfo*>(smem + p.off_q);  // [2][TM]
  ItemRec* items = reinterpret_cast<ItemRec*>(smem + p.off_items);
  uint2* irec = reinterpret_cast<uint2*>(items + NITEM);  // [NITEM][MAXS] (slab | flags << 30, bitmap)
  u64* thr_sh = reinterpret_cast<u64*>(smem + p.off_thr);    // [2][TM] (item << 32 | k-th bound bits)
  u64* mrg = reinterpret_cast<u64*>(smem + p.off_mrg);       // [TM][KP] half-list hand-over
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.off_bar);  // [MAXST] producer -> MMA (tx bytes)
  uint64_t* meta_full = full + MAXST;                              // [MAXST] producer -> MMA (stage metadata)
  uint64_t* d_full = meta_full + MAXST;                            // [NB] MMA commit -> epilogue, producer
  uint64_t* grp_free = d_full + NB;                                // [NB] epilogue -> MMA
  uint64_t* a_full = grp_free + NB;                                 // [2] loaders -> MMA, epilogue
  uint64_t* a_free = a_full + 2;                                   // [2] MMA commit -> loaders
  uint64_t* q_read = a_free + 2;                                   // [NQI] epilogue -> loaders (QInfo consumed)
  uint64_t* q_full = q_read + NQI;                                 // [NQI] loaders -> epilogue (QInfo written)
  uint64_t* item_full = q_full + NQI;                              // [NITEM] scheduler -> all
  uint64_t* item_empty = item_full + NITEM;                        // [NITEM] epilogue -> scheduler
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(item_empty + NITEM);
  auto stage_x = [&](int s) { return reinterpret_cast<uint16_t*>(smem + (size_t)s * p.stage_bytes); };
  auto stage_nrm = [&](int s) {
    return reinterpret_cast<float*>(smem + (size_t)s * p.stage_bytes + (size_t)GN * Dh * 2);
  };
  auto stage_id = [&](int s) {
    return reinterpret_cast<uint32_t*>(smem + (size_t)s * p.stage_bytes + (size_t)GN * Dh * 2 + GN * 4);
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef SIVF_TC_PROF
  long long pw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long tstart = clock64();
#endif
  if (threadIdx.x == 0) {
    for (int i = 0; i < MAXST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&meta_full[i], 1);
    }
    for (int b = 0; b < NB; ++b) {
      mbar_init(&d_full[b], 2);
      mbar_init(&grp_free[b], NEPI);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&a_full[b], NLD);
      mbar_init(&a_free[b], 1);
    }
    for (int b = 0; b < NQI; ++b) {
      mbar_init(&q_read[b], NEPI);
      mbar_init(&q_full[b], NLD);
    }
    for (int i = 0; i < NITEM; ++i) {
      mbar_init(&item_full[i], 1);
      mbar_init(&item_empty[i], NEPI);
    }
    fence_mbar_init();
  }
  for (int t = threadIdx.x; t < 2 * TM; t += blockDim.x) thr_sh[t] = ~0ull;  // tag matches no item
  if (warp == W_MMA) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;

  if (warp == W_SCHED) {
    // ------------------------------------------------------------ scheduler
    // claims work items and walks each list's slab directory ahead of the
    // producer (up to NITEM - 1 items ahead): the dependent loads (item ->
    // directory -> bitmap -> flag) leave the TMA issue path
    const int ntiles = st.ictr[a.phase == 1 ? I_NTILES0 : I_NTILES];
    const unsigned lt = (1u << lane) - 1u;
    for (uint32_t i = 0;; ++i) {
      const int slot = (int)(i % NITEM);
      if (lane == 0) PW(0, mbar_wait(&item_empty[slot], ((i / NITEM) & 1u) ^ 1u));
      int w = 0;
      if (lane == 0) w = atomicAdd(&st.ictr[a.phase == 2 ? I_WORK2 : I_WORK], 1);
      w = __shfl_sync(kFull, w, 0);
      ItemRec r{-1, 0, 0, 0, -1, 0, 0, 0};
      if (w < ntiles) {
        const int l = a.work_l[w];
        const int len = st.dir_len[l];
        const int32_t* dir = st.dir_arena + st.dir_off[l];
        uint2* rec = irec + slot * MAXS;
        int npre = 0, j0 = 0;
        for (; j0 < len; j0 += 32) {
          const int j = j0 + lane;
          int sl = 0;
          uint32_t bm = 0u;
          if (j < len) {
            sl = dir[j];
            bm = st.bitmap[sl];
          }
          const unsigned live = __ballot_sync(kFull, bm != 0u);
          if (npre + __popc(live) > MAXS) break;  // the producer walks the rest
          if (bm) {
            const uint32_t fl = st.slab_flag[sl] & 3u;
            rec[npre + __popc(live & lt)] = make_uint2((uint32_t)sl | (fl << 30), bm);
          }
          npre += __popc(live);
        }
        r = ItemRec{l, a.work_p0[w], a.work_n[w], npre, j0 < len ? j0 : -1, len, 0, 0};
      }
      __syncwarp();
      if (lane == 0) {
        items[slot] = r;
        mbar_arrive(&item_full[slot]);
      }
      if (w >= ntiles) break;
    }
  } else if (warp == W_TMA) {
    // ------------------------------------------------------------ producer
    uint32_t gseq = 0;
    // group slabs are held lane-distributed: lanes 0-3 the group being filled,
    // lanes 4-7 the completed group waiting to learn whether it is the item's last
    int my_s = 0;
    uint32_t my_bm = 0u, my_fl = 0u;
    auto emit = [&](int base, int nvalid, int last) {
      const int stg = (int)(gseq % (uint32_t)nst);
      // the stage is free once group gseq - nst has completed: its accumulator
      // commit (d_full, the group's only tcgen05.commit) also frees its stage;
      // nst <= NB, so that barrier cannot have moved on to a later phase
      if (lane == 0 && gseq >= (uint32_t)nst) {
        const uint32_t g0 = gseq - (uint32_t)nst;
        PW(1, mbar_wait(&d_full[g0 % NB], (g0 / NB) & 1u));
      }
      if (lane == 0) TR(0, gseq, clock64());
      __syncwarp();
      const int sl = __shfl_sync(kFull, my_s, base + (lane & 3));
      const uint32_t bmv = __shfl_sync(kFull, my_bm, base + (lane & 3));
      const uint32_t flv = __shfl_sync(kFull, my_fl, base + (lane & 3));
      StageMeta& m = smeta[stg];
      if (lane < GS) {
        m.slab[lane] = lane < nvalid ? sl : -1;
        m.bm[lane] = lane < nvalid ? bmv : 0u;
        m.flag[lane] = lane < nvalid ? flv : 0u;
      }
      if (lane == 0) m.last = last;
      __syncwarp();
      const uint32_t sbytes = (uint32_t)(kSlot * Dh * 2);
      if (lane == 0) {
        mbar_arrive(&meta_full[stg]);
        mbar_arrive_expect_tx(&full[stg], (a.dbg & 8) ? 0u : (uint32_t)nvalid * (sbytes + 2u * kSlot * 4u));
      }
      __syncwarp();
      if (a.dbg & 8) nvalid = 0;  // experiment: no B traffic
      // padding positions are not copied: their stale (finite) or uninitialised
      // columns only reach D columns whose slot norm is the NaN mask
      if (lane < nvalid) {
        bulk_g2s(stage_x(stg) + (size_t)lane * kSlot * Dh, st.payload16 + (size_t)sl * kSlot * Dh, sbytes, &full[stg]);
        bulk_g2s(stage_nrm(stg) + lane * kSlot, st.slab_norm + (size_t)sl * kSlot, kSlot * 4, &full[stg]);
        bulk_g2s(stage_id(stg) + lane * kSlot, st.slab_ids + (size_t)sl * kSlot, kSlot * 4, &full[stg]);
      }
      ++gseq;
    };
    int cnt = 0;
    bool has_pend = false;
    auto feed = [&](int ss, uint32_t sbm, uint32_t sfl) {  // warp-uniform arguments
      if (cnt == GS) {
        if (has_pend) emit(4, GS, 0);
        const int ps = __shfl_sync(kFull, my_s, lane & 3);
        const uint32_t pb = __shfl_sync(kFull, my_bm, lane & 3), pf = __shfl_sync(kFull, my_fl, lane & 3);
        if (lane >= 4 && lane < 8) {
          my_s = ps;
          my_bm = pb;
          my_fl = pf;
        }
        has_pend = true;
        cnt = 0;
      }
      if (lane == cnt) {
        my_s = ss;
        my_bm = sbm;
        my_fl = sfl;
      }
      ++cnt;
    };
    for (uint32_t i = 0;; ++i) {
      const int slot = (int)(i % NITEM);
      PW(4, mbar_wait(&item_full[slot], (i / NITEM) & 1u));
      const ItemRec rec = items[slot];
      if (rec.l < 0) break;
      cnt = 0;
      has_pend = false;
      const uint2* rr = irec + slot * MAXS;
      for (int r = 0; r < rec.npre; ++r) {
        const uint2 x = rr[r];
        feed((int)(x.x & 0x3fffffffu), x.y, x.x >> 30);
      }
      if (rec.dir_pos >= 0) {  // long list: walk the rest of the directory here
        const int32_t* dir = st.dir_arena + st.dir_off[rec.l];
        for (int j0 = rec.dir_pos; j0 < rec.len; j0 += 32) {
          const int j = j0 + lane;
          int s = 0;
          uint32_t bm = 0u, fl = 0u;
          if (j < rec.len) {
            s = dir[j];
            bm = st.bitmap[s];
            if (bm) fl = st.slab_flag[s] & 3u;
          }
          unsigned live = __ballot_sync(kFull, bm != 0u);
          while (live) {
            const int src = __ffs(live) - 1;
            live &= live - 1;
            feed(__shfl_sync(kFull, s, src), __shfl_sync(kFull, bm, src), __shfl_sync(kFull, fl, src));
          }
        }
      }
      if (cnt > 0) {
        if (has_pend) emit(4, GS, 0);
        emit(0, cnt, 1);
      } else if (has_pend) {
        emit(4, GS, 1);
      } else {
        emit(0, 0, 1);  // no live slab: one fully masked group keeps the roles in step
      }
    }
  } else if (warp == W_MMA) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = umma_idesc_f16(TM, GN);
    uint32_t gseq = 0;
    for (uint32_t i = 0;; ++i) {
      const int slot = (int)(i % NITEM);
      PW(6, mbar_wait(&item_full[slot], (i / NITEM) & 1u));
      const ItemRec rec = items[slot];
      if (rec.l < 0) break;
      const uint32_t ab = i & 1u;
      PW(1, mbar_wait(&a_full[ab], (i >> 1) & 1u));
      for (;;) {
        const int stg = (int)(gseq % (uint32_t)nst);
        const uint32_t b = gseq % NB;
        PW(0, mbar_wait(&meta_full[stg], (gseq / (uint32_t)nst) & 1u));
        const StageMeta& sm = smeta[stg];
        float xnv[GS];
        uint32_t idv[GS];
        PW(2, mbar_wait(&full[stg], (gseq / (uint32_t)nst) & 1u));
        if (lane == 0) TR(1, gseq, clock64());
#pragma unroll
        for (int j = 0; j < GS; ++j) {  // staged with the payload (garbage at padding positions: masked)
          xnv[j] = stage_nrm(stg)[j * kSlot + lane];
          idv[j] = stage_id(stg)[j * kSlot + lane];
        }
        PW(3, mbar_wait(&grp_free[b], ((gseq / NB) & 1u) ^ 1u));
        if (lane == 0) TR(2, gseq, clock64());
        GroupMeta& g = gm[b];
#ifdef SIVF_TC_PROF
        long long _tm0 = clock64();
#endif
#pragma unroll
        for (int j = 0; j < GS; ++j) {
          const bool v = ((sm.bm[j] >> lane) & 1u) != 0u;
          const float xn = xnv[j];
          g.xnm[j * kSlot + lane] = v ? xn : __int_as_float(0x7fc00000);
          g.id[j * kSlot + lane] = idv[j];
          const uint32_t mx = __reduce_max_sync(kFull, v ? __float_as_uint(fmaxf(xn, 0.f)) : 0u);
          if (lane == 0) {
            g.xnmax[j] = __uint_as_float(mx);
            g.flag[j] = sm.flag[j];
            g.slab[j] = sm.slab[j];
          }
        }
        const int last = sm.last;
        if (lane == 0) g.last = last;
        __syncwarp();
#ifdef SIVF_TC_PROF
        pw[5] += clock64() - _tm0;
        _tm0 = clock64();
#endif
        if (lane == 0) {
          tc_fence_after();
          const uint32_t bsm = smem_u32(stage_x(stg));
          const uint32_t dt = tbase + 128u + b * 128u, at = tbase + ab * 64u;
          // kind::f16: A (fp16 query tile) in TMEM, 8 columns per K = 16 step;
          // B (fp16 slab copies) K-major SWIZZLE_NONE, LBO = 128 B, SBO = 16 Dh B
          for (int kk = 0; kk < ((a.dbg & 4) ? 0 : (Dh >> 4)); ++kk)
            umma_f16_ts(dt, at + (uint32_t)(8 * kk), umma_sdesc(bsm + (uint32_t)kk * 256u, 128u, (uint32_t)Dh * 16u),
                        idesc, kk > 0 ? 1u : 0u);
          umma_commit(&d_full[b]);    // accumulator ready and stage stg free (one commit per group:
                                      // each tcgen05.commit costs ~200 cycles of tensor pipe, mma_probe)
          mbar_arrive(&d_full[b]);    // group metadata written
          if (last) umma_commit(&a_free[ab]);  // A[ab] may be overwritten once these MMAs are done
        }
        __syncwarp();
#ifdef SIVF_TC_PROF
        pw[4] += clock64() - _tm0;
#endif
        ++gseq;
        if (last) break;
      }
    }
  } else if (warp < W_EPI0) {
    // ------------------------------------------------------------ query loaders
    // thread = query row (TMEM lane); rows are loaded 64 dims at a time, the
    // first half before A[ab] is free (its latency hides behind the wait),
    // then ||q||^2 (fp32), the integrality and fp16-range flags and
    // tcgen05.st of the fp16 (RN) row, two halves per column
    const int qw = warp & 3, row = 32 * qw + lane;
    const bool vec = (st.D & 3) == 0;
    const int nc8 = Dh >> 3;
    for (uint32_t i = 0;; ++i) {
      const int slot = (int)(i % NITEM);
      mbar_wait(&item_full[slot], (i / NITEM) & 1u);
      const ItemRec rec = items[slot];
      if (rec.l < 0) break;
      const uint32_t ab = i & 1u;
      const bool rv = row < rec.nqt;
      const bool wv = 32 * qw < rec.nqt && !(a.dbg & 16);  // warp-uniform: the warp has a real row
      const int pair = rv ? a.inv_pairs[rec.p0 + row] : -1;
      const float* qr = a.Q + (int64_t)(rv ? pair / a.nprobe : 0) * st.D;
      const uint32_t ta = tbase + ((uint32_t)(32 * qw) << 16) + ab * 64u;
      float nrm = 0.f;
      uint32_t integ = 1u, over = 0u;
#ifdef SIVF_TC_PROF
      long long _tl0 = clock64();
#endif
      for (int h0 = 0; h0 < nc8; h0 += 8) {
        float x[8][8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int d0 = 8 * (h0 + u);
          if (wv && rv && vec && d0 + 7 < st.D) {
            const float4 lo = __ldg(reinterpret_cast<const float4*>(qr + d0));
            const float4 hi = __ldg(reinterpret_cast<const float4*>(qr + d0 + 4));
            x[u][0] = lo.x, x[u][1] = lo.y, x[u][2] = lo.z, x[u][3] = lo.w;
            x[u][4] = hi.x, x[u][5] = hi.y, x[u][6] = hi.z, x[u][7] = hi.w;
          } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) x[u][e] = (rv && h0 + u < nc8 && d0 + e < st.D) ? __ldg(qr + d0 + e) : 0.f;
          }
        }
        if (h0 == 0) {
          PW(4, mbar_wait(&a_free[ab], ((i >> 1) & 1u) ^ 1u));
          tc_fence_after();
        }
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
          if (h0 + u < nc8) {  // nc8 is even: 16 dims = 8 columns
            uint32_t hv[8];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const float xe = x[u + (e >> 3)][e & 7];
              nrm = fmaf(xe, xe, nrm);
              integ &= (xe == rintf(xe) ? 1u : 0u) & (fabsf(xe) <= 2048.f ? 1u : 0u);
              over |= fabsf(xe) <= 65504.f ? 0u : 1u;
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const __half2 h2 = __floats2half2_rn(x[u + (c >> 2)][2 * (c & 3)], x[u + (c >> 2)][2 * (c & 3) + 1]);
              hv[c] = *reinterpret_cast<const uint32_t*>(&h2);
            }
            if (wv) tmem_st8(ta + (uint32_t)(4 * (h0 + u)), hv);
          }
        }
      }
#ifdef SIVF_TC_PROF
      pw[1] += clock64() - _tl0;
      _tl0 = clock64();
#endif
      tmem_st_wait();
#ifdef SIVF_TC_PROF
      pw[2] += clock64() - _tl0;
#endif
      const int qb = (int)(i % NQI);
      PW(5, mbar_wait(&q_read[qb], ((i / NQI) & 1u) ^ 1u));  // item i - NQI's QInfo has been read
      qinfo[qb * TM + row] = QInfo{nrm, pair, integ, over};
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&a_full[ab]);
        mbar_arrive(&q_full[qb]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // thread = (query row, slab half h): slabs 2h, 2h+1 of every group; the two
    // halves of a row keep separate top-k lists (merged at the item's end) and
    // share their k-th distance bounds through shared memory every group
    const int qw = warp & 3, row = 32 * qw + lane, h = (warp - W_EPI0) >> 2;
    // certified band of the fp16 filter (u = 2^-11, RN): eps1 bounds the
    // relative error of q.x from the operand roundings (2u + u^2 <= 2^-9 +
    // 2^-19, tf32-safe margin kept) and fp32 accumulation (Dh 2^-23); esub the
    // absolute error of fp16 subnormals (|v| < 2^-14: error <= 2^-25 per value,
    // sum <= 2^-25 sqrt(Dh) (||q|| + ||x||)), times 2 for d and 2 for safety
    const float eps1 = 0x1p-9f + 0x1p-19f + (float)Dh * 0x1p-23f;
    const float eps2 = (float)(2 * Dp + 10) * 0x1p-24f;
    const float esub = 0x1p-23f * 1.001f * sqrtf((float)Dh);
    uint32_t gseq = 0;
    for (uint32_t i = 0;; ++i) {
      const int slot = (int)(i % NITEM);
      PW(4, mbar_wait(&item_full[slot], (i / NITEM) & 1u));
      const ItemRec rec = items[slot];
      if (rec.l < 0) break;
      const uint32_t ab = i & 1u;
      PW(1, mbar_wait(&q_full[i % NQI], (i / NQI) & 1u));
      const QInfo qi = qinfo[(i % NQI) * TM + row];
      __syncwarp();
      if (lane == 0) mbar_arrive(&q_read[i % NQI]);
      const bool rv = row < rec.nqt;
      const bool wact = 32 * qw < rec.nqt;
      const int qglob = rv ? qi.pair / a.nprobe : 0;
      const float qn = qi.qn, sqn = sqrtf(qn);
      float thr = rv ? __uint_as_float(__ldcg(a.gthr + qglob)) : -INFINITY;
      float gnext = thr, tpub = thr;
      u64 keys[KP];
#pragma unroll
      for (int t = 0; t < KP; ++t) keys[t] = t < KP - k ? 0ull : kPadKey;  // k-th = keys[KP-1]
      u64 kth = kPadKey;
      for (;;) {
        const uint32_t b = gseq % NB;
        PW(5, mbar_wait(&d_full[b], (gseq / NB) & 1u));
        if (lane == 0 && warp == W_EPI0 + 2) TR(3, gseq, clock64());
        if (lane == 0 && warp == W_EPI0 + 6) TR(5, gseq, clock64());
        tc_fence_after();
        const GroupMeta& g = gm[b];
        if (wact) {
          const u64 ps = thr_sh[(1 - h) * TM + row];  // partner half's bound, tagged with its item
          if ((uint32_t)(ps >> 32) == i) thr = fminf(thr, __uint_as_float((uint32_t)ps));
          thr = fminf(thr, gnext);  // other items of the same query (read one group ago)
          if (rv) gnext = __uint_as_float(__ldcg(a.gthr + qglob));
          // one chunk = one slab = 32 TMEM columns of this row
          auto chunk = [&](const int j, const uint32_t(&v)[32]) {
            const float xm = g.xnmax[j], sxm = sqrtf(xm);
            const float rs = sqn + sxm;
            const bool ex = qi.qint != 0u && (g.flag[j] & kFlagIntegral) != 0u && rs * rs < 16000000.f;
            // no finite fp16 copy of the query or the slab: every valid slot is re-ranked exactly
            const bool unsafe = qi.qover != 0u || (g.flag[j] & kFlagF16Over) != 0u;
            float E = 0.f;
            if (!ex) {
              const float cs = sqn * sxm;
              E = 2.f * (2.f * eps1 * cs + eps2 * (qn + xm + 2.f * cs)) + esub * rs;
            }
            float tadj = ex ? __fsub_ru(thr, qn) : __fadd_ru(__fsub_ru(thr, qn), E);
            const float4* x4 = reinterpret_cast<const float4*>(g.xnm + 32 * j);
            float m8[8];
#pragma unroll
            for (int c4 = 0; c4 < 8; ++c4) {
              const float4 xx = x4[c4];
              const float t0 = fmaf(-2.f, __uint_as_float(v[4 * c4 + 0]), xx.x);
              const float t1 = fmaf(-2.f, __uint_as_float(v[4 * c4 + 1]), xx.y);
              const float t2 = fmaf(-2.f, __uint_as_float(v[4 * c4 + 2]), xx.z);
              const float t3 = fmaf(-2.f, __uint_as_float(v[4 * c4 + 3]), xx.w);
              m8[c4] = fminf(fminf(t0, t1), fminf(t2, t3));
            }
            const float mn = fminf(fminf(fminf(m8[0], m8[1]), fminf(m8[2], m8[3])),
                                   fminf(fminf(m8[4], m8[5]), fminf(m8[6], m8[7])));
            if (!unsafe && (!(mn <= tadj) || (a.dbg & 1))) return;
            // slow path (per lane): survivors of this slab, exact distance, register top-k
#ifdef SIVF_TC_PROF
            long long _ts = clock64();
#endif
#ifdef SIVF_TC_PROF
            SCNT_ADD(&g_scnt[0], 1ull);
#endif
            uint32_t pm = 0u;
            if (unsafe) {
#pragma unroll
              for (int c = 0; c < 32; ++c) pm |= (g.xnm[32 * j + c] == g.xnm[32 * j + c] ? 1u : 0u) << c;  // valid
            } else
#pragma unroll
            for (int c4 = 0; c4 < 8; ++c4) {
              if (!(m8[c4] <= tadj)) continue;  // the quad's minimum already fails
              const float4 xx = x4[c4];
              pm |= (fmaf(-2.f, __uint_as_float(v[4 * c4 + 0]), xx.x) <= tadj ? 1u : 0u) << (4 * c4);
              pm |= (fmaf(-2.f, __uint_as_float(v[4 * c4 + 1]), xx.y) <= tadj ? 1u : 0u) << (4 * c4 + 1);
              pm |= (fmaf(-2.f, __uint_as_float(v[4 * c4 + 2]), xx.z) <= tadj ? 1u : 0u) << (4 * c4 + 2);
              pm |= (fmaf(-2.f, __uint_as_float(v[4 * c4 + 3]), xx.w) <= tadj ? 1u : 0u) << (4 * c4 + 3);
            }
#ifdef SIVF_TC_PROF
            SCNT_ADD(&g_scnt[1], (unsigned long long)__popc(pm));
#endif
            while (pm) {
              const int c = __ffs(pm) - 1;
              pm &= pm - 1;
              const float t = fmaf(-2.f, __uint_as_float(pick32(v, c)), g.xnm[32 * j + c]);
              if (!unsafe && !(t <= tadj)) continue;  // the threshold may have tightened
              float d;
              if (ex) {
                d = qn + t;  // exact: every term an integer < 2^24
              } else {
                const float* xs = st.payload + (size_t)g.slab[j] * kSlot * Dp;
                const float* qr = a.Q + (int64_t)qglob * st.D;
                float acc = 0.f;
                for (int i4 = 0; i4 < nq4; ++i4) {
                  const float4 xv = __ldg(reinterpret_cast<const float4*>(xs + pay_off(Dp, c, i4)));
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
              d = fmaxf(d, 0.f);
              if (!(d <= thr)) continue;
              const u64 key = make_key(d, g.id[32 * j + c]);
              if (key >= kth) continue;
              topk_reg_insert<KP>(keys, key);
              kth = keys[KP - 1];
              if (kth != kPadKey) {
                thr = fminf(thr, key_dist(kth));
                tadj = ex ? __fsub_ru(thr, qn) : __fadd_ru(__fsub_ru(thr, qn), E);
              }
#ifdef SIVF_TC_PROF
              pw[7]++;
              SCNT_ADD(&g_scnt[2], 1ull);
#endif
            }
#ifdef SIVF_TC_PROF
            pw[6] += clock64() - _ts;
#endif
          };
          const uint32_t dcol = tbase + ((uint32_t)(32 * qw) << 16) + 128u + b * 128u + (uint32_t)(64 * h);
#ifdef SIVF_TC_PROF
          long long _tg = clock64();
#endif
#pragma unroll 1
          for (int jj = 0; jj < 2; ++jj) {
            uint32_t v[32];
#ifdef SIVF_TC_PROF
            long long _tq = clock64();
#endif
            if (!(a.dbg & 32)) {
              tmem_ld32(dcol + 32u * (uint32_t)jj, v);
              tmem_ld_wait();
            } else {
#pragma unroll
              for (int c = 0; c < 32; ++c) v[c] = 0x7f800000u;
            }
#ifdef SIVF_TC_PROF
            pw[3] += clock64() - _tq;
#endif
            if (!(a.dbg & 2)) chunk(2 * h + jj, v);
          }
#ifdef SIVF_TC_PROF
          pw[0] += clock64() - _tg;
#endif
          thr_sh[h * TM + row] = ((u64)i << 32) | __float_as_uint(thr);
          if (rv && thr < tpub) {  // share the bound with the query's other items right away
            atomicMin(a.gthr + qglob, __float_as_uint(thr));
            tpub = thr;
          }
        }
        const int last = g.last;
        if (lane == 0 && warp == W_EPI0 + 2) TR(4, gseq, clock64());
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&grp_free[b]);
        ++gseq;
        if (last) break;
      }
      // merge the two halves of each row: h = 1 hands its list over in smem
      if (h == 1 && rv) {
#pragma unroll
        for (int t = 0; t < KP; ++t) mrg[row * KP + t] = keys[t];
      }
      PW(2, named_bar_sync(1 + qw, 64));
      if (h == 0 && rv) {
        for (int t = KP - k; t < KP; ++t) {
          const u64 key = mrg[row * KP + t];
          if (key >= kth) break;  // sorted: the rest cannot enter
          topk_reg_insert<KP>(keys, key);
          kth = keys[KP - 1];
        }
#pragma unroll
        for (int t = 0; t < KP; ++t)
          if (t >= KP - k) a.partial[(size_t)qi.pair * k + (t - (KP - k))] = keys[t];
        if (kth != kPadKey) atomicMin(&a.gthr[qglob], __float_as_uint(key_dist(kth)));
      }
      named_bar_sync(1 + qw, 64);
      if (lane == 0) {
        mbar_arrive(&item_empty[slot]);
      }
    }
  }
#ifdef SIVF_TC_PROF
  if (blockIdx.x < 2 && lane == 0)
    printf("blk %d warp %d total %lld | p0 %lld p1 %lld p2 %lld p3 %lld p4 %lld p5 %lld slow %lld ins %lld\n",
           blockIdx.x, warp, clock64() - tstart, pw[0], pw[1], pw[2], pw[3], pw[4], pw[5], pw[6], pw[7]);
#endif
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == W_MMA) tmem_dealloc(tbase, 512);
}


// Seed of the per-query bound gthr[q] on its final k-th distance: exact
// distances from q to the live slots of the first `nseed` live slabs of its
// nearest probed list (probes are sorted, rank 0 first).  Any k real
// candidates bound the final k-th distance from above, so the bound only
// prunes work, never results.  The difference form here and the scan's
// distances may round differently (each within (Dp+2) 2^-24 relative of the
// exact value), so the bound is inflated by (1 + (Dp+2) 2^-23), rounded up.
// Warp per query; lane = slot; slab payload loads are 4 full 128-B lines per chunk.
__global__ void __launch_bounds__(128) k_seed_bound(DevState st, const float* __restrict__ Q, int64_t nq,
                                                    int nprobe, const int32_t* __restrict__ probes, int nseed,
                                                    int k, uint32_t* __restrict__ gthr) {
  __shared__ __align__(16) float qs[4][128];
  __shared__ u64 tops[4][64];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t q = (int64_t)blockIdx.x * 4 + w;
  if (q >= nq) return;  // warp-uniform
  const int Dp = st.Dp, nq4 = Dp >> 2;
  for (int d = lane; d < Dp; d += 32) qs[w][d] = d < st.D ? __ldg(Q + q * st.D + d) : 0.f;
  u64* top = tops[w];
  u64* tmp = top + 32;
  warp_topk_init(top, k);
  const int l = probes[q * nprobe];
  const int len = st.dir_len[l];
  const int32_t* dir = st.dir_arena + st.dir_off[l];
  const float infl = 1.f + (float)(Dp + 2) * 0x1p-23f;
  int used = 0;
  for (int j = 0; j < len && used < nseed; ++j) {
    const int s = dir[j];
    const uint32_t bm = st.bitmap[s];
    if (!bm) continue;
    ++used;
    const float* xs = st.payload + (size_t)s * kSlot * Dp;
    const float4* q4 = reinterpret_cast<const float4*>(qs[w]);
    float acc = 0.f;
#pragma unroll 8
    for (int c4 = 0; c4 < nq4; ++c4) {
      const float4 xv = __ldg(reinterpret_cast<const float4*>(xs + pay_off(Dp, lane, c4)));
      const float4 qv = q4[c4];
      float t;
      t = qv.x - xv.x; acc = fmaf(t, t, acc);
      t = qv.y - xv.y; acc = fmaf(t, t, acc);
      t = qv.z - xv.z; acc = fmaf(t, t, acc);
      t = qv.w - xv.w; acc = fmaf(t, t, acc);
    }
    const bool valid = (bm >> lane) & 1u;
    warp_topk_insert(top, tmp, k, valid ? make_key(__fmul_ru(acc, infl), st.slab_ids[(size_t)s * kSlot + lane])
                                        : kPadKey);
  }
  const u64 kth = top[k - 1];
  if (lane == 0 && kth != kPadKey) atomicMin(&gthr[q], __float_as_uint(key_dist(kth)));
}

// register top-k width: the insertion network costs O(KP) per survivor
inline int scan_kp(int k) { return k <= 10 ? 10 : k <= 16 ? 16 : 32; }

int tc_stages(const Index& ix, int KP) {
  const size_t sb = tc_plan(ix.st.Dh, 0, KP).stage_bytes;
  const size_t fixed = tc_plan(ix.st.Dh, 0, KP).total;
  if (ix.smem_optin < fixed) return 0;
  int n = (int)((ix.smem_optin - fixed) / sb);
  return n > NB ? NB : n;  // the producer reuses the accumulator barriers: nst <= NB
}

}  // namespace

bool scan_tc_supported(const Index& ix, int k) {
  return ix.st.Dh > 0 && ix.st.Dh <= 128 && k <= 32 && tc_stages(ix, scan_kp(k)) >= 2;
}

cudaError_t setup_scan_tc(Index& ix) {
  if (ix.st.Dh == 0 || ix.st.Dh > 128) return cudaSuccess;
  cudaError_t e = cudaSuccess;
  if (tc_stages(ix, 10) >= 2)
    e = cudaFuncSetAttribute(k_scan_tc<10>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)tc_plan(ix.st.Dh, tc_stages(ix, 10), 10).total);
  if (e == cudaSuccess && tc_stages(ix, 16) >= 2)
    e = cudaFuncSetAttribute(k_scan_tc<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)tc_plan(ix.st.Dh, tc_stages(ix, 16), 16).total);
  if (e == cudaSuccess && tc_stages(ix, 32) >= 2)
    e = cudaFuncSetAttribute(k_scan_tc<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)tc_plan(ix.st.Dh, tc_stages(ix, 32), 32).total);
  return e;
}

cudaError_t launch_scan_tc(Index& ix, const float* d_q, int k, int nprobe, cudaStream_t s, int phase) {
  Scratch& sc = ix.sc;
  const int KP = scan_kp(k);
  const int nst = tc_stages(ix, KP);
  TcArgs a{ix.st, d_q, nprobe, k, nst, sc.inv_pairs, sc.work_l, sc.work_p0, sc.work_n, sc.partial, sc.gthr, phase, ix.dbg};
  const size_t smem = tc_plan(ix.st.Dh, nst, KP).total;
  if (KP == 10) k_scan_tc<10><<<ix.num_sms, TTHREADS, smem, s>>>(a);
  else if (KP == 16) k_scan_tc<16><<<ix.num_sms, TTHREADS, smem, s>>>(a);
  else k_scan_tc<32><<<ix.num_sms, TTHREADS, smem, s>>>(a);
  ix.launches += 1;
  return cudaGetLastError();
}

int scan_tc_tile() { return TM; }

cudaError_t launch_seed_bound(Index& ix, const float* d_q, int64_t nq, int k, int nprobe, cudaStream_t s) {
  if (ix.seed_slabs <= 0 || nq <= 0 || ix.st.Dp > 128 || k > 32) return cudaSuccess;
  k_seed_bound<<<ceil_div(nq, 4), 128, 0, s>>>(ix.st, d_q, nq, nprobe, ix.sc.probes, ix.seed_slabs, k, ix.sc.gthr);
  ix.launches += 1;
  return cudaGetLastError();
}

}  // namespace sivf

#ifdef SIVF_TC_PROF
extern "C" int sivf_debug_scnt(unsigned long long* host, int reset) {
  int rc = (int)cudaMemcpyFromSymbol(host, sivf::g_scnt, sizeof(unsigned long long) * 4);
  if (reset) {
    unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(sivf::g_scnt, z, sizeof(z));
  }
  return rc;
}
extern "C" int sivf_debug_trace(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, sivf::g_tr, sizeof(long long) * 6 * 1024);
}
#endif
