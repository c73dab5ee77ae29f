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
// operand must be K-major SWIZZLE_NONE with a uniform 8-row-group stride.  A
// slab's scan record (rec16_bytes(), written by k_append) is exactly that:
// 4 row groups of [Dh/8][8 slots][8 halves] core matrices, each followed by
// its 8 slots' norms and ids (SBO = 16 Dh + 64 B, LBO = 128 B), so each slab of
// a group is ONE contiguous cp.async.bulk into consecutive stage slots and the
// four together are the N = 128 operand, norms and ids included.  No gather,
// no shared-memory transpose (bulk copies stream 2x faster than TMA
// tile::gather4 from L2, tools/g4_probe.cu).
//
// Roles (1 persistent CTA per SM, 16 warps, no CTA-wide barrier after setup;
// every hand-off is an mbarrier):
//   warp 0      scheduler: claims work items (up to NITEM - 1 ahead, in an
//               item ring) and walks each list's slab directory ahead of
//               the producer, keeping the live slabs (bitmap != 0, Eq.
//               slot_valid at slab granularity) with their flags
//   warp 14     producer: per group of 4 live slabs, lanes 0-3 each issue
//               one bulk copy of a slab record into an nst-stage ring
//               (nst <= MAXST, as many as fit); a stage is refilled once the
//               epilogue of the group that used it is done
//   warp 15     group metadata: once a stage lands, NaN-masks the slot norms
//               in place by the bitmap and computes each slab's max norm
//   warp 1      MMA: one lane issues Dh/16 tcgen05.mma per group into one of
//               NB = 3 TMEM accumulators; one tcgen05.commit per group (each
//               costs ~200 cycles of tensor pipe) signals the epilogue
//   warps 2-5   query loaders: the next item's 128 query rows as fp16 into
//               the spare one of two TMEM A buffers (double-buffered across
//               items), with ||q||^2 (fp32), the integrality and fp16-range
//               flags (QInfo ring: up to NQI items ahead of the epilogue)
//   warps 6-13  epilogue: two sets of 4 warps, set h takes the groups g with
//               g & 1 == h (consecutive groups in flight at once); thread =
//               query row, 4 chunks of 32 columns per group; per chunk,
//               t = ||x||^2 - 2 q.x is one FFMA and the filter one FMNMX per
//               candidate; only chunks whose min passes the row's threshold
//               take the per-lane slow path (exact distance, then a sorted
//               register top-k of (dist, id) keys); the two sets' lists of a
//               row merge at the item's end
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
constexpr int MAXST = 8;  // stage ring depth cap (a stage is freed by the epilogue, not by the MMA commit)
constexpr int NLD = 4, NEPI = 8;
constexpr int W_SCHED = 0, W_MMA = 1, W_LD0 = 2, W_EPI0 = W_LD0 + NLD, W_TMA = W_EPI0 + NEPI, W_META = W_TMA + 1;
constexpr int TTHREADS = 32 * (W_META + 1);
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
            // bit2 skip the MMAs, bit3 skip the B copies, bit4 skip the A loads, bit7 no per-group bound
            // sharing, bit8 the epilogue only waits and frees, bit9 the metadata warp only forwards
};

struct ItemRec {
  int32_t l, p0, nqt;  // l < 0: no more work
  int32_t npre;        // live slabs prefetched into the slot's record array
  int32_t dir_pos;     // directory position where the prefetch stopped (-1: complete)
  int32_t len, pad[2];
};
// Per stage: written by the producer (slab, bm, flag, nvalid, last) before the
// stage's full barrier, and by the meta warp (xnm, xnmax, sxmax) before
// meta_ready.  The masked norms live here, not in the bulk-copied records: no
// generic-proxy write ever touches the async-proxy copy destination.
struct StageMeta {
  float xnm[GN];     // ||x||^2 per slot, NaN where the validity bit is clear
  int32_t slab[GS];  // -1: padding position
  uint32_t bm[GS];
  uint32_t flag[GS];
  float xnmax[GS];   // max ||x||^2 over the slab's valid slots
  float sxmax[GS];   // sqrt(xnmax)
  int32_t nvalid, last, pad[2];
};
struct QInfo {
  float qn;
  int32_t pair;
  uint32_t qint;  // every value an integer with |v| <= 2048 (exact in fp16)
  uint32_t qover; // some |v| > 65504: no finite fp16 copy, every candidate is re-ranked
  float thr0;     // the query's k-th distance bound (gthr) read by the loader: the epilogue
                  // starts the item without a global load on its path (re-read every group)
};

struct TcPlan {
  size_t stage_bytes, off_meta, off_q, off_items, off_thr, off_mrg, off_vst, off_ring, off_bar, total;
};
__host__ __device__ inline TcPlan tc_plan(int Dh, int nst, int KP) {
  TcPlan p;
  p.stage_bytes = ((size_t)GS * rec16_bytes(Dh) + 1023) & ~(size_t)1023;  // GS slab scan records (rec16_bytes)
  p.off_meta = (size_t)nst * p.stage_bytes;
  p.off_q = p.off_meta + MAXST * sizeof(StageMeta);
  p.off_items = p.off_q + NQI * TM * sizeof(QInfo);
  p.off_thr = p.off_items + NITEM * (sizeof(ItemRec) + MAXS * sizeof(uint2));
  p.off_mrg = p.off_thr + 2 * TM * 8;
  p.off_vst = p.off_mrg + (size_t)TM * KP * 8;
  p.off_ring = p.off_vst + (size_t)2 * TM * kSlot * 4;  // slow-path chunk rows [2 sets][TM][32]
  p.off_bar = p.off_ring + 128 * sizeof(uint2);
  p.total = p.off_bar + (3 * MAXST + 2 * NB + 4 + 2 * NQI + 2 * NITEM + 2) * 8 + 1024;  // + alignment slack
  return p;
}

#ifdef SIVF_TC_WATCHDOG
// debug builds: a wait that spins too long reports (block, warp, barrier, parity) and traps
__device__ __forceinline__ void scan_wait(uint64_t* bar, uint32_t phase, int tag) {
  for (long long it = 0;; ++it) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    if (ok) return;
    if (it == (1ll << 22)) {
      printf("scan watchdog: block %d warp %d lane %d tag %d parity %u\n", blockIdx.x, threadIdx.x >> 5,
             threadIdx.x & 31, tag, phase);
      __trap();
    }
  }
}
#define MBW(bar, ph, tag) scan_wait(bar, ph, tag)
#elif defined(SIVF_TC_SLEEPWAIT)
#define MBW(bar, ph, tag) mbar_wait_sleep(bar, ph)
#else
#define MBW(bar, ph, tag) mbar_wait(bar, ph)
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
__device__ __forceinline__ void named_bar_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
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

// Pipeline (one persistent CTA per SM, 16 warps; every hand-off is an mbarrier):
//   group g uses stage g % nst (fp16 payload, slot norms, ids; StageMeta) and
//   TMEM accumulator g % NB.  producer -> full[stage] -> meta warp (NaN mask of
//   the norms by the bitmap, xnmax) -> meta_ready[stage]; MMA warp waits
//   full[stage] + acc_free[acc] -> MMAs -> one commit -> d_full[acc]; the
//   epilogue set g & 1 processes group g (all 128 columns of its rows) while
//   the other set processes g + 1, then both arrive on acc_free and stage_free
//   (the stage is refilled only after its group's epilogue, so the producer
//   can run nst groups ahead of the epilogue, nst up to MAXST).
// CONC: concurrent mode (DevState::conc, NEXT-2): acquire loads of directory entries and
// bitmaps, the async-proxy fence before record copies, L2-coherent payload loads
template <int KP, bool CONC>
__global__ void __launch_bounds__(TTHREADS, 1) k_scan_tc(TcArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const DevState& st = a.st;
  const int Dp = st.Dp, nq4 = Dp >> 2, Dh = st.Dh, nst = a.nst, k = a.k;
  const TcPlan p = tc_plan(Dh, nst, KP);
  StageMeta* smeta = reinterpret_cast<StageMeta*>(smem + p.off_meta);
  QInfo* qinfo = reinterpret_cast<QInfo*>(smem + p.off_q);  // [NQI][TM]
  ItemRec* items = reinterpret_cast<ItemRec*>(smem + p.off_items);
  uint2* irec = reinterpret_cast<uint2*>(items + NITEM);  // [NITEM][MAXS] (slab | flags << 30, bitmap)
  u64* thr_sh = reinterpret_cast<u64*>(smem + p.off_thr);    // [2][TM] (item << 32 | k-th bound bits)
  u64* mrg = reinterpret_cast<u64*>(smem + p.off_mrg);       // [TM][KP] half-list hand-over
  uint32_t* vst = reinterpret_cast<uint32_t*>(smem + p.off_vst);  // [2][TM][32] a slow chunk's raw q.x
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.off_bar);  // [MAXST] producer -> MMA, meta (tx bytes)
  uint64_t* meta_ready = full + MAXST;                             // [MAXST] meta warp -> epilogue
  uint64_t* stage_free = meta_ready + MAXST;                       // [MAXST] epilogue -> producer
  uint64_t* d_full = stage_free + MAXST;                           // [NB] MMA commit -> epilogue
  uint64_t* acc_free = d_full + NB;                                // [NB] epilogue -> MMA
  uint64_t* a_full = acc_free + NB;                                // [2] loaders -> MMA
  uint64_t* a_free = a_full + 2;                                   // [2] MMA commit -> loaders
  uint64_t* q_read = a_free + 2;                                   // [NQI] epilogue -> loaders (QInfo consumed)
  uint64_t* q_full = q_read + NQI;                                 // [NQI] loaders -> epilogue (QInfo written)
  uint64_t* item_full = q_full + NQI;                              // [NITEM] scheduler -> all
  uint64_t* item_empty = item_full + NITEM;                        // [NITEM] epilogue -> scheduler
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(item_empty + NITEM);
  // stage s: GS slab scan records back to back (slab j at j * rbytes)
  auto stage_x = [&](int s) { return smem + (size_t)s * p.stage_bytes; };
  const uint32_t rbytes = (uint32_t)rec16_bytes(Dh), sbo = (uint32_t)rec16_sbo(Dh);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef SIVF_TC_PROF
  long long pw[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const long long tstart = clock64();
#endif
  if (threadIdx.x == 0) {
    for (int i = 0; i < MAXST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&meta_ready[i], 1);
      mbar_init(&stage_free[i], NEPI);
    }
    for (int b = 0; b < NB; ++b) {
      mbar_init(&d_full[b], 1);
      mbar_init(&acc_free[b], NEPI / 2);  // the processing set only (see the epilogue)
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
    // directory -> bitmap -> flag) leave the copy issue path
    const int ntiles = st.sctr[a.phase == 1 ? I_NTILES0 : I_NTILES];
    const unsigned lt = (1u << lane) - 1u;
    for (uint32_t i = 0;; ++i) {
      const int slot = (int)(i % NITEM);
      if (lane == 0) PW(0, MBW(&item_empty[slot], ((i / NITEM) & 1u) ^ 1u, 1));
      int w = 0;
      if (lane == 0) w = atomicAdd(&st.sctr[a.phase == 2 ? I_WORK2 : I_WORK], 1);
      w = __shfl_sync(kFull, w, 0);
      ItemRec r{-1, 0, 0, 0, -1, 0, 0, 0};
      if (w < ntiles) {
        const int l = a.work_l[w];
        const int len = ld_state_s32(&st.dir_len[l], CONC);
        const int32_t* dir = st.dir_arena + st.dir_off[l];
        uint2* rec = irec + slot * MAXS;
        int npre = 0, j0 = 0;
        for (; j0 < len; j0 += 32) {
          const int j = j0 + lane;
          int sl = 0;
          uint32_t bm = 0u;
          if (j < len) {
            sl = ld_state_s32(&dir[j], CONC);
            bm = ld_state_u32(&st.bitmap[sl], CONC);
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
    // lane-parallel: one bulk copy per slab (its whole scan record) by lanes
    // 0..GS-1.  Live slab records go through a 128-entry ring: the item's
    // prefetched records, then (long lists) the rest of its directory; a group
    // is emitted as not-last only while at least one more record follows it
    uint2* pring = reinterpret_cast<uint2*>(smem + p.off_ring);
    const unsigned lt = (1u << lane) - 1u;
    uint32_t gseq = 0;
    auto emit = [&](uint32_t head, int nvalid, int last) {  // records pring[head, head + nvalid)
      const int stg = (int)(gseq % (uint32_t)nst);
      if (lane == 0) PW(1, MBW(&stage_free[stg], ((gseq / (uint32_t)nst) & 1u) ^ 1u, 2));
      if (lane == 0) TR(0, gseq, clock64());
      __syncwarp();
      StageMeta& m = smeta[stg];
      const uint2 r = lane < nvalid ? pring[(head + (uint32_t)lane) & 127u] : make_uint2(0u, 0u);
      const int sl = (int)(r.x & 0x3fffffffu);
      if (lane < GS) {
        m.slab[lane] = lane < nvalid ? sl : -1;
        m.bm[lane] = r.y;
        m.flag[lane] = r.x >> 30;
      }
      if (lane == 0) {
        m.nvalid = nvalid;
        m.last = last;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&full[stg], (a.dbg & 8) ? 0u : (uint32_t)nvalid * rbytes);
      __syncwarp();
      if (CONC) fence_proxy_async_global();  // the bitmap acquire orders the record copies (NEXT-2)
      if (lane < nvalid && !(a.dbg & 8))
        bulk_g2s(stage_x(stg) + (size_t)lane * rbytes, reinterpret_cast<const unsigned char*>(st.payload16) +
                                                           (size_t)sl * rbytes, rbytes, &full[stg]);
      ++gseq;
    };
    for (uint32_t i = 0;; ++i) {
      const int slot = (int)(i % NITEM);
      PW(4, MBW(&item_full[slot], (i / NITEM) & 1u, 3));
      const ItemRec rec = items[slot];
      if (rec.l < 0) break;
      uint32_t head = 0u, tail = 0u;  // warp-uniform ring cursors
      const uint2* rr = irec + slot * MAXS;
      for (int r0 = 0; r0 < rec.npre; r0 += 32)
        if (r0 + lane < rec.npre) pring[(uint32_t)(r0 + lane) & 127u] = rr[r0 + lane];
      tail = (uint32_t)rec.npre;
      __syncwarp();
      while (tail - head > (uint32_t)GS) {
        emit(head, GS, 0);
        head += GS;
      }
      if (rec.dir_pos >= 0) {  // long list: walk the rest of the directory here
        const int32_t* dir = st.dir_arena + st.dir_off[rec.l];
        for (int j0 = rec.dir_pos; j0 < rec.len; j0 += 32) {
          const int j = j0 + lane;
          int sl = 0;
          uint32_t bm = 0u, fl = 0u;
          if (j < rec.len) {
            sl = ld_state_s32(&dir[j], CONC);
            bm = ld_state_u32(&st.bitmap[sl], CONC);
            if (bm) fl = st.slab_flag[sl] & 3u;
          }
          const unsigned live = __ballot_sync(kFull, bm != 0u);
          if (bm) pring[(tail + (uint32_t)__popc(live & lt)) & 127u] = make_uint2((uint32_t)sl | (fl << 30), bm);
          tail += (uint32_t)__popc(live);
          __syncwarp();
          while (tail - head > (uint32_t)GS) {
            emit(head, GS, 0);
            head += GS;
          }
        }
      }
      emit(head, (int)(tail - head), 1);  // 0..GS records (0: the item has no live slab, an empty group)
    }
  } else if (warp == W_META) {
    // ------------------------------------------------------------ group metadata
    // per group, after its copies land: slot norms NaN-masked in place by the
    // validity bitmap (Eq. slot_valid) and the per-slab max ||x||^2 for the
    // epilogue's error bound, off the MMA issue path
    uint32_t gseq = 0;
    for (uint32_t i = 0;; ++i) {
      const int slot = (int)(i % NITEM);
      MBW(&item_full[slot], (i / NITEM) & 1u, 4);
      if (items[slot].l < 0) break;
      for (;;) {
        const int stg = (int)(gseq % (uint32_t)nst);
        PW(0, MBW(&full[stg], (gseq / (uint32_t)nst) & 1u, 5));
        StageMeta& m = smeta[stg];
        const int nv = (a.dbg & 512) ? 0 : m.nvalid;
        const unsigned char* sb = stage_x(stg) + rec16_norm_off(Dh, lane);
        float xn[GS];
        uint32_t mx[GS];
#pragma unroll
        for (int j = 0; j < GS; ++j) {  // loads first, then the reductions: independent chains
          const bool v = j < nv && ((m.bm[j] >> lane) & 1u) != 0u;
          xn[j] = v ? *reinterpret_cast<const float*>(sb + (size_t)j * rbytes) : __int_as_float(0x7fc00000);
        }
#pragma unroll
        for (int j = 0; j < GS; ++j) {
          m.xnm[j * kSlot + lane] = xn[j];
          mx[j] = __reduce_max_sync(kFull, xn[j] == xn[j] ? __float_as_uint(fmaxf(xn[j], 0.f)) : 0u);
        }
        if (lane < GS) {
          const float x = __uint_as_float(lane == 0 ? mx[0] : lane == 1 ? mx[1] : lane == 2 ? mx[2] : mx[3]);
          m.xnmax[lane] = x;
          m.sxmax[lane] = sqrtf(x);
        }
        const int last = m.last;
        __syncwarp();
        if (lane == 0) mbar_arrive(&meta_ready[stg]);
        ++gseq;
        if (last) break;
      }
    }
  } else if (warp == W_MMA) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = umma_idesc_f16(TM, GN);
    uint32_t gseq = 0;
    for (uint32_t i = 0;; ++i) {
      const int slot = (int)(i % NITEM);
      PW(6, MBW(&item_full[slot], (i / NITEM) & 1u, 6));
      const ItemRec rec = items[slot];
      if (rec.l < 0) break;
      const uint32_t ab = i & 1u;
      PW(1, MBW(&a_full[ab], (i >> 1) & 1u, 7));
      for (;;) {
        const int stg = (int)(gseq % (uint32_t)nst);
        const uint32_t b = gseq % NB;
        PW(2, MBW(&full[stg], (gseq / (uint32_t)nst) & 1u, 8));
        const int last = smeta[stg].last, nv = smeta[stg].nvalid;
        PW(3, MBW(&acc_free[b], ((gseq / NB) & 1u) ^ 1u, 9));
        if (lane == 0) TR(1, gseq, clock64());
#ifdef SIVF_TC_PROF
        long long _tm0 = clock64();
#endif
        if (lane == 0) {
          tc_fence_after();
          const uint32_t bsm = smem_u32(stage_x(stg));
          const uint32_t dt = tbase + 128u + b * 128u, at = tbase + ab * 64u;
          // kind::f16: A (fp16 query tile) in TMEM, 8 columns per K = 16 step;
          // B (fp16 slab records) K-major SWIZZLE_NONE, LBO = 128 B, SBO = 16 Dh + 64 B
          const int nk = ((a.dbg & 4) || nv == 0) ? 0 : (Dh >> 4);
          for (int kk = 0; kk < nk; ++kk)
            umma_f16_ts(dt, at + (uint32_t)(8 * kk), umma_sdesc(bsm + (uint32_t)kk * 256u, 128u, sbo),
                        idesc, kk > 0 ? 1u : 0u);
          umma_commit(&d_full[b]);  // accumulator ready (one commit per group)
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
      MBW(&item_full[slot], (i / NITEM) & 1u, 10);
      const ItemRec rec = items[slot];
      if (rec.l < 0) break;
      const uint32_t ab = i & 1u;
      // TMEM lane 32 qw + lane holds the item's row 4 lane + qw: a partial tile's rows
      // spread over the four lane quarters (the epilogue warps share its work evenly)
      const int trow = 4 * lane + qw;
      const bool rv = trow < rec.nqt;
      const bool wv = qw < rec.nqt && !(a.dbg & 16);  // warp-uniform: the warp has a real row
      const int pair = rv ? a.inv_pairs[rec.p0 + trow] : -1;
      const uint32_t thr0 = rv ? __ldcg(a.gthr + pair / a.nprobe) : 0xFF800000u;  // consumed at the QInfo write
      const float* qr = a.Q + (int64_t)(rv ? pair / a.nprobe : 0) * st.D;
      const uint32_t ta = tbase + ((uint32_t)(32 * qw) << 16) + ab * 64u;
      float nrm = 0.f;
      uint32_t integ = 1u, over = 0u;
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
          PW(4, MBW(&a_free[ab], ((i >> 1) & 1u) ^ 1u, 11));
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
      tmem_st_wait();
      const int qb = (int)(i % NQI);
      PW(5, MBW(&q_read[qb], ((i / NQI) & 1u) ^ 1u, 12));  // item i - NQI's QInfo has been read
      qinfo[qb * TM + row] = QInfo{nrm, pair, integ, over, __uint_as_float(thr0)};
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&a_full[ab]);
        mbar_arrive(&q_full[qb]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // two sets of 4 warps; set h processes the groups g with g & 1 == h, thread
    // = query row, all 4 slabs (128 columns) of the group: the two sets work
    // on consecutive groups concurrently.  Each set keeps its own per-row
    // top-k (merged at the item's end) and the two share their k-th distance
    // bounds through shared memory every group
    const int qw = warp & 3, row = 32 * qw + lane, h = (warp - W_EPI0) >> 2;
    // certified band of the fp16 filter (u = 2^-11, RN): eps1 bounds the
    // relative error of q.x from the operand roundings (2u + u^2 <= 2^-9 +
    // 2^-19, tf32-safe margin kept) and fp32 accumulation (Dh 2^-23); esub the
    // absolute error of fp16 subnormals (|v| < 2^-14: error <= 2^-25 per value,
    // sum <= 2^-25 sqrt(Dh) (||q|| + ||x||)), times 2 for d and 2 for safety
    const float eps1 = 0x1p-9f + 0x1p-19f + (float)Dh * 0x1p-23f;
    const float eps2 = (float)(2 * Dp + 10) * 0x1p-24f;
    const float esub = 0x1p-23f * 1.001f * sqrtf((float)Dh);
    const int dbg = a.dbg;
    uint32_t gseq = 0;
    // item-end hand-over of a row's list between the sets: barrier 1 + qw (h = 1's list
    // is in mrg) and 5 + qw (h = 0 has consumed mrg); each side only waits for the
    // other's arrival, so h = 1 goes on to its next item while h = 0 merges
    if (h == 0) named_bar_arrive(5 + qw, 64);  // mrg starts free
    for (uint32_t i = 0;; ++i) {
      const int slot = (int)(i % NITEM);
      PW(4, MBW(&item_full[slot], (i / NITEM) & 1u, 13));
      const ItemRec rec = items[slot];
      if (rec.l < 0) break;
      PW(1, MBW(&q_full[i % NQI], (i / NQI) & 1u, 14));
      const QInfo qi = qinfo[(i % NQI) * TM + row];
      __syncwarp();
      if (lane == 0) mbar_arrive(&q_read[i % NQI]);
      const bool rv = 4 * lane + qw < rec.nqt;  // the item's row 4 lane + qw (see the loaders)
      const bool wact = qw < rec.nqt;
      const int qglob = rv ? qi.pair / a.nprobe : 0;
      const float qn = qi.qn, sqn = sqrtf(qn);
      float thr = rv ? qi.thr0 : -INFINITY;
      // the current bound, read now: consumed at the first group (after its barrier
      // waits), fresher than the loader's copy
      float gnext = rv ? __uint_as_float(__ldcg(a.gthr + qglob)) : thr, tpub = thr;
      u64 keys[KP];
#pragma unroll
      for (int t = 0; t < KP; ++t) keys[t] = t < KP - k ? 0ull : kPadKey;  // k-th = keys[KP-1]
      u64 kth = kPadKey;
      for (;;) {
        const uint32_t b = gseq % NB;
        const int stg = (int)(gseq % (uint32_t)nst);
        const bool mine = (gseq & 1u) == (uint32_t)h;
        PW(5, MBW(&meta_ready[stg], (gseq / (uint32_t)nst) & 1u, 15));
        const StageMeta& m = smeta[stg];
        const int last = m.last;
        if (mine) {
          PW(6, MBW(&d_full[b], (gseq / NB) & 1u, 16));
          if (lane == 0 && warp == W_EPI0 + 2) TR(3, gseq, clock64());
          tc_fence_after();
          const int nv = m.nvalid;
          if (wact && nv > 0 && !(dbg & 256)) {
#ifdef SIVF_TC_PROF
            long long _tb = clock64();
#endif
            const u64 ps = thr_sh[(1 - h) * TM + row];  // other set's bound, tagged with its item
            if ((uint32_t)(ps >> 32) == i) thr = fminf(thr, __uint_as_float((uint32_t)ps));
            thr = fminf(thr, gnext);  // other items of the same query (read one group ago)
            if (rv && !(dbg & 128)) gnext = __uint_as_float(__ldcg(a.gthr + qglob));
            const unsigned char* sbase = stage_x(stg);
#ifdef SIVF_TC_PROF
            __syncwarp();
            if (thr == 12345.f) pw[7] += 1;  // consume thr: the wait on the bound loads is timed here
            pw[8] += clock64() - _tb;
#endif
            // one chunk = one slab = 32 TMEM columns of this row
            auto chunk = [&](const int j, const uint32_t(&v)[32]) {
              const unsigned char* rb = sbase + (size_t)j * rbytes;  // slab j's record
              const uint32_t fl = m.flag[j];
              const float sxm = m.sxmax[j];
              const float rs = sqn + sxm;
              const bool ex = qi.qint != 0u && (fl & kFlagIntegral) != 0u && rs * rs < 16000000.f;
              // no finite fp16 copy of the query or the slab: every valid slot is re-ranked exactly
              const bool unsafe = qi.qover != 0u || (fl & kFlagF16Over) != 0u;
              float E = 0.f;
              if (!ex) {
                const float xm = m.xnmax[j];
                const float cs = sqn * sxm;
                E = 2.f * (2.f * eps1 * cs + eps2 * (qn + xm + 2.f * cs)) + esub * rs;
              }
              float tadj = ex ? __fsub_ru(thr, qn) : __fadd_ru(__fsub_ru(thr, qn), E);
              // norms of slots 4 c4 .. 4 c4 + 3, NaN where the slot is not valid
              const float4* xq = reinterpret_cast<const float4*>(m.xnm + kSlot * j);
              auto x4 = [&](int c4) { return xq[c4]; };
              float m8[8];
#pragma unroll
              for (int c4 = 0; c4 < 8; ++c4) {
                const float4 xx = x4(c4);
                const float t0 = fmaf(-2.f, __uint_as_float(v[4 * c4 + 0]), xx.x);
                const float t1 = fmaf(-2.f, __uint_as_float(v[4 * c4 + 1]), xx.y);
                const float t2 = fmaf(-2.f, __uint_as_float(v[4 * c4 + 2]), xx.z);
                const float t3 = fmaf(-2.f, __uint_as_float(v[4 * c4 + 3]), xx.w);
                m8[c4] = fminf(fminf(t0, t1), fminf(t2, t3));
              }
              const float mn = fminf(fminf(fminf(m8[0], m8[1]), fminf(m8[2], m8[3])),
                                     fminf(fminf(m8[4], m8[5]), fminf(m8[6], m8[7])));
              if (!unsafe && (!(mn <= tadj) || (dbg & 1))) return;
              // slow path (per lane): survivors of this slab, exact distance, register top-k
#ifdef SIVF_TC_PROF
              long long _ts = clock64();
              SCNT_ADD(&g_scnt[0], 1ull);
              const bool cold = !(thr < INFINITY);
#endif
              // the chunk's 32 raw products to this thread's shared row (16-B quads
              // XOR-swizzled by the row: conflict-free), read back per survivor
              uint32_t* vrow = vst + (size_t)(h * TM + row) * kSlot;
#pragma unroll
              for (int c4 = 0; c4 < 8; ++c4)
                *reinterpret_cast<uint4*>(vrow + 4 * (c4 ^ (row & 7))) =
                    make_uint4(v[4 * c4], v[4 * c4 + 1], v[4 * c4 + 2], v[4 * c4 + 3]);
              uint32_t pm = 0u;
              if (unsafe) {
                pm = m.bm[j];  // every valid slot
              } else {
#pragma unroll
                for (int c4 = 0; c4 < 8; ++c4) {
                  if (!(m8[c4] <= tadj)) continue;  // the quad's minimum already fails
                  const float4 xx = x4(c4);
                  pm |= (fmaf(-2.f, __uint_as_float(v[4 * c4 + 0]), xx.x) <= tadj ? 1u : 0u) << (4 * c4);
                  pm |= (fmaf(-2.f, __uint_as_float(v[4 * c4 + 1]), xx.y) <= tadj ? 1u : 0u) << (4 * c4 + 1);
                  pm |= (fmaf(-2.f, __uint_as_float(v[4 * c4 + 2]), xx.z) <= tadj ? 1u : 0u) << (4 * c4 + 2);
                  pm |= (fmaf(-2.f, __uint_as_float(v[4 * c4 + 3]), xx.w) <= tadj ? 1u : 0u) << (4 * c4 + 3);
                }
              }
#ifdef SIVF_TC_PROF
              SCNT_ADD(&g_scnt[1], (unsigned long long)__popc(pm));
#endif
              while (pm) {
                const int c = __ffs(pm) - 1;
                pm &= pm - 1;
                // independent shared loads first: product, norm, id
                const uint32_t pv = vrow[4 * ((c >> 2) ^ (row & 7)) + (c & 3)];
                const float xn = m.xnm[kSlot * j + c];
                const uint32_t cid = *reinterpret_cast<const uint32_t*>(rb + rec16_id_off(Dh, c));
                const float t = fmaf(-2.f, __uint_as_float(pv), xn);
                if (!unsafe && !(t <= tadj)) continue;  // the threshold may have tightened
                float d;
                if (ex) {
                  d = qn + t;  // exact: every term an integer < 2^24
                } else {
                  const float* xs = st.payload + (size_t)m.slab[j] * kSlot * Dp;
                  const float* qr = a.Q + (int64_t)qglob * st.D;
                  float acc = 0.f;
                  for (int i4 = 0; i4 < nq4; ++i4) {
                    const float4* xp = reinterpret_cast<const float4*>(xs + pay_off(Dp, c, i4));
                    // concurrent mode: L2-coherent loads (a texture-cache line read earlier in
                    // this launch may predate the slot's publication)
                    const float4 xv = CONC ? __ldcg(xp) : __ldg(xp);
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
                const u64 key = make_key(d, cid);
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
                if (cold) SCNT_ADD(&g_scnt[3], 1ull);
#endif
              }
#ifdef SIVF_TC_PROF
              pw[2] += clock64() - _ts;
#endif
            };
            const uint32_t dcol = tbase + ((uint32_t)(32 * qw) << 16) + 128u + b * 128u;
#ifdef SIVF_TC_PROF
            long long _tg = clock64();
#endif
#pragma unroll 1
            for (int j = 0; j < nv; ++j) {
              uint32_t v[32];
              tmem_ld32(dcol + 32u * (uint32_t)j, v);
              tmem_ld_wait();
              if (!(dbg & 2)) chunk(j, v);
            }
#ifdef SIVF_TC_PROF
            pw[0] += clock64() - _tg;
#endif
            thr_sh[h * TM + row] = ((u64)i << 32) | __float_as_uint(thr);
            if (rv && thr < tpub && !(dbg & 128)) {  // share the bound with the query's other items right away
              atomicMin(a.gthr + qglob, __float_as_uint(thr));
              tpub = thr;
            }
          }
          if (lane == 0 && warp == W_EPI0 + 2) TR(4, gseq, clock64());
          tc_fence_before();
          __syncwarp();
          // only the processing set frees the accumulator: an early arrival of
          // the other set could land in the previous phase of the barrier (its
          // arrival for group g is not ordered after the completion of g - NB)
          if (lane == 0) mbar_arrive(&acc_free[b]);
        }
        __syncwarp();
        // both sets free the stage, each after reading its metadata: every
        // arrival for group g follows meta_ready(g), hence the refill for g,
        // hence the completion of the stage's phase for g - nst
        if (lane == 0) mbar_arrive(&stage_free[stg]);
        ++gseq;
        if (last) break;
      }
#ifdef SIVF_TC_PROF
      long long _te = clock64();
#endif
      // merge the two sets' lists of each row: h = 1 hands its list over in smem
      if (h == 1) {
        named_bar_sync(5 + qw, 64);  // the previous item's list has been merged
        if (rv) {
#pragma unroll
          for (int t = 0; t < KP; ++t) mrg[row * KP + t] = keys[t];
        }
        named_bar_arrive(1 + qw, 64);
      } else {
        PW(3, named_bar_sync(1 + qw, 64));
      }
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
      if (h == 0) named_bar_arrive(5 + qw, 64);  // mrg consumed
      if (lane == 0) {
        mbar_arrive(&item_empty[slot]);
      }
#ifdef SIVF_TC_PROF
      pw[9] += clock64() - _te;
#endif
    }
    if (h == 1) named_bar_sync(5 + qw, 64);  // h = 0's last "mrg consumed" arrival
  }
#ifdef SIVF_TC_PROF
  if (blockIdx.x < 2 && lane == 0)
    printf("blk %d warp %d total %lld | p0 %lld p1 %lld p2 %lld p3 %lld p4 %lld p5 %lld p6 %lld ins %lld p8 %lld p9 %lld\n",
           blockIdx.x, warp, clock64() - tstart, pw[0], pw[1], pw[2], pw[3], pw[4], pw[5], pw[6], pw[7], pw[8], pw[9]);
#endif
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == W_MMA) tmem_dealloc(tbase, 512);
}


// Per-list seed of the per-query bound (SIVF_OPT_SEED_LIST): block per list l;
// the first live slab of l holding >= k valid slots is staged once in shared
// memory, and every query whose NEAREST probed list is l (its rank-0 pair, found in
// the inverse map's entry l) gets the k-th smallest of its exact distances to
// those slots.  Any k real candidates bound the final k-th distance from above,
// so this prunes work only, never results.  The distances are the scan's exact
// re-rank form (fp32 differences, fmaf squares; on integer data it and
// ||q||^2 + t are exact) summed in four interleaved partial sums: two orders of a
// sum of D non-negative terms differ by at most D 2^-23 relative, so the k-th value
// is inflated by (1 + (Dp+2) 2^-23), rounded up, and bounds the scan's own values
// of those k candidates.  One slab per list (~10 queries
// each at SIFT1M / nprobe 32) instead of one per query: ~100x fewer payload bytes
// than k_seed_bound.
__global__ void __launch_bounds__(256) k_seed_list(DevState st, const float* __restrict__ Q, int nprobe, int k,
                                                   const int32_t* __restrict__ inv_off,
                                                   const int32_t* __restrict__ inv_cnt,
                                                   const int32_t* __restrict__ inv_pairs, uint32_t* __restrict__ gthr) {
  __shared__ float xs[kSlot][129];  // Dp <= 128 (+1: conflict-free rows)
  __shared__ float qs[8][128];
  __shared__ int32_t q0[256];
  __shared__ int s_slab, s_n0;
  __shared__ uint32_t s_bm;
  const int l = blockIdx.x, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cnt = inv_cnt[l];
  if (cnt == 0) return;  // block-uniform
  const int Dp = st.Dp;
  if (threadIdx.x == 0) s_n0 = 0;
  __syncthreads();
  if (w == 0) {  // the list's first live slab with >= k valid slots (beside the pair scan)
    const int len = st.dir_len[l];
    const int32_t* dir = st.dir_arena + st.dir_off[l];
    int slab = -1;
    uint32_t bmf = 0u;
    for (int j0 = 0; j0 < len && slab < 0; j0 += 32) {
      const int j = j0 + lane;
      int sl = 0;
      uint32_t bm = 0u;
      if (j < len) {
        sl = dir[j];
        bm = st.bitmap[sl];
      }
      const unsigned ok = __ballot_sync(kFull, __popc(bm) >= k);
      if (ok) {
        const int src = __ffs(ok) - 1;
        slab = __shfl_sync(kFull, sl, src);
        bmf = __shfl_sync(kFull, bm, src);
      }
    }
    if (lane == 0) {
      s_slab = slab;
      s_bm = bmf;
    }
  } else {  // the queries whose nearest probed list is l (rank-0 pairs of entry l)
    const int off = inv_off[l];
    for (int i = threadIdx.x - 32; i < cnt; i += blockDim.x - 32) {
      const int p = inv_pairs[off + i];
      if (p % nprobe == 0) {
        const int pos = atomicAdd(&s_n0, 1);
        if (pos < 256) q0[pos] = p / nprobe;
      }
    }
  }
  __syncthreads();
  const int slab = s_slab;
  if (s_n0 == 0 || slab < 0) return;  // block-uniform (e.g. no query starts here at nlist 16384)
  const int n0 = min(s_n0, 256);
  // each warp's first query row is fetched together with the slab (two DRAM round
  // trips overlapped instead of chained)
  if (w < n0)
    for (int d = lane; d < Dp; d += 32) qs[w][d] = d < st.D ? __ldg(Q + (int64_t)q0[w] * st.D + d) : 0.f;
  const float* xsrc = st.payload + (size_t)slab * kSlot * Dp;
  for (int i = threadIdx.x; i < kSlot * (Dp >> 2); i += blockDim.x) {
    const int n = i & 31, c4 = i >> 5;
    const float4 v = __ldg(reinterpret_cast<const float4*>(xsrc + pay_off(Dp, n, c4)));
    xs[n][4 * c4] = v.x, xs[n][4 * c4 + 1] = v.y, xs[n][4 * c4 + 2] = v.z, xs[n][4 * c4 + 3] = v.w;
  }
  __syncthreads();
  const uint32_t bm = s_bm;
  const float infl = 1.f + (float)(Dp + 2) * 0x1p-23f;
  for (int t = w; t < n0; t += 8) {
    const int q = q0[t];
    if (t != w)  // (the first one is already staged)
      for (int d = lane; d < Dp; d += 32) qs[w][d] = d < st.D ? __ldg(Q + (int64_t)q * st.D + d) : 0.f;
    __syncwarp();
    // four independent partial sums (any order: the inflation below covers the
    // reordering against the scan's sequential sum, (Dp+2) 2^-23 relative)
    float a4[4] = {0.f, 0.f, 0.f, 0.f};
    for (int d = 0; d < Dp; d += 4) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float tt = qs[w][d + e] - xs[lane][d + e];
        a4[e] = fmaf(tt, tt, a4[e]);
      }
    }
    const float acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
    const uint32_t key = ((bm >> lane) & 1u) ? __float_as_uint(acc) : 0x7f800000u;  // >= 0: bit order
    // the k-th smallest over the 32 slots: bitonic sort of the keys across the warp
    uint32_t v = key;
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1)
#pragma unroll
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        const uint32_t o = __shfl_xor_sync(kFull, v, stride);
        const bool up = (lane & size) == 0 || size == 32, lower = (lane & stride) == 0;
        v = (lower == up) ? min(v, o) : max(v, o);
      }
    const uint32_t kth = __shfl_sync(kFull, v, k - 1);
    if (lane == 0 && kth < 0x7f800000u) atomicMin(gthr + q, __float_as_uint(__fmul_ru(__uint_as_float(kth), infl)));
    __syncwarp();
  }
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
  if (ix.tc_max_stages > 0 && n > ix.tc_max_stages) n = ix.tc_max_stages;  // experiments (SIVF_OPT_TC_STAGES)
  return n > MAXST ? MAXST : n;
}

}  // namespace

bool scan_tc_supported(const Index& ix, int k) {
  return ix.st.Dh > 0 && ix.st.Dh <= 128 && k <= 32 && tc_stages(ix, scan_kp(k)) >= 2;
}

cudaError_t setup_scan_tc(Index& ix) {
  if (ix.st.Dh == 0 || ix.st.Dh > 128) return cudaSuccess;
  cudaError_t e = cudaSuccess;
#define SIVF_TC_ATTR(KPV)                                                                                   \
  if (e == cudaSuccess && tc_stages(ix, KPV) >= 2) {                                                        \
    const int sm = (int)tc_plan(ix.st.Dh, tc_stages(ix, KPV), KPV).total;                                   \
    e = cudaFuncSetAttribute(k_scan_tc<KPV, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);       \
    if (e == cudaSuccess)                                                                                   \
      e = cudaFuncSetAttribute(k_scan_tc<KPV, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);      \
  }
  SIVF_TC_ATTR(10)
  SIVF_TC_ATTR(16)
  SIVF_TC_ATTR(32)
#undef SIVF_TC_ATTR
  return e;
}

cudaError_t launch_scan_tc(Index& ix, const float* d_q, int k, int nprobe, cudaStream_t s, int phase) {
  Scratch& sc = ix.sc;
  const int KP = scan_kp(k);
  const int nst = tc_stages(ix, KP);
  TcArgs a{ix.st, d_q, nprobe, k, nst, sc.inv_pairs, sc.work_l, sc.work_p0, sc.work_n, sc.partial, sc.gthr, phase, ix.dbg};
  const size_t smem = tc_plan(ix.st.Dh, nst, KP).total;
  const bool conc = ix.st.conc != 0;
  if (KP == 10) {
    if (conc) k_scan_tc<10, true><<<ix.num_sms, TTHREADS, smem, s>>>(a);
    else k_scan_tc<10, false><<<ix.num_sms, TTHREADS, smem, s>>>(a);
  } else if (KP == 16) {
    if (conc) k_scan_tc<16, true><<<ix.num_sms, TTHREADS, smem, s>>>(a);
    else k_scan_tc<16, false><<<ix.num_sms, TTHREADS, smem, s>>>(a);
  } else {
    if (conc) k_scan_tc<32, true><<<ix.num_sms, TTHREADS, smem, s>>>(a);
    else k_scan_tc<32, false><<<ix.num_sms, TTHREADS, smem, s>>>(a);
  }
  ix.launches += 1;
  return cudaGetLastError();
}

int scan_tc_tile() { return TM; }

cudaError_t launch_seed_bound(Index& ix, const float* d_q, int64_t nq, int k, int nprobe, cudaStream_t s) {
  // (only with >= 4 queries per list on average: a block per list must amortise its
  // directory walk and slab load; the sliding step's 1k queries or nlist 16384 do not)
  if (ix.seed_list && nq >= 4 * (int64_t)ix.st.nlist && ix.st.Dp <= 128 && k <= 32 && !ix.st.conc) {
    k_seed_list<<<ix.st.nlist, 256, 0, s>>>(ix.st, d_q, nprobe, k, ix.sc.inv_off, ix.sc.inv_cnt, ix.sc.inv_pairs,
                                            ix.sc.gthr);
    ix.launches += 1;
  }
  if (ix.seed_slabs <= 0 || nq <= 0 || ix.st.Dp > 128 || k > 32) return cudaGetLastError();
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
