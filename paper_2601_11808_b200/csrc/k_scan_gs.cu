// k_scan_gs.cu — slab scan for D > 128 (the GIST1M-shaped configuration, any k)
// on the 5th-generation tensor cores.
//
// Eq. l2 for a work item (list l x a tile of <= 128 queries
// probing l) is a dense contraction: d(q, x) = ||q||^2 + ||x||^2 - 2 q.x.  For
// D > 128 neither the query tile nor a group of slabs fits on chip at once, so
// this is a K-chunked GEMM: per group of 4 live slabs (N = 128 slots) the
// 64-dim chunks of the query tile (A) and of the slabs (B) stream through a
// 3-stage shared-memory ring and accumulate in TMEM (kind::f16 M = 128,
// N = 128, K = 16 per instruction, A and B from shared memory).
//
// Precision (BASELINE.json: distances within 1e-4 relative, ids equal except
// near-ties): both operands are split fp16 -- x 2^e = hi + lo per vector
// (k_append, recg_off(); the query tile likewise, k_gs_prep) -- and
// q.x = 2^-(e_q + e_x) (qh.xh + qh.xl + ql.xh): three MMAs per K step, the
// dropped ql.xl term and the roundings of the low parts are ~2^-22 |q| |x|,
// the fp32 accumulation (D + 2) 2^-24 sum |q_i x_i| (~1e-6 relative on
// GIST-shaped data, where ||q||^2 + ||x||^2 is a few times d).  The fp32
// payload stays the source of truth (C35); this copy is derived from it.
//
// Selection: the epilogue writes each (query, probed list) row of distances
// (invalid slots +inf, Eq. slot_valid) into a dense buffer; k_gs_select then
// takes each query's top-k over its nprobe rows (warp per query, P:353-355
// with the merge fused).  Items whose rows do not fit the buffer (lists far
// longer than average) take k_gs_fallback (CUDA cores, per-pair top-k) and
// k_gs_select merges those pairs' partial lists instead.
//
// Roles (1 persistent CTA per SM, 6 warps, every hand-off an mbarrier):
//   warp 0     producer: claims items, walks the list's directory (live slabs
//              only, their ids into the item's header in the dense buffer),
//              per group: the slots' norms and scales into the metadata ring,
//              per chunk: one 32-KB bulk copy of the A chunk (hi | lo) and one
//              2-KB copy per (slab, row group) of the B chunk (hi | lo)
//   warp 1     MMA: 4 K steps x 3 MMAs per chunk, a commit per chunk frees
//              the stage, a commit per group fills one of 2 accumulators
//   warps 2-5  epilogue: thread = query row; d = ||q||^2 + ||x||^2 - 2 s q.x
//              per slot, 128 B stores of each slab's 32 distances
#include <cuda.h>
#include <cuda_fp16.h>

#include "sivf_host.h"

namespace sivf {

namespace {

constexpr int GQ = 128;          // queries per work item (UMMA M)
constexpr int GG = 8;            // slabs per group (UMMA N = 256: each streamed A chunk serves 8 slabs)
constexpr int NSTG = 4;          // stage ring depth
constexpr int NBG = 2;           // TMEM accumulators (GN = 256 columns each)
constexpr int GN = GG * 32;      // columns per group
constexpr int NGM = 4;           // group metadata ring
constexpr int ACH = GQ * kGsKch * 4;  // A chunk bytes: 128 rows x 32 dims x 2 B x (hi, lo)
constexpr int BPS = kGsKch * 128;       // B chunk bytes per slab: 4 row groups x [hi | lo] pieces
constexpr int STG = ACH + GG * BPS;  // stage: A chunk + B chunk (8 slabs x 4 row groups x 1 KB)
constexpr int GS_THREADS = 6 * 32;

struct GsMeta {
  float xn[GG * kSlot];  // ||x||^2 per slot (bulk copy of slab_norm)
  float xs[GG * kSlot];  // 2^-e_x per slot (bulk copy of slab_xs)
  int32_t slab[GG];
  uint32_t bm[GG];
  int32_t item, pos0, nv, pad;  // item < 0: no more work; pos0: live position of the group's first slab
};

struct GsArgs {
  DevState st;
  const float* Q;
  int nprobe, k;
  const int32_t* inv_pairs;
  const int32_t* work_l;
  const int32_t* work_p0;
  const int32_t* work_n;
  const uint16_t* gs_a;
  const float* gs_qn;
  const float* gs_qs;
  const int64_t* doff;
  const int32_t* dlen;
  int32_t* nlive;
  float* dense;
};

__host__ __device__ inline int64_t gs_hdr(int dlen) { return (int64_t)((dlen + 3) & ~3); }

constexpr size_t kGsSmem = (size_t)NSTG * STG + NGM * sizeof(GsMeta) + 128 * 8 + (2 * NSTG + 2 * NBG + 2 * NGM) * 8 +
                           16 + 1024;

// Per work item (list, <= 128 queries), in order: its region of the dense
// buffer (the live slabs' ids, then one row of 32 dlen distances per query;
// dlen = the list's directory length now) or -1 when it does not fit.
__global__ void __launch_bounds__(1024) k_gs_offsets(DevState st, const int32_t* __restrict__ work_l,
                                                     const int32_t* __restrict__ work_n, int64_t cap,
                                                     int64_t* __restrict__ doff, int32_t* __restrict__ dlen) {
  __shared__ int64_t ws[32];
  __shared__ int64_t carry;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int ntiles = st.sctr[I_NTILES];
  if (t == 0) carry = 0;
  __syncthreads();
  for (int i0 = 0; i0 < ntiles; i0 += 1024) {
    const int i = i0 + t;
    int dl = 0;
    int64_t sz = 0;
    if (i < ntiles) {
      dl = ld_state_s32(&st.dir_len[work_l[i]], st.conc);
      sz = gs_hdr(dl) + (int64_t)work_n[i] * kSlot * dl;
    }
    int64_t v = sz;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t a = __shfl_up_sync(kFull, v, o);
      if (lane >= o) v += a;
    }
    if (lane == 31) ws[w] = v;
    __syncthreads();
    if (w == 0) {
      int64_t x = ws[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t a = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += a;
      }
      ws[lane] = x;
    }
    __syncthreads();
    if (i < ntiles) {
      const int64_t off = carry + (w ? ws[w - 1] : 0) + v - sz;
      doff[i] = off + sz <= cap ? off : -1;
      dlen[i] = dl;
    }
    __syncthreads();
    if (t == 0) carry += ws[31];
    __syncthreads();
  }
}

// Split-fp16 copy of each query, once per query (its work items gather it below):
// x 2^e = hi + lo (e from the row's largest |v|, as k_append does for the slabs),
// ||q||^2 and 2^-e_q.  Warp per query.
__global__ void __launch_bounds__(256) k_gs_qsplit(DevState st, const float* __restrict__ Q, int64_t nq,
                                                   uint16_t* __restrict__ qh, uint16_t* __restrict__ ql,
                                                   float* __restrict__ qqn, float* __restrict__ qqs) {
  const int lane = threadIdx.x & 31;
  const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (q >= nq) return;  // warp-uniform
  const float* qr = Q + q * st.D;
  const int Dg = st.Dg;
  float mx = 0.f, nrm = 0.f;
  for (int d = lane; d < st.D; d += 32) {
    const float v = __ldg(qr + d);
    mx = fmaxf(mx, fabsf(v));
    nrm = fmaf(v, v, nrm);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
    nrm += __shfl_xor_sync(kFull, nrm, o);
  }
  int e = 0;
  if (mx > 0.f && mx <= 3.4e38f) {
    int ex;
    frexpf(mx, &ex);
    e = 15 - ex;
    e = e < -120 ? -120 : e > 120 ? 120 : e;
  }
  if (lane == 0) {
    qqn[q] = nrm;
    qqs[q] = ldexpf(1.f, -e);
  }
  for (int d = 2 * lane; d < Dg; d += 64) {
    const float s0 = ldexpf(d < st.D ? __ldg(qr + d) : 0.f, e), s1 = ldexpf(d + 1 < st.D ? __ldg(qr + d + 1) : 0.f, e);
    const __half h0 = __float2half_rn(s0), h1 = __float2half_rn(s1);
    const __half l0 = __float2half_rn(s0 - __half2float(h0)), l1 = __float2half_rn(s1 - __half2float(h1));
    *reinterpret_cast<__half2*>(qh + q * Dg + d) = __halves2half2(h0, h1);
    *reinterpret_cast<__half2*>(ql + q * Dg + d) = __halves2half2(l0, l1);
  }
}

// Split-fp16 query tile of each dense work item: A[item][chunk] = [hi: 16 row
// groups x K-cores x 8 rows x 8 halves][lo: same] (K-major SWIZZLE_NONE,
// LBO = 128 B, SBO = K-cores x 128 B), gathered from the per-query split copies
// (16-B K-cores), and ||q||^2, 2^-e_q per row.  Rows >= nqt are not written (their
// accumulator rows are never read).  Thread = row: the warp's stores of one K-core
// are 4 contiguous 128-B core matrices.
__global__ void __launch_bounds__(GQ) k_gs_prep(GsArgs a, uint16_t* __restrict__ gs_a, float* __restrict__ gs_qn,
                                                float* __restrict__ gs_qs, const uint16_t* __restrict__ qh,
                                                const uint16_t* __restrict__ ql, const float* __restrict__ qqn,
                                                const float* __restrict__ qqs) {
  const DevState& st = a.st;
  const int ntiles = st.sctr[I_NTILES];
  const int row = threadIdx.x, Dg = st.Dg, nch = Dg / kGsKch;
  constexpr int KC8 = kGsKch / 8;  // K-cores per chunk
  for (int w = blockIdx.x; w < ntiles; w += gridDim.x) {
    if (a.doff[w] < 0 || row >= a.work_n[w]) continue;
    const int q = a.inv_pairs[a.work_p0[w] + row] / a.nprobe;
    gs_qn[(size_t)w * GQ + row] = qqn[q];
    gs_qs[(size_t)w * GQ + row] = qqs[q];
    const uint4* sh = reinterpret_cast<const uint4*>(qh + (size_t)q * Dg);
    const uint4* sl = reinterpret_cast<const uint4*>(ql + (size_t)q * Dg);
    unsigned char* A = reinterpret_cast<unsigned char*>(gs_a) + (size_t)w * nch * ACH + (row >> 3) * (KC8 * 128) +
                       (row & 7) * 16;
#pragma unroll 4
    for (int c8 = 0; c8 < (Dg >> 3); ++c8) {
      const uint4 hv = __ldg(sh + c8), lv = __ldg(sl + c8);
      unsigned char* p = A + (size_t)(c8 / KC8) * ACH + (c8 % KC8) * 128;
      *reinterpret_cast<uint4*>(p) = hv;
      *reinterpret_cast<uint4*>(p + ACH / 2) = lv;
    }
  }
}

__global__ void __launch_bounds__(GS_THREADS, 1) k_scan_gs(GsArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const DevState& st = a.st;
  const int conc = st.conc, nch = st.Dg / kGsKch;
  GsMeta* gm = reinterpret_cast<GsMeta*>(smem + (size_t)NSTG * STG);
  uint2* pring = reinterpret_cast<uint2*>(gm + NGM);  // [128] live (slab, bitmap) records
  uint64_t* full = reinterpret_cast<uint64_t*>(pring + 128);  // [NSTG] producer -> MMA (tx bytes)
  uint64_t* empty = full + NSTG;                               // [NSTG] MMA commit -> producer
  uint64_t* d_full = empty + NSTG;                             // [NBG] MMA commit -> epilogue
  uint64_t* acc_free = d_full + NBG;                           // [NBG] epilogue -> MMA
  uint64_t* gm_full = acc_free + NBG;                          // [NGM] producer -> MMA, epilogue (tx bytes)
  uint64_t* gm_free = gm_full + NGM;                           // [NGM] epilogue -> producer
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(gm_free + NGM);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NSTG; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int b = 0; b < NBG; ++b) {
      mbar_init(&d_full[b], 1);
      mbar_init(&acc_free[b], 4);
    }
    for (int g = 0; g < NGM; ++g) {
      mbar_init(&gm_full[g], 1);
      mbar_init(&gm_free[g], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, NBG * GN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    const int ntiles = st.sctr[I_NTILES];
    const unsigned lt = (1u << lane) - 1u;
    uint32_t gseq = 0, cseq = 0;
    for (;;) {
      int w = 0;
      if (lane == 0) w = atomicAdd(&st.sctr[I_WORK], 1);
      w = __shfl_sync(kFull, w, 0);
      if (w >= ntiles) break;
      const int64_t doff = a.doff[w];
      if (doff < 0) continue;  // k_gs_fallback's item
      const int l = a.work_l[w];
      int len = ld_state_s32(&st.dir_len[l], conc);
      if (len > a.dlen[w]) len = a.dlen[w];  // concurrent growth: the region holds dlen slabs
      const int32_t* dir = st.dir_arena + st.dir_off[l];
      int32_t* hdr = reinterpret_cast<int32_t*>(a.dense + doff);
      uint32_t head = 0u, tail = 0u;
      auto emit = [&](int nv) {  // group = records pring[head, head + nv)
        const int gi = (int)(gseq % NGM);
        if (lane == 0) mbar_wait(&gm_free[gi], ((gseq / NGM) & 1u) ^ 1u);
        __syncwarp();
        GsMeta& m = gm[gi];
        const uint2 r = lane < nv ? pring[(head + (uint32_t)lane) & 127u] : make_uint2(0u, 0u);
        if (lane < GG) {
          m.slab[lane] = lane < nv ? (int32_t)r.x : -1;
          m.bm[lane] = r.y;
        }
        if (lane == 0) {
          m.item = w;
          m.pos0 = (int32_t)head;
          m.nv = nv;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(&gm_full[gi], (uint32_t)nv * 2u * kSlot * 4u);
        __syncwarp();
        if (conc) fence_proxy_async_global();  // the bitmap acquire orders the copies (NEXT-2)
        if (lane < nv) {
          bulk_g2s(m.xn + kSlot * lane, st.slab_norm + (size_t)r.x * kSlot, kSlot * 4, &gm_full[gi]);
          bulk_g2s(m.xs + kSlot * lane, st.slab_xs + (size_t)r.x * kSlot, kSlot * 4, &gm_full[gi]);
        }
        const uint32_t sr = r.x;  // lane < nv: slab of the group's position `lane`
        for (int c = 0; c < nch; ++c, ++cseq) {
          const int stg = (int)(cseq % NSTG);
          if (lane == 0) mbar_wait(&empty[stg], ((cseq / NSTG) & 1u) ^ 1u);
          __syncwarp();
          unsigned char* sb = smem + (size_t)stg * STG;
          if (lane == 0) {
            mbar_arrive_expect_tx(&full[stg], (uint32_t)ACH + (uint32_t)nv * (uint32_t)BPS);
            bulk_g2s(sb, reinterpret_cast<const unsigned char*>(a.gs_a) + ((size_t)w * nch + c) * ACH, ACH, &full[stg]);
          }
          __syncwarp();
          if (lane < nv)  // slab `lane`'s chunk c: its 4 row-group pieces, one copy (chunk-major record)
            bulk_g2s(sb + ACH + lane * BPS,
                     reinterpret_cast<const unsigned char*>(st.payload_g) + (size_t)sr * recg_bytes(st.Dg) +
                         (size_t)c * BPS,
                     BPS, &full[stg]);
        }
        ++gseq;
      };
      for (int j0 = 0; j0 < len; j0 += 32) {
        const int j = j0 + lane;
        int sl = 0;
        uint32_t bm = 0u;
        if (j < len) {
          sl = ld_state_s32(&dir[j], conc);
          bm = ld_state_u32(&st.bitmap[sl], conc);
        }
        const unsigned live = __ballot_sync(kFull, bm != 0u);
        if (bm) {
          const uint32_t p = tail + (uint32_t)__popc(live & lt);
          pring[p & 127u] = make_uint2((uint32_t)sl, bm);
          hdr[p] = sl;  // live position p -> slab (k_gs_select maps slots to ids through it)
        }
        tail += (uint32_t)__popc(live);
        __syncwarp();
        while (tail - head >= (uint32_t)GG) {
          emit(GG);
          head += GG;
        }
      }
      if (tail > head) {
        emit((int)(tail - head));
        head = tail;
      }
      if (lane == 0) a.nlive[w] = (int32_t)tail;
    }
    // end of work: a group record with item = -1
    const int gi = (int)(gseq % NGM);
    if (lane == 0) {
      mbar_wait(&gm_free[gi], ((gseq / NGM) & 1u) ^ 1u);
      gm[gi].item = -1;
      mbar_arrive(&gm_full[gi]);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = umma_idesc_f16(GQ, GG * kSlot);
    uint32_t gseq = 0, cseq = 0;
    for (;;) {
      const int gi = (int)(gseq % NGM);
      mbar_wait(&gm_full[gi], (gseq / NGM) & 1u);
      if (gm[gi].item < 0) break;
      const uint32_t b = gseq % NBG;
      mbar_wait(&acc_free[b], ((gseq / NBG) & 1u) ^ 1u);
      tc_fence_after();
      const uint32_t dt = tbase + b * (uint32_t)GN;
      for (int c = 0; c < nch; ++c, ++cseq) {
        const int stg = (int)(cseq % NSTG);
        mbar_wait(&full[stg], (cseq / NSTG) & 1u);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t A = smem_u32(smem + (size_t)stg * STG), B = A + ACH;
#pragma unroll
          for (int kk = 0; kk < kGsKch / 16; ++kk) {
            const uint64_t ah = umma_sdesc(A + 256u * kk, 128u, kGsKch * 16u),
                           al = umma_sdesc(A + ACH / 2 + 256u * kk, 128u, kGsKch * 16u);
            const uint64_t bh = umma_sdesc(B + 256u * kk, 128u, kGsKch * 32u),
                           bl = umma_sdesc(B + kGsKch * 16u + 256u * kk, 128u, kGsKch * 32u);
            umma_f16_ss(dt, ah, bh, idesc, (c | kk) != 0 ? 1u : 0u);
            umma_f16_ss(dt, ah, bl, idesc, 1u);
            umma_f16_ss(dt, al, bh, idesc, 1u);
          }
          umma_commit(&empty[stg]);  // the stage may be refilled once these MMAs are done
        }
        __syncwarp();
      }
      if (lane == 0) umma_commit(&d_full[b]);
      __syncwarp();
      ++gseq;
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int qw = warp & 3, row = 32 * qw + lane;
    uint32_t gseq = 0;
    for (;;) {
      const int gi = (int)(gseq % NGM);
      mbar_wait(&gm_full[gi], (gseq / NGM) & 1u);
      const GsMeta& m = gm[gi];
      const int item = m.item;
      if (item < 0) break;
      const uint32_t b = gseq % NBG;
      mbar_wait(&d_full[b], (gseq / NBG) & 1u);
      tc_fence_after();
      const bool rv = row < a.work_n[item];
      const int dl = a.dlen[item];
      const float qn = rv ? a.gs_qn[(size_t)item * GQ + row] : 0.f;
      const float qs = rv ? a.gs_qs[(size_t)item * GQ + row] : 0.f;
      float* rowp = a.dense + a.doff[item] + gs_hdr(dl) + (int64_t)row * kSlot * dl;
      for (int j = 0; j < m.nv; ++j) {
        uint32_t v[32];
        tmem_ld32(tbase + ((uint32_t)(32 * qw) << 16) + b * (uint32_t)GN + 32u * (uint32_t)j, v);
        tmem_ld_wait();
        if (rv) {
          const uint32_t bm = m.bm[j];
          float4* dst = reinterpret_cast<float4*>(rowp + (int64_t)(m.pos0 + j) * kSlot);
#pragma unroll
          for (int c4 = 0; c4 < 8; ++c4) {
            float o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int c = 4 * c4 + e;
              const float qx = __uint_as_float(v[c]) * (qs * m.xs[kSlot * j + c]);  // exact rescale (powers of 2)
              const float d = fmaf(-2.f, qx, qn + m.xn[kSlot * j + c]);
              o[e] = ((bm >> c) & 1u) ? fmaxf(d, 0.f) : __int_as_float(0x7f800000);  // Eq. slot_valid
            }
            dst[c4] = make_float4(o[0], o[1], o[2], o[3]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&acc_free[b]);
        mbar_arrive(&gm_free[gi]);
      }
      ++gseq;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tbase, NBG * GN);
}

// Items without a dense region: per-pair top-k on CUDA cores (warp per pair,
// lane = slot, difference form, warp_topk_insert), into the pair's partial list.
__global__ void __launch_bounds__(256) k_gs_fallback(GsArgs a, unsigned long long* __restrict__ partial) {
  __shared__ u64 sm[8][256];
  const DevState& st = a.st;
  const int ntiles = st.sctr[I_NTILES];
  const int wp = threadIdx.x >> 5, lane = threadIdx.x & 31, k = a.k, Dp = st.Dp;
  u64* top = sm[wp];
  u64* tmp = top + k;
  for (int w = blockIdx.x; w < ntiles; w += gridDim.x) {
    if (a.doff[w] >= 0) continue;
    const int l = a.work_l[w], n = a.work_n[w];
    const int len = ld_state_s32(&st.dir_len[l], st.conc);
    const int32_t* dir = st.dir_arena + st.dir_off[l];
    for (int r = wp; r < n; r += 8) {
      const int pair = a.inv_pairs[a.work_p0[w] + r];
      const float* qr = a.Q + (int64_t)(pair / a.nprobe) * st.D;
      warp_topk_init(top, k);
      for (int j = 0; j < len; ++j) {
        const int s = ld_state_s32(&dir[j], st.conc);
        const uint32_t bm = ld_state_u32(&st.bitmap[s], st.conc);
        if (!bm) continue;
        const float* xs = st.payload + (size_t)s * kSlot * Dp;
        float acc = 0.f;
        for (int c4 = 0; c4 < (Dp >> 2); ++c4) {
          const float4 x = st.conc ? __ldcg(reinterpret_cast<const float4*>(xs + pay_off(Dp, lane, c4)))
                                   : __ldg(reinterpret_cast<const float4*>(xs + pay_off(Dp, lane, c4)));
          float qv[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) qv[e] = 4 * c4 + e < st.D ? __ldg(qr + 4 * c4 + e) : 0.f;
          float t;
          t = qv[0] - x.x; acc = fmaf(t, t, acc);
          t = qv[1] - x.y; acc = fmaf(t, t, acc);
          t = qv[2] - x.z; acc = fmaf(t, t, acc);
          t = qv[3] - x.w; acc = fmaf(t, t, acc);
        }
        const bool valid = (bm >> lane) & 1u;  // Eq. slot_valid
        warp_topk_insert(top, tmp, k, valid ? make_key(acc, st.slab_ids[(size_t)s * kSlot + lane]) : kPadKey);
      }
      for (int j = lane; j < k; j += 32) partial[(size_t)pair * k + j] = top[j];
      __syncwarp();
    }
  }
}

// Warp per query: top-k of its nprobe rows (dense) or partial lists (fallback
// items), by (dist, id) (C4), padded (+inf, -1) (C5).  The running top-k lives in
// registers, key 32 r + lane in tk[r] (R registers per lane, k <= 32 R); a
// candidate vector with few survivors of the k-th-key filter is inserted one key at
// a time (ballots for the position, one shuffle shift per register), a crowded one
// by a warp sort and a bitonic merge (R = 1) or through the shared-memory list
// (warp_topk_insert, R > 1).
template <int R>
__global__ void __launch_bounds__(128) k_gs_select(GsArgs a, const int32_t* __restrict__ pair_pos,
                                                   const int32_t* __restrict__ item_of,
                                                   const unsigned long long* __restrict__ partial, int64_t nq,
                                                   float* __restrict__ dist, int64_t* __restrict__ ids) {
  __shared__ u64 sm[4][R == 1 ? 1 : 64 * R];
  const int wp = threadIdx.x >> 5, lane = threadIdx.x & 31, k = a.k;
  const int64_t q = (int64_t)blockIdx.x * 4 + wp;
  if (q >= nq) return;  // warp-uniform
  const DevState& st = a.st;
  u64* top = sm[wp];
  u64* tmp = top + k;
  u64 tk[R];
#pragma unroll
  for (int r = 0; r < R; ++r) tk[r] = kPadKey;
  u64 kth = kPadKey;  // the k-th smallest key (warp-uniform)
  const int rk = (k - 1) >> 5, lk = (k - 1) & 31;
  auto kth_of = [&]() {
    u64 v = tk[0];
#pragma unroll
    for (int r = 1; r < R; ++r) v = r == rk ? tk[r] : v;
    return __shfl_sync(kFull, v, lk);
  };
  // offer one candidate per lane (kPadKey: none)
  auto offer = [&](u64 cand) {
    unsigned m = __ballot_sync(kFull, cand < kth);
    if (!m) return;
    if (__popc(m) > 4) {
      if (R == 1) {
        const u64 v = warp_sort32(cand < kth ? cand : kPadKey);  // ascending
        u64 w = umin64(tk[0], __shfl_sync(kFull, v, 31 - lane));  // the 32 smallest, bitonic
#pragma unroll
        for (int j = 16; j > 0; j >>= 1) {
          const u64 o = __shfl_xor_sync(kFull, w, j);
          w = (lane & j) ? umax64(w, o) : umin64(w, o);
        }
        tk[0] = lane < k ? w : kPadKey;
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (32 * r + lane < k) top[32 * r + lane] = tk[r];
        __syncwarp();
        warp_topk_insert(top, tmp, k, cand);
#pragma unroll
        for (int r = 0; r < R; ++r) tk[r] = 32 * r + lane < k ? top[32 * r + lane] : kPadKey;
        __syncwarp();
      }
    } else {
      while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const u64 c = __shfl_sync(kFull, cand, src);
        if (!(c < kth)) continue;  // warp-uniform (kth tightened)
        int pos = 0;
        u64 up[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          pos += __popc(__ballot_sync(kFull, tk[r] < c));
          up[r] = __shfl_up_sync(kFull, tk[r], 1);  // key 32 r + lane - 1 (lane > 0)
        }
#pragma unroll
        for (int r = R - 1; r > 0; --r) {
          const u64 carry = __shfl_sync(kFull, tk[r - 1], 31);
          if (lane == 0) up[r] = carry;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int p = 32 * r + lane;
          tk[r] = p == pos ? c : (p > pos ? up[r] : tk[r]);
          if (p >= k) tk[r] = kPadKey;
        }
        kth = kth_of();
      }
    }
    kth = kth_of();
  };
  // per-probe metadata for 32 probes at once (lane r: probe r0 + r): one round of
  // dependent loads per 32 probes instead of one per probe
  int m_pos = 0, m_w = 0, m_dl = 0, m_nl = 0, m_p0 = 0;
  long long m_doff = -1;
  for (int r = 0; r < a.nprobe; ++r) {
    const int pair = (int)(q * a.nprobe + r);
    if ((r & 31) == 0) {
      if (r + lane < a.nprobe) {
        m_pos = pair_pos[pair + lane];
        m_w = item_of[m_pos];
        m_doff = a.doff[m_w];
        m_dl = a.dlen[m_w];
        m_nl = a.nlive[m_w];
        m_p0 = a.work_p0[m_w];
      }
    }
    const int src = r & 31;
    const int pos = __shfl_sync(kFull, m_pos, src);
    const int64_t doff = (int64_t)__shfl_sync(kFull, m_doff, src);
    if (doff < 0) {
      for (int j0 = 0; j0 < k; j0 += 32) offer(j0 + lane < k ? partial[(size_t)pair * k + j0 + lane] : kPadKey);
      continue;
    }
    const int dl = __shfl_sync(kFull, m_dl, src), nl = __shfl_sync(kFull, m_nl, src);
    const int32_t* hdr = reinterpret_cast<const int32_t*>(a.dense + doff);
    const float* rowp = a.dense + doff + gs_hdr(dl) + (int64_t)(pos - __shfl_sync(kFull, m_p0, src)) * kSlot * dl;
    // R = 1: software-pipelined (the next PB slabs' distances are in flight while these
    // are filtered); R > 1: the registers go to the top-k, one batch at a time
    constexpr int PB = R == 1 ? 8 : 4;
    float dn[PB];
    if (R == 1) {
#pragma unroll
      for (int u = 0; u < PB; ++u) dn[u] = u < nl ? __ldcs(rowp + (int64_t)u * kSlot + lane) : INFINITY;
    }
    for (int j0 = 0; j0 < nl; j0 += PB) {
      float d4[PB];
#pragma unroll
      for (int u = 0; u < PB; ++u) {
        if (R == 1) {
          d4[u] = dn[u];
          dn[u] = j0 + PB + u < nl ? __ldcs(rowp + (int64_t)(j0 + PB + u) * kSlot + lane) : INFINITY;
        } else {
          d4[u] = j0 + u < nl ? __ldcs(rowp + (int64_t)(j0 + u) * kSlot + lane) : INFINITY;
        }
      }
#pragma unroll
      for (int u = 0; u < PB; ++u) {
        const uint32_t kth_hi = (uint32_t)(kth >> 32);
        const bool pass = d4[u] < INFINITY && __float_as_uint(d4[u]) <= kth_hi;
        if (!__ballot_sync(kFull, pass)) continue;
        offer(pass ? make_key(d4[u], st.slab_ids[(size_t)hdr[j0 + u] * kSlot + lane]) : kPadKey);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int j = 32 * r + lane;
    if (j < k) {
      const bool pad = tk[r] == kPadKey;
      dist[q * k + j] = pad ? __int_as_float(0x7f800000) : key_dist(tk[r]);
      ids[q * k + j] = pad ? -1 : (int64_t)key_id(tk[r]);
    }
  }
}

}  // namespace

bool scan_gs_supported(const Index& ix) { return ix.st.Dg > 0 && ix.smem_optin >= kGsSmem; }

cudaError_t setup_scan_gs(Index& ix) {
  if (!scan_gs_supported(ix)) return cudaSuccess;
  return cudaFuncSetAttribute(k_scan_gs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGsSmem);
}

// After the search front (work items of <= 128 queries, nb = 1): offsets,
// query tiles, the GEMM scan, the fallback items; then (merge phase) the
// per-query selection straight into (dist, ids).
cudaError_t launch_scan_gs(Index& ix, const float* d_q, int64_t nq, int k, int nprobe, cudaStream_t s) {
  Scratch& sc = ix.sc;
  GsArgs a{ix.st,      d_q,       nprobe,    k,         sc.inv_pairs, sc.work_l, sc.work_p0, sc.work_n,
           sc.gs_a,    sc.gs_qn,  sc.gs_qs,  sc.item_doff, sc.item_dlen, sc.item_nlive, sc.dense};
  k_gs_offsets<<<1, 1024, 0, s>>>(ix.st, sc.work_l, sc.work_n, sc.dense_cap, sc.item_doff, sc.item_dlen);
  k_gs_qsplit<<<(unsigned)ceil_div(nq * 32, (int64_t)256), 256, 0, s>>>(ix.st, d_q, nq, sc.gs_qh, sc.gs_ql, sc.gs_qqn,
                                                                       sc.gs_qqs);
  k_gs_prep<<<4 * ix.num_sms, GQ, 0, s>>>(a, sc.gs_a, sc.gs_qn, sc.gs_qs, sc.gs_qh, sc.gs_ql, sc.gs_qqn, sc.gs_qqs);
  k_scan_gs<<<ix.num_sms, GS_THREADS, kGsSmem, s>>>(a);
  k_gs_fallback<<<2 * ix.num_sms, 256, 0, s>>>(a, sc.partial);
  ix.launches += 5;
  return cudaGetLastError();
}

cudaError_t launch_select_gs(Index& ix, const float* d_q, int64_t nq, int k, int nprobe, float* d_dist,
                             int64_t* d_ids, cudaStream_t s) {
  Scratch& sc = ix.sc;
  GsArgs a{ix.st,      d_q,       nprobe,    k,         sc.inv_pairs, sc.work_l, sc.work_p0, sc.work_n,
           sc.gs_a,    sc.gs_qn,  sc.gs_qs,  sc.item_doff, sc.item_dlen, sc.item_nlive, sc.dense};
  if (k <= 32)
    k_gs_select<1><<<ceil_div(nq, 4), 128, 0, s>>>(a, sc.pair_pos, sc.item_of, sc.partial, nq, d_dist, d_ids);
  else
    k_gs_select<4><<<ceil_div(nq, 4), 128, 0, s>>>(a, sc.pair_pos, sc.item_of, sc.partial, nq, d_dist, d_ids);
  ix.launches += 1;
  return cudaGetLastError();
}

}  // namespace sivf
