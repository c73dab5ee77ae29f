// k_coarse_tc.cu — coarse quantisation on the 5th-generation tensor cores.
//
// Insert assigns each vector to its nearest centroid and search
// probes the nprobe nearest lists.  Both must equal the exact
// definition bit for bit: the m smallest keys (dist32(x, c_l), l) with dist32
// the canonical fp32 distance (readings C1-C3, C34).  The distance matrix is
// the only dense contraction on the path, so it runs on tcgen05:
//
//   k_rows_tiles   X [n][D] row-major -> tiles [n/128][Dp/4][128][4] (the
//                  K-major SWIZZLE_NONE UMMA layout: 8-row x 16-B core
//                  matrices) + ||x||^2
//   k_cent_tiles   centroids -> tiles [nlist/256][Dp/4][256][4] + ||c||^2,
//                  ||c|| (on every centroid update)
//   k_coarse_gemm  one CTA per 128-row tile: a bulk-copy producer streams
//                  32-dim K-chunks of the row tile and of each 256-centroid
//                  N-tile through a 4-stage mbarrier ring; one thread issues
//                  tcgen05.mma kind::tf32 (M=128, N=256, K=8) into one of two
//                  TMEM accumulators (double buffered across N-tiles); 8
//                  epilogue warps (thread = (row, column half)) read the fp32
//                  dot products with tcgen05.ld and form A = ||x||^2 + ||c||^2
//                  - 2 x.c and a certified bound E >= |A - dist32| (below).
//                  Each keeps the m smallest upper bounds A+E of its half in
//                  registers (U = the m-th, exchanged with the partner half
//                  through shared memory: any m upper bounds bound the m-th
//                  smallest dist32 from above) and appends every list whose
//                  lower bound A-E <= min(U, U_partner) to the row's buffer.
//   k_coarse_rerank warp per row: U* = m-th smallest upper bound over the
//                  candidates (every list with A+E <= U* is a candidate, so
//                  this is the exact m-th smallest upper bound); candidates
//                  with A-E <= U* are compacted and get the canonical dist32
//                  (sequential, __fsub/__fmul/__fadd_rn, never contracted); a
//                  warp top-m by (dist32, list) gives the exact argmin
//                  (insert) or probe set (search).
//
// Why the band is exact: U_(m) = m-th smallest upper bound >= m-th smallest
// dist32, so every member of the exact top-m (ties included) has lower bound
// <= its dist32 <= U_(m) <= U, hence is a candidate, and the re-rank orders
// candidates by the exact key.  A row whose buffer overflows re-ranks all lists.
//
// Split tf32 products: x = xh + xl, c = ch + cl with xh, ch tf32-exact (low 13
// mantissa bits cleared) and |xl| < u|x|, |cl| < u|c|; the tensor cores compute
// xh.ch + xh.cl + xl.ch (3 MMAs per K step into one fp32 accumulator).
// Error bound (u = 2^-10 tf32 operand precision, w = 2^-23 = 2x the fp32
// unit roundoff, S = ||x|| ||c|| >= sum |x_k c_k|):
//   |2 x.c_tc - 2 x.c|   <= 2 [3u^2(1+u) + (3 Dp + 2) w] S       (operands, fp32 accumulation)
//   norms + the 2 roundings of A            <= (D + 6) w (||x||^2 + ||c||^2) + 4 w S
//   |dist32 - d|                            <= (D + 2) w/2 d       (Higham, non-negative terms)
// E = 2 (E0 + e3 (max(A,0) + E0)),  E0 = e1 S + e2 (||x||^2 + ||c||^2),
// e1 = 2(3u^2+4u^3) + 2(3Dp+4)w, e2 = (D+6)w, e3 = (D+3)w (safety factor 2); with
// max(A,0) <= ||x||^2 + ||c||^2 + 2S + E0 this is <= ka S + kb (||x||^2 + ||c||^2),
// ka = 2(1+2e3)e1 + 4e3, kb = 2(1+2e3)e2 + 2e3 (both rounded up), the form
// evaluated per element.  A violation could only show up as a wrong assignment or
// probe set; the GPU tests compare both with the oracle bit for bit, including
// adversarial 1-ulp near-ties.
#include <cuda.h>

#include "sivf_host.h"

namespace sivf {

namespace {

constexpr int TM = 128;        // rows per tile (UMMA M, TMEM lanes)
constexpr int TN = 256;        // centroids per N-tile (UMMA N)
constexpr int KC = 16;         // dims per pipeline stage (hi and lo halves of each operand)
constexpr int NSTG = 4;        // stage ring depth
constexpr int W_PROD = 0, W_MMA = 1, W_EPI0 = 2, NEPI = 8;
constexpr int CTHREADS = 32 * (W_EPI0 + NEPI);
constexpr size_t kStageA = (size_t)2 * TM * KC * 4;  // 16 KB: [hi | lo]
constexpr size_t kStageB = (size_t)2 * TN * KC * 4;  // 32 KB: [hi | lo]

struct CoarseArgs {
  const float* x_tiles;   // [ntile][hi, lo][Dp/4][128][4]
  const float* xnorm;     // [n]
  const float* c_tiles;   // [nct][hi, lo][Dp/4][256][4]
  const float* cnorm;     // [nct*256] ||c||^2 (NaN for padding columns)
  const float* ccsa;      // [nct*256] ka * ||c||
  const float* ccnb;      // [nct*256] kb * ||c||^2
  int64_t n;
  int Dp, nlist, m, cap;
  float kb;
  unsigned long long* cand;  // [n][cap] lower-bound keys (bits(max(A-E,0)) << 32 | list)
  float* cand_ub;            // [n][cap] upper bounds A+E
  int32_t* cand_cnt;         // [n] appended candidates (> cap: overflow)
  float* mat;                // KP == 0: A = ||x||^2 + ||c||^2 - 2 x.c_tc, [n][nlist] row-major
  int ntpc;                  // N-tiles per CTA (blockIdx.y selects the range); KP != 0: all
};

__host__ __device__ constexpr int coarse_nstg(int KP) { return KP == 0 ? 3 : NSTG; }
__host__ __device__ constexpr size_t coarse_xchg_bytes(int KP) {
  return KP == 0 ? (size_t)NEPI * 32 * 32 * 4 : (size_t)TM * 32 * 4;  // store tiles | half-row top-32
}
__host__ __device__ constexpr size_t coarse_smem_bytes(int KP = 1) {
  return (size_t)coarse_nstg(KP) * (kStageA + kStageB)  // operand ring
         + 2 * 3 * TN * 4                    // per-N-tile column constants (double buffered)
         + coarse_xchg_bytes(KP)             // exchange area
         + TM * 4 + 2 * TM * 4               // candidate counters, half-row bounds
         + 256 + 1024;                       // barriers, TMEM base, alignment slack
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
}

// Ascending bitonic sort of 32 register floats (no NaN: callers map NaN to +inf).
__device__ __forceinline__ void sort32(float (&x)[32]) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int l = i ^ j;
        if (l > i) {
          const float a = x[i], b = x[l];
          const bool asc = (i & k) == 0;
          x[i] = asc ? fminf(a, b) : fmaxf(a, b);
          x[l] = asc ? fmaxf(a, b) : fminf(a, b);
        }
      }
}
// keys (ascending) <- the 32 smallest of keys and c (c ascending), ascending.
__device__ __forceinline__ void merge_lower32(float (&keys)[32], const float* c) {
#pragma unroll
  for (int i = 0; i < 32; ++i) keys[i] = fminf(keys[i], c[31 - i]);  // bitonic
#pragma unroll
  for (int j = 16; j > 0; j >>= 1)
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int l = i ^ j;
      if (l > i) {
        const float a = keys[i], b = keys[l];
        keys[i] = fminf(a, b);
        keys[l] = fmaxf(a, b);
      }
    }
}

// KP = 1 (assignment, m = 1): one pass; the running minimum upper bound of the
// row half (and of its partner half) is the threshold for appending.
// KP = 32 (probes, m <= 32): two passes over the N-tiles.  Pass 1 keeps the
// exact 32 smallest upper bounds of each row half (register sort-merge per 32
// columns), the halves merge them, and U = the m-th smallest over the row;
// pass 2 recomputes the products and appends exactly the lists with A-E <= U.
template <int KP>
__global__ void __launch_bounds__(CTHREADS, 1) k_coarse_gemm(const __grid_constant__ CUtensorMap tmat, CoarseArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 128B-swizzle tiles
  constexpr int NS = coarse_nstg(KP);
  float* sA = reinterpret_cast<float*>(smem);                                  // [NS][16 KB]
  float* sB = reinterpret_cast<float*>(smem + NS * kStageA);                   // [NS][32 KB]
  float* colc = reinterpret_cast<float*>(smem + NS * (kStageA + kStageB));     // [2][3][TN]
  float* xchg = colc + 2 * 3 * TN;                                             // see coarse_xchg_bytes
  int* cnt_sm = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(xchg) + coarse_xchg_bytes(KP));  // [TM]
  float* thr_sh = reinterpret_cast<float*>(cnt_sm + TM);                       // [2][TM]
  uint64_t* full = reinterpret_cast<uint64_t*>(thr_sh + 2 * TM);
  uint64_t* empty = full + NS;
  uint64_t* acc_full = empty + NS;     // [2]
  uint64_t* acc_empty = acc_full + 2;  // [2]
  uint32_t* tmem_base_sm = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x;
  const int Dp = a.Dp, nq4 = Dp >> 2;
  const int nchunk = (Dp + KC - 1) / KC;
  const int jbeg = blockIdx.y * a.ntpc;
  const int ntn = min((a.nlist + TN - 1) / TN - jbeg, a.ntpc);  // N-tiles of this CTA: [jbeg, jbeg + ntn)
  constexpr int NPASS = KP <= 1 ? 1 : 2;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], NEPI);
    }
    fence_mbar_init();
  }
  if (threadIdx.x < TM) {
    cnt_sm[threadIdx.x] = 0;
    thr_sh[threadIdx.x] = INFINITY;
    thr_sh[TM + threadIdx.x] = INFINITY;
  }
  if (warp == W_MMA) tmem_alloc(tmem_base_sm, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_base_sm;

  if (warp == W_PROD) {
    if (lane == 0) {
      const float* xa = a.x_tiles + (size_t)tile * 2 * nq4 * TM * 4;
      uint32_t seq = 0;
      for (int t = 0; t < NPASS * ntn; ++t) {
        const float* cb = a.c_tiles + (size_t)(jbeg + t % ntn) * 2 * nq4 * TN * 4;
        for (int c = 0; c < nchunk; ++c, ++seq) {
          const int st = (int)(seq % NS);
          mbar_wait(&empty[st], ((seq / NS) & 1u) ^ 1u);
          const int kc = min(KC, Dp - c * KC);
          const uint32_t ba = (uint32_t)kc * TM * 4, bb = (uint32_t)kc * TN * 4;
          mbar_arrive_expect_tx(&full[st], 2 * (ba + bb));
          float* da = sA + (size_t)st * (kStageA / 4);
          float* db = sB + (size_t)st * (kStageB / 4);
          bulk_g2s(da, xa + (size_t)c * KC * TM, ba, &full[st]);                                  // x hi
          bulk_g2s(da + TM * KC, xa + (size_t)nq4 * TM * 4 + (size_t)c * KC * TM, ba, &full[st]);   // x lo
          bulk_g2s(db, cb + (size_t)c * KC * TN, bb, &full[st]);                                  // c hi
          bulk_g2s(db + TN * KC, cb + (size_t)nq4 * TN * 4 + (size_t)c * KC * TN, bb, &full[st]);   // c lo
        }
      }
    }
  } else if (warp == W_MMA) {
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_tf32(TM, TN);
      uint32_t seq = 0;
      for (int t = 0; t < NPASS * ntn; ++t) {
        const uint32_t b = (uint32_t)t & 1u, use = (uint32_t)t >> 1;
        mbar_wait(&acc_empty[b], (use & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t dt = tbase + b * TN;
        for (int c = 0; c < nchunk; ++c, ++seq) {
          const int st = (int)(seq % NS);
          mbar_wait(&full[st], (seq / NS) & 1u);
          tc_fence_after();
          const int kc = min(KC, Dp - c * KC);
          const uint32_t a0 = smem_u32(sA + (size_t)st * (kStageA / 4));
          const uint32_t b0 = smem_u32(sB + (size_t)st * (kStageB / 4));
          // split tf32 ("3xTF32"): x.c ~ xh.ch + xh.cl + xl.ch (the bound E below)
          for (int kk = 0; kk < (kc >> 3); ++kk) {
            const uint32_t ah = a0 + (uint32_t)kk * 2u * TM * 16u, al = ah + (uint32_t)(TM * KC * 4);
            const uint32_t bh = b0 + (uint32_t)kk * 2u * TN * 16u, bl = bh + (uint32_t)(TN * KC * 4);
            umma_tf32_ss(dt, umma_sdesc(ah, TM * 16u, 128u), umma_sdesc(bh, TN * 16u, 128u), idesc,
                         (c > 0 || kk > 0) ? 1u : 0u);
            umma_tf32_ss(dt, umma_sdesc(ah, TM * 16u, 128u), umma_sdesc(bl, TN * 16u, 128u), idesc, 1u);
            umma_tf32_ss(dt, umma_sdesc(al, TM * 16u, 128u), umma_sdesc(bh, TN * 16u, 128u), idesc, 1u);
          }
          umma_commit(&empty[st]);  // stage reusable once these MMAs have read it
        }
        umma_commit(&acc_full[b]);
      }
    }
  } else {
    // ------------------------------------------------ epilogue: thread = (row, column half)
    const int ew = warp - W_EPI0;   // 0..7
    const int q = warp & 3;         // TMEM lane quarter this warp may access
    const int h = ew >> 2;          // column half of each N-tile
    const int r = 32 * q + lane;
    const int et = 32 * ew + lane;  // 0..255
    const int64_t row = (int64_t)tile * TM + r;
    const bool rv = row < a.n;
    const float qn = rv ? a.xnorm[row] : 0.f;
    const float sq = sqrtf(qn), qnb = a.kb * qn;
    float keys[KP > 0 ? KP : 1];
#pragma unroll
    for (int i = 0; i < KP; ++i) keys[i] = i < KP - a.m ? -INFINITY : INFINITY;
    float Uo = INFINITY;  // KP == 1: running min upper bound; KP == 32: final U (after pass 1)
    unsigned long long* crow = a.cand + (size_t)(rv ? row : 0) * a.cap;
    float* urow = a.cand_ub + (size_t)(rv ? row : 0) * a.cap;
    for (int t = 0; t < NPASS * ntn; ++t) {
      const int j = jbeg + t % ntn;
      const bool append_pass = NPASS == 1 || t >= ntn;
      if constexpr (NPASS == 2) {
        if (t == ntn) {
        // end of pass 1: merge the two half lists of each row -> exact m-th smallest upper bound
        if (h == 1)
#pragma unroll
          for (int i = 0; i < 32; ++i) xchg[r * 32 + i] = keys[i];
        asm volatile("bar.sync 1, %0;" ::"n"(32 * NEPI));
        if (h == 0) {
          // the partner's m real bounds sit at [32 - m, 32) behind its -inf prefill
          float c[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) c[i] = i < a.m ? xchg[r * 32 + (32 - a.m) + i] : INFINITY;
          merge_lower32(*reinterpret_cast<float(*)[32]>(keys), c);
          thr_sh[r] = keys[31];
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * NEPI));
        Uo = thr_sh[r];
        }
      }
      const uint32_t b = (uint32_t)t & 1u, use = (uint32_t)t >> 1;
      float* cc = colc + b * 3 * TN;
      {
        const int col = j * TN + et;
        cc[et] = __ldg(a.cnorm + col);
        cc[TN + et] = __ldg(a.ccsa + col);
        cc[2 * TN + et] = __ldg(a.ccnb + col);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * NEPI));
      mbar_wait(&acc_full[b], use & 1u);
      tc_fence_after();
      float T = NPASS == 1 ? fminf(Uo, thr_sh[(1 - h) * TM + r]) : Uo;
#pragma unroll 1
      for (int c32 = 0; c32 < 4; ++c32) {
        uint32_t v[32];
        const int cb = h * (TN / 2) + 32 * c32;  // column within the N-tile
        __syncwarp();
        tmem_ld32(tbase + ((uint32_t)(32 * q) << 16) + b * TN + (uint32_t)cb, v);
        tmem_ld_wait();
        if constexpr (KP == 0) {
          // store A = ||x||^2 + ||c||^2 - 2 x.c_tc for the per-row selection: the
          // warp's 32 rows x 32 columns go to a 128B-swizzled shared tile (conflict-free
          // 16-B stores), then one TMA tensor store (rows >= n land in unused scratch
          // rows; columns >= nlist are clipped by the tensor map)
          float* T = xchg + (size_t)ew * 32 * 32;
#pragma unroll
          for (int c16 = 0; c16 < 8; ++c16) {
            const float4 cn = *reinterpret_cast<const float4*>(cc + cb + 4 * c16);
            float4 o;
            o.x = fmaf(-2.f, __uint_as_float(v[4 * c16 + 0]), qn + cn.x);
            o.y = fmaf(-2.f, __uint_as_float(v[4 * c16 + 1]), qn + cn.y);
            o.z = fmaf(-2.f, __uint_as_float(v[4 * c16 + 2]), qn + cn.z);
            o.w = fmaf(-2.f, __uint_as_float(v[4 * c16 + 3]), qn + cn.w);
            *reinterpret_cast<float4*>(T + lane * 32 + ((c16 ^ (lane & 7)) * 4)) = o;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmat, T, j * TN + cb, tile * TM + 32 * q);
            bulk_commit();
            bulk_wait_read0();  // the tile may be rewritten by the next chunk
          }
          __syncwarp();
          continue;
        }
        if constexpr (NPASS == 2) {
          if (!append_pass) {
          // pass 1 (KP == 32): exact per-half top-32 of the upper bounds
          float ub[32];
          float mn = INFINITY;
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const float A = fmaf(-2.f, __uint_as_float(v[e]), qn + cc[cb + e]);
            const float E = fmaf(sq, cc[TN + cb + e], qnb + cc[2 * TN + cb + e]);
            ub[e] = rv ? fminf(A + E, INFINITY) : INFINITY;  // NaN (padding column) -> +inf
            mn = fminf(mn, ub[e]);
          }
          if (__any_sync(kFull, mn < keys[KP - 1])) {
            sort32(ub);
            merge_lower32(*reinterpret_cast<float(*)[32]>(keys), ub);
          }
          continue;
          }
        }
        if (rv) {
#pragma unroll
          for (int e4 = 0; e4 < 8; ++e4) {
            const float4 cn = *reinterpret_cast<const float4*>(cc + cb + 4 * e4);
            const float4 cs = *reinterpret_cast<const float4*>(cc + TN + cb + 4 * e4);
            const float4 cq = *reinterpret_cast<const float4*>(cc + 2 * TN + cb + 4 * e4);
            const float cna[4] = {cn.x, cn.y, cn.z, cn.w};
            const float csa[4] = {cs.x, cs.y, cs.z, cs.w};
            const float cqa[4] = {cq.x, cq.y, cq.z, cq.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float A = fmaf(-2.f, __uint_as_float(v[4 * e4 + e]), qn + cna[e]);
              const float E = fmaf(sq, csa[e], qnb + cqa[e]);
              const float lb = A - E;
              if (lb <= T) {  // NaN (padding column) never passes
                const float ub = A + E;
                if (NPASS == 1 && ub < Uo) {
                  Uo = ub;
                  T = fminf(T, Uo);
                }
                // N-split grid (gridDim.y > 1): the row's CTAs share one global counter
                const int slot = gridDim.y > 1 ? atomicAdd(&a.cand_cnt[row], 1) : atomicAdd(&cnt_sm[r], 1);
                if (slot < a.cap) {
                  crow[slot] = ((unsigned long long)__float_as_uint(fmaxf(lb, 0.f)) << 32) |
                               (uint32_t)(j * TN + cb + 4 * e4 + e);
                  urow[slot] = ub;
                }
              }
            }
          }
        }
      }
      if (NPASS == 1) thr_sh[h * TM + r] = Uo;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[b]);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * NEPI));
    if (KP != 0 && gridDim.y == 1 && h == 0 && rv) a.cand_cnt[row] = cnt_sm[r];
  }
  if (KP == 0 && warp >= W_EPI0 && lane == 0) bulk_wait0();  // stores complete before exit
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == W_MMA) tmem_dealloc(tbase, 512);
}

// The tf32 part of x (low 13 mantissa bits cleared): exactly representable in tf32,
// so the tensor core takes it unchanged whether it truncates or rounds; x - hi is
// exact in fp32 and |x - hi| < 2^-10 |x|.
__device__ __forceinline__ float4 tf32_hi(float4 v) {
  return make_float4(__uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u),
                     __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u),
                     __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u),
                     __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u));
}

// X [n][D] row-major -> [n/128][hi, lo][Dp/4][128][4] zero padded; ||x||^2 (fp32, any order).
// 4 threads per row (quarters of the row, loads issued 8 ahead), partial norms
// combined through shared memory.
__global__ void __launch_bounds__(4 * TM) k_rows_tiles(const float* __restrict__ X, int64_t n, int D, int Dp,
                                                       float* __restrict__ out, float* __restrict__ norm) {
  __shared__ float part[4][TM];
  const int r = threadIdx.x & (TM - 1), qt = threadIdx.x >> 7;
  const int64_t row = (int64_t)blockIdx.x * TM + r;
  const int nq4 = Dp >> 2;
  const int c0 = (nq4 * qt) >> 2, c1 = (nq4 * (qt + 1)) >> 2;
  float4* o = reinterpret_cast<float4*>(out) + (size_t)blockIdx.x * 2 * nq4 * TM + r;
  float4* ol = o + (size_t)nq4 * TM;
  const float* xr = X + (row < n ? row : 0) * (int64_t)D;
  const bool vec = (D & 3) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
  float nrm = 0.f;
#pragma unroll 8
  for (int c4 = c0; c4 < c1; ++c4) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row < n) {
      if (vec && 4 * c4 + 3 < D) {
        v = __ldg(reinterpret_cast<const float4*>(xr) + c4);
      } else {
        float t[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) t[e] = 4 * c4 + e < D ? __ldg(xr + 4 * c4 + e) : 0.f;
        v = make_float4(t[0], t[1], t[2], t[3]);
      }
    }
    const float4 hi = tf32_hi(v);
    o[(size_t)c4 * TM] = hi;
    ol[(size_t)c4 * TM] = make_float4(v.x - hi.x, v.y - hi.y, v.z - hi.z, v.w - hi.w);  // exact
    nrm = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, nrm))));
  }
  part[qt][r] = nrm;
  __syncthreads();
  if (qt == 0 && row < n) norm[row] = (part[0][r] + part[1][r]) + (part[2][r] + part[3][r]);
}

// centroids [nlist][Dp] -> [nlist/256][Dp/4][256][4] zero padded; per column
// ||c||^2 (NaN for padding: such columns never become candidates), ka ||c||, kb ||c||^2.
__global__ void __launch_bounds__(TN) k_cent_tiles(const float* __restrict__ C, int nlist, int Dp, float ka,
                                                   float kb, float* __restrict__ out, float* __restrict__ cnorm,
                                                   float* __restrict__ ccsa, float* __restrict__ ccnb) {
  const int r = threadIdx.x;
  const int l = blockIdx.x * TN + r;
  const int nq4 = Dp >> 2;
  float4* o = reinterpret_cast<float4*>(out) + (size_t)blockIdx.x * 2 * nq4 * TN + r;
  float4* ol = o + (size_t)nq4 * TN;
  const float4* cr = reinterpret_cast<const float4*>(C + (size_t)(l < nlist ? l : 0) * Dp);
  float nrm = 0.f;
  for (int c4 = 0; c4 < nq4; ++c4) {
    const float4 v = l < nlist ? cr[c4] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 hi = tf32_hi(v);
    o[(size_t)c4 * TN] = hi;
    ol[(size_t)c4 * TN] = make_float4(v.x - hi.x, v.y - hi.y, v.z - hi.z, v.w - hi.w);  // exact
    nrm = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, nrm))));
  }
  cnorm[l] = l < nlist ? nrm : __int_as_float(0x7fc00000);
  ccsa[l] = ka * sqrtf(nrm);
  ccnb[l] = kb * nrm;
}

// Canonical dist32 (reading C1) of the smem row xs against global row cr: the
// same sequential order as the definition; loads are issued 8 x 16 B ahead of
// the dependent add chain.
__device__ __forceinline__ float dist32_rows(const float* __restrict__ xs, const float* __restrict__ cr, int D,
                                            bool vec) {
  float s = 0.f;
  int k = 0;
  if (vec) {
    for (; k + 32 <= D; k += 32) {
      float4 cv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) cv[j] = __ldg(reinterpret_cast<const float4*>(cr + k) + j);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 xv = *reinterpret_cast<const float4*>(xs + k + 4 * j);
        float t;
        t = __fsub_rn(xv.x, cv[j].x); s = __fadd_rn(s, __fmul_rn(t, t));
        t = __fsub_rn(xv.y, cv[j].y); s = __fadd_rn(s, __fmul_rn(t, t));
        t = __fsub_rn(xv.z, cv[j].z); s = __fadd_rn(s, __fmul_rn(t, t));
        t = __fsub_rn(xv.w, cv[j].w); s = __fadd_rn(s, __fmul_rn(t, t));
      }
    }
  }
  for (; k < D; ++k) {
    const float t = __fsub_rn(xs[k], __ldg(cr + k));
    s = __fadd_rn(s, __fmul_rn(t, t));
  }
  return s;
}

// Two canonical dist32 chains interleaved (independent sequential sums: the
// latency of one 128-long add chain hides the other's).
__device__ __forceinline__ void dist32_rows2(const float* __restrict__ xs, const float* __restrict__ c0,
                                             const float* __restrict__ c1, int D, bool vec, float& d0, float& d1) {
  float s0 = 0.f, s1 = 0.f;
  int k = 0;
  if (vec) {
    for (; k + 16 <= D; k += 16) {
      float4 a[4], b[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        a[j] = __ldg(reinterpret_cast<const float4*>(c0 + k) + j);
        b[j] = __ldg(reinterpret_cast<const float4*>(c1 + k) + j);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float4 xv = *reinterpret_cast<const float4*>(xs + k + 4 * j);
        float t, u;
        t = __fsub_rn(xv.x, a[j].x); u = __fsub_rn(xv.x, b[j].x);
        s0 = __fadd_rn(s0, __fmul_rn(t, t)); s1 = __fadd_rn(s1, __fmul_rn(u, u));
        t = __fsub_rn(xv.y, a[j].y); u = __fsub_rn(xv.y, b[j].y);
        s0 = __fadd_rn(s0, __fmul_rn(t, t)); s1 = __fadd_rn(s1, __fmul_rn(u, u));
        t = __fsub_rn(xv.z, a[j].z); u = __fsub_rn(xv.z, b[j].z);
        s0 = __fadd_rn(s0, __fmul_rn(t, t)); s1 = __fadd_rn(s1, __fmul_rn(u, u));
        t = __fsub_rn(xv.w, a[j].w); u = __fsub_rn(xv.w, b[j].w);
        s0 = __fadd_rn(s0, __fmul_rn(t, t)); s1 = __fadd_rn(s1, __fmul_rn(u, u));
      }
    }
  }
  for (; k < D; ++k) {
    const float t = __fsub_rn(xs[k], __ldg(c0 + k)), u = __fsub_rn(xs[k], __ldg(c1 + k));
    s0 = __fadd_rn(s0, __fmul_rn(t, t));
    s1 = __fadd_rn(s1, __fmul_rn(u, u));
  }
  d0 = s0;
  d1 = s1;
}

__host__ __device__ inline size_t rerank_smem_per_warp(int m, int cap, int Dp) {
  // 16-B aligned sections: keys (2m u64), survivors (cap rounded to 4), row (Dp, a multiple of 8)
  return sizeof(unsigned long long) * 2 * (size_t)m + sizeof(int32_t) * (size_t)((cap + 3) & ~3) +
         sizeof(float) * (size_t)Dp;
}

// Warp per row (see the file comment).  MODE 0: best[row] = smallest exact key
// (assignment); MODE 1: probes[row][0..m) = the m smallest, sorted.
template <int MODE>
__global__ void __launch_bounds__(128) k_coarse_rerank(const float* __restrict__ X, int64_t n, int D,
                                                       const float* __restrict__ C, int Dp, int nlist, int m,
                                                       const unsigned long long* __restrict__ cand,
                                                       const float* __restrict__ cand_ub,
                                                       const int32_t* __restrict__ cand_cnt, int cap,
                                                       unsigned long long* __restrict__ best,
                                                       int32_t* __restrict__ probes, int probes_ld) {
  extern __shared__ __align__(16) unsigned char sm_rr[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 4 + w;
  if (row >= n) return;  // warp-uniform
  unsigned char* base = sm_rr + (size_t)w * rerank_smem_per_warp(m, cap, Dp);
  unsigned long long* top = reinterpret_cast<unsigned long long*>(base);
  unsigned long long* tmp = top + m;
  int32_t* surv = reinterpret_cast<int32_t*>(tmp + m);
  float* xs = reinterpret_cast<float*>(surv + ((cap + 3) & ~3));
  const float* xr = X + row * (int64_t)D;
  for (int k = lane; k < D; k += 32) xs[k] = __ldg(xr + k);
  const bool vec = (Dp & 3) == 0;
  const int cnt = cand_cnt[row];
  const unsigned long long* crow = cand + (size_t)row * cap;
  const float* urow = cand_ub + (size_t)row * cap;
  const unsigned lt = (1u << lane) - 1u;

  // 1. survivors: every list if the buffer overflowed, else lower bound <= U*
  int ns = 0;
  if (cnt > cap) {
    ns = -1;
  } else {
    float U;
    if (MODE == 0) {
      float u = INFINITY;
      for (int i = lane; i < cnt; i += 32) u = fminf(u, urow[i]);
#pragma unroll
      for (int off = 16; off; off >>= 1) u = fminf(u, __shfl_xor_sync(kFull, u, off));
      U = u;
    } else {
      warp_topk_init(top, m);
      for (int i0 = 0; i0 < cnt; i0 += 32) {
        const int i = i0 + lane;
        warp_topk_insert(top, tmp, m, i < cnt ? make_key(fmaxf(urow[i], 0.f), (uint32_t)i) : kPadKey);
      }
      U = key_dist(top[m - 1]);  // +inf if fewer than m candidates
    }
    for (int i0 = 0; i0 < cnt; i0 += 32) {
      const int i = i0 + lane;
      int l = 0;
      bool pass = false;
      if (i < cnt) {
        const unsigned long long ck = crow[i];
        l = (int)(ck & 0xffffffffu);
        pass = __uint_as_float((uint32_t)(ck >> 32)) <= U;
      }
      const unsigned pm = __ballot_sync(kFull, pass);
      if (pass) surv[ns + __popc(pm & lt)] = l;
      ns += __popc(pm);
    }
    __syncwarp();
  }
  // 2. exact dist32 of the survivors, exact top-m by (dist32, list)
  const int total = ns < 0 ? nlist : ns;
  unsigned long long bestk = ~0ull;
  if (MODE == 1) warp_topk_init(top, m);
  for (int i0 = 0; i0 < total; i0 += 32) {
    const int i = i0 + lane;
    unsigned long long key = kPadKey;
    if (i < total) {
      const int l = ns < 0 ? i : surv[i];
      key = make_key(dist32_rows(xs, C + (size_t)l * Dp, D, vec), (uint32_t)l);
    }
    if (MODE == 0) bestk = umin64(bestk, key);
    else warp_topk_insert(top, tmp, m, key);
  }
  if (MODE == 0) {
#pragma unroll
    for (int off = 16; off; off >>= 1) bestk = umin64(bestk, __shfl_xor_sync(kFull, bestk, off));
    if (lane == 0) best[row] = bestk;
  } else {
    for (int j = lane; j < m; j += 32) probes[row * probes_ld + j] = (int32_t)key_id(top[j]);
  }
}


// Per-row selection over the stored A matrix (warp per row; lane owns the
// columns lane + 32 i).  With E the certified bound of the file comment:
//   U = the m-th smallest upper bound max(A + E, 0),
//   candidates = {l : A_l - E_l <= U} (every member of the exact top-m, ties
//       included, has lower bound <= its dist32 <= U),
// then the canonical dist32 of each candidate and the exact top-m by
// (dist32, l).  MODE 0: best[row] = smallest key (assignment); MODE 1:
// probes[row][0..m) sorted.  More than CCAP candidates: every list is re-ranked.
// U and the candidates are found on a superset S of few columns: with U' the
// m-th smallest A and Emax >= every E_l of the row, U <= U' + Emax and every
// candidate has A_l <= U + E_l <= U' + 2 Emax, so S = {l : A_l <= U' + 2 Emax}
// (rounded up) holds every column that decides U and every candidate; E, the
// bounds and U are then evaluated exactly as on the full row, on S only.
constexpr int CCAP = 256;
// Fused first step of the search's inverse probe map (k_search.cu k_inv_count): per
// probe rank j of a row, one count in bucket (j >= r0) of its list; the row's k-th
// distance bound reset to +inf.  cnt == nullptr: not fused.
struct InvCount {
  int32_t* cnt;
  uint32_t* gthr;
  int nb, r0;
  int keep = 0;  // experiments (SIVF_OPT_DEBUG bit 6): keep the previous search's bounds
};
__device__ __forceinline__ void inv_count_row(const InvCount& ic, int nlist, int64_t row, int j, int32_t l) {
  if (!ic.cnt) return;
  atomicAdd(&ic.cnt[((ic.nb == 2 && j >= ic.r0) ? nlist : 0) + l], 1);
  if (j == 0 && !ic.keep) ic.gthr[row] = 0x7F800000u;
}
#ifdef SIVF_TC_PROF
__device__ unsigned g_selhist[2][64];
__device__ unsigned long long g_selclk[2][8];
#define SELCLK(i)                                                             \
  do {                                                                        \
    const long long _t = clock64();                                           \
    if (lane == 0) atomicAdd(&g_selclk[MODE][i], (unsigned long long)(_t - _t0)); \
    _t0 = _t;                                                                 \
  } while (0)
#else
#define SELCLK(i) \
  do {            \
  } while (0)
#endif
constexpr int SELW = 8;  // rows (warps) per block
__host__ __device__ inline size_t select_smem_per_warp(int Dp) {
  return (size_t)Dp * 4 + 5 * CCAP * 4 + 2 * 32 * 8;
}
constexpr int QCAP = SELW * 64;  // block re-rank queue: <= 64 uncertain candidates per row
__host__ __device__ inline size_t select_smem(int Dp, int nlist, int mode = 1) {
  (void)mode;
  return SELW * select_smem_per_warp(Dp) + (size_t)2 * nlist * 4 + 16;
}
// order-preserving map of a (non-NaN) float to uint32
__device__ __forceinline__ uint32_t fkey(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}
// the m-th smallest (1 <= m <= 32) of the warp's values v0 (all lanes) and, when
// two, v1, with 0xFFFFFFFF padding: two warp bitonic sorts and one bitonic merge
__device__ __forceinline__ uint32_t warp_mth64(uint32_t a0, uint32_t a1, bool two, int m) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const uint32_t o0 = __shfl_xor_sync(kFull, a0, stride);
      const uint32_t o1 = two ? __shfl_xor_sync(kFull, a1, stride) : 0u;
      const bool up = (lane & size) == 0 || size == 32, lower = (lane & stride) == 0;
      a0 = (lower == up) ? min(a0, o0) : max(a0, o0);
      if (two) a1 = (lower == up) ? min(a1, o1) : max(a1, o1);
    }
  }
  uint32_t b = two ? min(a0, __shfl_sync(kFull, a1, 31 - lane)) : a0;  // bitonic: the 32 smallest
  if (two) {
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) {
      const uint32_t o = __shfl_xor_sync(kFull, b, j);
      b = (lane & j) ? max(b, o) : min(b, o);
    }
  }
  return __shfl_sync(kFull, b, m - 1);
}
// the (j+1)-th smallest (0 <= j < 64) of the warp's 64 values v0, v1 (0xFFFFFFFF padding):
// a full bitonic sort of 64 (two warp sorts and a merge network across both halves)
__device__ __forceinline__ uint32_t warp_kth64(uint32_t a0, uint32_t a1, int j) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const uint32_t o0 = __shfl_xor_sync(kFull, a0, stride), o1 = __shfl_xor_sync(kFull, a1, stride);
      const bool up = (lane & size) == 0, lower = (lane & stride) == 0;
      // a0 sorted ascending (size 32 stage: ascending), a1 descending: together bitonic
      const bool up0 = up || size == 32, up1 = up && size != 32;
      a0 = (lower == up0) ? min(a0, o0) : max(a0, o0);
      a1 = (lower == up1) ? min(a1, o1) : max(a1, o1);
    }
  }
  // a0 ascending, a1 descending: a bitonic sequence of 64; half-cleaner across halves
  const uint32_t lo = min(a0, a1), hi = max(a0, a1);
  uint32_t b0 = lo, b1 = hi;  // b0 holds the 32 smallest (bitonic), b1 the 32 largest (bitonic)
#pragma unroll
  for (int stride = 16; stride > 0; stride >>= 1) {
    const uint32_t o0 = __shfl_xor_sync(kFull, b0, stride), o1 = __shfl_xor_sync(kFull, b1, stride);
    const bool lower = (lane & stride) == 0;
    b0 = lower ? min(b0, o0) : max(b0, o0);
    b1 = lower ? min(b1, o1) : max(b1, o1);
  }
  return j < 32 ? __shfl_sync(kFull, b0, j) : __shfl_sync(kFull, b1, j - 32);
}
template <int NPL, int MODE>
__global__ void __launch_bounds__(32 * SELW, 3) k_coarse_select(const float* __restrict__ mat,
                                                             const float* __restrict__ X, int64_t n, int D,
                                                             int nlist, int m, const float* __restrict__ xnorm,
                                                             const float* __restrict__ ccsa,
                                                             const float* __restrict__ ccnb, float kb,
                                                             const float* __restrict__ C, int Dp,
                                                             unsigned long long* __restrict__ best,
                                                             int32_t* __restrict__ probes, int probes_ld,
                                                             int need_dist, InvCount ic) {
  extern __shared__ __align__(16) unsigned char sm_sel[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* csa_s = reinterpret_cast<float*>(sm_sel + SELW * select_smem_per_warp(Dp));
  float* cnb_s = csa_s + nlist;
  uint32_t* cmax = reinterpret_cast<uint32_t*>(cnb_s + nlist);  // [2] max csa, max cnb (bits; >= 0)
  __shared__ int q_cnt;            // block re-rank queue (MODE 1): entries (warp, list) -> dist32
  __shared__ uint8_t q_w[QCAP];
  __shared__ int32_t q_l[QCAP];
  __shared__ float q_d[QCAP];
  if (threadIdx.x < 2) cmax[threadIdx.x] = 0u;
  if (threadIdx.x == 0) q_cnt = 0;
  __syncthreads();
  uint32_t ma = 0u, mb = 0u;
  for (int c = threadIdx.x; c < nlist; c += blockDim.x) {
    const float va = __ldg(ccsa + c), vb = __ldg(ccnb + c);
    csa_s[c] = va;
    cnb_s[c] = vb;
    ma = max(ma, __float_as_uint(va));
    mb = max(mb, __float_as_uint(vb));
  }
  ma = __reduce_max_sync(kFull, ma);
  mb = __reduce_max_sync(kFull, mb);
  if (lane == 0) {
    atomicMax(&cmax[0], ma);
    atomicMax(&cmax[1], mb);
  }
  __syncthreads();
  const int64_t row = (int64_t)blockIdx.x * SELW + w;
  unsigned char* base = sm_sel + (size_t)w * select_smem_per_warp(Dp);
  float* xs = reinterpret_cast<float*>(base);
  int32_t* cand = reinterpret_cast<int32_t*>(xs + Dp);
  float* capx = reinterpret_cast<float*>(cand + CCAP);  // approximate distance of each candidate
  int32_t* scol = reinterpret_cast<int32_t*>(capx + CCAP);  // the superset S (columns)
  float* clb = reinterpret_cast<float*>(scol + CCAP);       // candidate lower / upper bounds
  float* cub = clb + CCAP;
  unsigned long long* top = reinterpret_cast<unsigned long long*>(cub + CCAP);
  unsigned long long* tmp = top + 32;
  const bool vec = (Dp & 3) == 0;
  int path = 0;                 // MODE 1: 1 = batched exact re-rank of the uncertain candidates
  int qbase = 0, nu = 0, nce = 0, ncand = 0;
  uint32_t lbm = 0u;            // (m+1)-th smallest lower-bound key among the candidates
  do {  // MODE 1 leaves by break (the block barriers below), MODE 0 may return
  if (row >= n) break;  // warp-uniform
#ifdef SIVF_TC_PROF
  long long _t0 = clock64();
#endif
  // lane owns the columns lane + 32 i (coalesced 128-B row segments)
  const float* arow = mat + (size_t)row * nlist;
  float A[NPL];
#pragma unroll
  for (int i = 0; i < NPL; ++i) A[i] = lane + 32 * i < nlist ? __ldcs(arow + lane + 32 * i) : INFINITY;
  const float qn = xnorm[row], sq = sqrtf(qn), qnb = kb * qn;
  auto Ecol = [&](int c) { return fmaf(sq, csa_s[c], qnb + cnb_s[c]); };  // the per-column form
  const float Emax = __fmaf_ru(sq, __uint_as_float(cmax[0]), __fadd_ru(qnb, __uint_as_float(cmax[1])));
  const float* xr = X + row * (int64_t)D;
  // the row itself is staged only for an exact re-rank (most assignment rows have a
  // single certain candidate and never read it)
  auto load_xs = [&]() {
    for (int k = lane; k < Dp; k += 32) xs[k] = k < D ? __ldg(xr + k) : 0.f;
    __syncwarp();
  };
  const unsigned lt = (1u << lane) - 1u;
  SELCLK(0);
  // 1. U' >= the m-th smallest A of the row, within 8 values above it (m = 1: the
  //    minimum); any such U' makes step 2's S a superset of every candidate
  float Up;
  {
    float mn = INFINITY;
#pragma unroll
    for (int i = 0; i < NPL; ++i) mn = fminf(mn, A[i]);
    if (m == 1) {
      Up = fkey_inv(__reduce_min_sync(kFull, fkey(mn)));
    } else {
      // >= 32 >= m values are <= the largest of the lanes' minima: compact those
      const uint32_t hi = __reduce_max_sync(kFull, fkey(mn));
      uint32_t* sv = reinterpret_cast<uint32_t*>(cand);  // scratch
      int nv = 0;
#pragma unroll
      for (int i = 0; i < NPL; ++i) {
        const uint32_t kk = fkey(A[i]);
        const bool keep = kk <= hi;
        const unsigned pm = __ballot_sync(kFull, keep);
        const int pos = nv + __popc(pm & lt);
        if (keep && pos < CCAP) sv[pos] = kk;
        nv += __popc(pm);
      }
      __syncwarp();
      if (nv <= 64) {
        Up = fkey_inv(warp_mth64(lane < nv ? sv[lane] : 0xFFFFFFFFu, lane + 32 < nv ? sv[lane + 32] : 0xFFFFFFFFu,
                                 nv > 32, m));
      } else {
        // bisection on the key bits over the compacted values (or the row)
        uint32_t lo = __reduce_min_sync(kFull, fkey(mn)), h2 = hi;
        if (nv <= CCAP) {
          uint32_t u[CCAP / 32];
#pragma unroll
          for (int t = 0; t < CCAP / 32; ++t) u[t] = lane + 32 * t < nv ? sv[lane + 32 * t] : 0xFFFFFFFFu;
          while (lo < h2) {
            const uint32_t mid = lo + ((h2 - lo) >> 1);
            int c = 0;
#pragma unroll
            for (int t = 0; t < CCAP / 32; ++t) c += u[t] <= mid ? 1 : 0;
            const int tot = (int)__reduce_add_sync(kFull, (unsigned)c);
            if (tot >= m) {
              h2 = mid;
              // any key with m..m+8 values at or below it bounds the m-th smallest from
              // above: the superset S below only grows by those few columns
              if (tot <= m + 8) break;
            } else {
              lo = mid + 1;
            }
          }
        } else {
          while (lo < h2) {
            const uint32_t mid = lo + ((h2 - lo) >> 1);
            int c = 0;
#pragma unroll
            for (int i = 0; i < NPL; ++i) c += fkey(A[i]) <= mid ? 1 : 0;
            const int tot = (int)__reduce_add_sync(kFull, (unsigned)c);
            if (tot >= m) {
              h2 = mid;
              if (tot <= m + 8) break;  // as above
            } else {
              lo = mid + 1;
            }
          }
        }
        Up = fkey_inv(h2);
      }
      __syncwarp();
    }
  }
  // 2. the superset S = {l : A_l <= U' + 2 Emax} (rounded up, with slack)
  const float thr = __fadd_ru(__fadd_ru(__fadd_ru(Up, Emax), Emax), fabsf(Up) * 0x1p-20f + Emax * 0x1p-10f);
  int ns = 0;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const bool keep = A[i] <= thr;
    const unsigned pm = __ballot_sync(kFull, keep);
    const int pos = ns + __popc(pm & lt);
    if (keep && pos < CCAP) scol[pos] = lane + 32 * i;
    ns += __popc(pm);
  }
  __syncwarp();
  const bool sall = ns > CCAP;  // S too large: the whole row (the lane's register columns)
  SELCLK(1);
  // 3. U = the m-th smallest upper bound max(A + E, 0), over S
  uint32_t Ub;
  {
    auto ub_of = [&](float a, int c) { return __float_as_uint(fmaxf(a + Ecol(c), 0.f)); };
    if (!sall && ns <= 64) {
      uint32_t u0 = 0xFFFFFFFFu, u1 = 0xFFFFFFFFu;
      if (lane < ns) u0 = ub_of(__ldcs(arow + scol[lane]), scol[lane]);
      if (lane + 32 < ns) u1 = ub_of(__ldcs(arow + scol[lane + 32]), scol[lane + 32]);
      Ub = (m == 1) ? __reduce_min_sync(kFull, min(u0, u1)) : warp_mth64(u0, u1, ns > 32, m);
    } else {
      uint32_t lo = 0xFFFFFFFFu, hi = 0u;
      auto each = [&](auto&& f) {
        if (sall) {
#pragma unroll
          for (int i = 0; i < NPL; ++i)
            if (lane + 32 * i < nlist) f(ub_of(A[i], lane + 32 * i));
        } else {
          for (int t = lane; t < ns; t += 32) f(ub_of(__ldcs(arow + scol[t]), scol[t]));
        }
      };
      each([&](uint32_t u) {
        lo = min(lo, u);
        hi = max(hi, u);
      });
      lo = __reduce_min_sync(kFull, lo);
      hi = __reduce_max_sync(kFull, hi);
      while (lo < hi) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        int c = 0;
        each([&](uint32_t u) { c += u <= mid ? 1 : 0; });
        const int tot = (int)__reduce_add_sync(kFull, (unsigned)c);
        if (tot >= m) {
          hi = mid;
          // U >= the m-th smallest upper bound: the candidates below stay a superset of
          // the exact top-m (a few more may need the exact re-rank)
          if (tot <= m + 2) break;
        } else {
          lo = mid + 1;
        }
      }
      Ub = hi;
    }
  }
  SELCLK(2);
  const float U = __uint_as_float(Ub);
  // 4. candidates: lower bound <= U, from S
  int nc = 0;
  if (sall) {
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
      const int c = lane + 32 * i;
      const float e = c < nlist ? Ecol(c) : 0.f;
      const bool pass = c < nlist && A[i] - e <= U;
      const unsigned pm = __ballot_sync(kFull, pass);
      const int pos = nc + __popc(pm & lt);
      if (pass && pos < CCAP) {
        cand[pos] = c;
        capx[pos] = fmaxf(A[i], 0.f);  // the midpoint of the band
        clb[pos] = A[i] - e;
        cub[pos] = fmaxf(A[i] + e, 0.f);
      }
      nc += __popc(pm);
    }
  } else {
    for (int t0 = 0; t0 < ns; t0 += 32) {
      const int t = t0 + lane;
      int c = 0;
      float a = INFINITY;
      if (t < ns) {
        c = scol[t];
        a = __ldcs(arow + c);
      }
      const float e = t < ns ? Ecol(c) : 0.f;
      const bool pass = t < ns && a - e <= U;
      const unsigned pm = __ballot_sync(kFull, pass);
      const int pos = nc + __popc(pm & lt);
      if (pass && pos < CCAP) {
        cand[pos] = c;
        capx[pos] = fmaxf(a, 0.f);
        clb[pos] = a - e;
        cub[pos] = fmaxf(a + e, 0.f);
      }
      nc += __popc(pm);
    }
  }
  __syncwarp();
#ifdef SIVF_TC_PROF
  if (lane == 0) atomicAdd(&g_selhist[MODE][nc < 63 ? nc : 63], 1u);
#endif
  SELCLK(3);
  const bool all = nc > CCAP;
  const int total = all ? nlist : nc;
  unsigned long long bestk = ~0ull;
  if (MODE == 0 && nc == 1 && !need_dist) {
    // a single candidate is certainly the argmin; the insert path needs only the list
    if (lane == 0) best[row] = (unsigned long long)(uint32_t)cand[0];
    return;
  }
  if (MODE == 1 && nc == m) {
    // exactly m candidates: the probe SET is certain (reading C3); order by the
    // approximate distance (nearest-first only steers the scan's work order)
    unsigned long long k0 = lane < nc ? make_key(capx[lane], (uint32_t)cand[lane]) : kPadKey;
    k0 = warp_sort32(k0);
    if (lane < m) {
      probes[row * probes_ld + lane] = (int32_t)key_id(k0);
      inv_count_row(ic, nlist, row, lane, (int32_t)key_id(k0));
    }
    SELCLK(4);
    break;
  }
  if (MODE == 1 && total <= 64) {
    // m < nc <= 64 candidates.  Candidate t is certainly in the top-m when fewer
    // than m others can reach it: ub_t < L, L the (m+1)-th smallest lower bound
    // (every list with lb <= ub_t is then among the m smallest lower bounds, t
    // included).  Only the other (uncertain) candidates need the canonical dist32;
    // they go to the block's re-rank queue (their exact keys pick the remaining
    // m - #certain slots after the block barrier)
    const uint32_t k0 = lane < nc ? fkey(clb[lane]) : 0xFFFFFFFFu;
    const uint32_t k1 = lane + 32 < nc ? fkey(clb[lane + 32]) : 0xFFFFFFFFu;
    lbm = warp_kth64(k0, k1, m);  // 0-based m: the (m+1)-th smallest
    const bool u0 = lane < nc && !(fkey(cub[lane]) < lbm);
    const bool u1 = lane + 32 < nc && !(fkey(cub[lane + 32]) < lbm);
    const unsigned b0 = __ballot_sync(kFull, u0), b1 = __ballot_sync(kFull, u1);
    nu = __popc(b0) + __popc(b1);
    nce = nc - nu;
    ncand = nc;
    if (lane == 0) qbase = atomicAdd(&q_cnt, nu);
    qbase = __shfl_sync(kFull, qbase, 0);
    if (u0) {
      const int e = qbase + __popc(b0 & lt);
      q_w[e] = (uint8_t)w;
      q_l[e] = cand[lane];
    }
    if (u1) {
      const int e = qbase + __popc(b0) + __popc(b1 & lt);
      q_w[e] = (uint8_t)w;
      q_l[e] = cand[lane + 32];
    }
    load_xs();  // read by the block's re-rank queue after the barrier
    path = 1;
    SELCLK(5);
    break;
  }
  load_xs();
  if (MODE == 1) warp_topk_init(top, m);
  for (int i0 = 0; i0 < total; i0 += 32) {
    const int i = i0 + lane;
    unsigned long long key = kPadKey;
    if (i < total) {
      const int l = all ? i : cand[i];
      key = make_key(dist32_rows(xs, C + (size_t)l * Dp, D, vec), (uint32_t)l);
    }
    if (MODE == 0) bestk = umin64(bestk, key);
    else warp_topk_insert(top, tmp, m, key);
  }
  if (MODE == 0) {
#pragma unroll
    for (int off = 16; off; off >>= 1) bestk = umin64(bestk, __shfl_xor_sync(kFull, bestk, off));
    if (lane == 0) best[row] = bestk;
  } else {
    for (int j = lane; j < m; j += 32) {
      probes[row * probes_ld + j] = (int32_t)key_id(top[j]);
      inv_count_row(ic, nlist, row, j, (int32_t)key_id(top[j]));
    }
  }
  } while (0);
  if (MODE == 1) {
    __syncthreads();  // the queue is complete
    const int qn = q_cnt;
    for (int e = threadIdx.x; e < qn; e += blockDim.x) {
      const float* xw = reinterpret_cast<const float*>(sm_sel + (size_t)q_w[e] * select_smem_per_warp(Dp));
      q_d[e] = dist32_rows(xw, C + (size_t)q_l[e] * Dp, D, vec);
    }
    __syncthreads();
    if (path == 1) {
      // the m - nce best uncertain by (dist32, list), then all m probes sorted
      // (certain ones by their approximate distance: the order only steers the scan)
      unsigned long long e0 = lane < nu ? make_key(q_d[qbase + lane], (uint32_t)q_l[qbase + lane]) : kPadKey;
      unsigned long long e1 = lane + 32 < nu ? make_key(q_d[qbase + lane + 32], (uint32_t)q_l[qbase + lane + 32]) : kPadKey;
      e0 = warp_sort32(e0);
      if (nu > 32) {
        e1 = warp_sort32(e1);
        e0 = umin64(e0, __shfl_sync(kFull, e1, 31 - lane));
#pragma unroll
        for (int j = 16; j > 0; j >>= 1) {
          const unsigned long long o = __shfl_xor_sync(kFull, e0, j);
          e0 = (lane & j) ? umax64(e0, o) : umin64(e0, o);
        }
      }
      // lane j < m - nce holds the j-th chosen uncertain key; the certain ones are
      // compacted behind them
      unsigned long long fk = lane < m - nce ? e0 : kPadKey;
      int pos = m - nce;
      const unsigned lt = (1u << lane) - 1u;
      for (int t0 = 0; t0 < ncand; t0 += 32) {
        const int t = t0 + lane;
        const bool cert = t < ncand && fkey(cub[t]) < lbm;
        const unsigned bm = __ballot_sync(kFull, cert);
        const int p = pos + __popc(bm & lt);
        // route the certain key to lane p (p < m <= 32)
        const unsigned long long ck = cert ? make_key(capx[t], (uint32_t)cand[t]) : kPadKey;
        for (int src = 0; src < 32; ++src) {
          if (!((bm >> src) & 1u)) continue;
          const unsigned long long v = __shfl_sync(kFull, ck, src);
          const int ps = __shfl_sync(kFull, p, src);
          if (lane == ps) fk = v;
        }
        pos += __popc(bm);
      }
      fk = warp_sort32(fk);
      if (lane < m) {
        probes[row * probes_ld + lane] = (int32_t)key_id(fk);
        inv_count_row(ic, nlist, row, lane, (int32_t)key_id(fk));
      }
    }
  }
}

struct Bound {
  float ka, kb;
};

Bound coarse_bound(int D, int Dp) {
  const double u = 0x1p-10, w = 0x1p-23;
  // split tf32: per product |err| <= 3 u^2 (1 + u) |x_k c_k| (x_h c_l, x_l c_h through one
  // more tf32 conversion each, x_l c_l dropped); 3 Dp products accumulated in fp32
  const double e1 = 2.0 * (3.0 * u * u + 4.0 * u * u * u) + 2.0 * (3 * Dp + 4) * w;
  const double e2 = (D + 6) * w, e3 = (D + 3) * w;
  const double ka = 2.0 * (1.0 + 2.0 * e3) * e1 + 4.0 * e3;
  const double kb = 2.0 * (1.0 + 2.0 * e3) * e2 + 2.0 * e3;
  const double up = 1.0 + (D + 16) * w;  // fp32 evaluation of E and of the norms / sqrt
  return Bound{(float)(ka * up), (float)(kb * up)};
}

}  // namespace

// ---------------------------------------------------------------- host side
bool coarse_tc_supported(const Index& ix, int m) {
  const int cap = m == 1 ? ix.sc.cand_cap_assign : ix.sc.cand_cap_probe;
  return ix.use_tc_coarse && m >= 1 && m <= 32 && coarse_smem_bytes() <= ix.smem_optin &&
         4 * rerank_smem_per_warp(m, cap, ix.st.Dp) <= 48 * 1024;
}

typedef CUresult (*EncodeTiledFn2)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

cudaError_t setup_coarse_tc(Index& ix) {
  // TMA descriptor of the coarse matrix [coarse_rows][nlist] fp32 (store box 32 x 32, 128B swizzle)
  ix.coarse_tmap_ok = false;
  if ((ix.st.nlist & 3) == 0 && ix.sc.coarse_rows >= TM) {
    EncodeTiledFn2 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q) ==
            cudaSuccess &&
        enc) {
      const cuuint64_t gdim[2] = {(cuuint64_t)ix.st.nlist, (cuuint64_t)ix.sc.coarse_rows};
      const cuuint64_t gstr[1] = {(cuuint64_t)ix.st.nlist * 4};
      const cuuint32_t box[2] = {32, 32};
      const cuuint32_t estr[2] = {1, 1};
      ix.coarse_tmap_ok =
          enc(reinterpret_cast<CUtensorMap*>(ix.coarse_tmap), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, ix.sc.coarse, gdim,
              gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
      ix.qcoarse_tmap_ok = false;
      if (ix.coarse_tmap_ok && ix.sc.q_rows >= TM) {
        const cuuint64_t qdim[2] = {(cuuint64_t)ix.st.nlist, (cuuint64_t)ix.sc.q_rows};
        ix.qcoarse_tmap_ok =
            enc(reinterpret_cast<CUtensorMap*>(ix.qcoarse_tmap), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, ix.sc.qcoarse,
                qdim, gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
      }
    } else {
      cudaGetLastError();
    }
  }
  cudaError_t e = cudaFuncSetAttribute(k_coarse_gemm<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)coarse_smem_bytes(0));
  // the per-row selection path (nlist <= 1024): its shared memory grows with Dp and
  // nlist; beyond the opt-in limit the path is switched off (the fused two-pass
  // epilogue serves instead) rather than failing sivf_create
  if (ix.st.nlist > 1024 || select_smem(ix.st.Dp, ix.st.nlist) > ix.smem_optin) {
    ix.coarse_select = ix.coarse_select_ok = false;
  } else if (e == cudaSuccess) {
    const int sel = (int)select_smem(ix.st.Dp, ix.st.nlist);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_coarse_select<8, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sel);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_coarse_select<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sel);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_coarse_select<16, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sel);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_coarse_select<16, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sel);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_coarse_select<32, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sel);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_coarse_select<32, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sel);
  }
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_coarse_gemm<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)coarse_smem_bytes());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_coarse_gemm<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)coarse_smem_bytes());
  return e;
}

cudaError_t refresh_centroid_tiles(Index& ix, cudaStream_t s) {
  const int nct = (int)ceil_div(ix.st.nlist, TN);
  const Bound bd = coarse_bound(ix.st.D, ix.st.Dp);
  k_cent_tiles<<<nct, TN, 0, s>>>(ix.st.centroids, ix.st.nlist, ix.st.Dp, bd.ka, bd.kb, ix.sc.c_tiles,
                                  ix.sc.c_norm, ix.sc.c_csa, ix.sc.c_cnb);
  ix.launches += 1;
  return cudaGetLastError();
}

// The search front (probe selection) may overlap an insert's assignment when it takes the
// k_coarse_select path on its own scratch set.
bool coarse_front_concurrent_ok(const Index& ix, int32_t nprobe) {
  return coarse_tc_supported(ix, nprobe) && ix.coarse_select && ix.coarse_tmap_ok && ix.qcoarse_tmap_ok &&
         ix.st.nlist <= 1024 && ix.sc.q_rows >= TM;
}

int coarse_tc_tile_rows() { return TM; }
int coarse_tc_tile_cols() { return TN; }

// Exact top-m (m <= 32) of rows X[0..n) on tensor cores.  probes == nullptr:
// assignment (m == 1) into best[i]; else probes[i * m + j].  Rows are
// processed in chunks of sc.tc_rows.
cudaError_t launch_coarse_tc(Index& ix, const float* d_x, int64_t n, int m, unsigned long long* best,
                             int32_t* probes, cudaStream_t s, bool need_dist) {
  Scratch& sc = ix.sc;
  const DevState& st = ix.st;
  const int D = st.D, Dp = st.Dp;
  const Bound bd = coarse_bound(D, Dp);
  // capacity per row: assignment calls (up to max(batch, queries) rows) get the small cap
  const int cap = probes == nullptr ? sc.cand_cap_assign : sc.cand_cap_probe;
  const int ntn = (int)ceil_div(st.nlist, TN);
  // Fast path: store A, then a per-row selection (k_coarse_select) — nlist <= 1024
  // and chunks of >= 128 rows of the coarse scratch matrix.
  // the search front may run concurrently with an insert's assignment: it then uses
  // its own scratch set (q*), sized for max_queries rows
  const bool alt = ix.coarse_alt;
  float* const xt = alt ? sc.qx_tiles : sc.x_tiles;
  float* const xn = alt ? sc.qx_norm : sc.x_norm;
  float* const mat = alt ? sc.qcoarse : sc.coarse;
  const void* const tmat = alt ? (const void*)ix.qcoarse_tmap : (const void*)ix.coarse_tmap;
  const int64_t R = alt ? sc.q_rows
                        : (sc.tc_rows < sc.coarse_rows / TM * TM ? sc.tc_rows : sc.coarse_rows / TM * TM);
  if (ix.coarse_select && ix.coarse_tmap_ok && st.nlist <= 1024 && R >= TM) {
    const size_t ssm = select_smem(Dp, st.nlist), ssm0 = select_smem(Dp, st.nlist, 0);
    for (int64_t r0 = 0; r0 < n; r0 += R) {
      const int64_t nr = n - r0 < R ? n - r0 : R;
      const float* xr = d_x + r0 * D;
      const int64_t ntile = ceil_div(nr, TM);
      k_rows_tiles<<<ntile, 4 * TM, 0, s>>>(xr, nr, D, Dp, xt, xn);
      // split the N-tiles over CTAs until every SM has a CTA
      // (from half the SMs in row tiles on, one CTA per row tile: the extra waves and
      // per-CTA fills of a split cost more than it gains, tools/ncg_sweep.py)
      int ncg = 2 * ntile >= ix.num_sms ? 1 : (int)ceil_div(ix.num_sms, ntile);
      if ((ix.dbg >> 16) & 7) ncg = (ix.dbg >> 16) & 7;  // experiments (SIVF_OPT_DEBUG bits 16-18)
      if (ncg > ntn) ncg = ntn;
      const int ntpc = (int)ceil_div(ntn, ncg);
      CoarseArgs a{xt, xn, sc.c_tiles, sc.c_norm, sc.c_csa, sc.c_cnb, nr, Dp, st.nlist, m, 0,
                   bd.kb, nullptr, nullptr, nullptr, mat, ntpc};
      k_coarse_gemm<0><<<dim3((unsigned)ntile, (unsigned)ceil_div(ntn, ntpc)), CTHREADS, coarse_smem_bytes(0), s>>>(
          *reinterpret_cast<const CUtensorMap*>(tmat), a);
      const dim3 g((unsigned)ceil_div(nr, SELW));
#define SIVF_SEL(NPL)                                                                                          \
  if (probes == nullptr)                                                                                       \
    k_coarse_select<NPL, 0><<<g, 32 * SELW, ssm0, s>>>(mat, xr, nr, D, st.nlist, m, xn, sc.c_csa,  \
                                                       sc.c_cnb, bd.kb, st.centroids, Dp, best + r0, nullptr, 0,  \
                                                       need_dist, InvCount{nullptr, nullptr, 1, 0});              \
  else                                                                                                         \
    k_coarse_select<NPL, 1><<<g, 32 * SELW, ssm, s>>>(mat, xr, nr, D, st.nlist, m, xn, sc.c_csa,  \
                                                       sc.c_cnb, bd.kb, st.centroids, Dp, nullptr, probes + r0 * m, m, 1, \
                                                       InvCount{ix.fuse_inv_cnt, ix.sc.gthr + r0, ix.fuse_nb, ix.fuse_r0, (ix.dbg >> 6) & 1});
      if (st.nlist <= 256) {
        SIVF_SEL(8)
      } else if (st.nlist <= 512) {
        SIVF_SEL(16)
      } else {
        SIVF_SEL(32)
      }
#undef SIVF_SEL
      ix.launches += 3;
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
    if (ix.fuse_inv_cnt) ix.fuse_inv_done = true;
    return cudaSuccess;
  }
  const size_t rsm = 4 * rerank_smem_per_warp(m, cap, Dp);
  for (int64_t r0 = 0; r0 < n; r0 += sc.tc_rows) {
    const int64_t nr = n - r0 < sc.tc_rows ? n - r0 : sc.tc_rows;
    const float* xr = d_x + r0 * D;
    const int64_t ntile = ceil_div(nr, TM);
    k_rows_tiles<<<ntile, 4 * TM, 0, s>>>(xr, nr, D, Dp, sc.x_tiles, sc.x_norm);
    // Fewer row tiles than SMs (a search batch, a query slice, a small insert batch):
    // split the N-tiles over ncg CTAs per row tile (the wave count times the N-tiles
    // per CTA is minimised).  Each CTA bounds with its own range's m-th smallest upper
    // bound U_R >= the row's U_(m), so every list with lower bound <= U_(m) is still
    // appended (a superset; >= m per range) and k_coarse_rerank's exact U* over the
    // candidates is unchanged.  ncg * m stays within half the candidate capacity.
    // Only for probe selection (m > 1) on a few row tiles (a query slice of the
    // query-sharded coarse step): with m = 1 every range's running minimum starts
    // loose and the appended candidates overflow the small assignment buffers, and at
    // >= half of the SMs in row tiles the extra per-CTA pipeline fills cost more
    // than the split gains (measured, tools/coarse_cmp.py).
    int ncg = 1;
    if (m > 1 && ntile * 2 <= ix.num_sms) {
      int64_t best = -1;
      for (int c = 1; c <= ntn && c * 2 * m <= cap && c <= 16; c *= 2) {
        const int64_t t = ceil_div((int64_t)ntile * c, (int64_t)ix.num_sms) * ceil_div((int64_t)ntn, (int64_t)c);
        if (best < 0 || t < best) best = t, ncg = c;
      }
    }
    const int ntpc = (int)ceil_div((int64_t)ntn, (int64_t)ncg);
    ncg = (int)ceil_div((int64_t)ntn, (int64_t)ntpc);
    if (ncg > 1) cudaMemsetAsync(sc.cand_cnt, 0, sizeof(int32_t) * nr, s);
    CoarseArgs a{sc.x_tiles, sc.x_norm, sc.c_tiles, sc.c_norm, sc.c_csa, sc.c_cnb, nr, Dp, st.nlist, m, cap,
                 bd.kb, sc.cand, sc.cand_ubv, sc.cand_cnt, nullptr, ntpc};
    const dim3 grid((unsigned)ntile, (unsigned)ncg);
    if (m == 1)
      k_coarse_gemm<1><<<grid, CTHREADS, coarse_smem_bytes(), s>>>(*reinterpret_cast<const CUtensorMap*>(ix.coarse_tmap), a);
    else
      k_coarse_gemm<32><<<grid, CTHREADS, coarse_smem_bytes(), s>>>(*reinterpret_cast<const CUtensorMap*>(ix.coarse_tmap), a);
    if (probes == nullptr)
      k_coarse_rerank<0><<<ceil_div(nr, 4), 128, rsm, s>>>(xr, nr, D, st.centroids, Dp, st.nlist, m, sc.cand,
                                                          sc.cand_ubv, sc.cand_cnt, cap, best + r0, nullptr, 0);
    else
      k_coarse_rerank<1><<<ceil_div(nr, 4), 128, rsm, s>>>(xr, nr, D, st.centroids, Dp, st.nlist, m, sc.cand,
                                                          sc.cand_ubv, sc.cand_cnt, cap, nullptr,
                                                          probes + r0 * m, m);
    ix.launches += 3;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace sivf

#ifdef SIVF_TC_PROF
extern "C" int sivf_debug_selhist(unsigned* host) {
  return (int)cudaMemcpyFromSymbol(host, sivf::g_selhist, sizeof(unsigned) * 128);
}
extern "C" int sivf_debug_selclk(unsigned long long* host) {
  return (int)cudaMemcpyFromSymbol(host, sivf::g_selclk, sizeof(unsigned long long) * 16);
}
#endif
