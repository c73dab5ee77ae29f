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
// Error bound (u = 2^-10 tf32 operand truncation, w = 2^-23 = 2x the fp32
// unit roundoff, S = ||x|| ||c|| >= sum |x_k c_k|):
//   |2 x.c_tc - 2 x.c|   <= 2 [(2u + u^2) + (Dp + 2) w] S        (operands, fp32 accumulation)
//   norms + the 2 roundings of A            <= (D + 6) w (||x||^2 + ||c||^2) + 4 w S
//   |dist32 - d|                            <= (D + 2) w/2 d       (Higham, non-negative terms)
// E = 2 (E0 + e3 (max(A,0) + E0)),  E0 = e1 S + e2 (||x||^2 + ||c||^2),
// e1 = 2(2u+u^2) + 2(Dp+4)w, e2 = (D+6)w, e3 = (D+3)w (safety factor 2); with
// max(A,0) <= ||x||^2 + ||c||^2 + 2S + E0 this is <= ka S + kb (||x||^2 + ||c||^2),
// ka = 2(1+2e3)e1 + 4e3, kb = 2(1+2e3)e2 + 2e3 (both rounded up), the form
// evaluated per element.  A violation could only show up as a wrong assignment or
// probe set; the GPU tests compare both with the oracle bit for bit, including
// adversarial 1-ulp near-ties.
#include "sivf_host.h"

namespace sivf {

namespace {

constexpr int TM = 128;        // rows per tile (UMMA M, TMEM lanes)
constexpr int TN = 256;        // centroids per N-tile (UMMA N)
constexpr int KC = 32;         // dims per pipeline stage
constexpr int NSTG = 4;        // stage ring depth
constexpr int W_PROD = 0, W_MMA = 1, W_EPI0 = 2, NEPI = 8;
constexpr int CTHREADS = 32 * (W_EPI0 + NEPI);
constexpr size_t kStageA = (size_t)TM * KC * 4;  // 16 KB
constexpr size_t kStageB = (size_t)TN * KC * 4;  // 32 KB

struct CoarseArgs {
  const float* x_tiles;   // [ntile][Dp/4][128][4]
  const float* xnorm;     // [n]
  const float* c_tiles;   // [nct][Dp/4][256][4]
  const float* cnorm;     // [nct*256] ||c||^2 (NaN for padding columns)
  const float* ccsa;      // [nct*256] ka * ||c||
  const float* ccnb;      // [nct*256] kb * ||c||^2
  int64_t n;
  int Dp, nlist, m, cap;
  float kb;
  unsigned long long* cand;  // [n][cap] lower-bound keys (bits(max(A-E,0)) << 32 | list)
  float* cand_ub;            // [n][cap] upper bounds A+E
  int32_t* cand_cnt;         // [n] appended candidates (> cap: overflow)
};

__host__ __device__ constexpr size_t coarse_smem_bytes() {
  return (size_t)NSTG * (kStageA + kStageB)  // operand ring
         + 2 * 3 * TN * 4                    // per-N-tile column constants (double buffered)
         + TM * 32 * 4                       // half-row top-32 exchange
         + TM * 4 + 2 * TM * 4               // candidate counters, half-row bounds
         + 256;                              // barriers, TMEM base
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
__global__ void __launch_bounds__(CTHREADS, 1) k_coarse_gemm(CoarseArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  float* sA = reinterpret_cast<float*>(smem);                                  // [NSTG][16 KB]
  float* sB = reinterpret_cast<float*>(smem + NSTG * kStageA);                 // [NSTG][32 KB]
  float* colc = reinterpret_cast<float*>(smem + NSTG * (kStageA + kStageB));   // [2][3][TN]
  float* xchg = colc + 2 * 3 * TN;                                             // [TM][32]
  int* cnt_sm = reinterpret_cast<int*>(xchg + TM * 32);                        // [TM]
  float* thr_sh = reinterpret_cast<float*>(cnt_sm + TM);                       // [2][TM]
  uint64_t* full = reinterpret_cast<uint64_t*>(thr_sh + 2 * TM);
  uint64_t* empty = full + NSTG;
  uint64_t* acc_full = empty + NSTG;   // [2]
  uint64_t* acc_empty = acc_full + 2;  // [2]
  uint32_t* tmem_base_sm = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x;
  const int Dp = a.Dp, nq4 = Dp >> 2;
  const int nchunk = (Dp + KC - 1) / KC;
  const int ntn = (a.nlist + TN - 1) / TN;
  constexpr int NPASS = KP == 1 ? 1 : 2;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NSTG; ++i) {
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
      const float* xa = a.x_tiles + (size_t)tile * nq4 * TM * 4;
      uint32_t seq = 0;
      for (int t = 0; t < NPASS * ntn; ++t) {
        const float* cb = a.c_tiles + (size_t)(t % ntn) * nq4 * TN * 4;
        for (int c = 0; c < nchunk; ++c, ++seq) {
          const int st = (int)(seq % NSTG);
          mbar_wait(&empty[st], ((seq / NSTG) & 1u) ^ 1u);
          const int kc = min(KC, Dp - c * KC);
          const uint32_t ba = (uint32_t)kc * TM * 4, bb = (uint32_t)kc * TN * 4;
          mbar_arrive_expect_tx(&full[st], ba + bb);
          bulk_g2s(sA + (size_t)st * (kStageA / 4), xa + (size_t)c * KC * TM, ba, &full[st]);
          bulk_g2s(sB + (size_t)st * (kStageB / 4), cb + (size_t)c * KC * TN, bb, &full[st]);
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
          const int st = (int)(seq % NSTG);
          mbar_wait(&full[st], (seq / NSTG) & 1u);
          tc_fence_after();
          const int kc = min(KC, Dp - c * KC);
          const uint32_t a0 = smem_u32(sA + (size_t)st * (kStageA / 4));
          const uint32_t b0 = smem_u32(sB + (size_t)st * (kStageB / 4));
          for (int kk = 0; kk < (kc >> 3); ++kk)
            umma_tf32_ss(dt, umma_sdesc(a0 + (uint32_t)kk * 2u * TM * 16u, TM * 16u, 128u),
                         umma_sdesc(b0 + (uint32_t)kk * 2u * TN * 16u, TN * 16u, 128u), idesc,
                         (c > 0 || kk > 0) ? 1u : 0u);
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
    float keys[KP];
#pragma unroll
    for (int i = 0; i < KP; ++i) keys[i] = i < KP - a.m ? -INFINITY : INFINITY;
    float Uo = INFINITY;  // KP == 1: running min upper bound; KP == 32: final U (after pass 1)
    unsigned long long* crow = a.cand + (size_t)(rv ? row : 0) * a.cap;
    float* urow = a.cand_ub + (size_t)(rv ? row : 0) * a.cap;
    for (int t = 0; t < NPASS * ntn; ++t) {
      const int j = t % ntn;
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
                const int slot = atomicAdd(&cnt_sm[r], 1);
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
    if (h == 0 && rv) a.cand_cnt[row] = cnt_sm[r];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == W_MMA) tmem_dealloc(tbase, 512);
}

// X [n][D] row-major -> [n/128][Dp/4][128][4] zero padded; ||x||^2 (fp32, any order).
__global__ void __launch_bounds__(TM) k_rows_tiles(const float* __restrict__ X, int64_t n, int D, int Dp,
                                                   float* __restrict__ out, float* __restrict__ norm) {
  const int r = threadIdx.x;
  const int64_t row = (int64_t)blockIdx.x * TM + r;
  const int nq4 = Dp >> 2;
  float4* o = reinterpret_cast<float4*>(out) + (size_t)blockIdx.x * nq4 * TM + r;
  const float* xr = X + (row < n ? row : 0) * (int64_t)D;
  const bool vec = (D & 3) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
  float nrm = 0.f;
  for (int c4 = 0; c4 < nq4; ++c4) {
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
    o[(size_t)c4 * TM] = v;
    nrm = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, nrm))));
  }
  if (row < n) norm[row] = nrm;
}

// centroids [nlist][Dp] -> [nlist/256][Dp/4][256][4] zero padded; per column
// ||c||^2 (NaN for padding: such columns never become candidates), ka ||c||, kb ||c||^2.
__global__ void __launch_bounds__(TN) k_cent_tiles(const float* __restrict__ C, int nlist, int Dp, float ka,
                                                   float kb, float* __restrict__ out, float* __restrict__ cnorm,
                                                   float* __restrict__ ccsa, float* __restrict__ ccnb) {
  const int r = threadIdx.x;
  const int l = blockIdx.x * TN + r;
  const int nq4 = Dp >> 2;
  float4* o = reinterpret_cast<float4*>(out) + (size_t)blockIdx.x * nq4 * TN + r;
  const float4* cr = reinterpret_cast<const float4*>(C + (size_t)(l < nlist ? l : 0) * Dp);
  float nrm = 0.f;
  for (int c4 = 0; c4 < nq4; ++c4) {
    const float4 v = l < nlist ? cr[c4] : make_float4(0.f, 0.f, 0.f, 0.f);
    o[(size_t)c4 * TN] = v;
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

struct Bound {
  float ka, kb;
};

Bound coarse_bound(int D, int Dp) {
  const double u = 0x1p-10, w = 0x1p-23;
  const double e1 = 2.0 * (2.0 * u + u * u) + 2.0 * (Dp + 4) * w;
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

cudaError_t setup_coarse_tc(Index& ix) {
  cudaError_t e = cudaFuncSetAttribute(k_coarse_gemm<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
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

int coarse_tc_tile_rows() { return TM; }
int coarse_tc_tile_cols() { return TN; }

// Exact top-m (m <= 32) of rows X[0..n) on tensor cores.  probes == nullptr:
// assignment (m == 1) into best[i]; else probes[i * m + j].  Rows are
// processed in chunks of sc.tc_rows.
cudaError_t launch_coarse_tc(Index& ix, const float* d_x, int64_t n, int m, unsigned long long* best,
                             int32_t* probes, cudaStream_t s) {
  Scratch& sc = ix.sc;
  const DevState& st = ix.st;
  const int D = st.D, Dp = st.Dp;
  const Bound bd = coarse_bound(D, Dp);
  // capacity per row: assignment calls (up to max(batch, queries) rows) get the small cap
  const int cap = probes == nullptr ? sc.cand_cap_assign : sc.cand_cap_probe;
  const size_t rsm = 4 * rerank_smem_per_warp(m, cap, Dp);
  for (int64_t r0 = 0; r0 < n; r0 += sc.tc_rows) {
    const int64_t nr = n - r0 < sc.tc_rows ? n - r0 : sc.tc_rows;
    const float* xr = d_x + r0 * D;
    const int64_t ntile = ceil_div(nr, TM);
    k_rows_tiles<<<ntile, TM, 0, s>>>(xr, nr, D, Dp, sc.x_tiles, sc.x_norm);
    CoarseArgs a{sc.x_tiles, sc.x_norm, sc.c_tiles, sc.c_norm, sc.c_csa, sc.c_cnb, nr, Dp, st.nlist, m, cap,
                 bd.kb, sc.cand, sc.cand_ubv, sc.cand_cnt};
    if (m == 1)
      k_coarse_gemm<1><<<ntile, CTHREADS, coarse_smem_bytes(), s>>>(a);
    else
      k_coarse_gemm<32><<<ntile, CTHREADS, coarse_smem_bytes(), s>>>(a);
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
