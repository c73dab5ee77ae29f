// k_coarse.cu — exact coarse quantisation on CUDA cores (canonical dist32).
//
// The coarse step ("coarse quantization ... to obtain list assignments";
// P:338 "probes nprobe coarse lists") must agree bit-for-bit with the
// oracle's assignment and probe sets (BASELINE.json north_star; readings
// C1-C3).  Every (vector, centroid) distance here is the canonical dist32:
// fp32, ascending dimension order, t = x - c, s = s + t*t with each op
// individually rounded (__fsub_rn/__fmul_rn/__fadd_rn are never contracted).
// Zero padding of dims [D, Dp) adds exact zeros and leaves s unchanged.
//
// k_dist_exact: 64x64 output tile per CTA, 4x4 register tile per thread, K
// staged through shared memory in 32-dim slices.  MODE 0 fuses argmin over
// centroids (key = dist bits << 32 | list, one 64-bit atomicMin per row and
// CTA); MODE 1 writes the distance matrix for the probe selection.
#include "sivf_host.h"

namespace sivf {

namespace {

constexpr int BM = 64, BN = 64, BK = 32;

template <int MODE>
__global__ void __launch_bounds__(256) k_dist_exact(const float* __restrict__ X, int64_t n, int D,
                                                    const float* __restrict__ C, int Dp, int nlist,
                                                    unsigned long long* __restrict__ best, float* __restrict__ out,
                                                    int64_t out_ld) {
  __shared__ __align__(16) float Xs[BK][BM + 4];
  __shared__ __align__(16) float Cs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t row0 = (int64_t)blockIdx.y * BM;
  const int col0 = blockIdx.x * BN;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < Dp; k0 += BK) {
#pragma unroll
    for (int e = tid; e < BM * BK; e += 256) {
      int r = e / BK, kk = e % BK;
      int64_t row = row0 + r;
      int k = k0 + kk;
      Xs[kk][r] = (row < n && k < D) ? X[row * D + k] : 0.f;
      int col = col0 + r;
      Cs[kk][r] = (col < nlist && k < Dp) ? C[(int64_t)col * Dp + k] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < BK; ++kk) {
      float4 xv = *reinterpret_cast<const float4*>(&Xs[kk][ty * 4]);
      float4 cv = *reinterpret_cast<const float4*>(&Cs[kk][tx * 4]);
      float xa[4] = {xv.x, xv.y, xv.z, xv.w};
      float ca[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float t = __fsub_rn(xa[i], ca[j]);
          acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(t, t));
        }
    }
    __syncthreads();
  }

  if (MODE == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      unsigned long long key = ~0ull;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int col = col0 + tx * 4 + j;
        if (col < nlist) key = umin64(key, make_key(acc[i][j], (uint32_t)col));
      }
#pragma unroll
      for (int off = 8; off >= 1; off >>= 1) key = umin64(key, __shfl_xor_sync(kFull, key, off));
      int64_t row = row0 + ty * 4 + i;
      if (tx == 0 && row < n) atomicMin(&best[row], key);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int64_t row = row0 + ty * 4 + i;
      if (row >= n) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int col = col0 + tx * 4 + j;
        if (col < nlist) out[row * out_ld + col] = acc[i][j];
      }
    }
  }
}

// One warp per query: the nprobe smallest (dist32, list) keys of a row of the
// coarse distance matrix (reading C3: the SET matters; output is sorted).
__global__ void k_select_probes(const float* __restrict__ dist, int64_t nq, int64_t q_base, int nlist, int nprobe,
                                int32_t* __restrict__ probes, int probes_ld) {
  extern __shared__ __align__(16) unsigned long long sm_sel[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + w;
  unsigned long long* top = sm_sel + (size_t)w * 2 * nprobe;
  unsigned long long* tmp = top + nprobe;
  if (q >= nq) return;  // warp-uniform
  warp_topk_init(top, nprobe);
  const float* row = dist + q * nlist;
  for (int l0 = 0; l0 < nlist; l0 += 32) {
    int l = l0 + lane;
    uint64_t key = l < nlist ? make_key(row[l], (uint32_t)l) : kPadKey;
    warp_topk_insert(top, tmp, nprobe, key);
  }
  for (int j = lane; j < nprobe; j += 32) probes[(q_base + q) * probes_ld + j] = (int32_t)key_id(top[j]);
}

}  // namespace

// k_select_probes keeps 2 nprobe keys per warp (4 warps) in dynamic shared memory:
// 64 nprobe B, beyond the 48 KB default for nprobe > 768.
cudaError_t setup_coarse_exact(Index& ix) {
  const size_t need = sizeof(unsigned long long) * 2 * (size_t)ix.cfg.max_nprobe * 4;
  if (need <= 48 * 1024) return cudaSuccess;
  if (need > ix.smem_optin) return cudaErrorInvalidValue;
  return cudaFuncSetAttribute(k_select_probes, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need);
}

cudaError_t launch_assign_exact(Index& ix, const float* d_x, int64_t n, cudaStream_t s, bool need_dist) {
  if (n <= 0) return cudaSuccess;
  PhaseTimer pt(ix, SIVF_PH_ASSIGN, s);
  if (coarse_tc_supported(ix, 1)) return launch_coarse_tc(ix, d_x, n, 1, ix.sc.row_best, nullptr, s, need_dist);
  cudaMemsetAsync(ix.sc.row_best, 0xff, sizeof(unsigned long long) * n, s);
  dim3 grid(ceil_div(ix.st.nlist, BN), ceil_div(n, BM));
  k_dist_exact<0><<<grid, 256, 0, s>>>(d_x, n, ix.st.D, ix.st.centroids, ix.st.Dp, ix.st.nlist, ix.sc.row_best,
                                        nullptr, 0);
  ix.launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_probe_exact(Index& ix, const float* d_q, int64_t nq, int32_t nprobe, cudaStream_t s) {
  const int nlist = ix.st.nlist;
  const int64_t rows = ix.sc.coarse_rows;
  PhaseTimer pt(ix, SIVF_PH_COARSE, s);
  if (coarse_tc_supported(ix, nprobe)) return launch_coarse_tc(ix, d_q, nq, nprobe, nullptr, ix.sc.probes, s);
  for (int64_t q0 = 0; q0 < nq; q0 += rows) {
    int64_t m = nq - q0 < rows ? nq - q0 : rows;
    dim3 grid(ceil_div(nlist, BN), ceil_div(m, BM));
    k_dist_exact<1><<<grid, 256, 0, s>>>(d_q + q0 * ix.st.D, m, ix.st.D, ix.st.centroids, ix.st.Dp, nlist, nullptr,
                                          ix.sc.coarse, nlist);
    const int wpb = 4;
    size_t smem = sizeof(unsigned long long) * 2 * nprobe * wpb;
    k_select_probes<<<ceil_div(m, wpb), 32 * wpb, smem, s>>>(ix.sc.coarse, m, q0, nlist, nprobe, ix.sc.probes,
                                                             nprobe);
    ix.launches += 2;
  }
  return cudaGetLastError();
}

}  // namespace sivf
