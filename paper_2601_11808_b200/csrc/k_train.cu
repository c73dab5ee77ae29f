// k_train.cu — Lloyd k-means for the coarse quantizer (SURVEY §8(a) a1,
// reading C31; the paper assumes a trained quantizer).
//
// Per iteration: exact assignment by (dist32, list) (k_coarse.cu); empty
// clusters take the point of the largest cluster farthest from its centroid;
// stable member lists per cluster (k_insert.cu's chunk ranks); each centroid
// coordinate = fp32(sum_fp64 over members in ascending point order / count).
// Every step is deterministic, so the result is bit-identical to a
// sequential implementation of the same definition.
#include "sivf_host.h"

namespace sivf {

namespace {

__device__ __forceinline__ uint64_t km_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_iota(int32_t* p, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = (int32_t)i;
}

// Partial Fisher-Yates: for i < nlist, j = i + H(seed, i) mod (n - i), swap.
__global__ void k_fisher_yates(int32_t* perm, int64_t n, int nlist, uint64_t seed) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int64_t i = 0; i < nlist; ++i) {
    const uint64_t h = km_mix64(seed ^ km_mix64((uint64_t)i));
    const int64_t j = i + (int64_t)(h % (uint64_t)(n - i));
    const int32_t t = perm[i];
    perm[i] = perm[j];
    perm[j] = t;
  }
}

__global__ void k_init_centroids(const float* __restrict__ X, const int32_t* __restrict__ perm, int nlist, int D,
                                 int Dp, float* __restrict__ C) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)nlist * Dp) return;
  const int l = (int)(e / Dp), k = (int)(e % Dp);
  C[e] = k < D ? X[(int64_t)perm[l] * D + k] : 0.f;
}

// Empty-cluster rule, clusters in ascending order: largest cluster L (ties
// lowest index); its point with the largest assignment distance (ties lowest
// point index) moves to the empty cluster with distance 0.
__global__ void __launch_bounds__(1024) k_fix_empty(unsigned long long* __restrict__ best, int64_t n,
                                                    int32_t* __restrict__ cnt, int nlist) {
  __shared__ unsigned long long red[32];
  __shared__ int32_t empties[1024];
  __shared__ int32_t nemp;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  for (int e0 = 0; e0 < nlist; e0 += 1024) {
    if (t == 0) nemp = 0;
    __syncthreads();
    const int e = e0 + t;
    const bool emp = e < nlist && cnt[e] == 0;
    const unsigned b = __ballot_sync(kFull, emp);
    if (lane == 0) red[w] = b;
    __syncthreads();
    if (t == 0) {  // compact empties in ascending order
      int m = 0;
      for (int ww = 0; ww < 32; ++ww) {
        unsigned bb = (unsigned)red[ww];
        while (bb) {
          int bit = __ffs(bb) - 1;
          bb &= bb - 1;
          empties[m++] = e0 + ww * 32 + bit;
        }
      }
      nemp = m;
    }
    __syncthreads();
    for (int ei = 0; ei < nemp; ++ei) {
      // L = argmax cnt, ties lowest: key = (cnt << 32) | (~l) maximised
      unsigned long long kbest = 0;
      for (int l = t; l < nlist; l += 1024)
        kbest = umax64(kbest, ((unsigned long long)(uint32_t)cnt[l] << 32) | (0xffffffffu - (uint32_t)l));
      for (int off = 16; off; off >>= 1) kbest = umax64(kbest, __shfl_xor_sync(kFull, kbest, off));
      if (lane == 0) red[w] = kbest;
      __syncthreads();
      if (w == 0) {
        unsigned long long v = red[lane];
        for (int off = 16; off; off >>= 1) v = umax64(v, __shfl_xor_sync(kFull, v, off));
        if (lane == 0) red[0] = v;
      }
      __syncthreads();
      const uint32_t L = 0xffffffffu - (uint32_t)(red[0] & 0xffffffffu);
      __syncthreads();
      // p = argmax dist among members of L, ties lowest index: key = (dist bits << 32) | ~i
      unsigned long long pbest = 0;
      for (int64_t i = t; i < n; i += 1024) {
        const unsigned long long b2 = best[i];
        if ((uint32_t)(b2 & 0xffffffffu) == L)
          pbest = umax64(pbest, (b2 & 0xffffffff00000000ull) | (0xffffffffu - (uint32_t)i));
      }
      for (int off = 16; off; off >>= 1) pbest = umax64(pbest, __shfl_xor_sync(kFull, pbest, off));
      if (lane == 0) red[w] = pbest;
      __syncthreads();
      if (t == 0) {
        unsigned long long v = 0;
        for (int ww = 0; ww < 32; ++ww) v = umax64(v, red[ww]);
        const int64_t p = (int64_t)(0xffffffffu - (uint32_t)(v & 0xffffffffu));
        const int eidx = empties[ei];
        best[p] = (unsigned long long)(uint32_t)eidx;  // dist 0, list e
        cnt[L] -= 1;
        cnt[eidx] += 1;
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(1024) k_excl_scan(const int32_t* __restrict__ cnt, int nlist,
                                                    int32_t* __restrict__ off) {
  __shared__ int32_t ws[32];
  __shared__ int32_t carry;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t == 0) carry = 0;
  __syncthreads();
  for (int l0 = 0; l0 < nlist; l0 += 1024) {
    const int l = l0 + t;
    const int c = l < nlist ? cnt[l] : 0;
    int v = c;
    for (int o = 1; o < 32; o <<= 1) {
      int a = __shfl_up_sync(kFull, v, o);
      if (lane >= o) v += a;
    }
    if (lane == 31) ws[w] = v;
    __syncthreads();
    if (w == 0) {
      int x = ws[lane];
      for (int o = 1; o < 32; o <<= 1) {
        int a = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += a;
      }
      ws[lane] = x;
    }
    __syncthreads();
    if (l < nlist) off[l] = carry + (w ? ws[w - 1] : 0) + v - c;
    __syncthreads();
    if (t == 0) carry += ws[31];
    __syncthreads();
  }
  if (t == 0) off[nlist] = carry;
}

__global__ void k_members(const int32_t* __restrict__ list, const int32_t* __restrict__ rank,
                          const int32_t* __restrict__ hist, const int32_t* __restrict__ off, int64_t n, int nlist,
                          int32_t* __restrict__ members) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int l = list[i];
  members[off[l] + hist[(i >> 10) * nlist + l] + rank[i]] = (int32_t)i;
}

__global__ void k_centroid_update(const float* __restrict__ X, const int32_t* __restrict__ members,
                                  const int32_t* __restrict__ off, int nlist, int D, int Dp, float* __restrict__ C) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)nlist * D) return;
  const int l = (int)(e / D), k = (int)(e % D);
  const int b = off[l], en = off[l + 1];
  double s = 0.0;
  for (int m = b; m < en; ++m) s = __dadd_rn(s, (double)X[(int64_t)members[m] * D + k]);
  C[(int64_t)l * Dp + k] = __double2float_rn(__ddiv_rn(s, (double)(en - b)));
}

}  // namespace

cudaError_t launch_train(Index& ix, const float* d_x, int64_t n, int32_t niter, cudaStream_t s) {
  Scratch& sc = ix.sc;
  DevState& st = ix.st;
  const int nlist = st.nlist;
  k_iota<<<ceil_div(n, 256), 256, 0, s>>>(sc.train_perm, n);
  k_fisher_yates<<<1, 32, 0, s>>>(sc.train_perm, n, nlist, ix.cfg.seed);
  cudaMemsetAsync(st.centroids, 0, sizeof(float) * nlist * st.Dp, s);
  k_init_centroids<<<ceil_div((int64_t)nlist * st.Dp, 256), 256, 0, s>>>(d_x, sc.train_perm, nlist, st.D, st.Dp,
                                                                         st.centroids);
  ix.launches += 3;
  for (int it = 0; it < niter; ++it) {
    cudaError_t e = refresh_centroid_tiles(ix, s);
    if (e != cudaSuccess) return e;
    e = launch_assign_exact(ix, d_x, n, s);
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(sc.row_status, 0, sizeof(int32_t) * n, s);
    e = launch_stable_ranks(ix, n, 0, s);
    if (e != cudaSuccess) return e;
    k_fix_empty<<<1, 1024, 0, s>>>(sc.row_best, n, sc.list_cnt, nlist);
    e = launch_stable_ranks(ix, n, 0, s);  // ranks after the moves
    if (e != cudaSuccess) return e;
    k_excl_scan<<<1, 1024, 0, s>>>(sc.list_cnt, nlist, sc.train_off);
    k_members<<<ceil_div(n, 256), 256, 0, s>>>(sc.row_list, sc.row_rank, sc.chunk_hist, sc.train_off, n, nlist,
                                               sc.train_members);
    k_centroid_update<<<ceil_div((int64_t)nlist * st.D, 256), 256, 0, s>>>(d_x, sc.train_members, sc.train_off,
                                                                           nlist, st.D, st.Dp, st.centroids);
    ix.launches += 4;
  }
  return refresh_centroid_tiles(ix, s);
}

}  // namespace sivf
