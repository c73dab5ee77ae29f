// tc_probe.cu — standalone check of the tcgen05 building blocks used by the
// scan/coarse kernels: TMEM alloc, tcgen05.st of the A tile (queries, fp32 as
// tf32), tcgen05.mma kind::tf32 with A in TMEM and B (a 32-slot slab in the
// dim-interleaved [D/4][32][4] layout) in shared memory, tcgen05.ld of D.
// Also the SS variant (A in smem, same interleaved layout, 128 rows).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_probe tools/tc_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (sm100)
  // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
  return d;
}

__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4)            // c_format F32
       | (2u << 7)            // a_format TF32
       | (2u << 10)           // b_format TF32
       | ((uint32_t)(N >> 3) << 17)
       | ((uint32_t)(M >> 4) << 24);
}

template <int MODE>  // 0: A in TMEM (ts), 1: A in smem (ss)
__global__ void probe(const float* A, const float* B, float* D, int K, int N) {
  // A [128][K] row-major, B [N][K] row-major (N = 32*nslab), D [128][N]
  extern __shared__ __align__(128) unsigned char smem[];
  float* sB = reinterpret_cast<float*>(smem);                  // [K/4][N][4]
  float* sA = sB + (size_t)K * N;                               // [K/4][128][4]
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < N * K; e += blockDim.x) {
    int r = e / K, k = e % K;
    sB[((k >> 2) * N + r) * 4 + (k & 3)] = B[e];
  }
  for (int e = tid; e < 128 * K; e += blockDim.x) {
    int r = e / K, k = e % K;
    sA[((k >> 2) * 128 + r) * 4 + (k & 3)] = A[e];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tmem_base;
  const uint32_t a_col = 0, d_col = 256;
  if (MODE == 0) {
    // each of 4 warps writes its 32 lanes: A row (32*warp + lane), K columns
    const int row = 32 * warp + lane;
    for (int c0 = 0; c0 < K; c0 += 8) {
      uint32_t v[8];
      for (int j = 0; j < 8; ++j) v[j] = __float_as_uint(A[(size_t)row * K + c0 + j]);
      uint32_t taddr = tbase + ((uint32_t)(32 * warp) << 16) + a_col + c0;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                   "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(128, N);
    for (int kk = 0; kk < K / 8; ++kk) {
      uint64_t bdesc = make_sdesc(smem_u32(sB) + kk * 2 * N * 16, N * 16, 128);
      uint32_t acc = kk > 0;
      if (MODE == 0) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tbase + d_col),
                     "r"(tbase + a_col + kk * 8), "l"(bdesc), "r"(idesc), "r"(acc));
      } else {
        uint64_t adesc = make_sdesc(smem_u32(sA) + kk * 2 * 128 * 16, 128 * 16, 128);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase + d_col),
                     "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  // wait for MMA completion
  asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
      smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    const int row = 32 * warp + lane;
    for (int c0 = 0; c0 < N; c0 += 16) {
      uint32_t v[16];
      uint32_t taddr = tbase + ((uint32_t)(32 * warp) << 16) + d_col + c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                   : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int j = 0; j < 16; ++j) D[(size_t)row * N + c0 + j] = __uint_as_float(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
}

int main() {
  const int K = 128;
  int fails = 0;
  for (int mode = 0; mode < 2; ++mode)
    for (int N : {32, 64, 128}) {
      std::vector<float> A(128 * K), B((size_t)N * K), D((size_t)128 * N);
      srand(1 + N + mode);
      for (auto& x : A) x = (float)(rand() % 256);
      for (auto& x : B) x = (float)(rand() % 256);
      float *dA, *dB, *dD;
      cudaMalloc(&dA, A.size() * 4);
      cudaMalloc(&dB, B.size() * 4);
      cudaMalloc(&dD, D.size() * 4);
      cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
      cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
      cudaMemset(dD, 0, D.size() * 4);
      size_t smem = ((size_t)K * N + (size_t)128 * K) * 4;
      if (mode == 0) {
        cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        probe<0><<<1, 128, smem>>>(dA, dB, dD, K, N);
      } else {
        cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        probe<1><<<1, 128, smem>>>(dA, dB, dD, K, N);
      }
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      double maxerr = 0;
      int bad = 0;
      for (int i = 0; i < 128; ++i)
        for (int j = 0; j < N; ++j) {
          double ref = 0;
          for (int k = 0; k < K; ++k) ref += (double)A[i * K + k] * B[(size_t)j * K + k];
          double err = fabs(ref - D[(size_t)i * N + j]);
          if (err > maxerr) maxerr = err;
          if (err != 0) bad++;
        }
      printf("mode=%s N=%d err=%s maxerr=%g bad=%d  D[0]=%g ref0=%g\n", mode ? "ss" : "ts", N, cudaGetErrorString(e),
             maxerr, bad, D[0], [&] { double r = 0; for (int k = 0; k < K; ++k) r += (double)A[k] * B[k]; return r; }());
      fails += bad != 0 || e != cudaSuccess;
      cudaFree(dA);
      cudaFree(dB);
      cudaFree(dD);
    }
  printf("%s\n", fails ? "FAIL" : "ALL OK");
  return fails;
}
