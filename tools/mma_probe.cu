// mma_probe.cu — tcgen05.mma issue cost per instruction vs N, A source and kind.
// One CTA per SM issues R back-to-back MMAs into TMEM, commit, wait; cycles/MMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2601_11808_b200/csrc -I include -o tools/mma_probe tools/mma_probe.cu
#include <cstdio>
#include <cstdint>
#include "sivf_internal.cuh"
using namespace sivf;

__device__ __forceinline__ void umma_f16_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void umma_f16_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
               "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

// MODE: 0 tf32 ts, 1 tf32 ss, 2 bf16 ss, 3 bf16 ts
template <int MODE>
__global__ void probe(int N, int R, long long* out, int nchain) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 200 * 1024);
  uint32_t* tb = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 1.0f;
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(tb, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tb;
  if (threadIdx.x == 0) {
    const bool bf16 = MODE >= 2;
    uint32_t idesc = bf16 ? ((1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24))
                          : umma_idesc_tf32(128, N);
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 64 * 1024);
    long long t0 = clock64();
    for (int r = 0; r < R; ++r) {
      const int kk = r & 15;
      uint64_t bd = umma_sdesc(sb + (kk & 7) * 1024u, 512u, 128u);
      const uint32_t dcol = 128 + (uint32_t)(r % nchain) * (uint32_t)N;
      if (MODE == 0) umma_tf32_ts(tbase + dcol, tbase + 8 * kk, bd, idesc, r >= nchain);
      if (MODE == 1) umma_tf32_ss(tbase + 256, umma_sdesc(sa + (kk & 7) * 4096u, 2048u, 128u), bd, idesc, r > 0);
      if (MODE == 2) umma_f16_ss(tbase + 256, umma_sdesc(sa + (kk & 7) * 4096u, 2048u, 128u), bd, idesc, r > 0);
      if (MODE == 3) umma_f16_ts(tbase + 256, tbase + 8 * kk, bd, idesc, r > 0);
    }
    umma_commit(bar);
    mbar_wait(bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tbase, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  const char* names[4] = {"tf32 A=tmem", "tf32 A=smem", "bf16 A=smem", "bf16 A=tmem"};
  for (int nchain : {1, 2, 4, 8, 12})
  for (int mode = 0; mode < 1; ++mode)
    for (int N : {32, 64, 128}) {
      if (128 + nchain * N > 512) continue;
      size_t smem = 200 * 1024 + 64;
      const int R = 512;
      cudaError_t e;
      if (mode == 0) { cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); probe<0><<<148, 128, smem>>>(N, R, d, nchain); }
      if (mode == 1) { cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); probe<1><<<148, 128, smem>>>(N, R, d, 1); }
      if (mode == 2) { cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); probe<2><<<148, 128, smem>>>(N, R, d, 1); }
      if (mode == 3) { cudaFuncSetAttribute(probe<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); probe<3><<<148, 128, smem>>>(N, R, d, 1); }
      e = cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      double k = mode >= 2 ? 16 : 8;
      printf("chains=%2d %-12s N=%3d %s  %.1f cycles/MMA  %.0f MAC/cycle/SM\n", nchain, names[mode], N, cudaGetErrorString(e),
             (double)c / R, 128.0 * N * k / ((double)c / R));
      (void)nchain;
    }
  return 0;
}
