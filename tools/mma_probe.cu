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
  uint32_t* tb = reinterpret_cast<uint32_t*>(bar + 4);  // bar[2], bar[3]: per-group commits
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 1.0f;
  if (threadIdx.x == 0) { mbar_init(bar, 1); mbar_init(bar + 2, 1); mbar_init(bar + 3, 1); fence_mbar_init(); }
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
      if (MODE >= 6) {  // 6: commit per 16 same D; 7: D switch, no commit; 8: 1 commit + D switch; 9: commit per 32
        const uint32_t dsel = MODE == 6 ? 0u : (uint32_t)((r >> 4) & 3);
        umma_tf32_ss(tbase + dsel * 128u, umma_sdesc(sa + (kk & 15) * 256u, 128u, 4096u),
                     umma_sdesc(sb + (kk & 15) * 256u, 128u, 4096u), idesc, kk > 0);
        if (MODE == 6 && kk == 15) { umma_commit(bar + 2); umma_commit(bar + 3); }
        if (MODE == 8 && kk == 15) umma_commit(bar + 2);
        if (MODE == 9 && (r & 31) == 31) umma_commit(bar + 2);
      }
      if (MODE == 5) {  // the scan's issue pattern: 16 MMAs per group into one of 4 D buffers, commit per group
        umma_tf32_ss(tbase + (uint32_t)((r >> 4) & 3) * 128u, umma_sdesc(sa + (kk & 15) * 256u, 128u, 4096u),
                     umma_sdesc(sb + (kk & 15) * 256u, 128u, 4096u), idesc, kk > 0);
        if (kk == 15) { umma_commit(bar + 2); umma_commit(bar + 3); }
      }
      if (MODE == 4)  // the scan's layout: A and B [rows/8][Dp/4][8][16 B], LBO = 128, SBO = 4096
        umma_tf32_ss(tbase + 256, umma_sdesc(sa + (kk & 15) * 256u, 128u, 4096u),
                     umma_sdesc(sb + (kk & 15) * 256u, 128u, 4096u), idesc, r > 0);
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

// LDTM throughput: NW warps each issue R tcgen05.ld 32x32b.x32 (4 KB per warp-instruction)
__global__ void ldtm_probe(int R, long long* out) {
  __shared__ uint32_t tb[1];
  if (threadIdx.x < 32) tmem_alloc(tb, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tb[0];
  const int warp = threadIdx.x >> 5;
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int r = 0; r < R; ++r) {
    uint32_t v[32];
    tmem_ld32(tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((r * 32 + warp * 64) & 511), v);
    tmem_ld_wait();
    for (int i = 0; i < 32; ++i) acc += v[i];
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (acc == 0x1234567u) out[1] = acc;
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
  for (int mode = 0; mode < (nchain == 1 ? 4 : 1); ++mode)
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
  for (int nw : {4, 8, 16}) {
    const int R = 256;
    ldtm_probe<<<148, 32 * nw>>>(R, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("LDTM %2d warps: %s %.1f cycles per warp-load, %.1f B/cycle/SM\n", nw, cudaGetErrorString(e), (double)c / R,
           (double)nw * R * 4096 / c);
  }
  {
    size_t smem = 200 * 1024 + 64;
    cudaFuncSetAttribute(probe<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe<4><<<148, 128, smem>>>(128, 512, d, 1);
    cudaError_t e = cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("tf32 SS scan layout (LBO 128, SBO 4096) N=128: %s %.1f cycles/MMA\n", cudaGetErrorString(e), (double)c / 512);
    cudaFuncSetAttribute(probe<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe<5><<<148, 128, smem>>>(128, 512, d, 1);
    e = cudaDeviceSynchronize();
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("tf32 SS scan pattern (16 MMAs + 2 commits per group, 4 D buffers): %s %.1f cycles/MMA\n", cudaGetErrorString(e), (double)c / 512);
    cudaFuncSetAttribute(probe<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(probe<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(probe<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(probe<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const char* nm[4] = {"2 commits/16, same D", "D switch/16, no commit", "1 commit/16 + D switch", "1 commit/32 + D switch/16"};
    for (int m = 6; m <= 9; ++m) {
      if (m == 6) probe<6><<<148, 128, smem>>>(128, 512, d, 1);
      if (m == 7) probe<7><<<148, 128, smem>>>(128, 512, d, 1);
      if (m == 8) probe<8><<<148, 128, smem>>>(128, 512, d, 1);
      if (m == 9) probe<9><<<148, 128, smem>>>(128, 512, d, 1);
      e = cudaDeviceSynchronize();
      cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      printf("  %s: %s %.1f cycles/MMA\n", nm[m - 6], cudaGetErrorString(e), (double)c / 512);
    }
  }
  {  // tf32 SS at N = 256 (A smem, D 256 cols)
    size_t smem = 200 * 1024 + 64;
    cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int N : {128, 192, 256}) {
      probe<1><<<148, 128, smem>>>(N, 512, d, 1);
      cudaError_t e = cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      printf("tf32 A=smem N=%d: %s %.1f cycles/MMA %.0f MAC/cycle/SM\n", N, cudaGetErrorString(e), (double)c / 512, 128.0 * N * 8 / ((double)c / 512));
    }
  }
  return 0;
}
