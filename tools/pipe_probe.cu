// pipe_probe.cu — microbenchmark of the k_scan_tc stage pipeline in isolation:
// producer (cp.async.bulk 16 KB slabs) -> MMA (16 x tcgen05.mma tf32 128x32x8,
// A in TMEM) -> consumer (wait + tcgen05.ld) -> release.  Variants switch off
// the copy, the MMA or the TMEM load to find which link serialises a stage.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2601_11808_b200/csrc -I include -o tools/pipe_probe tools/pipe_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include "sivf_internal.cuh"
using namespace sivf;

constexpr int NS = 4, NCONS = 4;

template <bool COPY, bool MMA, bool LD, int SPLIT = 1>
__global__ void __launch_bounds__(32 * (2 + NCONS), 1) pipe(const float* slabs, int nslabs, int nstages,
                                                            long long* cycles) {
  extern __shared__ __align__(1024) unsigned char smem[];
  float* stage = reinterpret_cast<float*>(smem);                   // NS x 4096 floats
  uint64_t* full = reinterpret_cast<uint64_t*>(stage + NS * 4096);
  uint64_t* mmad = full + NS;
  uint64_t* empty = mmad + NS;
  uint32_t* tb = reinterpret_cast<uint32_t*>(empty + NS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) { mbar_init(&full[i], 1); mbar_init(&mmad[i], 1); mbar_init(&empty[i], NCONS); }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tb, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tb;
  long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    for (int it = 0; it < nstages; ++it) {
      const int stg = it % NS;
      mbar_wait(&empty[stg], ((it / NS) & 1u) ^ 1u);
      const int s = (blockIdx.x * 7919 + it * 104729) % nslabs;
      if (COPY) {
        mbar_arrive_expect_tx(&full[stg], 16384);
        for (int c = 0; c < SPLIT; ++c)
          bulk_g2s(stage + stg * 4096 + c * (4096 / SPLIT), slabs + (size_t)s * 4096 + c * (4096 / SPLIT),
                   16384 / SPLIT, &full[stg]);
      } else {
        mbar_arrive(&full[stg]);
      }
    }
  } else if (warp == 1 && lane == 0) {
    const uint32_t idesc = umma_idesc_tf32(128, 32);
    for (int it = 0; it < nstages; ++it) {
      const int stg = it % NS;
      mbar_wait(&full[stg], (it / NS) & 1u);
      tc_fence_after();
      if (MMA) {
        const uint32_t bsm = smem_u32(stage + stg * 4096);
        for (int kk = 0; kk < 16; ++kk)
          umma_tf32_ts(tbase + 128 + stg * 32, tbase + 8 * kk, umma_sdesc(bsm + kk * 1024u, 512u, 128u), idesc, kk > 0);
        umma_commit(&mmad[stg]);
      } else {
        mbar_arrive(&mmad[stg]);
      }
    }
  } else if (warp >= 2) {
    const int g = warp & 3;
    float acc = 0.f;
    for (int it = 0; it < nstages; ++it) {
      const int stg = it % NS;
      mbar_wait(&full[stg], (it / NS) & 1u);
      mbar_wait(&mmad[stg], (it / NS) & 1u);
      tc_fence_after();
      if (LD) {
        uint32_t v[16];
        tmem_ld16(tbase + ((uint32_t)(32 * g) << 16) + 128 + stg * 32, v);
        tmem_ld_wait();
        for (int j = 0; j < 16; ++j) acc += __uint_as_float(v[j]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stg]);
    }
    if (acc == 12345.f) cycles[1] = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd((unsigned long long*)cycles, (unsigned long long)(clock64() - t0));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tbase, 256);
}

template <bool C, bool M, bool L, int SP = 1>
void run(const char* name, const float* d, int nslabs, long long* dc) {
  const int nst = 2000, grid = 148;
  size_t smem = NS * 16384 + 3 * NS * 8 + 64;
  cudaFuncSetAttribute(pipe<C, M, L, SP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaMemset(dc, 0, 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  pipe<C, M, L, SP><<<grid, 32 * (2 + NCONS), smem>>>(d, nslabs, 50, dc);  // warm
  cudaDeviceSynchronize();
  cudaMemset(dc, 0, 16);
  cudaEventRecord(a);
  pipe<C, M, L, SP><<<grid, 32 * (2 + NCONS), smem>>>(d, nslabs, nst, dc);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, a, b);
  long long cyc; cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  printf("%-26s %s  %.3f ms  %.0f cycles/stage  %.1f GB/s\n", name, cudaGetErrorString(e), ms,
         (double)cyc / grid / nst, (double)grid * nst * 16384 / (ms * 1e-3) / 1e9);
}

int main() {
  const int nslabs = 64 * 1024;  // 1 GB of slabs (> L2)
  float* d; long long* dc;
  cudaMalloc(&d, (size_t)nslabs * 16384);
  cudaMemset(d, 0, (size_t)nslabs * 16384);
  cudaMalloc(&dc, 16);
  run<true, false, false, 32>("copy 32x512B", d, nslabs, dc);
  run<true, false, false, 8>("copy 8x2KB", d, nslabs, dc);
  run<true, false, false, 32>("copy 32x512B (L2)", d, 256, dc);
  run<false, false, false>("sync only", d, nslabs, dc);
  run<true, false, false>("copy", d, nslabs, dc);
  run<false, true, false>("mma", d, nslabs, dc);
  run<false, true, true>("mma+ld", d, nslabs, dc);
  run<true, true, false>("copy+mma", d, nslabs, dc);
  run<true, true, true>("copy+mma+ld", d, nslabs, dc);
  run<true, true, true>("copy+mma+ld (L2: 256 slabs)", d, 256, dc);
  return 0;
}
