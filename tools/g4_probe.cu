// g4_probe.cu — TMA tile::gather4 as the slab-group interleaver.
// The payload [num_slabs][Dp/4][32][4] viewed as a 2-D tensor of rows of 512 B
// (row = slab * Dp/4 + c4).  One gather4 of rows {s0,s1,s2,s3}*Dp/4 + c4 lands
// [4][128 floats] in shared memory = the [c4][4 slabs][32][4] interleaved UMMA
// B layout of k_scan_tc.  Checks the layout, then measures the streaming rate
// (random 4-slab groups, NST-stage ring, 1 CTA/SM) against 16-KB bulk copies.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2601_11808_b200/csrc -I include -o tools/g4_probe tools/g4_probe.cu
#include <cuda.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "sivf_internal.cuh"
using namespace sivf;

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ void g4(void* dst, const CUtensorMap* tm, int col, int r0, int r1, int r2, int r3,
                                   uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

constexpr int DP = 128, NQ4 = DP / 4, GB = 4 * 32 * DP * 4;  // 64 KB per group

__global__ void k_check(const __grid_constant__ CUtensorMap tm, float* out, const int* slabs) {
  extern __shared__ __align__(1024) unsigned char smem[];
  float* buf = reinterpret_cast<float*>(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + GB);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(bar, GB);
    for (int c4 = 0; c4 < NQ4; ++c4)
      g4(buf + c4 * 512, &tm, 0, slabs[0] * NQ4 + c4, slabs[1] * NQ4 + c4, slabs[2] * NQ4 + c4, slabs[3] * NQ4 + c4, bar);
  }
  mbar_wait(bar, 0);
  for (int i = threadIdx.x; i < GB / 4; i += blockDim.x) out[i] = buf[i];
}

template <bool GATHER>
__global__ void __launch_bounds__(64, 1) k_stream(const __grid_constant__ CUtensorMap tm, const float* payload,
                                                  int nslabs, int ngroups, int nst, unsigned* sink) {
  extern __shared__ __align__(1024) unsigned char smem[];
  float* st = reinterpret_cast<float*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)nst * GB);
  uint64_t* empty = full + nst;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0 && lane == 0) {
    for (int g = 0; g < ngroups; ++g) {
      const int s = g % nst;
      mbar_wait(&empty[s], ((g / nst) & 1u) ^ 1u);
      mbar_arrive_expect_tx(&full[s], GB);
      int sl[4];
      for (int j = 0; j < 4; ++j)
        sl[j] = (int)(((unsigned)(blockIdx.x * 7919 + g * 4 + j) * 2654435761u) % (unsigned)nslabs);
      float* dst = st + (size_t)s * (GB / 4);
      if (GATHER) {
        for (int c4 = 0; c4 < NQ4; ++c4)
          g4(dst + c4 * 512, &tm, 0, sl[0] * NQ4 + c4, sl[1] * NQ4 + c4, sl[2] * NQ4 + c4, sl[3] * NQ4 + c4, &full[s]);
      } else {
        for (int j = 0; j < 4; ++j) bulk_g2s(dst + j * 4096, payload + (size_t)sl[j] * 4096, 16384, &full[s]);
      }
    }
  } else if (warp == 1) {
    unsigned acc = 0;
    for (int g = 0; g < ngroups; ++g) {
      const int s = g % nst;
      mbar_wait(&full[s], (g / nst) & 1u);
      acc += __float_as_uint(st[(size_t)s * (GB / 4) + lane * 33]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 0x12345u) sink[0] = acc;
  }
}

// one warp per CTA copies each group with cp.async (16 B per lane, L2-only),
// writing the interleaved layout directly: lane = slot, dst = c4*2048 + j*512 + slot*16
template <int NW>
__global__ void __launch_bounds__(32 * (NW + 1), 1) k_stream_cpasync(const float* payload, int nslabs, int ngroups,
                                                                  int nst, unsigned* sink) {
  extern __shared__ __align__(1024) unsigned char smem[];
  float* st = reinterpret_cast<float*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)nst * GB);
  uint64_t* empty = full + nst;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) { mbar_init(&full[i], 32 * NW); mbar_init(&empty[i], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp < NW) {
    for (int g = 0; g < ngroups; ++g) {
      const int s = g % nst;
      mbar_wait(&empty[s], ((g / nst) & 1u) ^ 1u);
      const uint32_t dst = smem_u32(st + (size_t)s * (GB / 4));
#pragma unroll 1
      for (int j = warp; j < 4; j += NW) {
        const int sl = (int)(((unsigned)(blockIdx.x * 7919 + g * 4 + j) * 2654435761u) % (unsigned)nslabs);
        const float* src = payload + (size_t)sl * 4096 + lane * 4;
#pragma unroll 8
        for (int c4 = 0; c4 < NQ4; ++c4)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + c4 * 2048 + j * 512 + lane * 16),
                       "l"(src + c4 * 128)
                       : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[s])) : "memory");
    }
  } else if (warp == NW) {
    unsigned acc = 0;
    for (int g = 0; g < ngroups; ++g) {
      const int s = g % nst;
      mbar_wait(&full[s], (g / nst) & 1u);
      acc += __float_as_uint(st[(size_t)s * (GB / 4) + lane * 33]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 0x12345u) sink[0] = acc;
  }
}

int main() {
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  if (!enc) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
  const int nslabs = 46024;
  const size_t nfl = (size_t)nslabs * 32 * DP;
  std::vector<float> h(nfl);
  for (size_t i = 0; i < nfl; ++i) h[i] = (float)(i % 1000003);
  float* d;
  cudaMalloc(&d, nfl * 4);
  cudaMemcpy(d, h.data(), nfl * 4, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  cuuint64_t gdim[2] = {128, (cuuint64_t)nslabs * NQ4};
  cuuint64_t gstr[1] = {512};
  cuuint32_t estr[2] = {1, 1};
  for (int boxr : {1, 4}) {
    cuuint32_t box[2] = {128, (cuuint32_t)boxr};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, gdim, gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode box rows %d -> %d\n", boxr, (int)r);
    if (r != CUDA_SUCCESS) continue;
    int hs[4] = {17, 3, 40000, 17};
    int* ds;
    float* dout;
    cudaMalloc(&ds, 16);
    cudaMalloc(&dout, GB);
    cudaMemcpy(ds, hs, 16, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_check, cudaFuncAttributeMaxDynamicSharedMemorySize, GB + 64);
    k_check<<<1, 256, GB + 64>>>(tm, dout, ds);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> o(GB / 4);
    cudaMemcpy(o.data(), dout, GB, cudaMemcpyDeviceToHost);
    long bad = 0;
    for (int c4 = 0; c4 < NQ4; ++c4)
      for (int j = 0; j < 4; ++j)
        for (int t = 0; t < 128; ++t)
          bad += o[(c4 * 4 + j) * 128 + t] != h[((size_t)hs[j] * NQ4 + c4) * 128 + t];
    printf("  check: err=%s mismatches=%ld\n", cudaGetErrorString(e), bad);
    if (bad || e) continue;
    unsigned* sink;
    cudaMalloc(&sink, 4);
    for (int nst : {2, 3})
    for (int ns : {nslabs, 2000}) {
      const size_t sm = (size_t)nst * GB + 256;
      cudaFuncSetAttribute(k_stream<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      cudaFuncSetAttribute(k_stream<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      cudaFuncSetAttribute(k_stream_cpasync<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      cudaFuncSetAttribute(k_stream_cpasync<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      cudaFuncSetAttribute(k_stream_cpasync<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      const int ng = 200;
      for (int gather = 0; gather < 5; ++gather) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int rep = 0; rep < 3; ++rep) {
          cudaEventRecord(a);
          if (gather == 1) k_stream<true><<<148, 64, sm>>>(tm, d, ns, ng, nst, sink);
          else if (gather == 0) k_stream<false><<<148, 64, sm>>>(tm, d, ns, ng, nst, sink);
          else if (gather == 2) k_stream_cpasync<1><<<148, 64, sm>>>(d, ns, ng, nst, sink);
          else if (gather == 3) k_stream_cpasync<2><<<148, 96, sm>>>(d, ns, ng, nst, sink);
          else k_stream_cpasync<4><<<148, 160, sm>>>(d, ns, ng, nst, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (rep == 2)
            printf("  nst %d slabs %d %s: %.3f ms  %.0f GB/s  (err %s)\n", nst, ns,
                   gather == 1 ? "gather4" : gather == 0 ? "bulk16K" : gather == 2 ? "cpasync1w" : gather == 3 ? "cpasync2w" : "cpasync4w", ms,
                   148.0 * ng * GB / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
      }
    }
  }
  return 0;
}
