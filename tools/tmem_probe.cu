// tmem_probe.cu — TMEM -> register read throughput (tcgen05.ld) per SM on B200.
// One CTA per SM, NW warps; warp w reads TMEM lanes 32 (w % 4) .. +31.  Each
// iteration issues `batch` loads of 32x32b.x{16,32,64} (distinct columns) and
// then one tcgen05.wait::ld; bytes/cycle/SM = total bytes / elapsed SM cycles.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2601_11808_b200/csrc -I include -o tools/tmem_probe tools/tmem_probe.cu
#include <cstdint>
#include <cstdio>

#include "sivf_internal.cuh"
using namespace sivf;

__device__ __forceinline__ void ld64(uint32_t taddr, uint32_t (&v)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
      "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
      "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]), "=r"(v[32]),
        "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]), "=r"(v[38]), "=r"(v[39]), "=r"(v[40]),
        "=r"(v[41]), "=r"(v[42]), "=r"(v[43]), "=r"(v[44]), "=r"(v[45]), "=r"(v[46]), "=r"(v[47]), "=r"(v[48]),
        "=r"(v[49]), "=r"(v[50]), "=r"(v[51]), "=r"(v[52]), "=r"(v[53]), "=r"(v[54]), "=r"(v[55]), "=r"(v[56]),
        "=r"(v[57]), "=r"(v[58]), "=r"(v[59]), "=r"(v[60]), "=r"(v[61]), "=r"(v[62]), "=r"(v[63])
      : "r"(taddr)
      : "memory");
}

// SHAPE: 16 / 32 / 64 columns per load; BATCH loads before each wait
template <int SHAPE, int BATCH>
__global__ void probe(int R, long long* out, unsigned* sink) {
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(&tb, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = tb + ((uint32_t)(32 * (warp & 3)) << 16);
  unsigned acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < R; ++r) {
#pragma unroll
    for (int b = 0; b < BATCH; ++b) {
      const uint32_t col = (uint32_t)(((r * BATCH + b) * SHAPE) & 511);
      if (SHAPE == 16) {
        uint32_t v[16];
        tmem_ld16(base + col, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) acc ^= v[i];
      } else if (SHAPE == 32) {
        uint32_t v[32];
        tmem_ld32(base + col, v);
        if (b == BATCH - 1) tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += v[i];
      } else {
        uint32_t v[64];
        ld64(base + col, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 64; ++i) acc += v[i];
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tb, 512);
}

template <int SHAPE, int BATCH>
void run(int nw) {
  const int R = 2000;
  long long* d;
  unsigned* s;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&s, 4);
  probe<SHAPE, BATCH><<<148, 32 * nw>>>(R, d, s);
  probe<SHAPE, BATCH><<<148, 32 * nw>>>(R, d, s);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0, sum = 0;
  for (int i = 0; i < 148; ++i) {
    mx = h[i] > mx ? h[i] : mx;
    sum += h[i];
  }
  const double bytes = (double)nw * 32 * SHAPE * 4 * BATCH * R;
  printf("shape x%-2d batch %d warps %2d: %.1f B/cyc/SM (avg cycles %.0f) err=%d\n", SHAPE, BATCH, nw,
         bytes / ((double)sum / 148), (double)sum / 148, (int)e);
  cudaFree(d);
  cudaFree(s);
}

int main() {
  for (int nw : {4, 8, 16}) {
    run<16, 1>(nw);
    run<32, 1>(nw);
    run<32, 2>(nw);
    run<64, 1>(nw);
  }
  return 0;
}
