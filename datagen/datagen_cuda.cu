/* datagen_cuda.cu — device driver for sivf_datagen.h (harness code, not the
 * product: libsivfgen_cuda.so is loaded by bench.py / tests only).
 *
 * The same (seed, g) -> vector map as datagen_host.c, evaluated on the GPU so
 * that 100M-vector workloads (BASELINE configs[4]) need no host staging.  Every
 * fp32 op goes through __fmul_rn / __fadd_rn (sivf_datagen.h), so device and
 * host outputs are bit-identical (tests/test_datagen.py checks it on a GPU).
 * Vector i of a call is g = g0 + i * gstride (gstride = G for rank-local ids
 * of an id-sharded index).
 */
#include <cuda_runtime.h>
#include <stdint.h>

#include "sivf_datagen.h"

namespace {

constexpr int kThreads = 128;
constexpr int kMaxR = 64;

/* model tables: mu[M][D], A[M][D][r] */
__global__ void k_tables(sivfgen_params p, float* mu, float* A) {
  const int m = blockIdx.x;
  for (int k = threadIdx.x; k < p.dim; k += blockDim.x) {
    mu[(size_t)m * p.dim + k] = sivfgen_mu(&p, m, k);
    for (int j = 0; j < p.r; ++j) A[((size_t)m * p.dim + k) * p.r + j] = sivfgen_basis(&p, m, k, j);
  }
}

/* block per vector (grid-stride); threads = coordinates */
__global__ void __launch_bounds__(kThreads) k_range(sivfgen_params p, const float* __restrict__ mu,
                                                    const float* __restrict__ A, uint64_t g0, uint64_t gstride,
                                                    int64_t n, float* __restrict__ out) {
  __shared__ float z[kMaxR];
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const uint64_t g = g0 + (uint64_t)i * gstride;
    float* o = out + (size_t)i * p.dim;
    if (p.kind == SIVFGEN_UNIFORM) {
      for (int k = threadIdx.x; k < p.dim; k += blockDim.x) o[k] = sivfgen_uniform(p.seed, g, k);
      continue;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < p.r; j += blockDim.x) z[j] = sivfgen_N01(p.seed, g, 1000u + (uint64_t)j);
    __syncthreads();
    const int m = sivfgen_component(&p, g);
    for (int k = threadIdx.x; k < p.dim; k += blockDim.x)
      o[k] = sivfgen_coord(&p, g, k, mu[(size_t)m * p.dim + k], A + ((size_t)m * p.dim + k) * p.r, z);
  }
}

/* block per listed id (grid-stride) */
__global__ void __launch_bounds__(kThreads) k_list(sivfgen_params p, const float* __restrict__ mu,
                                                   const float* __restrict__ A, const uint64_t* __restrict__ gs,
                                                   int64_t n, float* __restrict__ out) {
  __shared__ float z[kMaxR];
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const uint64_t g = gs[i];
    float* o = out + (size_t)i * p.dim;
    if (p.kind == SIVFGEN_UNIFORM) {
      for (int k = threadIdx.x; k < p.dim; k += blockDim.x) o[k] = sivfgen_uniform(p.seed, g, k);
      continue;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < p.r; j += blockDim.x) z[j] = sivfgen_N01(p.seed, g, 1000u + (uint64_t)j);
    __syncthreads();
    const int m = sivfgen_component(&p, g);
    for (int k = threadIdx.x; k < p.dim; k += blockDim.x)
      o[k] = sivfgen_coord(&p, g, k, mu[(size_t)m * p.dim + k], A + ((size_t)m * p.dim + k) * p.r, z);
  }
}

}  // namespace

extern "C" {

typedef struct sivfgen_cuda_model {
  sivfgen_params p;
  float* mu;
  float* A;
} sivfgen_cuda_model;

/* Builds the model tables on the current device; returns NULL on error. */
sivfgen_cuda_model* sivfgen_cuda_model_new(const sivfgen_params* p) {
  if (!p || p->r > kMaxR) return nullptr;
  sivfgen_cuda_model* md = new sivfgen_cuda_model();
  md->p = *p;
  md->mu = nullptr;
  md->A = nullptr;
  if (p->kind != SIVFGEN_UNIFORM) {
    const size_t M = (size_t)p->M, D = (size_t)p->dim, r = (size_t)(p->r > 0 ? p->r : 1);
    if (cudaMalloc(&md->mu, sizeof(float) * M * D) != cudaSuccess ||
        cudaMalloc(&md->A, sizeof(float) * M * D * r) != cudaSuccess) {
      cudaFree(md->mu);
      delete md;
      return nullptr;
    }
    k_tables<<<p->M, 128>>>(md->p, md->mu, md->A);
    if (cudaDeviceSynchronize() != cudaSuccess) {
      cudaFree(md->mu);
      cudaFree(md->A);
      delete md;
      return nullptr;
    }
  }
  return md;
}

void sivfgen_cuda_model_free(sivfgen_cuda_model* md) {
  if (!md) return;
  cudaFree(md->mu);
  cudaFree(md->A);
  delete md;
}

/* out[i][:] = vector(g0 + i * gstride), i < n; d_out is a device pointer
   [n][dim]; asynchronous on `stream`.  Returns a cudaError_t. */
int sivfgen_cuda_range(const sivfgen_cuda_model* md, uint64_t g0, uint64_t gstride, int64_t n, float* d_out,
                       void* stream) {
  if (!md || n < 0 || (n > 0 && !d_out)) return (int)cudaErrorInvalidValue;
  if (n == 0) return 0;
  const int64_t grid = n < 148 * 64 ? n : 148 * 64;
  k_range<<<(unsigned)grid, kThreads, 0, (cudaStream_t)stream>>>(md->p, md->mu, md->A, g0, gstride, n, d_out);
  return (int)cudaGetLastError();
}

/* out[i][:] = vector(d_gs[i]), i < n (device ids list); asynchronous on `stream`. */
int sivfgen_cuda_list(const sivfgen_cuda_model* md, const uint64_t* d_gs, int64_t n, float* d_out, void* stream) {
  if (!md || n < 0 || (n > 0 && (!d_out || !d_gs))) return (int)cudaErrorInvalidValue;
  if (n == 0) return 0;
  const int64_t grid = n < 148 * 64 ? n : 148 * 64;
  k_list<<<(unsigned)grid, kThreads, 0, (cudaStream_t)stream>>>(md->p, md->mu, md->A, d_gs, n, d_out);
  return (int)cudaGetLastError();
}
}
