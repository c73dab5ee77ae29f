/* sivf_datagen.h — seeded synthetic workload generator (harness code).
 *
 * This module is shared by the CPU oracle tests, the GPU parity tests and
 * bench.py.  It holds NONE of the method's arithmetic (no distances, no
 * assignment, no index state): it only maps (seed, g) -> a float vector, so
 * that the oracle and the CUDA path can be fed identical inputs.
 *
 * Recipe ("Synthetic generator"): a low-rank Gaussian
 * mixture shaped like SIFT1M (integer-valued, clamped to [0,255]) or GIST1M
 * (non-negative floats), or the paper's uniform [0,1) data.
 *
 *   mix64(z)   splitmix64 finaliser (z += golden gamma first)
 *   H(s,a,b)   = mix64(s ^ mix64(a ^ mix64(b)))
 *   U22(s,a,b) = H(s,a,b) >> 42                        (22-bit uniform)
 *   N01(s,a,b) = (float(U22(s,a,4b)+..+U22(s,a,4b+3)) * 2^-22 - 2) * sqrt(3)
 *                (Irwin-Hall(4): mean 0, variance 1; the integer sum < 2^24
 *                 is exact in fp32 and so is "* 2^-22 - 2")
 *   component  m(g)     = H(s, g, 0) mod M
 *   centre     mu[m][k] = a * (U22(s, 2^50+m, k) * 2^-22)^2
 *   basis      A[m][k][j] = (b/sqrt(r)) * N01(s, 2^51 + m*D + k, j)
 *   vector g   x[k] = mu + sum_{j<r} A[k][j]*N01(s,g,1000+j)   (sequential j)
 *                     + sigma * N01(s,g,2000+k)
 *   SIFT: x = rint(clamp(x,0,255));  GIST: x = max(x,0);
 *   UNIFORM: x[k] = U22(s,g,3000+k) * 2^-22
 *
 * Every fp32 operation is a single correctly-rounded op (no FMA contraction):
 * host code must be compiled with -ffp-contract=off, device code uses
 * __fmul_rn/__fadd_rn.  Host and device therefore produce identical bits.
 */
#ifndef SIVF_DATAGEN_H
#define SIVF_DATAGEN_H

#include <stdint.h>
#include <math.h>

#if defined(__CUDACC__)
#define SIVFGEN_HD __host__ __device__ __forceinline__
#else
#define SIVFGEN_HD static inline
#endif

enum { SIVFGEN_SIFT = 0, SIVFGEN_GIST = 1, SIVFGEN_UNIFORM = 2 };

/* Index spaces for g: base vector g = id; query g = 2^40 + q;
   k-means training sample g = 2^41 + i. */
#define SIVFGEN_QUERY_BASE (1ull << 40)
#define SIVFGEN_TRAIN_BASE (1ull << 41)

SIVFGEN_HD uint64_t sivfgen_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

SIVFGEN_HD uint64_t sivfgen_H(uint64_t s, uint64_t a, uint64_t b) {
  return sivfgen_mix64(s ^ sivfgen_mix64(a ^ sivfgen_mix64(b)));
}

SIVFGEN_HD uint32_t sivfgen_U22(uint64_t s, uint64_t a, uint64_t b) {
  return (uint32_t)(sivfgen_H(s, a, b) >> 42);
}

SIVFGEN_HD float sivfgen_fmul(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fmul_rn(a, b);
#else
  return a * b;
#endif
}

SIVFGEN_HD float sivfgen_fadd(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fadd_rn(a, b);
#else
  return a + b;
#endif
}

SIVFGEN_HD float sivfgen_N01(uint64_t s, uint64_t a, uint64_t b) {
  uint32_t sum = sivfgen_U22(s, a, 4 * b) + sivfgen_U22(s, a, 4 * b + 1) +
                 sivfgen_U22(s, a, 4 * b + 2) + sivfgen_U22(s, a, 4 * b + 3);
  float t = sivfgen_fmul((float)sum, 0x1p-22f);
  t = sivfgen_fadd(t, -2.0f);
  return sivfgen_fmul(t, 1.7320508f);
}

SIVFGEN_HD float sivfgen_uniform(uint64_t s, uint64_t g, int k) {
  return sivfgen_fmul((float)sivfgen_U22(s, g, 3000u + (uint64_t)k), 0x1p-22f);
}

typedef struct {
  uint64_t seed;
  int32_t dim;     /* D */
  int32_t M;       /* mixture components */
  int32_t r;       /* latent rank */
  int32_t kind;    /* SIVFGEN_SIFT / GIST / UNIFORM */
  float a;         /* centre scale */
  float b_over_sqrt_r; /* basis scale, rounded once on the host */
  float sigma;     /* isotropic noise */
} sivfgen_params;

SIVFGEN_HD float sivfgen_mu(const sivfgen_params* p, int m, int k) {
  float u = sivfgen_fmul((float)sivfgen_U22(p->seed, (1ull << 50) + (uint64_t)m, (uint64_t)k), 0x1p-22f);
  return sivfgen_fmul(p->a, sivfgen_fmul(u, u));
}

SIVFGEN_HD float sivfgen_basis(const sivfgen_params* p, int m, int k, int j) {
  return sivfgen_fmul(p->b_over_sqrt_r,
                      sivfgen_N01(p->seed, (1ull << 51) + (uint64_t)m * (uint64_t)p->dim + (uint64_t)k, (uint64_t)j));
}

SIVFGEN_HD int sivfgen_component(const sivfgen_params* p, uint64_t g) {
  return (int)(sivfgen_H(p->seed, g, 0) % (uint64_t)p->M);
}

/* Finish one coordinate: k-th dim of vector g given its mixture value.
   z[] = latents N01(s,g,1000+j), A_k = basis row for (m,k) (length r). */
SIVFGEN_HD float sivfgen_coord(const sivfgen_params* p, uint64_t g, int k, float mu_k,
                               const float* A_k, const float* z) {
  float x = mu_k;
  for (int j = 0; j < p->r; ++j) x = sivfgen_fadd(x, sivfgen_fmul(A_k[j], z[j]));
  x = sivfgen_fadd(x, sivfgen_fmul(p->sigma, sivfgen_N01(p->seed, g, 2000u + (uint64_t)k)));
  if (p->kind == SIVFGEN_SIFT) {
    x = x < 0.f ? 0.f : (x > 255.f ? 255.f : x);
#if defined(__CUDA_ARCH__)
    x = rintf(x);
#else
    x = nearbyintf(x); /* FE_TONEAREST: round half to even, like rintf */
#endif
  } else {
    x = x < 0.f ? 0.f : x;
  }
  return x;
}

#endif /* SIVF_DATAGEN_H */
