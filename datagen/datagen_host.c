/* datagen_host.c — host (CPU) driver for sivf_datagen.h.
 * Harness code: produces the seeded synthetic vectors that both the oracle
 * and the CUDA path consume.  Compiled with -O2 -ffp-contract=off so that
 * every fp32 op is individually rounded (bit-identical to the device path).
 */
#include "sivf_datagen.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

typedef struct sivfgen_model {
  sivfgen_params p;
  float* mu; /* [M][D] */
  float* A;  /* [M][D][r] */
} sivfgen_model;

typedef struct {
  const sivfgen_model* m;
  const uint64_t* gs; /* optional explicit list */
  uint64_t g0;
  int64_t begin, end;
  float* out;
} job_t;

static void gen_one(const sivfgen_model* md, uint64_t g, float* out, float* z) {
  const sivfgen_params* p = &md->p;
  const int D = p->dim;
  if (p->kind == SIVFGEN_UNIFORM) {
    for (int k = 0; k < D; ++k) out[k] = sivfgen_uniform(p->seed, g, k);
    return;
  }
  int m = sivfgen_component(p, g);
  for (int j = 0; j < p->r; ++j) z[j] = sivfgen_N01(p->seed, g, 1000u + (uint64_t)j);
  const float* mu = md->mu + (size_t)m * D;
  const float* A = md->A + (size_t)m * D * p->r;
  for (int k = 0; k < D; ++k) out[k] = sivfgen_coord(p, g, k, mu[k], A + (size_t)k * p->r, z);
}

static void* worker(void* arg) {
  job_t* j = (job_t*)arg;
  float* z = (float*)malloc(sizeof(float) * (size_t)(j->m->p.r > 0 ? j->m->p.r : 1));
  const int D = j->m->p.dim;
  for (int64_t i = j->begin; i < j->end; ++i) {
    uint64_t g = j->gs ? j->gs[i] : j->g0 + (uint64_t)i;
    gen_one(j->m, g, j->out + (size_t)i * D, z);
  }
  free(z);
  return NULL;
}

static int hw_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  if (n < 1) n = 1;
  if (n > 128) n = 128;
  return (int)n;
}

sivfgen_model* sivfgen_model_new(const sivfgen_params* p) {
  sivfgen_model* md = (sivfgen_model*)calloc(1, sizeof(sivfgen_model));
  md->p = *p;
  if (p->kind != SIVFGEN_UNIFORM) {
    const int D = p->dim, M = p->M, r = p->r;
    md->mu = (float*)malloc(sizeof(float) * (size_t)M * D);
    md->A = (float*)malloc(sizeof(float) * (size_t)M * D * (r > 0 ? r : 1));
    for (int m = 0; m < M; ++m)
      for (int k = 0; k < D; ++k) {
        md->mu[(size_t)m * D + k] = sivfgen_mu(p, m, k);
        for (int j = 0; j < r; ++j) md->A[((size_t)m * D + k) * r + j] = sivfgen_basis(p, m, k, j);
      }
  }
  return md;
}

void sivfgen_model_free(sivfgen_model* md) {
  if (!md) return;
  free(md->mu);
  free(md->A);
  free(md);
}

static void run(const sivfgen_model* md, const uint64_t* gs, uint64_t g0, int64_t n, float* out,
                int nthreads) {
  if (n <= 0) return;
  if (nthreads <= 0) nthreads = hw_threads();
  int64_t per = 256;
  if ((int64_t)nthreads * per > n) nthreads = (int)((n + per - 1) / per);
  if (nthreads < 1) nthreads = 1;
  pthread_t th[128];
  job_t jobs[128];
  int64_t chunk = (n + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; ++t) {
    jobs[t].m = md;
    jobs[t].gs = gs;
    jobs[t].g0 = g0;
    jobs[t].begin = t * chunk;
    jobs[t].end = (t + 1) * chunk < n ? (t + 1) * chunk : n;
    jobs[t].out = out;
    if (t > 0) pthread_create(&th[t], NULL, worker, &jobs[t]);
  }
  worker(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* Vectors for g = g0 .. g0+n-1, row-major [n][dim]. */
void sivfgen_range(const sivfgen_model* md, uint64_t g0, int64_t n, float* out, int nthreads) {
  run(md, NULL, g0, n, out, nthreads);
}

/* Vectors for an explicit list of g values. */
void sivfgen_list(const sivfgen_model* md, const uint64_t* gs, int64_t n, float* out, int nthreads) {
  run(md, gs, 0, n, out, nthreads);
}

/* Raw primitives, exported for pinning tests. */
uint64_t sivfgen_mix64_x(uint64_t z) { return sivfgen_mix64(z); }
uint64_t sivfgen_H_x(uint64_t s, uint64_t a, uint64_t b) { return sivfgen_H(s, a, b); }
float sivfgen_N01_x(uint64_t s, uint64_t a, uint64_t b) { return sivfgen_N01(s, a, b); }
