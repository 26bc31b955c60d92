/* srj_c_demo.c -- the C ABI (include/srj.h) used from plain C + the CUDA
 * runtime, no Python: a 2-D Dirichlet Poisson problem relaxed with a
 * two-level weight cycle (one over-relaxed step, seven damped ones) through
 *   (1) the plan API: srj_layout -> srj_plan_create -> srj_plan_run (fused
 *       multi-step launches, per-step norms on the device), and
 *   (2) the kernel-level drop-in srj_wj_dense on the reference's dense layout,
 *       one step per call (what _WJ_KERNELS[2] does, grids.py:547-554),
 * and checked against a CPU loop restating the reference _wj2 arithmetic
 * (grids.py:351-376): all three fields and norm histories must be bitwise
 * equal.  Exit status 0 on success.
 *
 * Build: see __graft_entry__.build_examples(); run: examples/bin/srj_c_demo
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "srj.h"

#define N0 130
#define N1 257
#define STEPS 96

#define CK(x)                                                               \
  do {                                                                      \
    int rc_ = (x);                                                          \
    if (rc_ != SRJ_OK) {                                                    \
      fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, srj_last_error());   \
      return 1;                                                             \
    }                                                                       \
  } while (0)
#define CU(x)                                                               \
  do {                                                                      \
    cudaError_t e_ = (x);                                                   \
    if (e_ != cudaSuccess) {                                                \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));              \
      return 1;                                                             \
    }                                                                       \
  } while (0)

/* CPU restatement of one reference step (constant stencil, two buffers). */
static void cpu_step(const double *u, double *un, const double *s, double c, double a,
                     double omega, double *dmax, double *rmax) {
  const int w = N1 + 2;
  *dmax = 0.0;
  *rmax = 0.0;
  for (int i = 0; i < N0; ++i)
    for (int j = 0; j < N1; ++j) {
      const double uc = u[(i + 1) * w + j + 1];
      const double r = s[i * N1 + j] - ((((c * uc + a * u[i * w + j + 1]) + a * u[(i + 2) * w + j + 1]) +
                                         a * u[(i + 1) * w + j]) + a * u[(i + 1) * w + j + 2]);
      const double d = omega * r / c;
      un[(i + 1) * w + j + 1] = uc + d;
      if (fabs(d) > *dmax) *dmax = fabs(d);
      if (fabs(r) > *rmax) *rmax = fabs(r);
    }
}

int main(void) {
  const double c = 4.0, a = -1.0;
  const double weights[8] = {12.0, 0.8, 0.8, 0.8, 0.8, 0.8, 0.8, 0.8};
  const int64_t n[3] = {N0, N1, 0};
  const size_t gcells = (size_t)(N0 + 2) * (N1 + 2);
  double *u0 = calloc(gcells, sizeof(double)), *src = malloc(sizeof(double) * N0 * N1);
  for (int i = 0; i < N0; ++i)
    for (int j = 0; j < N1; ++j) src[i * N1 + j] = sin(0.05 * i) * cos(0.031 * j) + 1e-3 * ((i * 7 + j * 13) % 17);

  /* ---- CPU reference ---- */
  double *cu = calloc(gcells, sizeof(double)), *cn = calloc(gcells, sizeof(double));
  double cpu_norms[2 * STEPS];
  for (int k = 0; k < STEPS; ++k) {
    cpu_step(cu, cn, src, c, a, weights[k % 8], &cpu_norms[2 * k], &cpu_norms[2 * k + 1]);
    double *t = cu; cu = cn; cn = t;
  }

  /* ---- (1) plan API on the padded layout ---- */
  srj_layout_t lay;
  CK(srj_layout(2, n, 1, &lay));
  double *f[3], *dsrc, *dnorms;
  for (int b = 0; b < 3; ++b) {
    CU(cudaMalloc((void **)&f[b], sizeof(double) * lay.elems));
    CU(cudaMemset(f[b], 0, sizeof(double) * lay.elems));
  }
  CU(cudaMalloc((void **)&dsrc, sizeof(double) * lay.elems));
  CU(cudaMemset(dsrc, 0, sizeof(double) * lay.elems));
  CU(cudaMalloc((void **)&dnorms, sizeof(double) * 2 * STEPS));
  for (int b = 0; b < 3; ++b) CK(srj_upload_field(&lay, u0, f[b], NULL));
  CK(srj_upload_interior(&lay, src, dsrc, 8, NULL));
  srj_plan_desc desc;
  memset(&desc, 0, sizeof(desc));
  desc.layout = lay;
  desc.coef_mode = 0;
  desc.coef[0] = c;
  for (int k = 1; k < 5; ++k) desc.coef[k] = a;
  desc.source = dsrc;
  desc.physical_lo0 = desc.physical_hi0 = 1;
  srj_plan *plan;
  CK(srj_plan_create(&desc, &plan));
  int32_t fin = 0;
  CK(srj_plan_run(plan, f[0], f[1], f[2], weights, 8, 0, STEPS, 4, dnorms, &fin, NULL));
  double *plan_u = malloc(sizeof(double) * gcells), plan_norms[2 * STEPS];
  CK(srj_download_field(&lay, f[fin], plan_u, NULL));
  CU(cudaMemcpy(plan_norms, dnorms, sizeof(plan_norms), cudaMemcpyDeviceToHost));

  /* ---- (2) dense kernel-level entry point, one step per call ---- */
  double *du[2], *ds, *dc, *dlo[2], *dhi[2], *dn1;
  const size_t icells = (size_t)N0 * N1;
  double *cst = malloc(sizeof(double) * icells), *nb = malloc(sizeof(double) * icells);
  for (size_t q = 0; q < icells; ++q) { cst[q] = c; nb[q] = a; }
  for (int b = 0; b < 2; ++b) {
    CU(cudaMalloc((void **)&du[b], sizeof(double) * gcells));
    CU(cudaMemcpy(du[b], u0, sizeof(double) * gcells, cudaMemcpyHostToDevice));
    CU(cudaMalloc((void **)&dlo[b], sizeof(double) * icells));
    CU(cudaMalloc((void **)&dhi[b], sizeof(double) * icells));
    CU(cudaMemcpy(dlo[b], nb, sizeof(double) * icells, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(dhi[b], nb, sizeof(double) * icells, cudaMemcpyHostToDevice));
  }
  CU(cudaMalloc((void **)&ds, sizeof(double) * icells));
  CU(cudaMalloc((void **)&dc, sizeof(double) * icells));
  CU(cudaMalloc((void **)&dn1, sizeof(double) * 2));
  CU(cudaMemcpy(ds, src, sizeof(double) * icells, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(dc, cst, sizeof(double) * icells, cudaMemcpyHostToDevice));
  const double *lo[2] = {dlo[0], dlo[1]}, *hi[2] = {dhi[0], dhi[1]};
  double dense_norms[2 * STEPS];
  for (int k = 0; k < STEPS; ++k) {
    CK(srj_wj_dense(2, n, du[k % 2], du[(k + 1) % 2], ds, dc, lo, hi, NULL, weights[k % 8], dn1,
                    NULL));
    CU(cudaMemcpy(&dense_norms[2 * k], dn1, 2 * sizeof(double), cudaMemcpyDeviceToHost));
  }
  double *dense_u = malloc(sizeof(double) * gcells);
  CU(cudaMemcpy(dense_u, du[STEPS % 2], sizeof(double) * gcells, cudaMemcpyDeviceToHost));

  /* ---- bitwise comparison ---- */
  size_t bad_plan = 0, bad_dense = 0;
  for (size_t q = 0; q < gcells; ++q) {
    bad_plan += memcmp(&plan_u[q], &cu[q], 8) != 0;
    bad_dense += memcmp(&dense_u[q], &cu[q], 8) != 0;
  }
  const int norms_ok = memcmp(plan_norms, cpu_norms, sizeof(cpu_norms)) == 0 &&
                       memcmp(dense_norms, cpu_norms, sizeof(cpu_norms)) == 0;
  double sum = 0.0;
  for (size_t q = 0; q < gcells; ++q) sum += cu[q];
  printf("srj_c_demo: %dx%d, %d steps, plan mismatches %zu, dense mismatches %zu, norms %s, "
         "checksum %.17g, last dmax %.3e\n", N0, N1, STEPS, bad_plan, bad_dense,
         norms_ok ? "equal" : "DIFFER", sum, cpu_norms[2 * STEPS - 2]);
  srj_plan_destroy(plan);
  if (bad_plan || bad_dense || !norms_ok) return 2;
  printf("OK\n");
  return 0;
}
