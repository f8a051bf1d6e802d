/*
 * c_api_demo.c -- the differentiable MLS-MPM step through the plain C ABI (include/mpm.h),
 * no Python, no torch: a falling block of particles, forward n steps, backward from the
 * loss L = x-coordinate of the centre of mass, and the gradients.
 *
 * Build (after libmpm.so is built):
 *   gcc -std=c99 -O2 -I include examples/c_api_demo.c -L paper_1810_01054_b200 -lmpm \
 *       -Wl,-rpath,$PWD/paper_1810_01054_b200 -lm -o c_api_demo
 * Run on a GPU box: ./c_api_demo   (prints the gradients' closed-form check and exits 0/1)
 *
 * Without wall contact the centre of mass moves with the initial momentum and gravity only,
 * so dL/dx0_p = m_p / M and dL/dv0_p = T dt m_p / M exactly.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "mpm.h"

#define CHECK(call)                                                                \
  do {                                                                             \
    mpm_status s_ = (call);                                                        \
    if (s_ != MPM_OK) {                                                            \
      fprintf(stderr, "%s failed: %d (%s)\n", #call, (int)s_, mpm_last_error(ctx)); \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

int main(void) {
  const int res = 64, cells = 8, ppc_axis = 2, T = 50;
  const int n = cells * cells * cells * ppc_axis * ppc_axis * ppc_axis; /* 4096 particles */
  const float dx = 1.0f / res;
  float* x = malloc(sizeof(float) * n * 3);
  float* v = calloc((size_t)n * 3, sizeof(float));
  float* mass = malloc(sizeof(float) * n);
  float* vol = malloc(sizeof(float) * n);
  float* E = malloc(sizeof(float) * n);
  float* nu = malloc(sizeof(float) * n);
  int p = 0;
  for (int i = 0; i < cells * ppc_axis; ++i)
    for (int j = 0; j < cells * ppc_axis; ++j)
      for (int k = 0; k < cells * ppc_axis; ++k, ++p) {
        x[3 * p + 0] = (28 + (i + 0.5f) / ppc_axis) * dx; /* block of 8^3 cells at the centre */
        x[3 * p + 1] = (28 + (j + 0.5f) / ppc_axis) * dx;
        x[3 * p + 2] = (28 + (k + 0.5f) / ppc_axis) * dx;
        v[3 * p + 0] = 0.5f;
        mass[p] = vol[p] = dx * dx * dx / 8.0f; /* rho = 1, 8 particles per cell (R15) */
        E[p] = 1000.0f;
        nu[p] = 0.3f;
      }
  mpm_config cfg = {0};
  cfg.dim = 3;
  cfg.res = res;
  cfg.batch = 1;
  cfg.n_particles = n;
  cfg.max_steps = T;
  cfg.dt = 1e-4f;
  cfg.gravity[1] = -9.8f;
  cfg.bound = 3;
  cfg.friction[2] = 0.5f;
  mpm_ctx ctx = NULL;
  if (mpm_create(&cfg, &ctx) != MPM_OK) {
    fprintf(stderr, "mpm_create failed\n");
    return 1;
  }
  CHECK(mpm_set_state(ctx, x, v, NULL, NULL, mass, vol, E, nu, NULL)); /* F = I, C = 0 */
  CHECK(mpm_forward(ctx, T));
  float* seed = calloc((size_t)n * 3, sizeof(float));
  double M = 0.0;
  for (int q = 0; q < n; ++q) M += mass[q];
  for (int q = 0; q < n; ++q) seed[3 * q] = (float)(mass[q] / M); /* dL/dx_T for L = CoM_x */
  CHECK(mpm_backward(ctx, seed, NULL, NULL, NULL));
  float* dx0 = malloc(sizeof(float) * n * 3);
  float* dv0 = malloc(sizeof(float) * n * 3);
  CHECK(mpm_grad(ctx, dx0, dv0, NULL, NULL, NULL, NULL, NULL));
  double ex = 0.0, ev = 0.0, nx = 0.0, nv = 0.0;
  for (int q = 0; q < n; ++q)
    for (int a = 0; a < 3; ++a) {
      double rx = a == 0 ? mass[q] / M : 0.0, rv = a == 0 ? T * cfg.dt * mass[q] / M : 0.0;
      ex += (dx0[3 * q + a] - rx) * (dx0[3 * q + a] - rx);
      ev += (dv0[3 * q + a] - rv) * (dv0[3 * q + a] - rv);
      nx += rx * rx;
      nv += rv * rv;
    }
  ex = sqrt(ex / nx);
  ev = sqrt(ev / nv);
  printf("particles %d, steps %d: rel. error vs closed form  dL/dx0 %.3e  dL/dv0 %.3e\n", n, T, ex, ev);
  mpm_destroy(ctx);
  return (ex < 1e-3 && ev < 1e-3) ? 0 : 1;
}
