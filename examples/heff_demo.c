/*
 * heff_demo.c -- the C ABI used from plain C (no Python, no torch): build a two-site
 * H_eff for the N = 2 Heisenberg chain with trivial boundary environments (Eq. (1) of the
 * paper at N = 2), find its ground state with lanczos_ground, and split it
 * with heff_svd_split.  Expected: E0 = -3/4 (the singlet) and Schmidt values 1/sqrt(2).
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/heff_demo.c -L paper_2007_14822_b200 -lheff \
 *       -Wl,-rpath,$PWD/paper_2007_14822_b200 -lcudart -L /usr/local/cuda/lib64 -o heff_demo
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "heff.h"

#define CHECK(x)                                                                   \
  do {                                                                             \
    int rc_ = (x);                                                                 \
    if (rc_ != HEFF_OK) {                                                          \
      fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, heff_last_error());         \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

/* Heisenberg MPO of bond dimension 5 (reading R4): start channel 4, done channel 0 */
static void heisenberg_W(double W[5][2][2][5]) {
  const double I[2][2] = {{1, 0}, {0, 1}}, Sz[2][2] = {{0.5, 0}, {0, -0.5}};
  const double Sp[2][2] = {{0, 1}, {0, 0}}, Sm[2][2] = {{0, 0}, {1, 0}};
  memset(W, 0, sizeof(double) * 100);
  for (int s = 0; s < 2; ++s)
    for (int t = 0; t < 2; ++t) {
      W[0][s][t][0] = I[s][t];
      W[4][s][t][4] = I[s][t];
      W[4][s][t][1] = 0.5 * Sm[s][t];
      W[4][s][t][2] = 0.5 * Sp[s][t];
      W[4][s][t][3] = Sz[s][t];
      W[1][s][t][0] = Sp[s][t];
      W[2][s][t][0] = Sm[s][t];
      W[3][s][t][0] = Sz[s][t];
    }
}

int main(void) {
  double W[5][2][2][5], L[5] = {0, 0, 0, 0, 1}, R[5] = {1, 0, 0, 0, 0};
  double psi[4] = {0.3, -0.7, 0.5, 0.1};
  heisenberg_W(W);
  double *dW, *dL, *dR, *dpsi, *dQ, *dS, *dC;
  if (cudaMalloc((void**)&dW, sizeof W) || cudaMalloc((void**)&dL, sizeof L) || cudaMalloc((void**)&dR, sizeof R) ||
      cudaMalloc((void**)&dpsi, sizeof psi) || cudaMalloc((void**)&dQ, 4 * sizeof(double)) ||
      cudaMalloc((void**)&dS, 2 * sizeof(double)) || cudaMalloc((void**)&dC, 4 * sizeof(double))) {
    fprintf(stderr, "cudaMalloc failed (no GPU?)\n");
    return 2;
  }
  cudaMemcpy(dW, W, sizeof W, cudaMemcpyHostToDevice);
  cudaMemcpy(dL, L, sizeof L, cudaMemcpyHostToDevice);
  cudaMemcpy(dR, R, sizeof R, cudaMemcpyHostToDevice);
  cudaMemcpy(dpsi, psi, sizeof psi, cudaMemcpyHostToDevice);

  heff_dims dims = {1, 2, 2, 1, 5, 5, 5};  /* mL, d1, d2, mR, kL, kM, kR */
  heff_plan plan;
  CHECK(heff_create(&plan, &dims, dL, dW, dW, dR, NULL, NULL));
  heff_lanczos_opts opts = {20, 1, 1e-12, NULL, NULL, NULL};
  double energy = 0, resid = 0;
  int iters = 0;
  CHECK(lanczos_ground(plan, dpsi, &opts, &energy, &iters, &resid, NULL));
  CHECK(heff_destroy(plan));

  heff_trunc tr = {0.0, 0, 1};
  int64_t n = 0;
  double err = 0;
  int sweeps = 0;
  CHECK(heff_svd_split(2, 2, dpsi, &tr, 0, dQ, dS, dC, &n, &err, &sweeps, NULL));
  double S[2];
  cudaMemcpy(S, dS, sizeof S, cudaMemcpyDeviceToHost);
  printf("E0 = %.15f (exact -0.75) after %d Lanczos steps; Schmidt values %.15f %.15f (exact 1/sqrt(2))\n", energy,
         iters, S[0], S[1]);
  const int ok = fabs(energy + 0.75) < 1e-12 && fabs(S[0] - sqrt(0.5)) < 1e-12 && fabs(S[1] - sqrt(0.5)) < 1e-12;
  printf("%s\n", ok ? "OK" : "MISMATCH");
  return ok ? 0 : 1;
}
