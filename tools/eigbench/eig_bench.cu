// Microbenchmark of the split's pair eigen-solve (svd_pair_eig_kernel) on synthetic SPD
// 32x32 Grams: time per launch for npairs CTAs, and (instrumented copy) where the cycles of
// one Jacobi round go.  Tool only; build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
// -std=c++17 -I paper_2007_14822_b200/csrc tools/eigbench/eig_bench.cu -o tools/eigbench/eig_bench
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <random>
#ifndef EIG_NO_INSTR
#define HEFF_EIG_INSTR
#endif
#include "svd.cuh"
using namespace heff;

namespace heff {
// the index-table version of the kernel (before the position-permuted rewrite), for a bitwise comparison
__global__ void __launch_bounds__(kSvdEigThreads) svd_pair_eig_kernel_old(const double* __restrict__ Gp, int nslots,
                                                                     int64_t C, int gram_grid,
                                                                     double tol, double negl, int inner_sweeps,
                                                                     double* __restrict__ Qg, int* __restrict__ flag,
                                                                     unsigned long long* __restrict__ stat_maxoff,
                                                                     int* __restrict__ stat_nrot) {
  __shared__ double Gs[2][kSvdPair][kSvdPair + 1];   // ping-pong: round rr reads Gs[rr&1], writes Gs[~]
  __shared__ double Q[kSvdPair][kSvdPair + 1];
  __shared__ double2 s_cs[2][16], s_nn[2][16];       // (c, s) and the rotated diagonal per pair
  __shared__ int s_on[2][16];
  __shared__ int s_neg[kSvdPair];
  __shared__ unsigned char s_pa[31][16], s_pb[31][16], s_kof[31][kSvdPair], s_hi[31][kSvdPair];
  __shared__ uint32_t s_pk1[31][16], s_pk2[31][16];   // per (round, pair of the next round): index chains
  __shared__ unsigned char s_pk3[31][16];
  __shared__ int s_any[kSvdMaxInnerSweeps];          // did inner sweep i rotate anything
  __shared__ double s_off[kSvdEigThreads / 32];
  const int p = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double* gsrc = Gp + (int64_t)p * nslots * (kSvdPair * kSvdPair);
  const int64_t T = (int64_t)gridDim.x * C;  // gridDim.x = npairs
  const int nsum = svd_sk_owner((int64_t)p * C + C - 1, T, gram_grid) - svd_sk_owner((int64_t)p * C, T, gram_grid) + 1;
  for (int e = tid; e < kSvdPair * kSvdPair; e += blockDim.x) {
    double v = 0.0;
    for (int sp = 0; sp < nsum; ++sp) v += gsrc[(int64_t)sp * (kSvdPair * kSvdPair) + e];
    const int r = e >> 5, c = e & 31;
    Gs[0][r][c] = v;
    Q[r][c] = (r == c) ? 1.0 : 0.0;
  }
  for (int e = tid; e < 31 * 16; e += blockDim.x) {  // round-robin (circle method) over 32 columns
    const int rr = e >> 4, k = e & 15;
    auto idx = [&](int i) { return i == 0 ? 0 : ((i - 1 + rr) % 31) + 1; };
    const int a = idx(k), b = idx(31 - k);
    s_pa[rr][k] = (unsigned char)a;
    s_pb[rr][k] = (unsigned char)b;
    s_kof[rr][a] = s_kof[rr][b] = (unsigned char)k;   // which pair of round rr holds column a / b
    s_hi[rr][a] = 0;
    s_hi[rr][b] = 1;
  }
  __syncthreads();
  for (int e = tid; e < 31 * 16; e += blockDim.x) {  // the dependent index lookups of the rotation warp
    const int rr = e >> 4, t = e & 15, r1 = (rr + 1) % 31;
    const int a = s_pa[r1][t], b = s_pb[r1][t];
    const int ka = s_kof[rr][a], kb = s_kof[rr][b];
    s_pk1[rr][t] = (uint32_t)a | ((uint32_t)b << 8) | ((uint32_t)ka << 16) | ((uint32_t)kb << 24);
    s_pk2[rr][t] = (uint32_t)s_pa[rr][ka] | ((uint32_t)s_pb[rr][ka] << 8) | ((uint32_t)s_pa[rr][kb] << 16) |
                   ((uint32_t)s_pb[rr][kb] << 24);
    s_pk3[rr][t] = (unsigned char)(s_hi[rr][a] | (s_hi[rr][b] << 1));
  }
  if (tid < kSvdPair) s_neg[tid] = !(Gs[0][tid][tid] > negl);
  __syncthreads();
  double off = 0.0;
  for (int e = tid; e < kSvdPair * kSvdPair; e += blockDim.x) {
    const int r = e >> 5, c = e & 31;
    if (r < c && !s_neg[r] && !s_neg[c]) off = fmax(off, fabs(Gs[0][r][c]) / sqrt(Gs[0][r][r] * Gs[0][c][c]));
  }
  for (int o = 16; o > 0; o >>= 1) off = fmax(off, __shfl_xor_sync(0xffffffffu, off, o));
  if (lane == 0) s_off[warp] = off;
  __syncthreads();
  off = s_off[0];
  for (int w = 1; w < kSvdEigThreads / 32; ++w) off = fmax(off, s_off[w]);
  const bool rotate = off > tol;
  if (tid == 0) {
    flag[p] = rotate ? 1 : 0;
    atomicMax(stat_maxoff, (unsigned long long)__double_as_longlong(off));
    if (rotate) atomicAdd(stat_nrot, 1);
  }
  if (!rotate) return;

  // Cyclic two-sided Jacobi, one barrier per round: in round rr every thread writes its
  // 2x2 block of the rotated G into the other buffer and updates Q, while threads 0..15
  // already compute round rr+1's rotations from the OLD G and round rr's rotations.
  // Rotations live as (c, s) pairs -- the identity (1, 0) for a skipped pair, so the block
  // update is branch-free -- plus the exact rotated diagonal (na, nb) and an on flag.
  auto put_rot = [&](int buf, int k, const SvdRot& r) {
    s_cs[buf][k] = make_double2(r.c, r.s);
    s_nn[buf][k] = make_double2(r.na, r.nb);
    s_on[buf][k] = r.on;
  };
  auto rot2 = [](double& x00, double& x01, double& x10, double& x11, double2 rk, double2 rkk) {
    const double y00 = rkk.x * x00 - rkk.y * x01, y01 = rkk.y * x00 + rkk.x * x01;   // columns (pair kk)
    const double y10 = rkk.x * x10 - rkk.y * x11, y11 = rkk.y * x10 + rkk.x * x11;
    x00 = rk.x * y00 - rk.y * y10;                                                  // rows (pair k)
    x10 = rk.y * y00 + rk.x * y10;
    x01 = rk.x * y01 - rk.y * y11;
    x11 = rk.y * y01 + rk.x * y11;
  };
  if (tid < 16) {
    const int a = s_pa[0][tid], b = s_pb[0][tid];
    put_rot(0, tid, svd_make_rot(Gs[0][a][a], Gs[0][b][b], Gs[0][a][b], !s_neg[a] && !s_neg[b], tol));
  }
  if (tid < kSvdMaxInnerSweeps) s_any[tid] = 0;
  __syncthreads();
  const int total_rounds = 31 * min(inner_sweeps, kSvdMaxInnerSweeps);
  for (int it = 0; it < total_rounds; ++it) {
    const int rr = it % 31, cur = it & 1, nxt = cur ^ 1;
    const int sweep = it / 31;
    double(*Go)[kSvdPair + 1] = Gs[cur];
    double(*Gn)[kSvdPair + 1] = Gs[nxt];
    if (tid < 256) {  // this thread's 2x2 block (pair k rows, pair kk columns)
      const int k = tid >> 4, kk = tid & 15;
      const int a = s_pa[rr][k], b = s_pb[rr][k], a2 = s_pa[rr][kk], b2 = s_pb[rr][kk];
      if (k == kk) {
        const double2 nn = s_nn[cur][k];
        Gn[a][a] = nn.x;
        Gn[b][b] = nn.y;
        Gn[a][b] = Gn[b][a] = s_on[cur][k] ? 0.0 : Go[a][b];
      } else {
        double x00 = Go[a][a2], x01 = Go[a][b2], x10 = Go[b][a2], x11 = Go[b][b2];
        rot2(x00, x01, x10, x11, s_cs[cur][k], s_cs[cur][kk]);
        Gn[a][a2] = x00; Gn[a][b2] = x01; Gn[b][a2] = x10; Gn[b][b2] = x11;
      }
      if (tid < 16 && s_on[cur][tid]) s_any[sweep] = 1;
    }
    for (int task = tid; task < 32 * 16; task += 256) {  // Q <- Q J (columns, in place)
      if (tid >= 256) break;
      const int k = task & 15, r = task >> 4;
      if (!s_on[cur][k]) continue;
      const double2 rk = s_cs[cur][k];
      const int a = s_pa[rr][k], b = s_pb[rr][k];
      const double qa = Q[r][a], qb = Q[r][b];
      Q[r][a] = rk.x * qa - rk.y * qb;
      Q[r][b] = rk.y * qa + rk.x * qb;
    }
    const int pl = tid - 256;  // the rotation warp: round rr+1's rotations from the rotated entries
    if (pl >= 0 && pl < 16 && it + 1 < total_rounds) {
      const uint32_t p1 = s_pk1[rr][pl], p2 = s_pk2[rr][pl];
      const int hh = s_pk3[rr][pl];
      const int a = p1 & 255, b = (p1 >> 8) & 255, ka = (p1 >> 16) & 255, kb = p1 >> 24;
      const int ax = p2 & 255, bx = (p2 >> 8) & 255, ay = (p2 >> 16) & 255, by = p2 >> 24;
      const int hx = hh & 1, hy = hh >> 1;
      const double2 nna = s_nn[cur][ka], nnb = s_nn[cur][kb];
      const double app = hx ? nna.y : nna.x;                   // rotated diagonals: exact values
      const double aqq = hy ? nnb.y : nnb.x;
      // rotated off-diagonal (a, b): a and b sit in different pairs of round rr
      double x00 = Go[ax][ay], x01 = Go[ax][by], x10 = Go[bx][ay], x11 = Go[bx][by];
      rot2(x00, x01, x10, x11, s_cs[cur][ka], s_cs[cur][kb]);
      const double apq = hx ? (hy ? x11 : x10) : (hy ? x01 : x00);
      put_rot(nxt, pl, svd_make_rot(app, aqq, apq, !s_neg[a] && !s_neg[b], tol));
    }
    __syncthreads();
    if (rr == 30 && !s_any[sweep]) break;  // end of an inner sweep that rotated nothing
  }
  double* q = Qg + (int64_t)p * (kSvdPair * kSvdPair);
  for (int e = tid; e < kSvdPair * kSvdPair; e += blockDim.x) q[e] = Q[e >> 5][e & 31];
}

}  // namespace heff

int main(int argc, char** argv) {
  const int npairs = argc > 1 ? atoi(argv[1]) : 16;
  const int reps = 200;
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  std::vector<double> G((size_t)npairs * 1024);
  for (int p = 0; p < npairs; ++p) {
    std::vector<double> A(64 * 32);
    for (auto& x : A) x = nd(rng);
    for (int i = 0; i < 32; ++i)
      for (int j = 0; j < 32; ++j) {
        double s = 0;
        for (int r = 0; r < 64; ++r) s += A[r * 32 + i] * A[r * 32 + j];
        G[(size_t)p * 1024 + i * 32 + j] = s;
      }
  }
  double *dG, *dQ;
  int *dflag, *dnrot;
  unsigned long long* dmax;
  cudaMalloc(&dG, G.size() * 8);
  cudaMalloc(&dQ, G.size() * 8);
  cudaMalloc(&dflag, npairs * 4);
  cudaMalloc(&dnrot, 4);
  cudaMalloc(&dmax, 8);
  cudaMemcpy(dG, G.data(), G.size() * 8, cudaMemcpyHostToDevice);
  const double tol = 4 * 2.2e-16 * 32, negl = 1e-300;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int inner : {1, 2}) {
    for (int w = 0; w < 5; ++w)
      svd_pair_eig_kernel<<<npairs, kSvdEigThreads>>>(dG, 1, 1, npairs, tol, negl, inner, dQ, dflag, dmax, dnrot);
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r)
      svd_pair_eig_kernel<<<npairs, kSvdEigThreads>>>(dG, 1, 1, npairs, tol, negl, inner, dQ, dflag, dmax, dnrot);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("npairs=%d inner=%d: %.2f us per launch (%s)\n", npairs, inner, 1e3 * ms / reps,
           cudaGetErrorString(cudaGetLastError()));
  }
  {  // bitwise comparison with the index-table kernel (also with negligible columns / near-diagonal pairs)
    std::vector<double> G2 = G;
    for (int p = 0; p < npairs; p += 3) {
      for (int i = 0; i < 32; ++i) G2[(size_t)p * 1024 + 5 * 32 + i] = G2[(size_t)p * 1024 + i * 32 + 5] = 0.0;  // column 5 zero
    }
    for (int p = 1; p < npairs; p += 3)
      for (int i = 0; i < 32; ++i)
        for (int j = 0; j < 32; ++j)
          if (i != j) G2[(size_t)p * 1024 + i * 32 + j] *= 1e-15;  // nearly converged pair
    int bad = 0;
    for (int variant = 0; variant < 2; ++variant) {
      cudaMemcpy(dG, (variant ? G2 : G).data(), G.size() * 8, cudaMemcpyHostToDevice);
      for (int inner : {1, 3}) {
        std::vector<double> q0(G.size()), q1(G.size());
        std::vector<int> f0(npairs), f1(npairs);
        svd_pair_eig_kernel_old<<<npairs, kSvdEigThreads>>>(dG, 1, 1, npairs, tol, negl, inner, dQ, dflag, dmax, dnrot);
        cudaMemcpy(q0.data(), dQ, G.size() * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(f0.data(), dflag, npairs * 4, cudaMemcpyDeviceToHost);
        cudaMemset(dQ, 0, G.size() * 8);
        svd_pair_eig_kernel<<<npairs, kSvdEigThreads>>>(dG, 1, 1, npairs, tol, negl, inner, dQ, dflag, dmax, dnrot);
        cudaMemcpy(q1.data(), dQ, G.size() * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(f1.data(), dflag, npairs * 4, cudaMemcpyDeviceToHost);
        for (int p = 0; p < npairs; ++p) {
          if (f0[p] != f1[p]) ++bad;
          if (f0[p] && memcmp(&q0[(size_t)p * 1024], &q1[(size_t)p * 1024], 8192) != 0) ++bad;
        }
      }
    }
    cudaMemcpy(dG, G.data(), G.size() * 8, cudaMemcpyHostToDevice);
    printf("bitwise comparison with the index-table kernel: %s (%d mismatching pairs)\n", bad ? "FAIL" : "identical", bad);
    for (int w = 0; w < 3; ++w)
      svd_pair_eig_kernel_old<<<npairs, kSvdEigThreads>>>(dG, 1, 1, npairs, tol, negl, 1, dQ, dflag, dmax, dnrot);
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r)
      svd_pair_eig_kernel_old<<<npairs, kSvdEigThreads>>>(dG, 1, 1, npairs, tol, negl, 1, dQ, dflag, dmax, dnrot);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("index-table kernel: %.2f us per launch\n", 1e3 * ms / reps);
  }
#ifdef HEFF_EIG_INSTR
  long long ins[4];
  svd_pair_eig_kernel<<<npairs, kSvdEigThreads>>>(dG, 1, 1, npairs, tol, negl, 1, dQ, dflag, dmax, dnrot);
  cudaMemcpyFromSymbol(ins, g_eig_instr, sizeof ins);
  printf("pair 0, one inner sweep (31 rounds): update thread %.0f clk/round, rotation lane %.0f clk/round, "
         "round %.0f clk, whole kernel from loop start %lld clk\n", ins[0] / 31.0, ins[1] / 30.0, ins[2] / 31.0, ins[3]);
#endif
  return 0;
}
