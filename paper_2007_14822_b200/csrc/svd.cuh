// svd.cuh -- the two-site split: truncated SVD of the two-site
// wavefunction Psi[(a s1)][(s2 b)] (Sec. 5) by block one-sided (Hestenes)
// Jacobi on FP64 tensor cores.
//
// The columns of a working copy X (Psi moving right, Psi^T moving left) are made mutually
// orthogonal by orthogonal rotations X <- X Q; at convergence X = U S (column norms = the
// singular values, normalised columns = the singular vectors) -- no V is accumulated, the
// next centre is one GEMM with the original Psi afterwards.
//
// Work unit: a PAIR of 16-column blocks (I, J).  Per round of the round-robin ordering all
// nblk/2 pairs are disjoint and run in parallel, two kernels per round:
//   svd_gram_kernel   G = [X_I X_J]^T [X_I X_J] (32 x 32), DMMA over a row range, one
//                     partial per (pair, row split); the 4 loaded values per lane feed 10
//                     DMMA (upper triangle of 4x4 tiles; columns permuted c = 4g + i so one
//                     lane loads 32 contiguous bytes).
//   svd_pair_eig_kernel one CTA per pair: sums the partials (fixed order), tests the pair
//                     for convergence (max |g_ij| / sqrt(g_ii g_jj) over non-negligible
//                     columns) and diagonalises G in shared memory by cyclic two-sided Jacobi
//                     (relative accuracy for graded G) -> Q (32 x 32).
//   svd_rotate_kernel streams a row range of each rotated pair through Y <- Y Q on DMMA,
//                     Q's fragments held in registers.
// Columns are re-sorted by norm at the start of every sweep.  All reductions are
// fixed-order: the result is bitwise deterministic.
//
// Layout: X is stored block-column-major, Xb[blk][r][16] (a block's rows are 128-byte
// contiguous lines), zero-padded to an even number of blocks.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "ptx.cuh"

namespace heff {

constexpr int kSvdB = 16;              // columns per block
constexpr int kSvdPair = 2 * kSvdB;    // columns per pair
constexpr int kSvdGramThreads = 256;
constexpr int kSvdRotThreads = 128;
// Inner sweeps per pair step (host policy, heff_svd_split): one inner sweep of the 32 x 32
// Gram is as good as its full diagonalisation for the outer convergence (prototype: 12 / 25
// outer sweeps for Gaussian / graded inputs with 1, 2, 3 or 30 inner sweeps; on the GPU with
// the LQ preconditioner: C2 / C3 DMRG states 18.0 / 28.8 ms with one inner sweep vs 20.8 /
// 36.6 ms switching to full diagonalisation below an off-diagonal of 1e-2) and much shorter
// on the critical path.  HEFF_SVD_INNER_THRESH=x switches to up to kSvdMaxInnerSweeps inner
// sweeps once the previous outer sweep's max off-diagonal is below x.
constexpr int kSvdMaxInnerSweeps = 12;

// ---------------------------------------------------------------- packing
// Moving right: X = Psi [R][ncols] -> Xb (zero beyond ncols).
__global__ void svd_pack_kernel(const double* __restrict__ psi, double* __restrict__ Xb, int64_t R, int64_t ncols,
                                int64_t nblk, double scale) {
  const int64_t total = nblk * R * kSvdB;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e & (kSvdB - 1));
    const int64_t rb = e >> 4;
    const int64_t blk = rb / R, r = rb - blk * R;
    const int64_t c = blk * kSvdB + j;
    Xb[e] = c < ncols ? scale * psi[r * ncols + c] : 0.0;
  }
}

// Moving left: X = Psi^T, Psi is [ncols][R] -> Xb[blk][r][16] = Psi[blk*16+j][r]; 32x32 tiles.
__global__ void svd_pack_t_kernel(const double* __restrict__ psi, double* __restrict__ Xb, int64_t R, int64_t ncols,
                                  double scale) {
  __shared__ double tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int k = ty; k < 32; k += 8) {
    const int64_t c = c0 + k, r = r0 + tx;
    tile[k][tx] = (c < ncols && r < R) ? scale * psi[c * R + r] : 0.0;
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int64_t r = r0 + k, c = c0 + tx;
    if (r < R) Xb[((c >> 4) * R + r) * kSvdB + (c & 15)] = tile[tx][k];
  }
}

// ---------------------------------------------------------------- max |x| and sum of squares (deterministic)
// part[blockIdx.x] = max |x| over the block's grid-stride range (NaN propagates)
__global__ void svd_maxabs_partial_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ part) {
  __shared__ double red[256];
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = fabs(x[i]);
    m = (v > m || v != v) ? v : m;
  }
  red[threadIdx.x] = m;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      const double o = red[threadIdx.x + w];
      if (o > red[threadIdx.x] || o != o) red[threadIdx.x] = o;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// sum of (scale x)^2 -- scale is a power of two that brings max |x| into [1, 2)
__global__ void svd_sumsq_partial_kernel(const double* __restrict__ x, int64_t n, double scale,
                                         double* __restrict__ part) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = scale * x[i];
    s = fma(v, v, s);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void svd_sum_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += part[i];
    *out = s;
  }
}

// ---------------------------------------------------------------- Gram partials
// Balanced persistent schedule (stream-K style): the work is npairs x C chunks of 128 rows
// (chunk = one pass of the 8 warps x 4 lanes-rows x 4 unrolled rows); CTA b owns the
// contiguous iteration range [T b / G, T (b+1) / G), T = npairs C, G = gridDim.x, so there
// is no wave-quantisation tail.  A pair split across CTAs gets one partial Gram per CTA in
// slot (b - b0(pair)); the eigen kernel sums the slots in order (deterministic).
__host__ __device__ __forceinline__ int64_t svd_sk_start(int64_t T, int64_t b, int64_t G) { return T * b / G; }
__host__ __device__ __forceinline__ int svd_sk_owner(int64_t it, int64_t T, int64_t G) {
  int64_t b = (it * G) / T;
  while (b + 1 < G && svd_sk_start(T, b + 1, G) <= it) ++b;
  while (b > 0 && svd_sk_start(T, b, G) > it) --b;
  return (int)b;
}

// G[4m+i][4n+j] tile accumulation of one 128-row chunk; lane (g, t) holds row (t) columns 4g..4g+3
__device__ __forceinline__ void svd_gram_load(const double* __restrict__ base, int64_t rb, int64_t r_end, int warp,
                                              int t, double (&v)[4][4]) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t r = rb + u * 32 + warp * 4 + t;
    if (r < r_end) {
      const double2* src = reinterpret_cast<const double2*>(base + r * kSvdB);
      const double2 a = __ldg(src), b = __ldg(src + 1);
      v[u][0] = a.x; v[u][1] = a.y; v[u][2] = b.x; v[u][3] = b.y;
    } else {
      v[u][0] = v[u][1] = v[u][2] = v[u][3] = 0.0;
    }
  }
}

__global__ void __launch_bounds__(kSvdGramThreads, 2) svd_gram_kernel(const double* __restrict__ Xb, int64_t R,
                                                                   const int2* __restrict__ pairs, int npairs,
                                                                   int nslots, double* __restrict__ Gp) {
  __shared__ double red[kSvdGramThreads / 32][10 * 64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int64_t C = (R + 127) / 128;
  const int64_t T = (int64_t)npairs * C, G = gridDim.x;
  int64_t it = svd_sk_start(T, blockIdx.x, G);
  const int64_t it_end = svd_sk_start(T, blockIdx.x + 1, G);
  while (it < it_end) {
    const int p = (int)(it / C);
    const int64_t ch0 = it - (int64_t)p * C;
    const int64_t ch1 = min(C, ch0 + (it_end - it));
    const int2 pr = pairs[p];
    const double* base = Xb + (int64_t)(g < 4 ? pr.x : pr.y) * R * kSvdB + (g & 3) * 4;
    double acc[10][2];
#pragma unroll
    for (int i = 0; i < 10; ++i) acc[i][0] = acc[i][1] = 0.0;
    double v[4][4], w[4][4];
    svd_gram_load(base, ch0 * 128, R, warp, t, v);
    for (int64_t ch = ch0; ch < ch1; ++ch) {
      if (ch + 1 < ch1) svd_gram_load(base, (ch + 1) * 128, R, warp, t, w);  // prefetch
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int idx = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = i; j < 4; ++j, ++idx) dmma_8x8x4(acc[idx][0], acc[idx][1], v[u][i], v[u][j]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int q = 0; q < 4; ++q) v[u][q] = w[u][q];
    }
    // partial of this pair -> slot (b - b0)
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      red[warp][i * 64 + lane * 2] = acc[i][0];
      red[warp][i * 64 + lane * 2 + 1] = acc[i][1];
    }
    __syncthreads();
    const int slot = (int)blockIdx.x - svd_sk_owner((int64_t)p * C, T, G);
    double* out = Gp + ((int64_t)p * nslots + slot) * (kSvdPair * kSvdPair);
    for (int e = threadIdx.x; e < 10 * 64; e += blockDim.x) {
      double sum = 0.0;
#pragma unroll
      for (int ww = 0; ww < kSvdGramThreads / 32; ++ww) sum += red[ww][e];
      const int idx = e >> 6, l = (e >> 1) & 31, h = e & 1;
      int i = 0, j = 0, k = idx;  // idx -> (i, j), i <= j, row-major over the upper triangle
      for (i = 0; i < 4; ++i) {
        if (k < 4 - i) { j = i + k; break; }
        k -= 4 - i;
      }
      const int gm = l >> 2, tn = l & 3;
      const int row = 4 * gm + i, col = 4 * (2 * tn + h) + j;
      out[row * kSvdPair + col] = sum;
      if (i != j) out[col * kSvdPair + row] = sum;
    }
    __syncthreads();
    it += ch1 - ch0;
  }
}

// ---------------------------------------------------------------- pair eigen-solve
// One CTA per pair: sum the Gram partials (fixed order), test the pair (max |g_ij| /
// sqrt(g_ii g_jj) over non-negligible columns), and if it is not converged diagonalise G by
// cyclic two-sided Jacobi in shared memory (parallel round-robin ordering, 16 disjoint
// rotations per round).  Each round is one parameter phase and one update phase: every
// 2x2 block (pair k rows, pair k' columns) of G <- J^T G J depends only on its old values,
// so a thread updates a whole block at once (the diagonal blocks get the exact rotated
// 2x2 values), and Q <- Q J by columns.  Output: Qg[p] (row-major 32x32), flag[p].
#ifdef HEFF_EIG_INSTR
__device__ long long g_eig_instr[4];
#endif
constexpr int kSvdEigThreads = 288;  // 8 warps of 2x2-block updates + 1 warp for the next round's rotations

// FP64 rsqrt / reciprocal: MUFU approximation + two Newton steps (full precision for the
// normal, positive arguments used here; any rounding in t only leaves a slightly larger
// residual off-diagonal -- the rotation itself stays orthogonal because c, s come from t)
__device__ __forceinline__ double svd_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}
__device__ __forceinline__ double svd_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * fma(-x, y, 2.0);
  y = y * fma(-x, y, 2.0);
  return y;
}

struct SvdRot {
  double c, s, na, nb;  // rotation and the exact rotated diagonal of the pair
  int on;
};

// Jacobi rotation of the 2x2 block [[app, apq], [apq, aqq]]: with th = aqq - app,
// om = 2 apq, r = sqrt(th^2 + om^2) and x = |th| / r (= |cos 2phi|),
//   c = sqrt((1 + x) / 2),  s = sign(th) om / (2 r c),  t = s / c = sign(th) om / (|th| + r)
// (the same rotation as t = sign(th) om / (|th| + r), c = 1 / sqrt(1 + t^2), with two
// dependent reciprocal square roots on the critical path instead of three transcendental
// steps; c is in [1/sqrt 2, 1], so the half-angle form is well conditioned).
__device__ __forceinline__ SvdRot svd_make_rot(double app, double aqq, double apq, bool active, double tol) {
  SvdRot r{1.0, 0.0, app, aqq, 0};
  if (active && apq * apq > (tol * tol) * (app * aqq)) {  // |apq| > tol sqrt(app aqq), no sqrt
    const double th = aqq - app, om = 2.0 * apq;
    const double ir = svd_rsqrt(fma(th, th, om * om));      // 1 / r
    const double y = fma(0.5 * fabs(th), ir, 0.5);          // c^2 = (1 + x) / 2
    const double ry = svd_rsqrt(y);                          // 1 / c
    const double so = (th >= 0.0 ? om : -om) * (0.5 * ir);   // sign(th) om / (2 r)
    const double tt = so * (ry * ry);                        // t = s / c
    r.c = y * ry;
    r.s = so * ry;
    r.na = app - tt * apq;
    r.nb = aqq + tt * apq;
    r.on = 1;
  }
  return r;
}

// new 2x2 block (rows of pair k, columns of pair kk) of J^T G J from the old one
__device__ __forceinline__ void svd_rot_block(double& x00, double& x01, double& x10, double& x11, const SvdRot& rk,
                                              const SvdRot& rkk) {
  if (rkk.on) {  // columns: [x.0 x.1] <- [x.0 x.1] [[c, s], [-s, c]]
    const double y00 = rkk.c * x00 - rkk.s * x01, y01 = rkk.s * x00 + rkk.c * x01;
    const double y10 = rkk.c * x10 - rkk.s * x11, y11 = rkk.s * x10 + rkk.c * x11;
    x00 = y00; x01 = y01; x10 = y10; x11 = y11;
  }
  if (rk.on) {   // rows: [x0. ; x1.] <- [[c, -s], [s, c]] [x0. ; x1.]
    const double y00 = rk.c * x00 - rk.s * x10, y10 = rk.s * x00 + rk.c * x10;
    const double y01 = rk.c * x01 - rk.s * x11, y11 = rk.s * x01 + rk.c * x11;
    x00 = y00; x01 = y01; x10 = y10; x11 = y11;
  }
}

// Position layout: G and Q are stored by POSITION, and pair k of every round is positions
// (k, 31-k).  After a round the column at position i moves to svd_np(i) (0 stays, 1 -> 31,
// i -> i-1): the circle method of round-robin ordering with the data moving instead of the
// index tables, so every thread's shared-memory addresses are fixed for the whole kernel.
// After 31 rounds every column is back at its own position.  (Same rotations, in the same
// order and arithmetic, as the index-table form: results are bitwise unchanged.)
__device__ __forceinline__ double svd_lds(uint32_t a) {
  double x;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(a) : "memory");
  return x;
}
__device__ __forceinline__ void svd_lds2(double& x, double& y, uint32_t a) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a) : "memory");
}
__device__ __forceinline__ void svd_sts(uint32_t a, double x) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(x) : "memory");
}
__device__ __forceinline__ int svd_np(int i) { return i == 0 ? 0 : (i == 1 ? 31 : i - 1); }
__device__ __forceinline__ int svd_np_inv(int i) { return i == 0 ? 0 : (i == 31 ? 1 : i + 1); }

__global__ void __launch_bounds__(kSvdEigThreads) svd_pair_eig_kernel(const double* __restrict__ Gp, int nslots,
                                                                     int64_t C, int gram_grid,
                                                                     double tol, double negl, int inner_sweeps,
                                                                     double* __restrict__ Qg, int* __restrict__ flag,
                                                                     unsigned long long* __restrict__ stat_maxoff,
                                                                     int* __restrict__ stat_nrot) {
  __shared__ double Gs[2][kSvdPair][kSvdPair + 1];   // ping-pong by round, position order
  __shared__ double Qs[2][kSvdPair][kSvdPair + 1];   // Q[row][position], ping-pong by round
  __shared__ double2 s_cs[2][16], s_nn[2][16];       // (c, s) and the rotated diagonal per pair
  __shared__ int s_on[2][16];
  __shared__ int s_neg[kSvdPair];                    // by column
  __shared__ int s_any[kSvdMaxInnerSweeps];          // did inner sweep i rotate anything
  __shared__ double s_off[kSvdEigThreads / 32];
  const int p = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  pdl_wait();                 // the Gram partials of this round
  const double* gsrc = Gp + (int64_t)p * nslots * (kSvdPair * kSvdPair);
  const int64_t T = (int64_t)gridDim.x * C;  // gridDim.x = npairs
  const int nsum = svd_sk_owner((int64_t)p * C + C - 1, T, gram_grid) - svd_sk_owner((int64_t)p * C, T, gram_grid) + 1;
  for (int e = tid; e < kSvdPair * kSvdPair; e += blockDim.x) {
    double v = 0.0;
    for (int sp = 0; sp < nsum; ++sp) v += gsrc[(int64_t)sp * (kSvdPair * kSvdPair) + e];
    const int r = e >> 5, c = e & 31;
    Gs[0][r][c] = v;
    Qs[0][r][c] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
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
  // 2x2 block of the rotated G (and two rotated Q entries per row pair) into the other
  // buffers at the columns' next positions, while the rotation warp already computes round
  // rr+1's rotations from the OLD G and round rr's rotations.  Rotations live as (c, s)
  // pairs -- the identity (1, 0) for a skipped pair, so the updates are branch-free -- plus
  // the exact rotated diagonal (na, nb) and an on flag.
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
  if (tid < 16)  // round 0: the column at position i is column i
    put_rot(0, tid, svd_make_rot(Gs[0][tid][tid], Gs[0][31 - tid][31 - tid], Gs[0][tid][31 - tid],
                                 !s_neg[tid] && !s_neg[31 - tid], tol));
  if (tid < kSvdMaxInnerSweeps) s_any[tid] = 0;
  __syncthreads();
  // update threads (tid < 256): G block (pair k rows, pair kk columns); Q rows k and k + 16 at pair kk
  const int k = (tid >> 4) & 15, kk = tid & 15;
  const int ra = k, rb = 31 - k, ca = kk, cb = 31 - kk;
  const int nra = svd_np(ra), nrb = svd_np(rb), nca = svd_np(ca), ncb = svd_np(cb);
  // rotation lane pl (tid 256..271): next round's pair pl = positions (pl, 31-pl), whose
  // columns sit this round at positions pa, pb, in pairs kA, kB (second element if hA / hB)
  const int pl = tid - 256;
  const int pa = svd_np_inv(pl & 15), pb = svd_np_inv(31 - (pl & 15));
  const int kA = min(pa, 31 - pa), kB = min(pb, 31 - pb);
  const bool hA = pa > 15, hB = pb > 15;
  // every shared-memory address below is a fixed byte offset from the round's buffer base
  constexpr uint32_t kBuf = kSvdPair * (kSvdPair + 1) * 8;
  auto soff = [](int r, int c) { return (uint32_t)((r * (kSvdPair + 1) + c) * 8); };
  const uint32_t sG = smem_u32(&Gs[0][0][0]), sQ = smem_u32(&Qs[0][0][0]);
  const uint32_t sCS = smem_u32(&s_cs[0][0]), sNN = smem_u32(&s_nn[0][0]);
  const uint32_t o_aa = soff(ra, ca), o_ab = soff(ra, cb), o_ba = soff(rb, ca), o_bb = soff(rb, cb);
  const uint32_t w_aa = soff(nra, nca), w_ab = soff(nra, ncb), w_ba = soff(nrb, nca), w_bb = soff(nrb, ncb);
  const uint32_t d_ab = soff(ra, rb), dw_aa = soff(nra, nra), dw_bb = soff(nrb, nrb), dw_ab = soff(nra, nrb),
                 dw_ba = soff(nrb, nra);
  const uint32_t q0a = soff(k, ca), q0b = soff(k, cb), q1a = soff(k + 16, ca), q1b = soff(k + 16, cb);
  const uint32_t qw0a = soff(k, nca), qw0b = soff(k, ncb), qw1a = soff(k + 16, nca), qw1b = soff(k + 16, ncb);
  const uint32_t x_00 = soff(kA, kB), x_01 = soff(kA, 31 - kB), x_10 = soff(31 - kA, kB), x_11 = soff(31 - kA, 31 - kB);
  const int total_rounds = 31 * min(inner_sweeps, kSvdMaxInnerSweeps);
  int cur = 0;
#ifdef HEFF_EIG_INSTR  // tools/eigbench: cycles per round (update thread 0, rotation lane 0, whole round)
  long long ins_t0 = clock64(), ins_upd = 0, ins_rot = 0, ins_round = 0;
#endif
  for (int it = 0; it < total_rounds; ++it) {
#ifdef HEFF_EIG_INSTR
    const long long ins_tb = clock64();
#endif
    const int rr = it % 31, nxt = cur ^ 1;
    const int sweep = it / 31;
    const uint32_t go = sG + cur * kBuf, gn = sG + nxt * kBuf, qo = sQ + cur * kBuf, qn = sQ + nxt * kBuf;
    const uint32_t cs = sCS + cur * 256, nnb_ = sNN + cur * 256;
    if (tid < 256) {
      double qx, qy;  // rotation of pair kk
      svd_lds2(qx, qy, cs + kk * 16);
      if (k == kk) {
        double nx, ny;
        svd_lds2(nx, ny, nnb_ + k * 16);
        const double o = s_on[cur][k] ? 0.0 : svd_lds(go + d_ab);
        svd_sts(gn + dw_aa, nx);
        svd_sts(gn + dw_bb, ny);
        svd_sts(gn + dw_ab, o);
        svd_sts(gn + dw_ba, o);
      } else {
        double x00 = svd_lds(go + o_aa), x01 = svd_lds(go + o_ab), x10 = svd_lds(go + o_ba), x11 = svd_lds(go + o_bb);
        double kx, ky;
        svd_lds2(kx, ky, cs + k * 16);
        rot2(x00, x01, x10, x11, make_double2(kx, ky), make_double2(qx, qy));
        svd_sts(gn + w_aa, x00);
        svd_sts(gn + w_ab, x01);
        svd_sts(gn + w_ba, x10);
        svd_sts(gn + w_bb, x11);
      }
      {  // Q <- Q J: columns of pair kk, rows k and k + 16
        const double a0 = svd_lds(qo + q0a), b0 = svd_lds(qo + q0b), a1 = svd_lds(qo + q1a), b1 = svd_lds(qo + q1b);
        svd_sts(qn + qw0a, qx * a0 - qy * b0);
        svd_sts(qn + qw0b, qy * a0 + qx * b0);
        svd_sts(qn + qw1a, qx * a1 - qy * b1);
        svd_sts(qn + qw1b, qy * a1 + qx * b1);
      }
      if (tid < 16 && s_on[cur][tid]) s_any[sweep] = 1;
#ifdef HEFF_EIG_INSTR
      if (tid == 0) ins_upd += clock64() - ins_tb;
#endif
    } else if (pl < 16 && it + 1 < total_rounds) {
      double nax, nay, nbx, nby, ckx, cky, ckkx, ckky;
      svd_lds2(nax, nay, nnb_ + kA * 16);
      svd_lds2(nbx, nby, nnb_ + kB * 16);
      svd_lds2(ckx, cky, cs + kA * 16);
      svd_lds2(ckkx, ckky, cs + kB * 16);
      const double app = hA ? nay : nax;                       // rotated diagonals: exact values
      const double aqq = hB ? nby : nbx;
      // rotated off-diagonal: the two columns sit in different pairs of round rr
      double x00 = svd_lds(go + x_00), x01 = svd_lds(go + x_01), x10 = svd_lds(go + x_10), x11 = svd_lds(go + x_11);
      rot2(x00, x01, x10, x11, make_double2(ckx, cky), make_double2(ckkx, ckky));
      const double apq = hA ? (hB ? x11 : x10) : (hB ? x01 : x00);
      // the columns at positions pl, 31-pl in round rr+1 (circle method)
      const int r1 = rr + 1 == 31 ? 0 : rr + 1;
      int ca1 = pl - 1 + r1, cb1 = 30 - pl + r1;
      ca1 = pl == 0 ? 0 : (ca1 >= 31 ? ca1 - 31 : ca1) + 1;
      cb1 = (cb1 >= 31 ? cb1 - 31 : cb1) + 1;
      put_rot(nxt, pl, svd_make_rot(app, aqq, apq, !s_neg[ca1] && !s_neg[cb1], tol));
#ifdef HEFF_EIG_INSTR
      if (pl == 0) ins_rot += clock64() - ins_tb;
#endif
    }
    __syncthreads();
#ifdef HEFF_EIG_INSTR
    ins_round += clock64() - ins_tb;
#endif
    cur = nxt;
    if (rr == 30 && !s_any[sweep]) break;  // end of an inner sweep that rotated nothing
  }
  double* q = Qg + (int64_t)p * (kSvdPair * kSvdPair);
  for (int e = tid; e < kSvdPair * kSvdPair; e += blockDim.x) q[e] = Qs[cur][e >> 5][e & 31];
#ifdef HEFF_EIG_INSTR
  if (p == 0 && tid == 0) { g_eig_instr[0] = ins_upd; g_eig_instr[2] = ins_round; g_eig_instr[3] = clock64() - ins_t0; }
  if (p == 0 && tid == 256) g_eig_instr[1] = ins_rot;
#endif
}

// ---------------------------------------------------------------- rotation
// Y <- Y Q on the rotated pairs.  A = Y (row g, k-slice kk of lane t = column 8t + kk),
// B = Q fragments held in registers, D tile n = output columns 8n + {2t, 2t+1}.
// Balanced persistent schedule over npairs x C2 groups of 32 rows (4 warps x 8 rows), the
// next group's rows prefetched into registers while the current one is on the DMMA pipe.
__device__ __forceinline__ void svd_rot_load(const double* __restrict__ src, bool ok, double (&y)[8]) {
  if (ok) {
    const double2* s2 = reinterpret_cast<const double2*>(src);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double2 v = s2[q];
      y[2 * q] = v.x;
      y[2 * q + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) y[q] = 0.0;
  }
}

__global__ void __launch_bounds__(kSvdRotThreads, 4) svd_rotate_kernel(double* __restrict__ Xb, int64_t R,
                                                                      const int2* __restrict__ pairs, int npairs,
                                                                      const double* __restrict__ Qg,
                                                                      const int* __restrict__ flag) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int64_t C2 = (R + 31) / 32;
  const int64_t T = (int64_t)npairs * C2, G = gridDim.x;
  int64_t it = svd_sk_start(T, blockIdx.x, G);
  const int64_t it_end = svd_sk_start(T, blockIdx.x + 1, G);
  while (it < it_end) {
    const int p = (int)(it / C2);
    const int64_t g0 = it - (int64_t)p * C2;
    const int64_t g1 = min(C2, g0 + (it_end - it));
    it += g1 - g0;
    if (!flag[p]) continue;
    const double* q = Qg + (int64_t)p * (kSvdPair * kSvdPair);
    double qf[8][4];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
#pragma unroll
      for (int n = 0; n < 4; ++n) qf[kk][n] = __ldg(q + (8 * t + kk) * kSvdPair + 8 * n + g);
    const int2 pr = pairs[p];
    double* XI = Xb + (int64_t)pr.x * R * kSvdB;
    double* XJ = Xb + (int64_t)pr.y * R * kSvdB;
    const double* src_base = (t < 2 ? XI : XJ) + (t & 1) * 8;
    double y[8], yn[8];
    int64_t row = g0 * 32 + warp * 8 + g;
    svd_rot_load(src_base + row * kSvdB, row < R, y);
    for (int64_t gi = g0; gi < g1; ++gi) {
      const int64_t nrow = row + 32;
      if (gi + 1 < g1) svd_rot_load(src_base + nrow * kSvdB, nrow < R, yn);  // prefetch
      double acc[4][2];
#pragma unroll
      for (int n = 0; n < 4; ++n) acc[n][0] = acc[n][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
#pragma unroll
        for (int n = 0; n < 4; ++n) dmma_8x8x4(acc[n][0], acc[n][1], y[kk], qf[kk][n]);
      if (row < R) {
#pragma unroll
        for (int n = 0; n < 4; ++n) {
          double* dst = (n < 2 ? XI : XJ) + row * kSvdB + (((8 * n) & 15) + 2 * t);
          *reinterpret_cast<double2*>(dst) = make_double2(acc[n][0], acc[n][1]);
        }
      }
#pragma unroll
      for (int qq = 0; qq < 8; ++qq) y[qq] = yn[qq];
      row = nrow;
    }
  }
}

// X columns permuted into descending-norm order at the start of a sweep (de Rijk-style
// ordering: the round-robin then meets the dominant columns first):
// dst[blk][r][j] = src column perm[blk*16 + j] (zero for padding columns >= ncols).
__global__ void svd_permute_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t R, int64_t ncols,
                                   int64_t nblk, const int* __restrict__ perm) {
  const int64_t total = nblk * R * kSvdB;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e & (kSvdB - 1));
    const int64_t rb = e >> 4;
    const int64_t blk = rb / R, r = rb - blk * R;
    const int64_t c = blk * kSvdB + j;
    double v = 0.0;
    if (c < ncols) {
      const int sc = perm[c];
      v = src[(((int64_t)(sc >> 4)) * R + r) * kSvdB + (sc & 15)];
    }
    dst[e] = v;
  }
}

// ---------------------------------------------------------------- extraction
// norms[c] = ||X[:, c]|| for c < ncols; one CTA (256 threads) per 16-column block
__global__ void svd_colnorm_kernel(const double* __restrict__ Xb, int64_t R, int64_t ncols, double* __restrict__ norms) {
  __shared__ double red[256];
  const int64_t blk = blockIdx.x;
  const int j = threadIdx.x & 15, rl = threadIdx.x >> 4;
  double s = 0.0;
  for (int64_t r = rl; r < R; r += 16) {
    const double x = Xb[(blk * R + r) * kSvdB + j];
    s = fma(x, x, s);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x < 16) {
    double tot = 0.0;
    for (int q = 0; q < 16; ++q) tot += red[q * 16 + threadIdx.x];
    const int64_t c = blk * kSvdB + threadIdx.x;
    if (c < ncols) norms[c] = sqrt(tot);
  }
}

// scale[k] = sign / s_k, sign making the largest-|.| entry of column perm[k] positive (first on ties)
// rowperm (nullable): X's row r is row rowperm[r] of the output factor (ties break on that index)
__global__ void svd_sign_kernel(const double* __restrict__ Xb, int64_t R, const int* __restrict__ perm,
                                const double* __restrict__ s, double* __restrict__ scale, const int* __restrict__ rowperm) {
  __shared__ double sv[256];
  __shared__ int64_t si[256], sx[256];
  const int k = blockIdx.x;
  const int c = perm[k];
  const double* col = Xb + (int64_t)(c >> 4) * R * kSvdB + (c & 15);
  double best = -1.0;
  int64_t bi = 0, bx = 0;  // output-row index (tie-break), X row
  for (int64_t r = threadIdx.x; r < R; r += blockDim.x) {
    const double a = fabs(col[r * kSvdB]);
    const int64_t ri = rowperm ? rowperm[r] : r;
    if (a > best || (a == best && ri < bi)) { best = a; bi = ri; bx = r; }
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  sx[threadIdx.x] = bx;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      const double o = sv[threadIdx.x + w];
      const int64_t oi = si[threadIdx.x + w];
      if (o > sv[threadIdx.x] || (o == sv[threadIdx.x] && oi < si[threadIdx.x])) {
        sv[threadIdx.x] = o;
        si[threadIdx.x] = oi;
        sx[threadIdx.x] = sx[threadIdx.x + w];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) scale[k] = (col[sx[0] * kSvdB] < 0.0 ? -1.0 : 1.0) / s[k];
}

// out[k][r] = X[r][perm k] * scale[k]   (k < n: grid.y; r < R)
__global__ void svd_gather_t_kernel(const double* __restrict__ Xb, int64_t R, const int* __restrict__ perm,
                                    const double* __restrict__ scale, double* __restrict__ out,
                                    const int* __restrict__ rowperm, int64_t n) {
  for (int64_t k = blockIdx.y; k < n; k += gridDim.y) {
    const int c = perm[k];
    const double sc = scale[k];
    const double* col = Xb + (int64_t)(c >> 4) * R * kSvdB + (c & 15);
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x)
      out[k * R + (rowperm ? rowperm[r] : r)] = col[r * kSvdB] * sc;
  }
}

// row norms^2 of a row-major matrix (one warp per row)
__global__ void svd_rownorm2_kernel(const double* __restrict__ A, int64_t rows, int64_t cols, double* __restrict__ out) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  double acc = 0.0;
  for (int64_t c = lane; c < cols; c += 32) {
    const double v = A[row * cols + c];
    acc = fma(v, v, acc);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[row] = acc;
}

// dst row r = src row perm[r] (row-major, cols per row)
__global__ void svd_gather_rows_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t rows,
                                       int64_t cols, const int* __restrict__ perm, double scale) {
  for (int64_t row = blockIdx.y; row < rows; row += gridDim.y) {
    const double* sr = src + (int64_t)perm[row] * cols;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += (int64_t)gridDim.x * blockDim.x)
      dst[row * cols + c] = scale * sr[c];
  }
}


// ---------------------------------------------------------------- TMA-fed Gram and rotation
// The same work as svd_gram_kernel / svd_rotate_kernel with the pair's rows streamed into a
// shared-memory ring by TMA (one 2-D tensor map over Xb viewed as [nblk*R rows][16 cols],
// 128-byte rows, 128-byte swizzle): one producer lane keeps STAGES chunks in flight, the
// DMMA warps read fragments from shared memory.  Rows past R inside a chunk belong to the
// next block (or are zero-filled past the end) and are masked.
constexpr int kSvdTmaRotRows = 64, kSvdTmaRotStages = 4, kSvdTmaRotWarps = 4;
constexpr int kSvdTmaGramRows = 128, kSvdTmaGramStages = 3, kSvdTmaGramWarps = 8;
constexpr int kSvdTmaRotSmem = kSvdTmaRotStages * 2 * kSvdTmaRotRows * 128 + 1024 + 64;
constexpr int kSvdTmaGramSmem = kSvdTmaGramStages * 2 * kSvdTmaGramRows * 128 + kSvdTmaGramWarps * 640 * 8 + 1024 + 64;

__device__ __forceinline__ uint32_t svd_swz(uint32_t buf, int row, int chunk) {
  return buf + row * 128 + ((chunk ^ (row & 7)) << 4);
}

__global__ void __launch_bounds__((kSvdTmaRotWarps + 1) * 32) svd_rotate_tma_kernel(
    const __grid_constant__ CUtensorMap xmap, double* __restrict__ Xb, int64_t R, const int2* __restrict__ pairs,
    int npairs, const double* __restrict__ Qg, const int* __restrict__ flag) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kStageBytes = 2 * kSvdTmaRotRows * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSvdTmaRotStages * kStageBytes);
  uint64_t* empty = full + kSvdTmaRotStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kSvdTmaRotStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kSvdTmaRotWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();                 // Q and flags of this round's eigen-solve
  const int64_t C2 = (R + kSvdTmaRotRows - 1) / kSvdTmaRotRows;
  const int64_t T = (int64_t)npairs * C2, G = gridDim.x;
  const int64_t it_begin = svd_sk_start(T, blockIdx.x, G), it_end = svd_sk_start(T, blockIdx.x + 1, G);
  int stage = 0;
  uint32_t phase = 0;
  if (warp == kSvdTmaRotWarps) {  // producer
    if (lane == 0) {
      tma_prefetch_desc(&xmap);
      for (int64_t it = it_begin; it < it_end;) {
        const int p = (int)(it / C2);
        const int64_t g0 = it - (int64_t)p * C2, g1 = min(C2, g0 + (it_end - it));
        it += g1 - g0;
        if (!flag[p]) continue;
        const int2 pr = pairs[p];
        for (int64_t ch = g0; ch < g1; ++ch) {
          mbar_wait(&empty[stage], phase ^ 1);
          unsigned char* sI = smem + stage * kStageBytes;
          mbar_arrive_expect_tx(&full[stage], kStageBytes);
          tma_load_2d(sI, &xmap, &full[stage], 0, (int32_t)((int64_t)pr.x * R + ch * kSvdTmaRotRows));
          tma_load_2d(sI + kStageBytes / 2, &xmap, &full[stage], 0, (int32_t)((int64_t)pr.y * R + ch * kSvdTmaRotRows));
          if (++stage == kSvdTmaRotStages) { stage = 0; phase ^= 1; }
        }
      }
    }
    return;
  }
  const int g = lane >> 2, t = lane & 3;
  const uint32_t sbase = smem_u32(smem);
  for (int64_t it = it_begin; it < it_end;) {
    const int p = (int)(it / C2);
    const int64_t g0 = it - (int64_t)p * C2, g1 = min(C2, g0 + (it_end - it));
    it += g1 - g0;
    if (!flag[p]) continue;
    const double* q = Qg + (int64_t)p * (kSvdPair * kSvdPair);
    double qf[8][4];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
#pragma unroll
      for (int n = 0; n < 4; ++n)  // k-slice kk of lane t = Y column 4t + kk (I) or 16 + 4t + kk - 4 (J)
        qf[kk][n] = __ldg(q + (kk < 4 ? 4 * t + kk : 12 + 4 * t + kk) * kSvdPair + 8 * n + g);
    const int2 pr = pairs[p];
    double* XI = Xb + (int64_t)pr.x * R * kSvdB;
    double* XJ = Xb + (int64_t)pr.y * R * kSvdB;
    for (int64_t ch = g0; ch < g1; ++ch) {
      mbar_wait(&full[stage], phase);
      // every quarter-warp reads one buffer at 8 distinct swizzled chunks: conflict-free
      const uint32_t bufI = sbase + stage * kStageBytes, bufJ = bufI + kStageBytes / 2;
      double y[2][8];
#pragma unroll
      for (int grp = 0; grp < 2; ++grp) {
        const int rl = warp * 16 + grp * 8 + g;
        lds128(y[grp][0], y[grp][1], svd_swz(bufI, rl, 2 * t));
        lds128(y[grp][2], y[grp][3], svd_swz(bufI, rl, 2 * t + 1));
        lds128(y[grp][4], y[grp][5], svd_swz(bufJ, rl, 2 * t));
        lds128(y[grp][6], y[grp][7], svd_swz(bufJ, rl, 2 * t + 1));
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == kSvdTmaRotStages) { stage = 0; phase ^= 1; }
#pragma unroll
      for (int grp = 0; grp < 2; ++grp) {
        const int64_t row = ch * kSvdTmaRotRows + warp * 16 + grp * 8 + g;
        double acc[4][2];
#pragma unroll
        for (int n = 0; n < 4; ++n) acc[n][0] = acc[n][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
#pragma unroll
          for (int n = 0; n < 4; ++n) dmma_8x8x4(acc[n][0], acc[n][1], y[grp][kk], qf[kk][n]);
        if (row < R) {
#pragma unroll
          for (int n = 0; n < 4; ++n) {
            double* dst = (n < 2 ? XI : XJ) + row * kSvdB + (((8 * n) & 15) + 2 * t);
            *reinterpret_cast<double2*>(dst) = make_double2(acc[n][0], acc[n][1]);
          }
        }
      }
    }
  }
}

__global__ void __launch_bounds__((kSvdTmaGramWarps + 1) * 32) svd_gram_tma_kernel(
    const __grid_constant__ CUtensorMap xmap, int64_t R, const int2* __restrict__ pairs, int npairs, int nslots,
    double* __restrict__ Gp) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kStageBytes = 2 * kSvdTmaGramRows * 128;
  double* red = reinterpret_cast<double*>(smem + kSvdTmaGramStages * kStageBytes);   // [warps][640]
  uint64_t* full = reinterpret_cast<uint64_t*>(red + kSvdTmaGramWarps * 640);
  uint64_t* empty = full + kSvdTmaGramStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kSvdTmaGramStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kSvdTmaGramWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();                 // Xb of the previous round's rotation; Gp free again
  const int64_t C = (R + kSvdTmaGramRows - 1) / kSvdTmaGramRows;
  const int64_t T = (int64_t)npairs * C, G = gridDim.x;
  const int64_t it_begin = svd_sk_start(T, blockIdx.x, G), it_end = svd_sk_start(T, blockIdx.x + 1, G);
  int stage = 0;
  uint32_t phase = 0;
  if (warp == kSvdTmaGramWarps) {  // producer
    if (lane == 0) {
      tma_prefetch_desc(&xmap);
      for (int64_t it = it_begin; it < it_end;) {
        const int p = (int)(it / C);
        const int64_t c0 = it - (int64_t)p * C, c1 = min(C, c0 + (it_end - it));
        it += c1 - c0;
        const int2 pr = pairs[p];
        for (int64_t ch = c0; ch < c1; ++ch) {
          mbar_wait(&empty[stage], phase ^ 1);
          unsigned char* sI = smem + stage * kStageBytes;
          mbar_arrive_expect_tx(&full[stage], kStageBytes);
          tma_load_2d(sI, &xmap, &full[stage], 0, (int32_t)((int64_t)pr.x * R + ch * kSvdTmaGramRows));
          tma_load_2d(sI + kStageBytes / 2, &xmap, &full[stage], 0, (int32_t)((int64_t)pr.y * R + ch * kSvdTmaGramRows));
          if (++stage == kSvdTmaGramStages) { stage = 0; phase ^= 1; }
        }
      }
    }
    // the producer joins the pair-boundary reductions below through named barrier 1? no:
    // it exits; the consumers synchronise among themselves with bar.sync 1, 256
    return;
  }
  const int g = lane >> 2, t = lane & 3;
  const uint32_t sbase = smem_u32(smem);
  for (int64_t it = it_begin; it < it_end;) {
    const int p = (int)(it / C);
    const int64_t c0 = it - (int64_t)p * C, c1 = min(C, c0 + (it_end - it));
    it += c1 - c0;
    double acc[10][2];
#pragma unroll
    for (int i = 0; i < 10; ++i) acc[i][0] = acc[i][1] = 0.0;
    for (int64_t ch = c0; ch < c1; ++ch) {
      mbar_wait(&full[stage], phase);
      const uint32_t buf = sbase + stage * kStageBytes + (g < 4 ? 0 : kStageBytes / 2);
      double v[4][4];
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        // the 4 rows of k-step ks: 8-row group ks/2, rows {0,1,4,5} + 2 (ks&1) of it, so the
        // swizzled chunks 2g', 2g'+1 of a quarter-warp land in 8 distinct bank groups
        const int rl = warp * 16 + (ks >> 1) * 8 + 2 * (ks & 1) + (t & 1) + 4 * (t >> 1);
        const bool ok = ch * kSvdTmaGramRows + rl < R;
        double a, b, c, d;
        lds128(a, b, svd_swz(buf, rl, 2 * (g & 3)));
        lds128(c, d, svd_swz(buf, rl, 2 * (g & 3) + 1));
        v[ks][0] = ok ? a : 0.0; v[ks][1] = ok ? b : 0.0; v[ks][2] = ok ? c : 0.0; v[ks][3] = ok ? d : 0.0;
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == kSvdTmaGramStages) { stage = 0; phase ^= 1; }
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        int idx = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = i; j < 4; ++j, ++idx) dmma_8x8x4(acc[idx][0], acc[idx][1], v[ks][i], v[ks][j]);
      }
    }
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      red[warp * 640 + i * 64 + lane * 2] = acc[i][0];
      red[warp * 640 + i * 64 + lane * 2 + 1] = acc[i][1];
    }
    asm volatile("bar.sync 1, %0;" ::"r"(kSvdTmaGramWarps * 32) : "memory");
    const int slot = (int)blockIdx.x - svd_sk_owner((int64_t)p * C, T, G);
    double* out = Gp + ((int64_t)p * nslots + slot) * (kSvdPair * kSvdPair);
    for (int e = threadIdx.x; e < 10 * 64; e += kSvdTmaGramWarps * 32) {
      double sum = 0.0;
#pragma unroll
      for (int ww = 0; ww < kSvdTmaGramWarps; ++ww) sum += red[ww * 640 + e];
      const int idx = e >> 6, l = (e >> 1) & 31, h = e & 1;
      int i = 0, j = 0, k = idx;
      for (i = 0; i < 4; ++i) {
        if (k < 4 - i) { j = i + k; break; }
        k -= 4 - i;
      }
      const int gm = l >> 2, tn = l & 3;
      const int row = 4 * gm + i, col = 4 * (2 * tn + h) + j;
      out[row * kSvdPair + col] = sum;
      if (i != j) out[col * kSvdPair + row] = sum;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(kSvdTmaGramWarps * 32) : "memory");
  }
}

// ---------------------------------------------------------------- U(1) block split helpers
// flag = 1 if Psi has a nonzero entry outside its charge blocks (qrow[r] != qcol[c])
__global__ void svd_qn_check_kernel(const double* __restrict__ psi, int64_t M, int64_t N, const int* __restrict__ qrow,
                                    const int* __restrict__ qcol, int* __restrict__ flag) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < M * N; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / N, c = e - r * N;
    if (qrow[r] != qcol[c] && psi[e] != 0.0) *flag = 1;
  }
}

// out[i][l] = psi[rows[i]][cols[l]]  (one charge block, dense Mc x Nc)
__global__ void svd_qn_gather_kernel(const double* __restrict__ psi, int64_t N, const int* __restrict__ rows,
                                     const int* __restrict__ cols, int64_t Mc, int64_t Nc, double* __restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < Mc * Nc; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / Nc, l = e - i * Nc;
    out[e] = psi[(int64_t)rows[i] * N + cols[l]];
  }
}

// Scatter the kept vectors of one block into the full factors.  jk[q] = (j, k): block vector j
// becomes new-bond index k.  dir 0: Q[rows[i]][k] = Qc[i][j] (pitch nc), C[k][cols[l]] = Cc[j][l];
// dir 1: Q[k][cols[l]] = Qc[j][l], C[rows[i]][k] = Cc[i][j] (pitch nc).  grid.y = kept count.
__global__ void svd_qn_scatter_kernel(const double* __restrict__ Qc, const double* __restrict__ Cc,
                                      const int2* __restrict__ jk, const int* __restrict__ rows,
                                      const int* __restrict__ cols, int64_t Mc, int64_t Nc, int64_t nc, int dir,
                                      double* __restrict__ Q, double* __restrict__ C, int64_t M, int64_t N,
                                      int64_t n, int nkept) {
  for (int q = blockIdx.y; q < nkept; q += gridDim.y) {
    const int2 p = jk[q];
    const int j = p.x, k = p.y;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < Mc; i += (int64_t)gridDim.x * blockDim.x) {
      if (dir == 0) Q[(int64_t)rows[i] * n + k] = Qc[i * nc + j];
      else C[(int64_t)rows[i] * n + k] = Cc[i * nc + j];
    }
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < Nc; l += (int64_t)gridDim.x * blockDim.x) {
      if (dir == 0) C[(int64_t)k * N + cols[l]] = Cc[(int64_t)j * Nc + l];
      else Q[(int64_t)k * N + cols[l]] = Qc[(int64_t)j * Nc + l];
    }
  }
}

// ---------------------------------------------------------------- small-matrix split (one CTA)
// For X of at most kSvdSmallMax rows and columns (DMRG bonds m <= 64 at d = 2) the whole
// split runs in ONE kernel with X resident in shared memory: scalar cyclic one-sided Jacobi
// (circle ordering, 8 warps, one warp per column pair, lanes over rows, warp-shuffle dot
// products), column norms, a rank sort, the truncation rule, the gauge and both factors --
// no host round trips, no per-round launches.  Same arithmetic contract as the large path:
// relative convergence test tol = 4 eps sqrt(R), power-of-two pre-scaling, readings R20-R22.
constexpr int kSvdSmallMax = 128;      // shared-memory capacity of svd_small_kernel
// heff_svd_split uses it up to here (HEFF_SVD_SMALL_N overrides, <= kSvdSmallMax).  Round 2
// measured both paths on random and graded (DMRG-like, 12 decades) inputs: the one-CTA kernel
// has no LQ preconditioner, so on graded spectra it needs 20-29 sweeps above 40 columns
// (64^2: 2.17 vs 1.18 ms, 96^2: 5.98 vs 1.78 ms on the block path) while it still wins on
// random ones up to 64; at 48^2 the two are equal on graded inputs (1.16 / 1.09 ms).
constexpr int kSvdSmallDispatch = 48;
constexpr int kSvdSmallThreads = 1024;
constexpr int kSvdSmallMaxSweeps = 80;

__device__ __forceinline__ double svd_warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// info: [0] n_kept, [1] trunc_err, [2] sweeps, [3] status (0 ok, 1 zero, 2 non-finite, 3 no convergence)
__global__ void __launch_bounds__(kSvdSmallThreads) svd_small_kernel(const double* __restrict__ psi, int M, int N,
                                                                    int dir, double cutoff, int64_t maxdim,
                                                                    int64_t mindim, double* __restrict__ Qout,
                                                                    double* __restrict__ S, double* __restrict__ Cout,
                                                                    double* __restrict__ info) {
  extern __shared__ double sm[];
  const int R = dir == 0 ? M : N, nc0 = dir == 0 ? N : M;
  const int nc = nc0 + (nc0 & 1);                 // even column count (zero pad)
  const int kmin = M < N ? M : N;
  double* X = sm;                                  // [nc][R] column-major: column c at X + c R
  double* nrm = X + (int64_t)nc * R;              // [nc]
  double* scl = nrm + kSvdSmallMax;               // [nc] 1/s with the gauge sign
  int* perm = reinterpret_cast<int*>(scl + kSvdSmallMax);   // [nc] sorted position -> column
  __shared__ double s_tol, s_negl, s_err, s_wmax[kSvdSmallThreads / 32];
  __shared__ int s_any, s_n, s_sweeps;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = kSvdSmallThreads / 32;
  // max |psi| -> exact power-of-two scale (NaN propagates)
  double m = 0.0;
  for (int e = tid; e < M * N; e += blockDim.x) {
    const double v = fabs(psi[e]);
    m = (v > m || v != v) ? v : m;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double w = __shfl_xor_sync(0xffffffffu, m, o);
    m = (w > m || w != w) ? w : m;
  }
  if (lane == 0) s_wmax[warp] = m;
  __syncthreads();
  double mxv = s_wmax[0];
  for (int w = 1; w < nwarps; ++w) mxv = (s_wmax[w] > mxv || s_wmax[w] != s_wmax[w]) ? s_wmax[w] : mxv;
  const double mx = mxv;
  if (!(mx < INFINITY)) {                           // NaN or inf
    if (tid == 0) info[3] = 2.0;
    return;
  }
  if (!(mx > 0.0)) {
    if (tid == 0) info[3] = 1.0;
    return;
  }
  const double sc = ldexp(1.0, -ilogb(mx));
  for (int e = tid; e < nc * R; e += blockDim.x) {
    const int c = e / R, r = e - c * R;
    double v = 0.0;
    if (c < nc0) v = dir == 0 ? psi[(int64_t)r * N + c] : psi[(int64_t)c * N + r];
    X[e] = sc * v;
  }
  __syncthreads();
  {  // ||X||_F^2: strided partials, warp sums, fixed-order total
    double f = 0.0;
    for (int e = tid; e < nc * R; e += blockDim.x) f = fma(X[e], X[e], f);
    f = svd_warp_sum(f);
    if (lane == 0) s_wmax[warp] = f;
  }
  __syncthreads();
  if (tid == 0) {
    double f = 0.0;
    for (int w = 0; w < nwarps; ++w) f += s_wmax[w];
    s_negl = 1e-30 * f;                                          // (1e-15 ||X||_F)^2
    s_tol = fmax(4.0 * 1.1102230246251565e-16 * sqrt((double)R), 8.0 * 1.1102230246251565e-16);
  }
  __syncthreads();
  const double tol = s_tol, negl = s_negl;
  int sweep = 0;
  for (; sweep < kSvdSmallMaxSweeps; ++sweep) {
    if (tid == 0) s_any = 0;
    __syncthreads();
    for (int rr = 0; rr < nc - 1; ++rr) {
      for (int k = warp; k < nc / 2; k += nwarps) {
        auto idx = [&](int i) {  // circle ordering without an integer division
          if (i == 0) return 0;
          int v = i - 1 + rr;
          if (v >= nc - 1) v -= nc - 1;
          return v + 1;
        };
        const int a = idx(k), b = idx(nc - 1 - k);
        double* xa = X + (int64_t)a * R;
        double* xb = X + (int64_t)b * R;
        double app = 0.0, aqq = 0.0, apq = 0.0;
        for (int r = lane; r < R; r += 32) {
          const double u = xa[r], v = xb[r];
          app = fma(u, u, app);
          aqq = fma(v, v, aqq);
          apq = fma(u, v, apq);
        }
        app = svd_warp_sum(app);
        aqq = svd_warp_sum(aqq);
        apq = svd_warp_sum(apq);
        if (app > negl && aqq > negl && apq * apq > (tol * tol) * (app * aqq)) {
          const double th = aqq - app, om = 2.0 * apq;
          const double h2 = fma(th, th, om * om);
          const double tt = (th >= 0.0 ? om : -om) * svd_rcp(fabs(th) + h2 * svd_rsqrt(h2));
          const double cs = svd_rsqrt(fma(tt, tt, 1.0)), sn = cs * tt;
          for (int r = lane; r < R; r += 32) {
            const double u = xa[r], v = xb[r];
            xa[r] = cs * u - sn * v;
            xb[r] = sn * u + cs * v;
          }
          if (lane == 0) s_any = 1;
        }
      }
      __syncthreads();
    }
    if (!s_any) break;
    __syncthreads();
  }
  if (tid == 0) s_sweeps = sweep + 1;
  if (sweep == kSvdSmallMaxSweeps) {
    if (tid == 0) { info[3] = 3.0; info[2] = kSvdSmallMaxSweeps; }
    return;
  }
  // column norms, rank sort (descending, ties by column index)
  for (int c = warp; c < nc; c += nwarps) {
    double f = 0.0;
    for (int r = lane; r < R; r += 32) f = fma(X[(int64_t)c * R + r], X[(int64_t)c * R + r], f);
    f = svd_warp_sum(f);
    if (lane == 0) nrm[c] = sqrt(f);
  }
  __syncthreads();
  for (int c = tid; c < nc; c += blockDim.x) {
    int rank = 0;
    for (int c2 = 0; c2 < nc; ++c2) rank += (nrm[c2] > nrm[c]) || (nrm[c2] == nrm[c] && c2 < c);
    perm[rank] = c;
  }
  __syncthreads();
  if (tid == 0) {  // truncation rule (R20/R21) on the kmin largest values
    double total = 0.0;
    for (int i = kmin - 1; i >= 0; --i) total += nrm[perm[i]] * nrm[perm[i]];
    const double s1 = nrm[perm[0]];
    int64_t rank = 0;
    while (rank < kmin && nrm[perm[rank]] > 1e-12 * s1) ++rank;
    int64_t n = kmin;
    double disc = 0.0;
    while (n > 1 && disc + nrm[perm[n - 1]] * nrm[perm[n - 1]] <= cutoff * total) {
      disc += nrm[perm[n - 1]] * nrm[perm[n - 1]];
      --n;
    }
    n = n < rank ? n : rank;
    const int64_t md = mindim < rank ? mindim : rank;
    n = n > md ? n : md;
    if (maxdim > 0 && n > maxdim) n = maxdim;
    double err = 0.0;
    for (int64_t i = kmin - 1; i >= n; --i) err += nrm[perm[i]] * nrm[perm[i]];
    s_n = (int)n;
    s_err = total > 0.0 ? err / total : 0.0;
  }
  __syncthreads();
  const int n = s_n;
  for (int i = tid; i < kmin; i += blockDim.x) S[i] = nrm[perm[i]] / sc;
  // gauge: largest |entry| of each kept vector positive (first such row on ties); 1/s scale
  for (int k = warp; k < n; k += nwarps) {
    const double* x = X + (int64_t)perm[k] * R;
    double best = -1.0;
    int bi = 0;
    for (int r = lane; r < R; r += 32) {
      const double v = fabs(x[r]);
      if (v > best) { best = v; bi = r; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) scl[k] = (x[bi] < 0.0 ? -1.0 : 1.0) / nrm[perm[k]];
  }
  __syncthreads();
  // factors: the orthonormal one from X, the centre by one small product with Psi
  if (dir == 0) {
    for (int e = tid; e < M * n; e += blockDim.x) {        // U [M][n]
      const int r = e / n, k = e - r * n;
      Qout[e] = X[(int64_t)perm[k] * R + r] * scl[k];
    }
    for (int e = tid; e < n * N; e += blockDim.x) {        // C = U^T Psi [n][N]
      const int k = e / N, j = e - k * N;
      const double* u = X + (int64_t)perm[k] * R;
      double acc = 0.0;
      for (int r = 0; r < M; ++r) acc = fma(u[r], psi[(int64_t)r * N + j], acc);
      Cout[e] = acc * scl[k];
    }
  } else {
    for (int e = tid; e < n * N; e += blockDim.x) {        // V^T [n][N]
      const int k = e / N, j = e - k * N;
      Qout[e] = X[(int64_t)perm[k] * R + j] * scl[k];
    }
    for (int e = tid; e < M * n; e += blockDim.x) {        // C = Psi V [M][n]
      const int i = e / n, k = e - i * n;
      const double* v = X + (int64_t)perm[k] * R;
      double acc = 0.0;
      for (int j = 0; j < N; ++j) acc = fma(psi[(int64_t)i * N + j], v[j], acc);
      Cout[e] = acc * scl[k];
    }
  }
  if (tid == 0) {
    info[0] = n;
    info[1] = s_err;
    info[2] = s_sweeps;
    info[3] = 0.0;
  }
}

}  // namespace heff
