// blas1.cuh -- Lanczos vector kernels: multi-dot c = V^T w, multi-axpy w -= V c,
// normalisation, all HBM-streaming with deterministic warp-shuffle reductions
// (fixed grid, fixed summation order, no fp64 atomics).
#pragma once
#include <cooperative_groups.h>
#include <cstdint>

#include "ptx.cuh"

namespace cg = cooperative_groups;

namespace heff {

constexpr int kRedThreads = 256;
constexpr int kDotQ = 8;  // vectors per multi-dot pass

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// partial[q][blockIdx.x] = sum over this block's grid-stride range of V[q][i] * w[i],
// q in [0, nq) (nq <= kDotQ).  V rows are ldv apart.
__global__ void __launch_bounds__(kRedThreads) multidot_partial_kernel(const double* __restrict__ V, int64_t ldv,
                                                                       int nq, const double* __restrict__ w,
                                                                       int64_t n, double* __restrict__ partial,
                                                                       int ldp) {
  double acc[kDotQ];
#pragma unroll
  for (int q = 0; q < kDotQ; ++q) acc[q] = 0.0;
  const bool vec = ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(V) | (uintptr_t)(ldv * 8)) & 15) == 0;
  const int64_t stride = (int64_t)gridDim.x * kRedThreads * 2;
  int64_t i = ((int64_t)blockIdx.x * kRedThreads + threadIdx.x) * 2;
  if (vec)  // two grid-stride steps per trip (their loads in flight together), same order
    for (; i + stride + 1 < n; i += 2 * stride) {
      const double2 x0 = __ldg(reinterpret_cast<const double2*>(w + i));
      const double2 x1 = __ldg(reinterpret_cast<const double2*>(w + i + stride));
#pragma unroll
      for (int q = 0; q < kDotQ; ++q)
        if (q < nq) {
          const double2 v0 = __ldcs(reinterpret_cast<const double2*>(V + q * ldv + i));
          const double2 v1 = __ldcs(reinterpret_cast<const double2*>(V + q * ldv + i + stride));
          acc[q] = fma(v0.x, x0.x, acc[q]);
          acc[q] = fma(v0.y, x0.y, acc[q]);
          acc[q] = fma(v1.x, x1.x, acc[q]);
          acc[q] = fma(v1.y, x1.y, acc[q]);
        }
    }
  for (; i < n; i += stride) {
    if (vec && i + 1 < n) {
      const double2 x = __ldg(reinterpret_cast<const double2*>(w + i));
#pragma unroll
      for (int q = 0; q < kDotQ; ++q)
        if (q < nq) {
          const double2 v = __ldcs(reinterpret_cast<const double2*>(V + q * ldv + i));
          acc[q] = fma(v.x, x.x, acc[q]);
          acc[q] = fma(v.y, x.y, acc[q]);
        }
    } else {
      for (int64_t ii = i; ii < min(i + 2, n); ++ii) {
        const double x = w[ii];
#pragma unroll
        for (int q = 0; q < kDotQ; ++q)
          if (q < nq) acc[q] = fma(V[q * ldv + ii], x, acc[q]);
      }
    }
  }
  __shared__ double red[kDotQ][kRedThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < kDotQ; ++q) {
    const double s = warp_sum(acc[q]);
    if (lane == 0) red[q][warp] = s;
  }
  __syncthreads();
  if (threadIdx.x < nq) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < kRedThreads / 32; ++k) s += red[threadIdx.x][k];
    partial[threadIdx.x * ldp + blockIdx.x] = s;
  }
}

// out[q] = sum_b partial[q][b] (fixed order: per-thread strided sums, then a warp tree).
// One block per q.  If `op` == 1, out[q] = sqrt(sum) (norm); `out_extra` gets 1/out.
__global__ void __launch_bounds__(kRedThreads) reduce_partial_kernel(const double* __restrict__ partial, int ldp,
                                                                     int nblocks, double* __restrict__ out,
                                                                     int op, double* __restrict__ out_extra) {
  const int q = blockIdx.x;
  double s = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += kRedThreads) s += partial[q * ldp + b];
  __shared__ double red[kRedThreads / 32];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < kRedThreads / 32; ++k) t += red[k];
    if (op == 1) {
      t = sqrt(t);
      if (out_extra) out_extra[q] = (t > 0.0) ? 1.0 / t : 0.0;
    }
    out[q] = t;
  }
}

// w[i] += sign * sum_q c[q] V[q][i]  for q < nq (nq <= 64 per launch; c read from device)
__global__ void __launch_bounds__(256) multiaxpy_kernel(const double* __restrict__ V, int64_t ldv, int nq,
                                                        const double* __restrict__ c, double sign,
                                                        double* __restrict__ w, int64_t n) {
  __shared__ double sc[64];
  if (threadIdx.x < nq) sc[threadIdx.x] = sign * c[threadIdx.x];
  __syncthreads();
  const bool vec = ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(V) | (uintptr_t)(ldv * 8)) & 15) == 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 2;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2; i < n; i += stride) {
    if (vec && i + 1 < n) {
      double2 x = *reinterpret_cast<double2*>(w + i);
      for (int q = 0; q < nq; ++q) {
        const double2 v = __ldcs(reinterpret_cast<const double2*>(V + q * ldv + i));
        x.x = fma(sc[q], v.x, x.x);
        x.y = fma(sc[q], v.y, x.y);
      }
      *reinterpret_cast<double2*>(w + i) = x;
    } else {
      for (int64_t ii = i; ii < min(i + 2, n); ++ii) {
        double x = w[ii];
        for (int q = 0; q < nq; ++q) x = fma(sc[q], V[q * ldv + ii], x);
        w[ii] = x;
      }
    }
  }
}

// y[i] = x[i] * s[0]   (s on the device, e.g. 1/beta)
__global__ void scale_kernel(const double* __restrict__ x, const double* __restrict__ s, double* __restrict__ y,
                             int64_t n) {
  const double f = *s;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i] * f;
}

// alpha[j] = Re(c1[j] + c2[j])  (the two CGS passes' coefficient on v_j; stride 2 for
// interleaved complex coefficients, whose real part is read)
__global__ void lanczos_alpha_kernel(const double* __restrict__ c1, const double* __restrict__ c2, int j,
                                     double* __restrict__ alpha, int stride) {
  if (threadIdx.x == 0 && blockIdx.x == 0) alpha[j] = c1[stride * j] + c2[stride * j];
}

// ---- complex (interleaved) vectors: <v,w> = sum conj(v) w -----------------------------
// partial[2q][b] / partial[2q+1][b] = Re / Im of block b's sum of conj(V_q[i]) w[i],
// i over n complex entries; V rows are ldv doubles apart (16-byte aligned).
__global__ void __launch_bounds__(kRedThreads) zmultidot_partial_kernel(const double* __restrict__ V, int64_t ldv,
                                                                        int nq, const double* __restrict__ w,
                                                                        int64_t n, double* __restrict__ partial,
                                                                        int ldp) {
  double re[kDotQ], im[kDotQ];
#pragma unroll
  for (int q = 0; q < kDotQ; ++q) re[q] = im[q] = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kRedThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kRedThreads) {
    const double2 x = __ldg(reinterpret_cast<const double2*>(w) + i);
#pragma unroll
    for (int q = 0; q < kDotQ; ++q)
      if (q < nq) {
        const double2 v = __ldcs(reinterpret_cast<const double2*>(V + q * ldv) + i);
        re[q] = fma(v.x, x.x, fma(v.y, x.y, re[q]));
        im[q] = fma(v.x, x.y, fma(-v.y, x.x, im[q]));
      }
  }
  __shared__ double red[2 * kDotQ][kRedThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < kDotQ; ++q) {
    const double a = warp_sum(re[q]), b = warp_sum(im[q]);
    if (lane == 0) {
      red[2 * q][warp] = a;
      red[2 * q + 1][warp] = b;
    }
  }
  __syncthreads();
  if (threadIdx.x < 2 * nq) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < kRedThreads / 32; ++k) t += red[threadIdx.x][k];
    partial[threadIdx.x * ldp + blockIdx.x] = t;
  }
}

// w[i] += sign * sum_q c_q V_q[i]; c interleaved complex (nq <= 64), w and V interleaved
__global__ void __launch_bounds__(256) zmultiaxpy_kernel(const double* __restrict__ V, int64_t ldv, int nq,
                                                         const double* __restrict__ c, double sign,
                                                         double* __restrict__ w, int64_t n) {
  __shared__ double sc[128];
  if (threadIdx.x < 2 * nq) sc[threadIdx.x] = sign * c[threadIdx.x];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 x = reinterpret_cast<double2*>(w)[i];
    for (int q = 0; q < nq; ++q) {
      const double2 v = __ldcs(reinterpret_cast<const double2*>(V + q * ldv) + i);
      const double cr = sc[2 * q], ci = sc[2 * q + 1];
      x.x = fma(cr, v.x, fma(-ci, v.y, x.x));
      x.y = fma(cr, v.y, fma(ci, v.x, x.y));
    }
    reinterpret_cast<double2*>(w)[i] = x;
  }
}

// planes[0][i] = Re z[i], planes[1][i] = Im z[i]  (and back)
__global__ void deinterleave_kernel(const double* __restrict__ z, double* __restrict__ re, double* __restrict__ im,
                                    int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = reinterpret_cast<const double2*>(z)[i];
    re[i] = v.x;
    im[i] = v.y;
  }
}

__global__ void interleave_kernel(const double* __restrict__ re, const double* __restrict__ im, double* __restrict__ z,
                                  int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    reinterpret_cast<double2*>(z)[i] = make_double2(re[i], im[i]);
}

// out = -x (the negated imaginary planes of the complex environments)
__global__ void negate_kernel(const double* __restrict__ x, double* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = -x[i];
}

// ------------------------------------------------------------------------------------
// One fused CGS2 Lanczos step (single device, no communicator), cooperative launch.
// Given w = H v_j and the basis V[0..j):
//   c1 = V^T w ; w -= V c1 ; c2 = V^T w ; w -= V c2 ; alpha = c1[j-1] + c2[j-1] ;
//   beta = ||w|| ; vnext = w / beta   (vnext may be null; then w holds w'' on return,
//   otherwise w holds w' and vnext the normalised w'')
// Each block owns one contiguous chunk of the vectors for all phases; the two
// grid-wide reductions are per-block partials + a grid sync + the same fixed-order sum in
// every block (deterministic, no atomics).  Replaces ~16 launches per step with one.
// partial: [2*jmax + 1][gridDim.x] (the second pass uses rows jmax .. jmax + j).
// ------------------------------------------------------------------------------------
constexpr int kStepThreads = 512;

// partial[q][b] <- block b's sum over its chunk of V[q][i] w[i], q < j (8 vectors per pass),
// and with `wnorm` also partial[j][b] <- its sum of w[i]^2 (accumulated in the first group).
// Every warp reduces its accumulators by shuffles; one barrier per group of 8; the first
// threads add the kStepThreads/32 warp sums in warp order (deterministic).
__device__ __forceinline__ void chunk_dots(const double* __restrict__ V, int64_t ldv, int j, bool wnorm,
                                           const double* __restrict__ w, int64_t lo, int64_t hi,
                                           double* __restrict__ partial, double (*red)[kStepThreads / 32]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int q0 = 0; q0 < j; q0 += kDotQ) {
    const int nq = min(kDotQ, j - q0);
    const bool nrm = wnorm && q0 == 0;
    double acc[kDotQ], accw = 0.0;
#pragma unroll
    for (int q = 0; q < kDotQ; ++q) acc[q] = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += kStepThreads) {
      const double x = w[i];
#pragma unroll
      for (int q = 0; q < kDotQ; ++q)
        if (q < nq) acc[q] = fma(V[(q0 + q) * ldv + i], x, acc[q]);
      accw = fma(x, x, accw);
    }
#pragma unroll
    for (int q = 0; q < kDotQ; ++q)
      if (q < nq) {
        const double v = warp_sum(acc[q]);
        if (lane == 0) red[q][warp] = v;
      }
    if (nrm) {
      accw = warp_sum(accw);
      if (lane == 0) red[kDotQ][warp] = accw;
    }
    __syncthreads();
    if (threadIdx.x < nq || (nrm && threadIdx.x == kDotQ)) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < kStepThreads / 32; ++k) t += red[threadIdx.x][k];
      partial[(threadIdx.x < nq ? q0 + threadIdx.x : j) * gridDim.x + blockIdx.x] = t;
    }
    __syncthreads();  // red is reused by the next group
  }
}

// Grid-wide sums s[q] = sum_b pp[q][b], q < j, computed identically in every block: warp
// (q mod warps) adds b = lane, lane + 32, ... then a shuffle tree (fixed order).
__device__ __forceinline__ void grid_sums(const double* __restrict__ pp, int j, int G, double* s_out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int q = warp; q < j; q += (int)(blockDim.x >> 5)) {
    double t = 0.0;
    for (int b = lane; b < G; b += 32) t += __ldcg(pp + (int64_t)q * G + b);
    t = warp_sum(t);
    if (lane == 0) s_out[q] = t;
  }
}

// Grid barrier of the CGS2 step kernels when they are launched as ordinary (not cooperative)
// kernels: one counter in global memory whose low 31 bits are 0 between barriers; block 0
// adds 2^31 - (G - 1), every other block 1, so the last arrival flips bit 31 and the low bits
// return to 0 (the counter is reusable across barriers and launches without a reset).
// Co-residency: the grid is at most the occupancy-limited resident grid, and its dependents
// launch only after every block has started, so no block waits on one that cannot start.
__device__ __forceinline__ void grid_barrier_flip(unsigned int* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
    __threadfence();
    const unsigned int old = atomicAdd(bar, inc);
    unsigned int cur;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
    } while (((old ^ cur) & 0x80000000u) == 0);
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kStepThreads) cgs2_step_kernel(const double* __restrict__ V, int64_t ldv, int j,
                                                                  double* __restrict__ w, int64_t n,
                                                                  double* __restrict__ partial, int jmax,
                                                                  double* __restrict__ c1, double* __restrict__ c2,
                                                                  double* __restrict__ alpha, double* __restrict__ beta,
                                                                  double* __restrict__ invb,
                                                                  double* __restrict__ vnext,
                                                                  unsigned int* __restrict__ gbar) {
  // gridDim.x == 1 (vectors of a few thousand entries): launched as an ordinary kernel and
  // the grid-wide barriers are block barriers (a cooperative launch costs ~10 us there);
  // gbar != null: an ordinary launch with grid_barrier_flip, else cooperative
  cg::grid_group grid = cg::this_grid();
  auto gsync = [&] {
    if (gridDim.x > 1) {
      if (gbar) grid_barrier_flip(gbar);
      else grid.sync();
    } else {
      __syncthreads();
    }
  };
  extern __shared__ double s_c[];  // [j + 1]
  pdl_wait();  // w comes from the matvec kernel before (launched with programmatic serialization)
  __shared__ double red[kDotQ + 1][kStepThreads / 32];
  const int G = gridDim.x;
  const int64_t chunk = ((n + G - 1) / G + 1) / 2 * 2;
  const int64_t lo = min(n, (int64_t)blockIdx.x * chunk), hi = min(n, lo + chunk);
  double* p1 = partial;
  double* p2 = partial + (int64_t)jmax * G;
  // Two grid barriers: the second pass's reduction also carries ||w'||^2 (w' = w after the
  // first update), and ||w''||^2 = ||w'||^2 - ||c2||^2 (V orthonormal: exact up to
  // O(eps ||c2||^2), and c2 = O(eps ||w||) after the first pass), so the norm needs no third
  // barrier and the last update writes v_{j+1} = w'' / beta directly.
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    double* pp = pass ? p2 : p1;
    double* cc = pass ? c2 : c1;
    chunk_dots(V, ldv, j, pass == 1, w, lo, hi, pp, red);
    gsync();
    grid_sums(pp, j + pass, G, s_c);  // the same fixed-order sums in every block
    __syncthreads();
    if (blockIdx.x == 0)
      for (int q = threadIdx.x; q < j; q += kStepThreads) cc[q] = s_c[q];
    double scale = 1.0;  // 1 / beta for the v_{j+1} store
    if (pass) {
      double nrm2 = s_c[j];
      for (int q = 0; q < j; ++q) nrm2 = fma(-s_c[q], s_c[q], nrm2);
      const double bt = nrm2 > 0.0 ? sqrt(nrm2) : 0.0;
      const double ib = bt > 0.0 ? 1.0 / bt : 0.0;
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        alpha[j - 1] = c1[j - 1] + s_c[j - 1];
        beta[j - 1] = bt;
        invb[j - 1] = ib;
      }
      if (vnext) scale = ib;
    }
    if (pass && vnext) {
#pragma unroll 1
      for (int64_t i = lo + threadIdx.x; i < hi; i += kStepThreads) {
        double x = w[i];
        for (int q = 0; q < j; ++q) x = fma(-s_c[q], V[q * ldv + i], x);
        vnext[i] = x * scale;
      }
    } else {
#pragma unroll 1
      for (int64_t i = lo + threadIdx.x; i < hi; i += kStepThreads) {
        double x = w[i];
        for (int q = 0; q < j; ++q) x = fma(-s_c[q], V[q * ldv + i], x);
        w[i] = x;
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// The same CGS2 step for short vectors (one block; n up to a few thousand entries).  The
// step is bound by dependent memory latency there (cgs2_step_kernel's one-block path:
// ~22 us + ~1 us per basis vector at n = 1024, ncu profiles/r02_c1_cgs2_ncu.md), so it is
// organised around few dependent waits: thread i owns entries i, i + 512, ...; the basis
// entries of 16 vectors are requested together (one latency per 16 vectors); the 16 partial
// dot products of a batch are reduced by warp shuffles, then across the 16 warps by one
// shuffle tree per vector (one warp per vector of the batch) -- fixed order, deterministic.
// Same outputs and formulas as cgs2_step_kernel (beta^2 = ||w'||^2 - ||c2||^2); the dot
// products are summed in a different fixed order.
// ------------------------------------------------------------------------------------
constexpr int kSmallStepThreads = 512;
constexpr int kSmallStepQ = 16;  // basis vectors per batch
constexpr int kSmallStepE = 8;   // entries per thread held in registers (n <= 4096)

__global__ void __launch_bounds__(kSmallStepThreads) cgs2_step_small_kernel(
    const double* __restrict__ V, int64_t ldv, int j, double* __restrict__ w, int64_t n, double* __restrict__ c1,
    double* __restrict__ c2, double* __restrict__ alpha, double* __restrict__ beta, double* __restrict__ invb,
    double* __restrict__ vnext) {
  extern __shared__ double s_c[];  // [j + 1]
  __shared__ double red[kSmallStepQ][kSmallStepThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tid = threadIdx.x;
  pdl_wait();  // w comes from the matvec kernel before (launched with programmatic serialization)
  double x[kSmallStepE];  // this thread's entries of w (then w')
#pragma unroll
  for (int e = 0; e < kSmallStepE; ++e) {
    const int64_t i = tid + (int64_t)e * kSmallStepThreads;
    x[e] = i < n ? w[i] : 0.0;
  }
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    // s_c[q] = V_q . w (q < j); in the second pass also s_c[j] = ||w'||^2
    const int nd = j + pass;
#pragma unroll 1
    for (int q0 = 0; q0 < nd; q0 += kSmallStepQ) {
      double acc[kSmallStepQ];
#pragma unroll
      for (int k = 0; k < kSmallStepQ; ++k) acc[k] = 0.0;
#pragma unroll
      for (int e = 0; e < kSmallStepE; ++e) {
        const int64_t i = tid + (int64_t)e * kSmallStepThreads;
        if (i < n) {
          double v[kSmallStepQ];
#pragma unroll
          for (int k = 0; k < kSmallStepQ; ++k)
            v[k] = (q0 + k < j) ? V[(int64_t)(q0 + k) * ldv + i] : x[e];  // q = j: w' itself
#pragma unroll
          for (int k = 0; k < kSmallStepQ; ++k) acc[k] = fma(v[k], x[e], acc[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < kSmallStepQ; ++k) {
        const double t = warp_sum(acc[k]);
        if (lane == 0) red[k][warp] = t;
      }
      __syncthreads();
      if (warp < kSmallStepQ && q0 + warp < nd) {
        constexpr int kW = kSmallStepThreads / 32;
        const double t = warp_sum(lane < kW ? red[warp][lane] : 0.0);
        if (lane == 0) s_c[q0 + warp] = t;
      }
      __syncthreads();
    }
    double* cc = pass ? c2 : c1;
    for (int q = tid; q < j; q += kSmallStepThreads) cc[q] = s_c[q];
    double scale = 1.0;
    if (pass) {
      double nrm2 = s_c[j];
      for (int q = 0; q < j; ++q) nrm2 = fma(-s_c[q], s_c[q], nrm2);
      const double bt = nrm2 > 0.0 ? sqrt(nrm2) : 0.0;
      const double ib = bt > 0.0 ? 1.0 / bt : 0.0;
      if (tid == 0) {
        alpha[j - 1] = c1[j - 1] + s_c[j - 1];
        beta[j - 1] = bt;
        invb[j - 1] = ib;
      }
      if (vnext) scale = ib;
    }
    // x -= V s_c, basis entries of 16 vectors in flight at a time
#pragma unroll 1
    for (int q0 = 0; q0 < j; q0 += kSmallStepQ) {
#pragma unroll
      for (int e = 0; e < kSmallStepE; ++e) {
        const int64_t i = tid + (int64_t)e * kSmallStepThreads;
        if (i < n) {
          double v[kSmallStepQ];
#pragma unroll
          for (int k = 0; k < kSmallStepQ; ++k) v[k] = (q0 + k < j) ? V[(int64_t)(q0 + k) * ldv + i] : 0.0;
#pragma unroll
          for (int k = 0; k < kSmallStepQ; ++k)
            if (q0 + k < j) x[e] = fma(-s_c[q0 + k], v[k], x[e]);
        }
      }
    }
    if (pass == 0 || !vnext) {
#pragma unroll
      for (int e = 0; e < kSmallStepE; ++e) {
        const int64_t i = tid + (int64_t)e * kSmallStepThreads;
        if (i < n) w[i] = x[e];
      }
    } else {
#pragma unroll
      for (int e = 0; e < kSmallStepE; ++e) {
        const int64_t i = tid + (int64_t)e * kSmallStepThreads;
        if (i < n) vnext[i] = x[e] * scale;
      }
    }
    __syncthreads();  // s_c is rewritten by the next pass
  }
}

// ------------------------------------------------------------------------------------
// The CGS2 step with the basis resident in shared memory (n <= 2048, j <= 31, j n 8 bytes
// <= kSmemStepMaxBytes: C1's whole Lanczos run).  The short-vector step is bound by
// dependent memory latency (one-block kernels: ~0.75 us per basis vector and step, i.e.
// ~4 round trips to L2 per vector -- measured with heff_debug_launch_probe), so here the
// j basis vectors arrive by j bulk copies (TMA, one mbarrier) right after the dependency
// wait -- one latency per step -- and both passes' dot products and updates read them from
// shared memory.  Each partial dot product is reduced by a warp shuffle tree, then across the
// 32 warps by warp q (one shuffle tree per vector, q <= 31): fixed order, deterministic.
// Same outputs and formulas as cgs2_step_kernel.
// ------------------------------------------------------------------------------------
constexpr int kSmemStepThreads = 1024;
constexpr int kSmemStepMaxJ = 31;
constexpr int kSmemStepMaxBytes = 200 * 1024;

__global__ void __launch_bounds__(kSmemStepThreads) cgs2_step_smem_kernel(
    const double* __restrict__ V, int64_t ldv, int j, double* __restrict__ w, int64_t n, double* __restrict__ c1,
    double* __restrict__ c2, double* __restrict__ alpha, double* __restrict__ beta, double* __restrict__ invb,
    double* __restrict__ vnext) {
  extern __shared__ __align__(16) double vs[];  // [j][np]
  __shared__ double red[kSmemStepMaxJ + 1][32];
  __shared__ double s_c[kSmemStepMaxJ + 1];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int np = (int)((n + 1) & ~int64_t(1));  // 16-byte rows (ldv >= np: the pitch is a multiple of 32)
  constexpr int E = 2;                            // entries per thread (n <= 2048)
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();  // w (matvec) and v_{j-1} (previous step) come from the kernels before
  if (tid == 0) {
    mbar_arrive_expect_tx(&bar, (uint32_t)(j * np * 8));
    for (int q = 0; q < j; ++q) bulk_load(vs + (int64_t)q * np, V + (int64_t)q * ldv, (uint32_t)(np * 8), &bar);
  }
  double x[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int64_t i = tid + (int64_t)e * kSmemStepThreads;
    x[e] = i < n ? w[i] : 0.0;
  }
  mbar_wait(&bar, 0);
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    const int nd = j + pass;  // pass 1 also ||w'||^2 (q = j)
#pragma unroll 4
    for (int q = 0; q < nd; ++q) {
      double t = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int64_t i = tid + (int64_t)e * kSmemStepThreads;
        if (i < n) t = fma(q < j ? vs[(int64_t)q * np + i] : x[e], x[e], t);
      }
      t = warp_sum(t);
      if (lane == 0) red[q][warp] = t;
    }
    __syncthreads();
    if (warp < nd) {
      const double t = warp_sum(red[warp][lane]);
      if (lane == 0) s_c[warp] = t;
    }
    __syncthreads();
    double* cc = pass ? c2 : c1;
    if (tid < j) cc[tid] = s_c[tid];
    double scale = 1.0;
    if (pass) {
      double nrm2 = s_c[j];
      for (int q = 0; q < j; ++q) nrm2 = fma(-s_c[q], s_c[q], nrm2);
      const double bt = nrm2 > 0.0 ? sqrt(nrm2) : 0.0;
      const double ib = bt > 0.0 ? 1.0 / bt : 0.0;
      if (tid == 0) {
        alpha[j - 1] = c1[j - 1] + s_c[j - 1];
        beta[j - 1] = bt;
        invb[j - 1] = ib;
      }
      if (vnext) scale = ib;
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int64_t i = tid + (int64_t)e * kSmemStepThreads;
      if (i < n) {
        double xe = x[e];
        for (int q = 0; q < j; ++q) xe = fma(-s_c[q], vs[(int64_t)q * np + i], xe);
        x[e] = xe;
        if (pass == 0 || !vnext)
          w[i] = xe;
        else
          vnext[i] = xe * scale;
      }
    }
    __syncthreads();  // s_c and red are rewritten by the next pass
  }
}

// ------------------------------------------------------------------------------------
// The cooperative CGS2 step in three passes over the basis instead of four (j <= kStep3MaxJ):
// pass A: c1 = V^T w;  pass B: w' = w - V c1 and, from the same basis entries held in
// registers, c2 = V^T w' and ||w'||^2;  pass C: v_{j+1} = (w' - V c2) / beta.  At C2 size the
// step streams the basis from HBM (~5-7 TB/s, profiles/r02_final_c2_lanczos20_ncu.md), so one
// pass less is a quarter less traffic.  Same formulas and the same two grid barriers as
// cgs2_step_kernel; per-block partial sums (warp shuffles, then the warps in order) and
// fixed-order grid sums: deterministic.
// ------------------------------------------------------------------------------------
constexpr int kStep3MaxJ = 24;
constexpr int kStep3SmallJ = 12;  // the two-blocks-per-SM instantiation
constexpr int kStep3Threads = 256;  // 1 block per SM: up to 255 registers for the basis entries

// acc[0..j) per thread (+ slot j already in red when nq = j + 1) -> pp[q * G + blockIdx.x] = the
// block's sum (warp shuffles, then the warps in order); a macro to keep acc in registers
#define HEFF_STEP3_BLOCK_PARTIALS(acc, nq, red, pp, G)                      \
  do {                                                                       \
    const int warp_ = threadIdx.x >> 5, lane_ = threadIdx.x & 31;            \
    _Pragma("unroll") for (int q_ = 0; q_ < kJ; ++q_) if (q_ < (nq) && q_ < j) { \
      const double v_ = warp_sum(acc[q_]);                                   \
      if (lane_ == 0) red[q_][warp_] = v_;                                   \
    }                                                                        \
    __syncthreads();                                                         \
    if ((int)threadIdx.x < (nq)) {                                           \
      double t_ = 0.0;                                                       \
      _Pragma("unroll") for (int k_ = 0; k_ < kStep3Threads / 32; ++k_) t_ += red[threadIdx.x][k_]; \
      (pp)[(int64_t)threadIdx.x * (G) + blockIdx.x] = t_;                    \
    }                                                                        \
  } while (0)

// JM: the largest j of the instantiation (the basis entries of a thread's element live in
// registers); MINB resident blocks per SM (<24, 1>: up to 255 registers; <12, 2>: twice the
// warps per SM for j <= 12, more loads in flight)
template <int JM, int MINB>
__global__ void __launch_bounds__(kStep3Threads, MINB) cgs2_step3_kernel(const double* __restrict__ V, int64_t ldv, int j,
                                                                   double* __restrict__ w, int64_t n,
                                                                   double* __restrict__ partial, int jmax,
                                                                   double* __restrict__ c1, double* __restrict__ c2,
                                                                   double* __restrict__ alpha, double* __restrict__ beta,
                                                                   double* __restrict__ invb,
                                                                   double* __restrict__ vnext,
                                                                   unsigned int* __restrict__ gbar, int unroll2) {
  constexpr int kJ = JM;
  cg::grid_group grid = cg::this_grid();
  auto gsync = [&] {  // gbar != null: ordinary launch (grid_barrier_flip), else cooperative
    if (gbar) grid_barrier_flip(gbar);
    else grid.sync();
  };
  __shared__ double s_c[kJ + 1];
  __shared__ double red[kJ + 1][kStep3Threads / 32];
  pdl_wait();  // w comes from the matvec kernel before
  const int G = gridDim.x;
  const int64_t chunk = ((n + G - 1) / G + 1) / 2 * 2;
  const int64_t lo = min(n, (int64_t)blockIdx.x * chunk), hi = min(n, lo + chunk);
  double* p1 = partial;
  double* p2 = partial + (int64_t)jmax * G;
  double acc[kJ + 1];
  // ---- pass A: c1 partials
#pragma unroll
  for (int q = 0; q <= kJ; ++q) acc[q] = 0.0;
  // Two of the thread's elements per iteration: both elements' loads are issued before
  // the FMAs (one block of 8 warps per SM leaves little else to hide their latency); each
  // accumulator still adds element i before element i + kStep3Threads (same sums, bitwise).
  int64_t i = lo + threadIdx.x;
  if (unroll2) {
    for (; i + kStep3Threads < hi; i += 2 * kStep3Threads) {
      const int64_t i1 = i + kStep3Threads;
      const double x0 = w[i], x1 = w[i1];
      double v0[kJ], v1[kJ];
#pragma unroll
      for (int q = 0; q < kJ; ++q)
        if (q < j) {
          v0[q] = V[(int64_t)q * ldv + i];
          v1[q] = V[(int64_t)q * ldv + i1];
        }
#pragma unroll
      for (int q = 0; q < kJ; ++q)
        if (q < j) acc[q] = fma(v1[q], x1, fma(v0[q], x0, acc[q]));
    }
  }
  for (; i < hi; i += kStep3Threads) {
    const double x = w[i];
#pragma unroll
    for (int q = 0; q < kJ; ++q)
      if (q < j) acc[q] = fma(V[(int64_t)q * ldv + i], x, acc[q]);
  }
  HEFF_STEP3_BLOCK_PARTIALS(acc, j, red, p1, G);
  gsync();
  grid_sums(p1, j, G, s_c);
  __syncthreads();
  if (blockIdx.x == 0)
    for (int q = threadIdx.x; q < j; q += kStep3Threads) c1[q] = s_c[q];
  // ---- pass B: w' = w - V c1; c2 partials and ||w'||^2 from the same basis entries
#pragma unroll
  for (int q = 0; q <= kJ; ++q) acc[q] = 0.0;
  double nacc = 0.0;
  i = lo + threadIdx.x;
  if (unroll2) {
    for (; i + kStep3Threads < hi; i += 2 * kStep3Threads) {
      const int64_t i1 = i + kStep3Threads;
      double v0[kJ], v1[kJ];
#pragma unroll
      for (int q = 0; q < kJ; ++q) {
        v0[q] = q < j ? V[(int64_t)q * ldv + i] : 0.0;
        v1[q] = q < j ? V[(int64_t)q * ldv + i1] : 0.0;
      }
      double x0 = w[i], x1 = w[i1];
#pragma unroll
      for (int q = 0; q < kJ; ++q)
        if (q < j) {
          x0 = fma(-s_c[q], v0[q], x0);
          x1 = fma(-s_c[q], v1[q], x1);
        }
      w[i] = x0;
      w[i1] = x1;
#pragma unroll
      for (int q = 0; q < kJ; ++q)
        if (q < j) acc[q] = fma(v1[q], x1, fma(v0[q], x0, acc[q]));
      nacc = fma(x1, x1, fma(x0, x0, nacc));
    }
  }
  for (; i < hi; i += kStep3Threads) {
    double v[kJ];
#pragma unroll
    for (int q = 0; q < kJ; ++q) v[q] = q < j ? V[(int64_t)q * ldv + i] : 0.0;
    double x = w[i];
#pragma unroll
    for (int q = 0; q < kJ; ++q)
      if (q < j) x = fma(-s_c[q], v[q], x);
    w[i] = x;
#pragma unroll
    for (int q = 0; q < kJ; ++q)
      if (q < j) acc[q] = fma(v[q], x, acc[q]);
    nacc = fma(x, x, nacc);
  }
  __syncthreads();  // red is rewritten
  {
    // ||w'||^2 into slot j of red (a register array indexed by j would go to local memory)
    const double v = warp_sum(nacc);
    if ((threadIdx.x & 31) == 0) red[j][threadIdx.x >> 5] = v;
  }
  HEFF_STEP3_BLOCK_PARTIALS(acc, j + 1, red, p2, G);
  gsync();
  grid_sums(p2, j + 1, G, s_c);
  __syncthreads();
  if (blockIdx.x == 0)
    for (int q = threadIdx.x; q < j; q += kStep3Threads) c2[q] = s_c[q];
  double nrm2 = s_c[j];
  for (int q = 0; q < j; ++q) nrm2 = fma(-s_c[q], s_c[q], nrm2);
  const double bt = nrm2 > 0.0 ? sqrt(nrm2) : 0.0;
  const double ib = bt > 0.0 ? 1.0 / bt : 0.0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    alpha[j - 1] = c1[j - 1] + s_c[j - 1];
    beta[j - 1] = bt;
    invb[j - 1] = ib;
  }
  // ---- pass C: v_{j+1} = (w' - V c2) / beta   (or w = w'' without vnext)
  i = lo + threadIdx.x;
  if (unroll2) {
    for (; i + kStep3Threads < hi; i += 2 * kStep3Threads) {
      const int64_t i1 = i + kStep3Threads;
      double v0[kJ], v1[kJ];
#pragma unroll
      for (int q = 0; q < kJ; ++q) {
        v0[q] = q < j ? V[(int64_t)q * ldv + i] : 0.0;
        v1[q] = q < j ? V[(int64_t)q * ldv + i1] : 0.0;
      }
      double x0 = w[i], x1 = w[i1];
#pragma unroll
      for (int q = 0; q < kJ; ++q)
        if (q < j) {
          x0 = fma(-s_c[q], v0[q], x0);
          x1 = fma(-s_c[q], v1[q], x1);
        }
      if (vnext) {
        vnext[i] = x0 * ib;
        vnext[i1] = x1 * ib;
      } else {
        w[i] = x0;
        w[i1] = x1;
      }
    }
  }
  for (; i < hi; i += kStep3Threads) {
    double v[kJ];
#pragma unroll
    for (int q = 0; q < kJ; ++q) v[q] = q < j ? V[(int64_t)q * ldv + i] : 0.0;
    double x = w[i];
#pragma unroll
    for (int q = 0; q < kJ; ++q)
      if (q < j) x = fma(-s_c[q], v[q], x);
    if (vnext)
      vnext[i] = x * ib;
    else
      w[i] = x;
  }
}

}  // namespace heff
