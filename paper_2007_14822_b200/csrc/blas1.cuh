// blas1.cuh -- Lanczos vector kernels: multi-dot c = V^T w, multi-axpy w -= V c,
// normalisation, all HBM-streaming with deterministic warp-shuffle reductions
// (fixed grid, fixed summation order, no fp64 atomics).
#pragma once
#include <cstdint>

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
  const int64_t stride = (int64_t)gridDim.x * kRedThreads * 2;
  for (int64_t i = ((int64_t)blockIdx.x * kRedThreads + threadIdx.x) * 2; i < n; i += stride) {
    if (i + 1 < n) {
      const double2 x = __ldg(reinterpret_cast<const double2*>(w + i));
#pragma unroll
      for (int q = 0; q < kDotQ; ++q)
        if (q < nq) {
          const double2 v = __ldcs(reinterpret_cast<const double2*>(V + q * ldv + i));
          acc[q] = fma(v.x, x.x, acc[q]);
          acc[q] = fma(v.y, x.y, acc[q]);
        }
    } else {
      const double x = w[i];
#pragma unroll
      for (int q = 0; q < kDotQ; ++q)
        if (q < nq) acc[q] = fma(V[q * ldv + i], x, acc[q]);
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
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 2;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2; i < n; i += stride) {
    if (i + 1 < n) {
      double2 x = *reinterpret_cast<double2*>(w + i);
      for (int q = 0; q < nq; ++q) {
        const double2 v = __ldcs(reinterpret_cast<const double2*>(V + q * ldv + i));
        x.x = fma(sc[q], v.x, x.x);
        x.y = fma(sc[q], v.y, x.y);
      }
      *reinterpret_cast<double2*>(w + i) = x;
    } else {
      double x = w[i];
      for (int q = 0; q < nq; ++q) x = fma(sc[q], V[q * ldv + i], x);
      w[i] = x;
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

// alpha[j] = c1[j] + c2[j]  (the two CGS passes' coefficient on v_j)
__global__ void lanczos_alpha_kernel(const double* __restrict__ c1, const double* __restrict__ c2, int j,
                                     double* __restrict__ alpha) {
  if (threadIdx.x == 0 && blockIdx.x == 0) alpha[j] = c1[j] + c2[j];
}

}  // namespace heff
