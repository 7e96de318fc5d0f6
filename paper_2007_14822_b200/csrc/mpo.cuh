// mpo.cuh -- the two small O(m^2 d^3 k^2) MPO steps of H_eff.psi, fused into one
// HBM-streaming kernel per order.
//
// Both MPO steps are applied at once through the two-site MPO
//   Wc[w,s1',s1,s2',s2,w2] = sum_w1 W1[w,s1',s1,w1] W2[w1,s2',s2,w2]
// held as a CSR list of its nonzeros (built once per plan on the host).  Order A maps,
// for every (a', b):   T3[a',s1',s2',w2,b] = sum Wc . T1[a',w,s1,s2,b]
// and order B maps, for every (a, b'):  V3[w,a,s1',s2',b'] = sum Wc . V1[a,s1,s2,b',w2].
// (Re-association of steps 2+3 of (D) in heff.h; exact up to rounding order.)
// Each block stages the k d^2 input column block of its (row, 128-column) tile in shared
// memory with coalesced loads, then writes every output row coalesced: one HBM read of
// the input and one write of the output, no intermediate T2.
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace heff {

constexpr int kMpoCols = 128;     // b (or b') columns per block
constexpr int kMpoSplit = 4;      // threads per column (each computes every kMpoSplit-th output row)
constexpr int kMpoThreads = kMpoCols * kMpoSplit;
constexpr int kMpoMaxRows = 200;  // k d1 d2 rows staged in shared memory (<= 200 KB)

// Order A.  T1: [mL][nin][mR] with nin = kL d1 d2 (rows (w,s1,s2));
//           T3: [mL][nout][mR] with nout = d1 d2 kR (rows (s1',s2',w2)).
// Block (b-tile, a'): the nin x width input tile arrives by nin 1-D bulk async copies
// (one thread issues them, one mbarrier counts the bytes), so the whole tile is in flight
// at once; odd row pitches fall back to plain coalesced loads.
template <int PLANES>
__global__ void __launch_bounds__(kMpoThreads) mpo_orderA_kernel(const double* __restrict__ T1, double* __restrict__ T3,
                                                              int64_t mR, int nin, int nout,
                                                              const int* __restrict__ rowptr,
                                                              const int* __restrict__ col,
                                                              const double* __restrict__ val,
                                                              const unsigned char* __restrict__ live,
                                                              int planes, int64_t in_plane, int64_t out_plane) {
  // PLANES == 2 (complex plans; `planes` must equal PLANES): rows [0, nin/2) come from the real plane of T1 and
  // [nin/2, nin) from the imaginary plane (in_plane doubles further); likewise for T3.
  // The CSR then holds the real 2x2 blocks [[Re, -Im], [Im, Re]] of the complex MPO.
  extern __shared__ __align__(16) double s_in[];  // [nin][kMpoCols]
  __shared__ uint64_t bar;
  pdl_wait();  // T1 from the GEMM before (programmatic dependent launch)
  const int64_t ap = blockIdx.y;
  // U(1) plans: blocks whose input and output are zero by symmetry are skipped (their T3
  // entries were zeroed once by heff_set_qn)
  if (live && !live[ap * gridDim.x + blockIdx.x]) return;
  const int nin_p = nin / PLANES, nout_p = nout / PLANES;
  const int64_t b0 = (int64_t)blockIdx.x * kMpoCols;
  const int width = (int)min((int64_t)kMpoCols, mR - b0);
  const double* in0 = T1 + ap * nin_p * mR + b0;  // row r of plane pl: in0 + pl in_plane + r' mR
  double* out0 = T3 + ap * nout_p * mR + b0;
  auto in_row = [&](int r) {
    if (PLANES == 1) return in0 + (int64_t)r * mR;
    const int pl = r >= nin_p;
    return in0 + pl * in_plane + (int64_t)(r - pl * nin_p) * mR;
  };
  const bool bulk = ((mR & 1) == 0) && ((width & 1) == 0);
  if (bulk) {
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // warp 0: lane 0 arms the barrier, the 32 lanes issue the row copies
      if (threadIdx.x == 0) mbar_arrive_expect_tx(&bar, (uint32_t)(nin * width * 8));
      __syncwarp();
      for (int r = threadIdx.x; r < nin; r += 32)
        bulk_load(s_in + r * kMpoCols, in_row(r), (uint32_t)(width * 8), &bar);
    }
    mbar_wait(&bar, 0);
  } else {
    for (int e = threadIdx.x; e < nin * kMpoCols; e += kMpoThreads) {
      const int r = e / kMpoCols, c = e - r * kMpoCols;
      if (c < width) s_in[e] = __ldcs(in_row(r) + c);
    }
    __syncthreads();
  }
  if (bulk && (PLANES == 1 || (out_plane & 1) == 0)) {
    // two adjacent columns per thread (width and the row pitch are even): 16-byte shared
    // loads and streaming stores, the CSR entries read once per column pair; 8 threads per
    // column pair step through the output rows.  Same fma order per element.
    constexpr int kPairs = kMpoCols / 2, kStep = kMpoThreads / kPairs;
    const int c2 = 2 * (threadIdx.x % kPairs);
    if (c2 >= width) return;
    for (int o = threadIdx.x / kPairs; o < nout; o += kStep) {
      double2 acc = make_double2(0.0, 0.0);
      const int e1 = __ldg(rowptr + o + 1);
      for (int e = __ldg(rowptr + o); e < e1; ++e) {
        const double v = __ldg(val + e);
        const double2 xin = *reinterpret_cast<const double2*>(s_in + __ldg(col + e) * kMpoCols + c2);
        acc.x = fma(v, xin.x, acc.x);
        acc.y = fma(v, xin.y, acc.y);
      }
      if (PLANES == 1) {
        __stcs(reinterpret_cast<double2*>(out0 + (int64_t)o * mR + c2), acc);
      } else {
        const int pl = o >= nout_p;
        __stcs(reinterpret_cast<double2*>(out0 + pl * out_plane + (int64_t)(o - pl * nout_p) * mR + c2), acc);
      }
    }
    return;
  }
  const int t = threadIdx.x % kMpoCols;
  if (t >= width) return;
  for (int o = threadIdx.x / kMpoCols; o < nout; o += kMpoSplit) {
    double acc = 0.0;
    const int e1 = __ldg(rowptr + o + 1);
    for (int e = __ldg(rowptr + o); e < e1; ++e) acc = fma(__ldg(val + e), s_in[__ldg(col + e) * kMpoCols + t], acc);
    if (PLANES == 1) {
      __stcs(out0 + (int64_t)o * mR + t, acc);
    } else {
      const int pl = o >= nout_p;
      __stcs(out0 + pl * out_plane + (int64_t)(o - pl * nout_p) * mR + t, acc);
    }
  }
}

// Small bonds (the whole order-A matvec in one launch, m up to ~48): one CTA per output row
// a' stages psi, R and L[a'] in shared memory and runs the three steps of (D) for that row --
// T1[(w s1 s2)][b] = sum_a L[a',w,a] psi[a,(s1 s2),b], the two-site MPO through the CSR,
// out[a',(s1' s2'),b'] = sum_{w2,b} T3[(s1' s2' w2)][b] R[b',w2,b] -- with plain FP64 FMAs.
// At these sizes the DMMA GEMM path is launch- and latency-bound (three launches of a few
// tiles each).  accumulate: out += instead of =.
constexpr int kSmallMvThreads = 256;
constexpr int kSmallMvMaxSmem = 200 * 1024;  // larger bonds: the GEMM path wins (measured)
__global__ void __launch_bounds__(kSmallMvThreads) heff_small_matvec_kernel(
    const double* __restrict__ L, const double* __restrict__ psi, const double* __restrict__ R,
    double* __restrict__ out, int mL, int dd, int mR, int kL, int kR, const int* __restrict__ rowptr,
    const int* __restrict__ col, const double* __restrict__ val, int accumulate) {
  extern __shared__ __align__(16) double sm[];
  const int nin = kL * dd, nout = dd * kR;
  double* s_psi = sm;                                // [mL][dd][mR]
  double* s_R = s_psi + (size_t)mL * dd * mR;        // [mR][kR][mR]
  double* s_L = s_R + (size_t)mR * kR * mR;          // [kL][mL]  (row a')
  double* s_T1 = s_L + (size_t)kL * mL;              // [nin][mR]
  double* s_T3 = s_T1 + (size_t)nin * mR;            // [nout][mR]
  pdl_wait();
  const int ap = blockIdx.x, tid = threadIdx.x;
  for (int e = tid; e < mL * dd * mR; e += kSmallMvThreads) s_psi[e] = psi[e];
  for (int e = tid; e < mR * kR * mR; e += kSmallMvThreads) s_R[e] = R[e];
  for (int e = tid; e < kL * mL; e += kSmallMvThreads) s_L[e] = L[(size_t)ap * kL * mL + e];
  __syncthreads();
  for (int e = tid; e < nin * mR; e += kSmallMvThreads) {  // T1 row (w, s) at column b
    const int r = e / mR, b = e - r * mR, w = r / dd, sp = r - w * dd;
    double acc = 0.0;
    for (int a = 0; a < mL; ++a) acc = fma(s_L[w * mL + a], s_psi[((size_t)a * dd + sp) * mR + b], acc);
    s_T1[e] = acc;
  }
  __syncthreads();
  for (int e = tid; e < nout * mR; e += kSmallMvThreads) {  // the two-site MPO
    const int o = e / mR, b = e - o * mR;
    double acc = 0.0;
    const int e1 = __ldg(rowptr + o + 1);
    for (int q = __ldg(rowptr + o); q < e1; ++q) acc = fma(__ldg(val + q), s_T1[__ldg(col + q) * mR + b], acc);
    s_T3[e] = acc;
  }
  __syncthreads();
  for (int e = tid; e < dd * mR; e += kSmallMvThreads) {  // out[a', s', b']
    const int sp = e / mR, bp = e - sp * mR;
    double acc = 0.0;
    for (int w2 = 0; w2 < kR; ++w2) {
      const double* t3 = s_T3 + (size_t)(sp * kR + w2) * mR;
      const double* r = s_R + ((size_t)bp * kR + w2) * mR;
      for (int b = 0; b < mR; ++b) acc = fma(t3[b], r[b], acc);
    }
    double* o = out + ((size_t)ap * dd + sp) * mR + bp;
    *o = accumulate ? *o + acc : acc;
  }
}

// Order B on a b'-shard of width nb.  V1: [mL][d1 d2][nb][kR]; V3: [kL][mL][d1 d2][nb].
// CSR rows o = (w,s1',s2') (nout = kL d1 d2).  The host stores each CSR column already as
// its shared-memory offset (s*kMpoCols + 0)*kR + w2 for input (s = (s1,s2), w2), so the
// [s][b'][w2] tile lands by dd bulk copies of contiguous width*kR runs.
__global__ void __launch_bounds__(kMpoThreads) mpo_orderB_kernel(const double* __restrict__ V1, double* __restrict__ V3,
                                                              int64_t mL, int64_t nb, int dd, int kR, int kL,
                                                              const int* __restrict__ rowptr,
                                                              const int* __restrict__ col,
                                                              const double* __restrict__ val) {
  extern __shared__ __align__(16) double s_in[];  // [(s1 s2)][kMpoCols][kR]
  __shared__ uint64_t bar;
  const int64_t a = blockIdx.y;
  const int64_t b0 = (int64_t)blockIdx.x * kMpoCols;
  const int width = (int)min((int64_t)kMpoCols, nb - b0);
  const int run = width * kR;  // doubles per (s1,s2) block
  const bool bulk = (((nb * kR) & 1) == 0) && (((b0 * kR) & 1) == 0) && ((run & 1) == 0);
  if (bulk) {
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      mbar_arrive_expect_tx(&bar, (uint32_t)(dd * run * 8));
      for (int s = 0; s < dd; ++s)
        bulk_load(s_in + s * kMpoCols * kR, V1 + ((a * dd + s) * nb + b0) * kR, (uint32_t)(run * 8), &bar);
    }
    mbar_wait(&bar, 0);
  } else {
    for (int s = 0; s < dd; ++s) {
      const double* src = V1 + ((a * dd + s) * nb + b0) * kR;
      for (int e = threadIdx.x; e < run; e += kMpoThreads) s_in[s * kMpoCols * kR + e] = __ldcs(src + e);
    }
    __syncthreads();
  }
  const int bl = threadIdx.x % kMpoCols;
  if (bl >= width) return;
  const int nout = kL * dd;
  const double* my = s_in + bl * kR;
  for (int o = threadIdx.x / kMpoCols; o < nout; o += kMpoSplit) {
    double acc = 0.0;
    const int e1 = __ldg(rowptr + o + 1);
    for (int e = __ldg(rowptr + o); e < e1; ++e) acc = fma(__ldg(val + e), my[__ldg(col + e)], acc);
    const int w = o / dd, s = o - w * dd;
    __stcs(V3 + ((w * mL + a) * dd + s) * nb + b0 + bl, acc);
  }
}

// Blocked-b gather layout [P][mL d1 d2][nb] -> natural [mL d1 d2][P nb] (after an
// all-gather of shards).  One thread per element, coalesced on the write side.
__global__ void relayout_blocked_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t rows,
                                        int64_t nb, int P) {
  const int64_t n = rows * nb * P;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / (nb * P);
    const int64_t rem = i - row * nb * P;
    const int64_t g = rem / nb, bl = rem - g * nb;
    dst[i] = src[(g * rows + row) * nb + bl];
  }
}

// dst[c][r] = src[r][c] for a rows x cols row-major matrix (32x32 shared-memory tiles,
// coalesced on both sides).  Used once per environment update for A-dagger.
__global__ void transpose_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t rows, int64_t cols) {
  __shared__ double tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[k][threadIdx.x] = src[r * cols + c];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t c = c0 + k, r = r0 + threadIdx.x;
    if (r < rows && c < cols) dst[c * rows + r] = tile[threadIdx.x][k];
  }
}

}  // namespace heff
