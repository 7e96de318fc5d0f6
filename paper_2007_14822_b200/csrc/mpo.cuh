// mpo.cuh -- the two small O(m^2 d^3 k^2) MPO steps of H_eff.psi, fused into one
// HBM-streaming kernel per order.
//
// Both MPO steps are applied at once through the two-site MPO
//   Wc[w,s1',s1,s2',s2,w2] = sum_w1 W1[w,s1',s1,w1] W2[w1,s2',s2,w2]
// held as a CSR list of its nonzeros (built once per plan on the device,
// mpo_csr_build_kernel).  Order A maps, for every (a', b):
//   T3[a',s1',s2',w2,b] = sum Wc . T1[a',w,s1,s2,b]
// and order B maps, for every (a, b'):  V3[w,a,s1',s2',b'] = sum Wc . V1[a,s1,s2,w2,b'].
// (Re-association of steps 2+3 of (D) in heff.h; exact up to rounding order.)
// Each block stages the k d^2 input column block of its (row, 128-column) tile in shared
// memory with coalesced loads, then writes every output row coalesced: one HBM read of
// the input and one write of the output, no intermediate T2.
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace heff {

constexpr int kMpoThreads = 512;
constexpr int kMpoMaxCols = 128;       // widest column tile
constexpr int kMpoMinCols = 16;        // narrowest column tile (16-byte bulk copies of 128-byte rows)
constexpr int kMpoSmemBytes = 200 * 1024;
constexpr int kMpoMaxRows = kMpoSmemBytes / (8 * kMpoMinCols);  // 1600 staged input rows

// Column-tile width of an MPO application with `nin` staged input rows: the widest of
// 128 / 64 / 32 / 16 whose nin x width fp64 tile fits the shared-memory budget (0: none).
// Wide tiles for the k d^2 <= 200 of every spin chain / cylinder; d = 4 Hubbard cylinders
// (k = 4W + 2, nin = 16 k up to ~1600) run 64..16-wide tiles.
__host__ __device__ constexpr int mpo_tile_cols(int64_t nin) {
  return nin * 8 * 128 <= kMpoSmemBytes ? 128
         : nin * 8 * 64 <= kMpoSmemBytes ? 64
         : nin * 8 * 32 <= kMpoSmemBytes ? 32
         : nin * 8 * 16 <= kMpoSmemBytes ? 16
                                         : 0;
}

// Where one MPO application reads and writes.  Block (x, y) stages input rows
// in + y in_blk + r in_row + [x TC, x TC + width) for r < nin (PLANES == 2: rows >= nin/2
// come from in_plane doubles further), applies the CSR, and writes output row o to
//   out + y out_blk + (o / out_grp) out_grp_stride + (o % out_grp) out_row  (+ out_plane).
//   order A: y = a', rows (w,s1,s2) of T1 -> rows (s1',s2',w2) of T3, row pitch mR;
//   order B: y = a,  rows (s1,s2,w2) of V1 -> rows (w,s1',s2') scattered into
//            V3[w][a][s1' s2'][b'] (out_grp = d1 d2), row pitch nb.
struct MpoIO {
  const double* in;
  double* out;
  int64_t ncol;            // columns per row (mR or nb)
  int nin, nout;           // rows staged / written per block (all planes)
  int64_t in_blk, in_row, in_plane;
  int64_t out_blk, out_row, out_grp_stride, out_plane;
  int out_grp;
};

// GROUPED: output rows scattered in groups (order B); otherwise one row pitch (order A,
// environments, complex planes) -- the kernel is issue-bound, so the common case carries no
// per-row group bookkeeping.
template <int PLANES, int TC, bool GROUPED>
__global__ void __launch_bounds__(kMpoThreads) mpo_apply_kernel(MpoIO io, const int* __restrict__ rowptr,
                                                                 const int* __restrict__ col,
                                                                 const double* __restrict__ val,
                                                                 const unsigned char* __restrict__ live) {
  // PLANES == 2 (complex plans): the CSR holds the real 2x2 blocks [[Re, -Im], [Im, Re]] of
  // the complex MPO over stacked [re; im] rows.
  extern __shared__ __align__(16) double s_in[];  // [nin][TC]
  __shared__ uint64_t bar;
  pdl_wait();  // the input comes from the GEMM before (programmatic dependent launch)
  const int64_t y = blockIdx.y;
  // U(1) plans: blocks whose input and output are zero by symmetry are skipped (their
  // output entries were zeroed once by heff_set_qn)
  if (live && !live[y * gridDim.x + blockIdx.x]) return;
  const int nin = io.nin, nout = io.nout;
  const int nin_p = nin / PLANES, nout_p = nout / PLANES;
  const int64_t b0 = (int64_t)blockIdx.x * TC;
  const int width = (int)min((int64_t)TC, io.ncol - b0);
  const double* in0 = io.in + y * io.in_blk + b0;
  double* out0 = io.out + y * io.out_blk + b0;
  auto in_row = [&](int r) {
    if (PLANES == 1) return in0 + (int64_t)r * io.in_row;
    const int pl = r >= nin_p;
    return in0 + pl * io.in_plane + (int64_t)(r - pl * nin_p) * io.in_row;
  };
  // output row address of row o: the rows a thread writes advance by a fixed step, so the
  // (plane, group, row-in-group) position is tracked incrementally -- no integer division per
  // row (an issue-bound kernel: a division per row cost 16% at C4)
  struct RowPos {
    int pl, q, g, rr;  // plane, row within the plane = g out_grp + rr
  };
  auto row_pos = [&](int o) {  // o: row over all planes
    RowPos r;
    r.pl = (PLANES == 2 && o >= nout_p) ? 1 : 0;
    r.q = o - r.pl * nout_p;
    r.g = GROUPED ? r.q / io.out_grp : 0;
    r.rr = r.q - r.g * io.out_grp;
    return r;
  };
  auto advance = [&](RowPos& r, int step) {
    r.q += step;
    if (GROUPED) {
      r.rr += step;
      while (r.rr >= io.out_grp) {
        r.rr -= io.out_grp;
        ++r.g;
      }
    }
    if (PLANES == 2 && r.pl == 0 && r.q >= nout_p) r = row_pos(r.q);  // into the imaginary plane (once)
  };
  auto out_row = [&](const RowPos& r) {
    if (!GROUPED) return out0 + r.pl * io.out_plane + (int64_t)r.q * io.out_row;
    return out0 + r.pl * io.out_plane + (int64_t)r.g * io.out_grp_stride + (int64_t)r.rr * io.out_row;
  };
  const bool even = ((io.in_row | io.in_blk | io.in_plane | width) & 1) == 0 &&
                    (reinterpret_cast<uintptr_t>(io.in) & 15) == 0;
  if (even) {
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // warp 0: lane 0 arms the barrier, the 32 lanes issue the row copies
      if (threadIdx.x == 0) mbar_arrive_expect_tx(&bar, (uint32_t)(nin * width * 8));
      __syncwarp();
      for (int r = threadIdx.x; r < nin; r += 32) bulk_load(s_in + r * TC, in_row(r), (uint32_t)(width * 8), &bar);
    }
    mbar_wait(&bar, 0);
  } else {
    for (int e = threadIdx.x; e < nin * TC; e += kMpoThreads) {
      const int r = e / TC, c = e - r * TC;
      if (c < width) s_in[e] = __ldcs(in_row(r) + c);
    }
    __syncthreads();
  }
  const bool out_even = ((io.out_row | io.out_blk | io.out_grp_stride | io.out_plane) & 1) == 0 &&
                        (reinterpret_cast<uintptr_t>(io.out) & 15) == 0;
  if (even && out_even) {
    // two adjacent columns per thread: 16-byte shared loads and streaming stores, the CSR
    // entries read once per column pair; kStep threads per column pair step through the
    // output rows.  Same fma order per element as the one-column path.
    constexpr int kPairs = TC / 2, kStep = kMpoThreads / kPairs;
    const int c2 = 2 * (threadIdx.x % kPairs);
    if (c2 >= width) return;
    RowPos rp = row_pos(threadIdx.x / kPairs);
    for (int o = threadIdx.x / kPairs; o < nout; o += kStep, advance(rp, kStep)) {
      double2 acc = make_double2(0.0, 0.0);
      const int e1 = __ldg(rowptr + o + 1);
      for (int e = __ldg(rowptr + o); e < e1; ++e) {
        const double v = __ldg(val + e);
        const double2 xin = *reinterpret_cast<const double2*>(s_in + __ldg(col + e) * TC + c2);
        acc.x = fma(v, xin.x, acc.x);
        acc.y = fma(v, xin.y, acc.y);
      }
      __stcs(reinterpret_cast<double2*>(out_row(rp) + c2), acc);
    }
    return;
  }
  const int t = threadIdx.x % TC;
  if (t >= width) return;
  RowPos rp = row_pos(threadIdx.x / TC);
  for (int o = threadIdx.x / TC; o < nout; o += kMpoThreads / TC, advance(rp, kMpoThreads / TC)) {
    double acc = 0.0;
    const int e1 = __ldg(rowptr + o + 1);
    for (int e = __ldg(rowptr + o); e < e1; ++e) acc = fma(__ldg(val + e), s_in[__ldg(col + e) * TC + t], acc);
    __stcs(out_row(rp) + t, acc);
  }
}

// ---- the two-site MPO as CSR, built on the device --------------------------------------
// Wc[w,s1',s1,s2',s2,w2] = sum_w1 W1[w,s1',s1,w1] W2[w1,s2',s2,w2] (steps 2+3 of (D)
// re-associated), one CSR row per output row of the MPO kernel, its nonzeros in input-row
// order (exact zeros dropped):
//   kCsrOrderA : rows (s1',s2',w2), columns (w,s1,s2)          -- T1 -> T3
//   kCsrOrderB : rows (w,s1',s2'),  columns (s1,s2,w2)         -- V1 -> V3
//   kCsrComplexA: order A over stacked [re; im] rows: real row o holds (c, Re), (nin + c, -Im),
//                 imaginary row nout + o holds (nin + c, Re), (c, Im)   (W1, W2 interleaved complex)
//   kCsrSingle : one site W[w,s',s,w'] (W2 unused): rows (s',w'), columns (w,s) -- the
//                left environment update's MPO step
//   kCsrSingleR: one site, rows (w,s), columns (s',w') -- the right environment update's
// One CTA walks the rows in order; every row's candidate entries are computed by the block
// and compacted in order (warp ballots + a block scan), so the CSR is identical to a
// sequential loop's.  rowptr[nrows + 1], col/val with room for nrows x ncols entries, *nnz.
enum { kCsrOrderA = 0, kCsrOrderB = 1, kCsrComplexA = 2, kCsrSingle = 3, kCsrSingleR = 4 };
constexpr int kCsrThreads = 1024;
static_assert(kCsrThreads == 32 * 32, "one scan warp covers all warp counts");

__global__ void __launch_bounds__(kCsrThreads) mpo_csr_build_kernel(const double* __restrict__ W1,
                                                                     const double* __restrict__ W2, int kL, int kM,
                                                                     int kR, int d1, int d2, int mode,
                                                                     int* __restrict__ rowptr, int* __restrict__ col,
                                                                     double* __restrict__ val, int* __restrict__ nnz) {
  __shared__ int s_warp[kCsrThreads / 32];
  __shared__ int s_run, s_chunk;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nin = kL * d1 * d2, nouts = d1 * d2 * kR;
  int nrows, nslots;
  switch (mode) {
    case kCsrOrderA: nrows = nouts; nslots = nin; break;
    case kCsrOrderB: nrows = nin; nslots = nouts; break;
    case kCsrComplexA: nrows = 2 * nouts; nslots = 2 * nin; break;
    case kCsrSingle: nrows = d1 * kR; nslots = kL * d1; break;
    default: nrows = kL * d1; nslots = d1 * kR; break;
  }
  auto w1 = [&](int w, int sp, int ss, int x, int c) {  // W1[w,s1',s1,x] (part c of a complex entry)
    const int64_t i = ((int64_t)(w * d1 + sp) * d1 + ss) * kM + x;
    return mode == kCsrComplexA ? W1[2 * i + c] : W1[i];
  };
  auto w2 = [&](int x, int sp, int ss, int w, int c) {
    const int64_t i = ((int64_t)(x * d2 + sp) * d2 + ss) * kR + w;
    return mode == kCsrComplexA ? W2[2 * i + c] : W2[i];
  };
  // entry of slot `c` in row `o`: value and CSR column
  auto entry = [&](int o, int c, int* cc) -> double {
    if (mode == kCsrSingle) {  // rows (s',w'), cols (w,s): W[w,s',s,w'] with W [kL][d1][d1][kR]
      const int sp = o / kR, wp = o - sp * kR, w = c / d1, ss = c - w * d1;
      *cc = c;
      return W1[((int64_t)(w * d1 + sp) * d1 + ss) * kR + wp];
    }
    if (mode == kCsrSingleR) {  // rows (w,s), cols (s',w')
      const int w = o / d1, ss = o - w * d1, sp = c / kR, wp = c - sp * kR;
      *cc = c;
      return W1[((int64_t)(w * d1 + sp) * d1 + ss) * kR + wp];
    }
    int s1p, s2p, w, s1, s2, wr, part = 0, im_row = 0;
    if (mode == kCsrOrderB) {  // rows (w,s1',s2'), cols (s1,s2,w2)
      w = o / (d1 * d2); s1p = (o / d2) % d1; s2p = o % d2;
      s1 = c / (d2 * kR); s2 = (c / kR) % d2; wr = c % kR;
      *cc = c;
    } else {
      int oo = o, ci = c;
      if (mode == kCsrComplexA) {
        im_row = o >= nouts;
        oo = o - im_row * nouts;
        part = c & 1;        // slot 2c': Re term, 2c'+1: Im term
        ci = c >> 1;
      }
      s1p = oo / (d2 * kR); s2p = (oo / kR) % d2; wr = oo % kR;
      w = ci / (d1 * d2); s1 = (ci / d2) % d1; s2 = ci % d2;
      *cc = (mode == kCsrComplexA && (part ^ im_row)) ? nin + ci : ci;
    }
    double re = 0.0, im = 0.0;
    for (int x = 0; x < kM; ++x) {
      const double ar = w1(w, s1p, s1, x, 0), br = w2(x, s2p, s2, wr, 0);
      if (mode == kCsrComplexA) {
        const double ai = w1(w, s1p, s1, x, 1), bi = w2(x, s2p, s2, wr, 1);
        re += ar * br - ai * bi;
        im += ar * bi + ai * br;
      } else {
        re += ar * br;
      }
    }
    if (mode != kCsrComplexA) return re;
    // real row: (c, Re), (nin + c, -Im); imaginary row: (nin + c, Re), (c, Im)
    return part == 0 ? re : (im_row ? im : -im);
  };
  if (tid == 0) {
    s_run = 0;
    rowptr[0] = 0;
  }
  __syncthreads();
  for (int o = 0; o < nrows; ++o) {
    for (int base = 0; base < nslots; base += kCsrThreads) {
      const int c = base + tid;
      int cc = 0;
      const double v = c < nslots ? entry(o, c, &cc) : 0.0;
      const bool nz = c < nslots && v != 0.0;
      const unsigned m = __ballot_sync(0xffffffffu, nz);
      if (lane == 0) s_warp[wid] = __popc(m);
      __syncthreads();
      if (wid == 0) {  // exclusive scan of the warp counts (kCsrThreads / 32 == 32 warps)
        const int x = s_warp[lane];
        int incl = x;
        for (int d = 1; d < 32; d <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, d);
          if (lane >= d) incl += y;
        }
        s_warp[lane] = incl - x;
        if (lane == 31) s_chunk = incl;
      }
      __syncthreads();
      const int run = s_run;
      if (nz) {
        const int pos = run + s_warp[wid] + __popc(m & ((1u << lane) - 1u));
        col[pos] = cc;
        val[pos] = v;
      }
      __syncthreads();
      if (tid == 0) s_run = run + s_chunk;
      __syncthreads();
    }
    if (tid == 0) rowptr[o + 1] = s_run;
    __syncthreads();
  }
  if (tid == 0) *nnz = s_run;
}

// Rows of R's b'-shard reordered for order B's GEMM_A: Rp[w2][b'][b] = R_g[b'][w2][b], so
// V1 = psi . Rp^T comes out as [(a s1 s2)][(w2 b')] -- for every a the MPO kernel's input
// rows (s1,s2,w2) are contiguous runs of b' (the order-A staging pattern).
__global__ void permute_r_shard_kernel(const double* __restrict__ R, double* __restrict__ Rp, int64_t nb, int kR,
                                       int64_t mR) {
  const int64_t row = blockIdx.x;  // output row (w2, b')
  const int64_t w2 = row / nb, bp = row - w2 * nb;
  const double2* src = reinterpret_cast<const double2*>(R + (bp * kR + w2) * mR);
  double2* dst = reinterpret_cast<double2*>(Rp + row * mR);
  if ((mR & 1) == 0) {
    for (int64_t i = threadIdx.x; i < mR / 2; i += blockDim.x) dst[i] = src[i];
  } else {
    const double* s1 = R + (bp * kR + w2) * mR;
    double* d1 = Rp + row * mR;
    for (int64_t i = threadIdx.x; i < mR; i += blockDim.x) d1[i] = s1[i];
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

// Blocked-b gather layout [P][rows][nb] -> natural [rows][P nb] (after an all-gather of
// shards).  One (row, shard) run of nb doubles per block iteration: 16-byte loads and
// stores when nb and both bases are even/aligned, no per-element index arithmetic.
__global__ void relayout_blocked_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t rows,
                                        int64_t nb, int P) {
  const bool v2 = ((nb & 1) == 0) && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  for (int64_t run = blockIdx.x; run < rows * P; run += gridDim.x) {
    const int64_t row = run / P, g = run - row * P;
    const double* s = src + (g * rows + row) * nb;
    double* d = dst + (row * P + g) * nb;
    if (v2) {
      const double2* s2 = reinterpret_cast<const double2*>(s);
      double2* d2 = reinterpret_cast<double2*>(d);
      for (int64_t i = threadIdx.x; i < nb / 2; i += blockDim.x) __stcs(d2 + i, __ldcs(s2 + i));
    } else {
      for (int64_t i = threadIdx.x; i < nb; i += blockDim.x) d[i] = s[i];
    }
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
