// lq.cuh -- Householder LQ factor (L only) of the split's working matrix: the Jacobi
// preconditioner of heff_svd_split.
//
// P = L Q (Q orthonormal rows, never formed), so P and L share U and S: one-sided Jacobi
// on the columns of L gives L W = U S directly.  L is the transposed R factor of P^T; its
// columns are graded (|l_ii| roughly decreasing), which is the case where one-sided Jacobi
// converges in few sweeps (the Drmac-Veselic preconditioning; unpreconditioned Jacobi
// needs ~2-3x more sweeps on spectra decaying over many decades, e.g. DMRG wavefunctions).
//
// Blocked right-looking Householder, 32 reflectors per panel:
//   lq_panel_kernel   factors the panel rows [j, j+nb) over columns [j, n) with a
//                     cooperative grid: every CTA keeps a 32 x <=128 column slice of the
//                     panel in shared memory; per reflector one grid barrier joins the
//                     partial dot products <x_r, x_i> (fixed-order sums: deterministic).
//   lq_panel_cluster_kernel the same panel on ONE thread-block cluster (<= 16 CTAs, each a
//                     32 x <= 512 column slice in shared memory): per reflector one cluster
//                     barrier, the partial dot products read from the peers' shared memory
//                     (DSMEM) -- instead of a grid barrier and a global-memory round trip.
//   lq_build_t_kernel the 32 x 32 triangular factor of the compact WY form
//                     H_1 ... H_nb = I - V T V^T from V V^T and the betas.
//   trailing rows     P_t <- P_t (I - V T V^T) by three DMMA GEMMs (heff_api.cu).
#pragma once
#include <cooperative_groups.h>
#include <cstdint>
#include <cuda_runtime.h>

#include "ptx.cuh"

namespace heff {

constexpr int kLqNb = 32;        // reflectors per panel
constexpr int kLqThreads = 256;
constexpr int kLqMaxCols = 128;  // panel columns per CTA (at most)
constexpr int kLqPitch = kLqMaxCols + 1;

// P: working matrix (row pitch ldp).  Panel: local rows [0, nbp) = global rows j.., local
// columns [0, L) = global columns j..  Vt: [nbp][ldv] (global column index), zero on entry.
// part: [2][gridDim.x][2 * kLqNb] scratch.  beta: [nbp].
__global__ void __launch_bounds__(kLqThreads) lq_panel_kernel(double* __restrict__ P, int64_t ldp, int64_t j,
                                                             int nbp, int64_t L, int cw, double* __restrict__ Vt,
                                                             int64_t ldv, double* __restrict__ beta,
                                                             double* __restrict__ part) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double S[kLqNb][kLqPitch];
  __shared__ double sh_g[kLqNb], sh_col[kLqNb];
  const int tid = threadIdx.x;
  const int64_t c0 = (int64_t)blockIdx.x * cw;
  const int64_t rem = L - c0;
  const int ncol = rem <= 0 ? 0 : (rem < cw ? (int)rem : cw);
  double* base = P + j * ldp + j;
  for (int e = tid; e < kLqNb * kLqMaxCols; e += blockDim.x) {
    const int r = e / kLqMaxCols, c = e % kLqMaxCols;
    S[r][c] = (r < nbp && c < ncol) ? base[(int64_t)r * ldp + c0 + c] : 0.0;
  }
  __syncthreads();
  const int nparts = gridDim.x;
  for (int i = 0; i < nbp; ++i) {
    double* pb = part + (int64_t)(i & 1) * nparts * (2 * kLqNb) + (int64_t)blockIdx.x * (2 * kLqNb);
    // partial <x_r, x_i> over this slice's columns >= i
    {
      const int r = tid >> 3, l = tid & 7;
      double acc = 0.0;
      if (r >= i && r < nbp)
        for (int c = l; c < ncol; c += 8)
          if (c0 + c >= i) acc = fma(S[r][c], S[i][c], acc);
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      if (l == 0) pb[r] = acc;
      if (tid < kLqNb && i >= c0 && i < c0 + ncol) pb[kLqNb + tid] = S[tid][i - c0];  // column i (owner)
    }
    grid.sync();
    const int owner = (int)(i / cw);
    {  // sum the CTAs' partials: 8 lanes per row r, CTA b on lane b % 8, then a fixed-order
       // shuffle tree (deterministic; 8 independent load streams instead of one)
      const int r = tid >> 3, l = tid & 7;
      const double* pp = part + (int64_t)(i & 1) * nparts * (2 * kLqNb);
      double g = 0.0;
      for (int b = l; b < nparts; b += 8) g += __ldcg(pp + (int64_t)b * (2 * kLqNb) + r);
      g += __shfl_xor_sync(0xffffffffu, g, 4);
      g += __shfl_xor_sync(0xffffffffu, g, 2);
      g += __shfl_xor_sync(0xffffffffu, g, 1);
      if (l == 0) sh_g[r] = g;
      if (tid < kLqNb) sh_col[tid] = __ldcg(pp + (int64_t)owner * (2 * kLqNb) + kLqNb + tid);
    }
    __syncthreads();
    const double norm2 = sh_g[i], x0 = sh_col[i];
    double alpha = 0.0, v0 = 0.0, bt = 0.0;
    if (norm2 > 0.0) {
      alpha = -copysign(sqrt(norm2), x0);
      v0 = x0 - alpha;
      bt = 1.0 / (norm2 - alpha * x0);  // 2 / v^T v with v^T v = 2 (norm2 - alpha x0)
    }
    // rows r > i: x_r <- x_r - beta <x_r, v> v, <x_r, v> = <x_r, x_i> - alpha x_r[i]
    for (int e = tid; e < kLqNb * kLqMaxCols; e += blockDim.x) {
      const int r = e / kLqMaxCols, c = e % kLqMaxCols;
      if (r <= i || r >= nbp || c >= ncol || c0 + c < i) continue;
      const double w = sh_g[r] - alpha * sh_col[r];
      const double vc = (c0 + c == i) ? v0 : S[i][c];
      S[r][c] = fma(-bt * w, vc, S[r][c]);
    }
    __syncthreads();
    for (int c = tid; c < ncol; c += blockDim.x) {  // row i: v into Vt, L entries into P
      const int64_t gc = c0 + c;
      if (gc < i) continue;
      Vt[(int64_t)i * ldv + j + gc] = (gc == i) ? v0 : S[i][c];
      S[i][c] = (gc == i) ? alpha : 0.0;
    }
    if (blockIdx.x == 0 && tid == 0) beta[i] = bt;
    __syncthreads();
  }
  for (int e = tid; e < kLqNb * kLqMaxCols; e += blockDim.x) {
    const int r = e / kLqMaxCols, c = e % kLqMaxCols;
    if (r < nbp && c < ncol) base[(int64_t)r * ldp + c0 + c] = S[r][c];
  }
}

// Cluster version of lq_panel_kernel (the same arithmetic and fixed-order sums over wider
// column slices: deterministic, equal to the grid version up to rounding).  gridDim.x = the
// cluster size; CTA `rank` owns columns [rank cw, rank cw + cw).  Dynamic shared memory:
// S[kLqNb][cw + 1] and part[2][2 kLqNb] (double-buffered by reflector: buffer i&1 is
// rewritten at reflector i+2, after every peer has passed barrier i+1, i.e. finished reading
// it).  512 threads: 16 lanes per row for the dot products, 8 row groups x 64 column lanes
// for the update; loops start at the first column >= i (no per-element tests), and the
// pivot entry of row i holds v0 during the update (no per-element select).
constexpr int kLqClThreads = 512;
constexpr int kLqClMaxCols = 512;  // panel columns per CTA
constexpr int kLqClMaxCtas = 16;   // cluster size (non-portable above 8)
constexpr int lq_cluster_smem(int cw) { return (kLqNb * (cw + 1) + 4 * kLqNb) * 8; }

__global__ void __launch_bounds__(kLqClThreads) lq_panel_cluster_kernel(double* __restrict__ P, int64_t ldp,
                                                                       int64_t j, int nbp, int64_t L, int cw,
                                                                       double* __restrict__ Vt, int64_t ldv,
                                                                       double* __restrict__ beta) {
  extern __shared__ double lq_sm[];
  const int pitch = cw + 1;
  double* S = lq_sm;                       // [kLqNb][pitch]
  double* part = lq_sm + kLqNb * pitch;    // [2][2 kLqNb]
  __shared__ double sh_g[kLqNb], sh_col[kLqNb];
  const int tid = threadIdx.x;
  const int rank = (int)cluster_ctarank();
  const int nparts = gridDim.x;
  const int64_t c0 = (int64_t)rank * cw;
  const int64_t rem = L - c0;
  const int ncol = rem <= 0 ? 0 : (rem < cw ? (int)rem : cw);
  double* base = P + j * ldp + j;
  const int tr = tid >> 6, tc = tid & 63;    // update / copy layout: 8 row groups x 64 column lanes
  const int dr = tid >> 4, dl = tid & 15;    // dot layout: row dr, 16 lanes
  for (int r = tr; r < kLqNb; r += 8) {
    const double* src = base + (int64_t)r * ldp + c0;
    double* dst = S + r * pitch;
    for (int c = tc; c < cw; c += 64) dst[c] = (r < nbp && c < ncol) ? src[c] : 0.0;
  }
  __syncthreads();
  const uint32_t part_u32 = smem_u32(part);
  for (int i = 0; i < nbp; ++i) {
    double* pb = part + (i & 1) * (2 * kLqNb);
    // first local column >= i (all of them when i < c0; none past ncol)
    const int64_t ioff = (int64_t)i - c0;
    const int cs = ioff <= 0 ? 0 : (ioff >= ncol ? ncol : (int)ioff);
    const bool own = i >= c0 && i < c0 + ncol;
    {  // partial <x_r, x_i> over this slice's columns >= i
      double acc0 = 0.0, acc1 = 0.0;
      if (dr >= i && dr < nbp) {
        const double* xr = S + dr * pitch;
        const double* xi = S + i * pitch;
        int c = cs + ((dl - cs) & 15);
        for (; c + 16 < ncol; c += 32) {
          acc0 = fma(xr[c], xi[c], acc0);
          acc1 = fma(xr[c + 16], xi[c + 16], acc1);
        }
        if (c < ncol) acc0 = fma(xr[c], xi[c], acc0);
      }
      double acc = acc0 + acc1;
      acc += __shfl_xor_sync(0xffffffffu, acc, 8);
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      if (dl == 0) pb[dr] = acc;
      if (own && tid < kLqNb) pb[kLqNb + tid] = S[tid * pitch + (i - c0)];  // column i (owner)
    }
    cluster_sync_all();
    const int owner = (int)(i / cw);
    if (tid < 8 * kLqNb) {  // the peers' partials in CTA order (8 lanes per row, fixed shuffle tree)
      const int r = tid >> 3, l = tid & 7;
      const uint32_t off = part_u32 + (uint32_t)(((i & 1) * (2 * kLqNb) + r) * 8);
      double g = 0.0;
      for (int b = l; b < nparts; b += 8) g += ld_dsmem_f64(mapa_shared(off, (uint32_t)b));
      g += __shfl_xor_sync(0xffffffffu, g, 4);
      g += __shfl_xor_sync(0xffffffffu, g, 2);
      g += __shfl_xor_sync(0xffffffffu, g, 1);
      if (l == 0) sh_g[r] = g;
    } else if (tid < 8 * kLqNb + kLqNb) {
      const int r = tid - 8 * kLqNb;
      sh_col[r] = ld_dsmem_f64(
          mapa_shared(part_u32 + (uint32_t)(((i & 1) * (2 * kLqNb) + kLqNb + r) * 8), (uint32_t)owner));
    }
    __syncthreads();
    const double norm2 = sh_g[i], x0 = sh_col[i];
    double alpha = 0.0, v0 = 0.0, bt = 0.0;
    if (norm2 > 0.0) {
      alpha = -copysign(sqrt(norm2), x0);
      v0 = x0 - alpha;
      bt = 1.0 / (norm2 - alpha * x0);  // 2 / v^T v with v^T v = 2 (norm2 - alpha x0)
    }
    if (own && tid == 0) S[i * pitch + (i - c0)] = v0;  // v = x_i - alpha e_i
    __syncthreads();
    // rows r > i: x_r <- x_r - beta <x_r, v> v, <x_r, v> = <x_r, x_i> - alpha x_r[i]
    {
      const double* v = S + i * pitch;
      const int cstart = cs + ((tc - cs) & 63);
      for (int r = i + 1 + tr; r < nbp; r += 8) {
        const double f = -bt * (sh_g[r] - alpha * sh_col[r]);
        double* xr = S + r * pitch;
        for (int c = cstart; c < ncol; c += 64) xr[c] = fma(f, v[c], xr[c]);
      }
    }
    __syncthreads();
    {  // row i: v into Vt, L entries (alpha on the diagonal, zeros right of it) into S
      double* vrow = Vt + (int64_t)i * ldv + j + c0;
      double* si = S + i * pitch;
      for (int c = cs + tid; c < ncol; c += kLqClThreads) {
        vrow[c] = si[c];
        si[c] = (c0 + c == i) ? alpha : 0.0;
      }
    }
    if (rank == 0 && tid == 0) beta[i] = bt;
    __syncthreads();
  }
  for (int r = tr; r < nbp; r += 8) {
    double* dst = base + (int64_t)r * ldp + c0;
    const double* src = S + r * pitch;
    for (int c = tc; c < ncol; c += 64) dst[c] = src[c];
  }
  cluster_sync_all();  // no CTA leaves while a peer may still read its partials
}

// T (upper triangular, nbp x nbp, row-major, written NEGATED for the update GEMM):
// T_ii = beta_i, T[0:i, i] = -beta_i T[0:i, 0:i] (V^T v_i)[0:i]   (forward, column-wise WY)
__global__ void lq_build_t_kernel(const double* __restrict__ VtV, const double* __restrict__ beta, int nbp,
                                  double* __restrict__ negT) {
  __shared__ double T[kLqNb][kLqNb + 1];
  __shared__ double G[kLqNb][kLqNb + 1];  // V^T V staged once (the recurrence reads it by column)
  const int l = threadIdx.x;  // 32 threads
  for (int c = 0; c < kLqNb; ++c) {
    T[l][c] = 0.0;
    G[c][l] = (c < nbp && l < nbp) ? VtV[c * nbp + l] : 0.0;
  }
  __syncwarp();
  for (int i = 0; i < nbp; ++i) {
    double s = 0.0;
    if (l < i)
      for (int p = l; p < i; ++p) s = fma(T[l][p], G[p][i], s);
    __syncwarp();
    if (l < i) T[l][i] = -beta[i] * s;
    if (l == i) T[i][i] = beta[i];
    __syncwarp();
  }
  for (int c = 0; c < nbp; ++c)
    if (l < nbp) negT[l * nbp + c] = -T[l][c];
}

// X (block-column layout, as svd_pack_kernel) from the lower trapezoid of P (rows R, the
// first k columns): X[r][c] = (c <= r && c < k) ? P[r][c] : 0
__global__ void lq_pack_lower_kernel(const double* __restrict__ P, int64_t ldp, double* __restrict__ Xb, int64_t R,
                                     int64_t k, int64_t nblk) {
  const int64_t total = nblk * R * 16;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int jj = (int)(e & 15);
    const int64_t rb = e >> 4;
    const int64_t blk = rb / R, r = rb - blk * R;
    const int64_t c = blk * 16 + jj;
    Xb[e] = (c < k && c <= r) ? P[r * ldp + c] : 0.0;
  }
}

}  // namespace heff
