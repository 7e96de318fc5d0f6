// split_api.cu -- libheff: the two-site split (heff_svd_split, heff_truncate_spectrum) and
// its U(1) version (heff_svd_split_qn).  C ABI in include/heff.h; kernels in svd.cuh and
// lq.cuh; shared host declarations in internal.h.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"
#include "lq.cuh"
#include "svd.cuh"

// --------------------------------------------------------------------------- two-site split
// NEXT-2: truncated SVD of Psi[(a s1)][(s2 b)] (Sec. 5) by
// block one-sided Jacobi (svd.cuh), then the sort / truncation rule (host, over min(M,N)
// norms), the gauge + gather kernels and one DMMA GEMM for the next centre.
struct SvdArena {
  double* buf = nullptr;
  size_t bytes = 0;
};
// per thread and per device (PerDev, internal.h)
static thread_local PerDev<SvdArena> t_svd_arena;
static thread_local PerDev<SplitWs> t_svd_splitws;
static thread_local PerDev<double*> t_small_info = {};  // svd_small_kernel's 4-double read-back

static int svd_reserve(size_t bytes) {
  SvdArena& a = t_svd_arena();
  if (a.bytes >= bytes) return HEFF_OK;
  cudaFree(a.buf);
  a.buf = nullptr;
  a.bytes = 0;
  CK(cudaMalloc(&a.buf, bytes));
  a.bytes = bytes;
  return HEFF_OK;
}

// round-robin (circle method) schedule of nblk (even) blocks: rounds nblk-1, nblk/2 pairs each
static std::vector<int2> svd_pair_schedule(int nblk) {
  std::vector<int> idx(nblk);
  for (int i = 0; i < nblk; ++i) idx[i] = i;
  std::vector<int2> out;
  out.reserve((size_t)(nblk - 1) * (nblk / 2));
  for (int r = 0; r < nblk - 1; ++r) {
    for (int k = 0; k < nblk / 2; ++k) out.push_back(make_int2(idx[k], idx[nblk - 1 - k]));
    const int last = idx[nblk - 1];
    for (int i = nblk - 1; i > 1; --i) idx[i] = idx[i - 1];
    idx[1] = last;
  }
  return out;
}

static std::mutex g_svd_init_mu;  // svd_init_once may race from the U(1) split's workers
static constexpr int kSvdMaxSweeps = 80;
static int g_lq_grid = 0;  // co-resident CTAs of lq_panel_kernel (cooperative launch)
static int g_lq_cl_max = 0;  // largest cluster of lq_panel_cluster_kernel that fits (0: none)
static int g_svd_gram_occ = 0, g_svd_rot_occ = 0;    // co-resident CTAs per SM
static int g_svd_tgram_occ = 0, g_svd_trot_occ = 0;  // (TMA-fed variants)
static constexpr double kSvdRankEps = 1e-12;   // reading R21
static constexpr double kSvdNegligible = 1e-15; // columns below this fraction of ||Psi||_F are not rotated

// The truncation rule of the split (readings R20/R21) on descending singular values.
static void truncate_rule(const double* sv, int64_t k, double cutoff, int64_t maxdim, int64_t mindim, int64_t* n_out,
                          double* err_out) {
  double total = 0.0;
  for (int64_t i = k - 1; i >= 0; --i) total += sv[i] * sv[i];
  int64_t rank = 0;
  while (rank < k && sv[rank] > kSvdRankEps * sv[0]) ++rank;
  int64_t n = k;
  double disc = 0.0;
  while (n > 1 && disc + sv[n - 1] * sv[n - 1] <= cutoff * total) {  // discard smallest while within cutoff
    disc += sv[n - 1] * sv[n - 1];
    --n;
  }
  n = std::min(n, rank);
  n = std::max(n, std::min(std::max<int64_t>(1, mindim), rank));
  if (maxdim > 0) n = std::min(n, maxdim);
  double err = 0.0;
  for (int64_t i = k - 1; i >= n; --i) err += sv[i] * sv[i];
  *n_out = n;
  *err_out = err / total;
}

extern "C" int heff_truncate_spectrum(const double* s, int64_t k, const heff_trunc* trunc, int64_t* n_kept,
                                      double* trunc_err) {
  if (!s || k < 1 || !n_kept || !trunc_err) return set_err(HEFF_EINVAL, "heff_truncate_spectrum: bad argument");
  const double cutoff = trunc ? trunc->cutoff : 0.0;
  if (!(cutoff >= 0.0)) return set_err(HEFF_EINVAL, "heff_truncate_spectrum: cutoff < 0");
  for (int64_t i = 0; i < k; ++i)
    if (!(s[i] >= 0.0) || (i > 0 && s[i] > s[i - 1]))
      return set_err(HEFF_EINVAL, "heff_truncate_spectrum: values must be descending and non-negative");
  if (!(s[0] > 0.0)) return set_err(HEFF_EZERO, "heff_truncate_spectrum: zero spectrum");
  truncate_rule(s, k, cutoff, trunc ? trunc->maxdim : 0, trunc ? trunc->mindim : 1, n_kept, trunc_err);
  return HEFF_OK;
}

// one-time occupancy queries / attributes of the split's kernels (thread-safe)
static int svd_init_once() {
  static std::atomic<uint64_t> done{0};  // bit d: device d (attributes are per device context)
  const uint64_t bit = uint64_t(1) << cur_device();
  if (done.load(std::memory_order_acquire) & bit) return HEFF_OK;
  std::lock_guard<std::mutex> lock(g_svd_init_mu);
  if (done.load(std::memory_order_acquire) & bit) return HEFF_OK;
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lq_panel_kernel, kLqThreads, 0));
  g_lq_grid = std::max(1, per_sm) * g_num_sms;
  CK(cudaFuncSetAttribute(lq_panel_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          lq_cluster_smem(kLqClMaxCols)));
  CK(cudaFuncSetAttribute(lq_panel_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  for (int cs = kLqClMaxCtas; cs >= 2 && g_lq_cl_max == 0; cs /= 2) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kLqClThreads);
    cfg.dynamicSmemBytes = lq_cluster_smem(kLqClMaxCols);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, lq_panel_cluster_kernel, &cfg) == cudaSuccess && ncl >= 1) g_lq_cl_max = cs;
  }
  (void)cudaGetLastError();
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_svd_gram_occ, svd_gram_kernel, kSvdGramThreads, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_svd_rot_occ, svd_rotate_kernel, kSvdRotThreads, 0));
  g_svd_gram_occ = std::max(1, g_svd_gram_occ);
  g_svd_rot_occ = std::max(1, g_svd_rot_occ);
  CK(cudaFuncSetAttribute(svd_rotate_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSvdTmaRotSmem));
  CK(cudaFuncSetAttribute(svd_gram_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSvdTmaGramSmem));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_svd_tgram_occ, svd_gram_tma_kernel, (kSvdTmaGramWarps + 1) * 32,
                                                   kSvdTmaGramSmem));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_svd_trot_occ, svd_rotate_tma_kernel, (kSvdTmaRotWarps + 1) * 32,
                                                   kSvdTmaRotSmem));
  g_svd_tgram_occ = std::max(1, g_svd_tgram_occ);
  g_svd_trot_occ = std::max(1, g_svd_trot_occ);
  CK(cudaFuncSetAttribute(svd_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)(sizeof(double) * ((size_t)kSvdSmallMax * kSvdSmallMax + 3 * kSvdSmallMax))));
  done.fetch_or(bit, std::memory_order_release);
  return HEFF_OK;
}

extern "C" int heff_svd_split(int64_t M, int64_t N, const double* psi, const heff_trunc* trunc, int dir, double* Qout,
                              double* S, double* Cout, int64_t* n_kept, double* trunc_err, int* sweeps_out,
                              heff_stream stream) {
  if (M < 1 || N < 1 || !psi || !Qout || !S || !Cout || !n_kept || !trunc_err || (dir != 0 && dir != 1))
    return set_err(HEFF_EINVAL, "heff_svd_split: bad argument");
  const double cutoff = trunc ? trunc->cutoff : 0.0;
  const int64_t maxdim = trunc ? trunc->maxdim : 0;
  const int64_t mindim = trunc ? std::max<int64_t>(1, trunc->mindim) : 1;
  if (!(cutoff >= 0.0)) return set_err(HEFF_EINVAL, "heff_svd_split: cutoff < 0");
  if (M * N >= (1ll << 40) || std::max(M, N) >= (1ll << 31)) return set_err(HEFF_EUNSUPPORTED, "heff_svd_split: too large");
  CKR(init_device_once());
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t R = dir == 0 ? M : N;          // rows of X
  const int64_t kmin = std::min(M, N);
  const int64_t colsP = dir == 0 ? N : M;      // columns of the working matrix P (Psi or Psi^T)
  CKR(svd_init_once());
  const char* sn = getenv("HEFF_SVD_SMALL_N");  // (read per call: tests switch it)
  const int64_t small_n = sn ? std::min<int64_t>(std::max(0, atoi(sn)), kSvdSmallMax) : (int64_t)kSvdSmallDispatch;
  if (R <= small_n && colsP <= small_n && getenv("HEFF_SVD_NO_SMALL") == nullptr) {
    // small matrix: the whole split in one CTA (svd_small_kernel)
    double*& d_info = t_small_info();
    if (!d_info) CK(cudaMalloc(&d_info, 4 * sizeof(double)));
    const int64_t ncp = colsP + (colsP & 1);
    const size_t smem = sizeof(double) * ((size_t)ncp * R + 3 * kSvdSmallMax);
    svd_small_kernel<<<1, kSvdSmallThreads, smem, s>>>(psi, (int)M, (int)N, dir, cutoff, maxdim, mindim, Qout, S, Cout,
                                                       d_info);
    CK(cudaGetLastError());
    double info[4];
    CK(cudaMemcpyAsync(info, d_info, sizeof info, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (info[3] == 1.0) return set_err(HEFF_EZERO, "heff_svd_split: psi is zero");
    if (info[3] == 2.0) return set_err(HEFF_EINVAL, "heff_svd_split: psi has a non-finite entry");
    if (info[3] == 3.0) return set_err(HEFF_ENOCONV, "heff_svd_split: Jacobi did not converge in %d sweeps",
                                       kSvdSmallMaxSweeps);
    *n_kept = (int64_t)info[0];
    *trunc_err = info[1];
    if (sweeps_out) *sweeps_out = (int)info[2];
    return HEFF_OK;
  }
  // LQ preconditioning (lq.cuh): Jacobi on the k = min(M,N) columns of L instead of P
  const bool precond = getenv("HEFF_SVD_NO_PRECOND") == nullptr && kmin > kSvdPair &&
                       (colsP + g_lq_grid - 1) / g_lq_grid <= kLqMaxCols;
  const int64_t ncols = precond ? kmin : colsP;  // columns of X (orthogonalised)
  int64_t nblk = (ncols + kSvdB - 1) / kSvdB;
  if (nblk & 1) ++nblk;
  if (nblk < 2) nblk = 2;
  const int npairs = (int)(nblk / 2), rounds = (int)(nblk - 1);
  // balanced persistent grids (svd.cuh): one wave of co-resident CTAs, work split evenly
  // TMA-fed Gram / rotation (svd.cuh) unless disabled; tensor-map row coordinates are int32
  const bool svd_tma = getenv("HEFF_SVD_NO_TMA") == nullptr && nblk * R < (1ll << 31);
  const int64_t gram_chunks = (R + 127) / 128;  // 128-row chunks in both Gram kernels
  const int gram_grid = (int)std::min<int64_t>((int64_t)(svd_tma ? g_svd_tgram_occ : g_svd_gram_occ) * g_num_sms,
                                               npairs * gram_chunks);
  int nslots = 1;  // CTAs touching one pair, at most
  for (int p = 0; p < npairs; ++p)
    nslots = std::max(nslots, svd_sk_owner((int64_t)p * gram_chunks + gram_chunks - 1, npairs * gram_chunks, gram_grid) -
                                  svd_sk_owner((int64_t)p * gram_chunks, npairs * gram_chunks, gram_grid) + 1);
  const int rot_grid = svd_tma ? (int)std::min<int64_t>((int64_t)g_svd_trot_occ * g_num_sms,
                                                         npairs * ((R + kSvdTmaRotRows - 1) / kSvdTmaRotRows))
                               : (int)std::min<int64_t>((int64_t)g_svd_rot_occ * g_num_sms, npairs * ((R + 31) / 32));
  const int red_blocks = 4 * g_num_sms;

  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  const size_t bX = al(sizeof(double) * nblk * kSvdB * R);
  const size_t bG = al(sizeof(double) * (size_t)npairs * nslots * kSvdPair * kSvdPair);
  const size_t bNorm = al(sizeof(double) * nblk * kSvdB);
  const size_t bPairs = al(sizeof(int2) * (size_t)rounds * npairs);
  const size_t bStat = al(sizeof(unsigned long long) * kSvdMaxSweeps + sizeof(int) * kSvdMaxSweeps);
  const size_t bRed = al(sizeof(double) * (red_blocks + 1));
  const size_t bPerm = al(sizeof(int) * kmin) + 2 * al(sizeof(double) * kmin);
  const size_t bUt = dir == 0 ? al(sizeof(double) * kmin * M) : 0;
  const size_t bQ = al(sizeof(double) * (size_t)npairs * kSvdPair * kSvdPair) + al(sizeof(int) * npairs);
  const size_t bSortPerm = al(sizeof(int) * nblk * kSvdB);
  const size_t bLq = precond ? al(sizeof(double) * R * colsP) + al(sizeof(double) * kLqNb * colsP) +
                                   al(sizeof(double) * R * kLqNb) +
                                   al(sizeof(double) * R * (dir == 1 ? std::max<int64_t>(kLqNb, colsP) : kLqNb)) +
                                   al(sizeof(int) * R) + 2 * al(sizeof(double) * kLqNb * kLqNb) +
                                   al(sizeof(double) * kLqNb) + al(sizeof(double) * 2 * g_lq_grid * 2 * kLqNb)
                             : 0;
  CKR(svd_reserve(2 * bX + bG + bNorm + bPairs + bStat + bRed + bPerm + bUt + bQ + bSortPerm + bLq));
  unsigned char* w = reinterpret_cast<unsigned char*>(t_svd_arena().buf);
  double *d_P = nullptr, *d_Vt = nullptr, *d_W = nullptr, *d_Y = nullptr, *d_VtV = nullptr, *d_negT = nullptr,
         *d_beta = nullptr, *d_part = nullptr;
  int* d_rowperm = nullptr;  // X row r = output row d_rowperm[r] (preconditioned path)
  if (precond) {
    d_P = reinterpret_cast<double*>(w); w += al(sizeof(double) * R * colsP);
    d_Vt = reinterpret_cast<double*>(w); w += al(sizeof(double) * kLqNb * colsP);
    d_W = reinterpret_cast<double*>(w); w += al(sizeof(double) * R * kLqNb);
    d_Y = reinterpret_cast<double*>(w); w += al(sizeof(double) * R * (dir == 1 ? std::max<int64_t>(kLqNb, colsP) : kLqNb));
    d_rowperm = reinterpret_cast<int*>(w); w += al(sizeof(int) * R);
    d_VtV = reinterpret_cast<double*>(w); w += al(sizeof(double) * kLqNb * kLqNb);
    d_negT = reinterpret_cast<double*>(w); w += al(sizeof(double) * kLqNb * kLqNb);
    d_beta = reinterpret_cast<double*>(w); w += al(sizeof(double) * kLqNb);
    d_part = reinterpret_cast<double*>(w); w += al(sizeof(double) * 2 * g_lq_grid * 2 * kLqNb);
  }
  double* Xb = reinterpret_cast<double*>(w); w += bX;
  double* Xb2 = reinterpret_cast<double*>(w); w += bX;
  double* d_Qg = reinterpret_cast<double*>(w); w += al(sizeof(double) * (size_t)npairs * kSvdPair * kSvdPair);
  int* d_flag = reinterpret_cast<int*>(w); w += al(sizeof(int) * npairs);
  int* d_sortperm = reinterpret_cast<int*>(w); w += bSortPerm;
  double* Gp = reinterpret_cast<double*>(w); w += bG;
  double* d_norm = reinterpret_cast<double*>(w); w += bNorm;
  int2* d_pairs = reinterpret_cast<int2*>(w); w += bPairs;
  unsigned long long* d_maxoff = reinterpret_cast<unsigned long long*>(w);
  int* d_nrot = reinterpret_cast<int*>(w + sizeof(unsigned long long) * kSvdMaxSweeps); w += bStat;
  double* d_red = reinterpret_cast<double*>(w); w += bRed;
  int* d_perm = reinterpret_cast<int*>(w); w += al(sizeof(int) * kmin);
  double* d_skept = reinterpret_cast<double*>(w); w += al(sizeof(double) * kmin);
  double* d_scale = reinterpret_cast<double*>(w); w += al(sizeof(double) * kmin);
  double* d_Ut = reinterpret_cast<double*>(w);

  const std::vector<int2> sched = svd_pair_schedule((int)nblk);
  CK(cudaMemcpyAsync(d_pairs, sched.data(), sizeof(int2) * sched.size(), cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(d_maxoff, 0, bStat, s));
  // Scale invariance: the working copy is scaled by a power of two (exact) that brings
  // max |Psi| into [1, 2), so no Gram product under- or overflows; S is scaled back.
  svd_maxabs_partial_kernel<<<red_blocks, 256, 0, s>>>(psi, M * N, d_red);
  std::vector<double> hmax(red_blocks);
  CK(cudaMemcpyAsync(hmax.data(), d_red, sizeof(double) * red_blocks, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  double maxabs = 0.0;
  for (double v : hmax) {
    if (!std::isfinite(v)) return set_err(HEFF_EINVAL, "heff_svd_split: psi has a non-finite entry");
    maxabs = std::max(maxabs, v);
  }
  if (!(maxabs > 0.0)) return set_err(HEFF_EZERO, "heff_svd_split: psi is zero");
  const double pscale = std::ldexp(1.0, -std::ilogb(maxabs));
  // ||scale Psi||_F^2 (deterministic two-pass) and the packed working copy
  svd_sumsq_partial_kernel<<<red_blocks, 256, 0, s>>>(psi, M * N, pscale, d_red);
  svd_sum_kernel<<<1, 32, 0, s>>>(d_red, red_blocks, d_red + red_blocks);
  // optional phase timing (HEFF_SVD_TIMING=1: LQ, Jacobi sweeps, extraction -> stderr)
  const bool timing = getenv("HEFF_SVD_TIMING") != nullptr;
  cudaEvent_t tev[4] = {nullptr, nullptr, nullptr, nullptr};
  if (timing)
    for (auto& e : tev) CK(cudaEventCreate(&e));
  if (timing) CK(cudaEventRecord(tev[0], s));
  if (precond) {
    // P = Pi Psi (moving right) or Pi Psi^T (moving left), R x colsP, rows sorted by
    // descending norm (static row pivoting of the LQ); P <- L by blocked Householder
    const double* src = psi;
    if (dir == 1) {
      CKR(launch_transpose(psi, d_Y, M, N, s));  // d_Y is R x colsP here
      src = d_Y;
    }
    svd_rownorm2_kernel<<<(unsigned)((R + 7) / 8), 256, 0, s>>>(src, R, colsP, d_W);
    std::vector<double> rn(R);
    CK(cudaMemcpyAsync(rn.data(), d_W, sizeof(double) * R, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    std::vector<int> rp(R);
    for (int64_t i = 0; i < R; ++i) rp[i] = (int)i;
    std::stable_sort(rp.begin(), rp.end(), [&](int a, int b) { return rn[a] > rn[b]; });
    CK(cudaMemcpyAsync(d_rowperm, rp.data(), sizeof(int) * R, cudaMemcpyHostToDevice, s));
    svd_gather_rows_kernel<<<dim3((unsigned)std::min<int64_t>((colsP + 255) / 256, 64), (unsigned)std::min<int64_t>(R, 65535)), 256, 0, s>>>(
        src, d_P, R, colsP, d_rowperm, pscale);
    CK(cudaGetLastError());
    int nl = 0;
    for (int64_t j = 0; j < kmin; j += kLqNb) {
      const int nbp = (int)std::min<int64_t>(kLqNb, kmin - j);
      const int64_t L = colsP - j;
      // few wide CTAs: a reflector's work per CTA is tiny (32 rows x <= 128 columns), the
      // grid barrier per reflector is the cost and grows with the CTA count
      const int64_t want = getenv("HEFF_LQ_NARROW") ? (L + 31) / 32 : (L + kLqMaxCols - 1) / kLqMaxCols;
      int grid = (int)std::min<int64_t>(g_lq_grid, want);
      int cw = (int)((L + grid - 1) / grid);
      grid = (int)((L + cw - 1) / cw);
      CK(cudaMemsetAsync(d_Vt, 0, sizeof(double) * kLqNb * colsP, s));
      double* Pp = d_P;
      int64_t ldp = colsP, jj = j, ldv = colsP;
      if (g_lq_cl_max > 0 && L <= (int64_t)g_lq_cl_max * kLqClMaxCols && getenv("HEFF_LQ_GRID") == nullptr) {
        // one cluster: a cluster barrier + DSMEM reads per reflector instead of a grid barrier
        int cs = (int)std::max<int64_t>(1, std::min<int64_t>(g_lq_cl_max, (L + 255) / 256));
        int ccw = (int)((L + cs - 1) / cs);
        ccw = (ccw + 7) / 8 * 8;
        cs = (int)((L + ccw - 1) / ccw);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(kLqClThreads);
        cfg.dynamicSmemBytes = lq_cluster_smem(ccw);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, lq_panel_cluster_kernel, Pp, ldp, jj, nbp, (int64_t)L, ccw, d_Vt, ldv, d_beta));
      } else {
        void* args[] = {&Pp, &ldp, &jj, (void*)&nbp, (void*)&L, &cw, &d_Vt, &ldv, &d_beta, &d_part};
        CK(cudaLaunchCooperativeKernel((const void*)lq_panel_kernel, dim3(grid), dim3(kLqThreads), args, 0, s));
      }
      GemmOp gv;  // V^T V = Vt Vt^T (K = L)
      gv.M = nbp; gv.N = nbp; gv.K = L; gv.A = d_Vt + j; gv.lda = colsP; gv.B = d_Vt + j; gv.ldb = colsP;
      gv.b_kmajor = true; gv.C = d_VtV; gv.ldc = nbp;
      CKR(launch_gemm(gv, 0, s, &nl, &t_svd_splitws()));
      lq_build_t_kernel<<<1, 32, 0, s>>>(d_VtV, d_beta, nbp, d_negT);
      const int64_t rT = R - j - nbp;
      if (rT > 0) {
        double* Pt = d_P + (j + nbp) * colsP + j;
        GemmOp g1;  // W = P_t V = P_t Vt^T
        g1.M = rT; g1.N = nbp; g1.K = L; g1.A = Pt; g1.lda = colsP; g1.B = d_Vt + j; g1.ldb = colsP;
        g1.b_kmajor = true; g1.C = d_W; g1.ldc = nbp;
        CKR(launch_gemm(g1, 0, s, &nl, &t_svd_splitws()));
        GemmOp g2;  // Y = W (-T)
        g2.M = rT; g2.N = nbp; g2.K = nbp; g2.A = d_W; g2.lda = nbp; g2.B = d_negT; g2.ldb = nbp;
        g2.b_kmajor = false; g2.C = d_Y; g2.ldc = nbp;
        CKR(launch_gemm(g2, 0, s, &nl, &t_svd_splitws()));
        GemmOp g3;  // P_t += Y Vt
        g3.M = rT; g3.N = L; g3.K = nbp; g3.A = d_Y; g3.lda = nbp; g3.B = d_Vt + j; g3.ldb = colsP;
        g3.b_kmajor = false; g3.C = Pt; g3.ldc = colsP; g3.accumulate = 1;
        CKR(launch_gemm(g3, 0, s, &nl, &t_svd_splitws()));
      }
    }
    lq_pack_lower_kernel<<<ew_grid(nblk * kSvdB * R), 256, 0, s>>>(d_P, colsP, Xb, R, kmin, nblk);
  } else if (dir == 0) {
    svd_pack_kernel<<<ew_grid(nblk * kSvdB * R), 256, 0, s>>>(psi, Xb, R, ncols, nblk, pscale);
  } else {
    dim3 grid((unsigned)((R + 31) / 32), (unsigned)(nblk * kSvdB / 32));
    svd_pack_t_kernel<<<grid, dim3(32, 8), 0, s>>>(psi, Xb, R, ncols, pscale);
  }
  CK(cudaGetLastError());
  double fro2 = 0.0;
  CK(cudaMemcpyAsync(&fro2, d_red + red_blocks, sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (!(fro2 > 0.0)) return set_err(HEFF_EZERO, "heff_svd_split: psi is zero");
  const double eps = 1.1102230246251565e-16;
  const double tol = std::max(4.0 * eps * std::sqrt((double)R), 8.0 * eps);
  const double negl = kSvdNegligible * kSvdNegligible * fro2;

  if (timing) CK(cudaEventRecord(tev[1], s));
  // Jacobi sweeps until a sweep rotates no pair
  int sweeps = 0;
  bool converged = false;
  const char* it_env = getenv("HEFF_SVD_INNER_THRESH");
  const double inner_thresh = it_env ? atof(it_env) : 0.0;  // default: one inner sweep throughout
  int inner = inner_thresh > 1.0 ? kSvdMaxInnerSweeps : 1;
  if (const char* f = getenv("HEFF_SVD_INNER_FORCE")) inner = atoi(f);
  const bool sort_cols = getenv("HEFF_SVD_NO_SORT") == nullptr;
  std::vector<double> nrm(nblk * kSvdB);
  std::vector<int> order(nblk * kSvdB);
  // The column norms of the current Xb are read back together with each sweep's convergence
  // scalars (one host synchronisation per sweep instead of two); they order the next sweep's
  // columns and, after the last sweep, are the singular values.
  const bool do_sort = sort_cols && ncols > kSvdPair;
  if (do_sort) {
    svd_colnorm_kernel<<<(unsigned)nblk, 256, 0, s>>>(Xb, R, ncols, d_norm);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(nrm.data(), d_norm, sizeof(double) * ncols, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  for (int sw = 0; sw < kSvdMaxSweeps && !converged; ++sw) {
    if (do_sort) {  // descending-norm column order for this sweep (norms read back above)
      for (int64_t i = 0; i < ncols; ++i) order[i] = (int)i;
      std::stable_sort(order.begin(), order.begin() + ncols, [&](int a, int b) { return nrm[a] > nrm[b]; });
      CK(cudaMemcpyAsync(d_sortperm, order.data(), sizeof(int) * ncols, cudaMemcpyHostToDevice, s));
      svd_permute_kernel<<<ew_grid(nblk * kSvdB * R), 256, 0, s>>>(Xb, Xb2, R, ncols, nblk, d_sortperm);
      std::swap(Xb, Xb2);
    }
    CUtensorMap xm_gram, xm_rot;  // Xb changes with the per-sweep column permutation
    if (svd_tma) {
      CKR(make_map(&xm_gram, Xb, nblk * R, kSvdB, kSvdB, kSvdB, kSvdTmaGramRows));
      CKR(make_map(&xm_rot, Xb, nblk * R, kSvdB, kSvdB, kSvdB, kSvdTmaRotRows));
    }
    for (int r = 0; r < rounds; ++r) {
      const int2* pr = d_pairs + (size_t)r * npairs;
      if (svd_tma)
        CK(launch_pdl(svd_gram_tma_kernel, dim3(gram_grid), dim3((kSvdTmaGramWarps + 1) * 32), kSvdTmaGramSmem, s,
                      xm_gram, R, pr, npairs, nslots, Gp));
      else
        svd_gram_kernel<<<gram_grid, kSvdGramThreads, 0, s>>>(Xb, R, pr, npairs, nslots, Gp);
      CK(launch_pdl(svd_pair_eig_kernel, dim3(npairs), dim3(kSvdEigThreads), 0, s, (const double*)Gp, nslots,
                    (int64_t)gram_chunks, gram_grid, tol, negl, inner, d_Qg, d_flag, d_maxoff + sw, d_nrot + sw));
      if (svd_tma)
        CK(launch_pdl(svd_rotate_tma_kernel, dim3(rot_grid), dim3((kSvdTmaRotWarps + 1) * 32), kSvdTmaRotSmem, s,
                      xm_rot, Xb, R, pr, npairs, (const double*)d_Qg, (const int*)d_flag));
      else
        svd_rotate_kernel<<<rot_grid, kSvdRotThreads, 0, s>>>(Xb, R, pr, npairs, d_Qg, d_flag);
    }
    CK(cudaGetLastError());
    int nrot = 0;
    unsigned long long offbits = 0;
    svd_colnorm_kernel<<<(unsigned)nblk, 256, 0, s>>>(Xb, R, ncols, d_norm);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&nrot, d_nrot + sw, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&offbits, d_maxoff + sw, sizeof(offbits), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(nrm.data(), d_norm, sizeof(double) * ncols, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    sweeps = sw + 1;
    converged = nrot == 0;
    double maxoff;
    memcpy(&maxoff, &offbits, sizeof maxoff);
    if (timing) {
      static thread_local std::chrono::steady_clock::time_point t_prev;
      const auto t_now = std::chrono::steady_clock::now();
      if (sw > 0)
        fprintf(stderr, "  sweep %d: %d of %lld pair steps rotated, max off-diagonal %.2e, %.2f ms\n", sw, nrot,
                (long long)npairs * rounds, maxoff, std::chrono::duration<double, std::milli>(t_now - t_prev).count());
      t_prev = t_now;
    }
    inner = maxoff < inner_thresh ? kSvdMaxInnerSweeps : 1;  // see svd.cuh kSvdMaxInnerSweeps
    if (const char* f = getenv("HEFF_SVD_INNER_FORCE")) inner = atoi(f);  // profiling knob
  }
  if (sweeps_out) *sweeps_out = sweeps;
  if (!converged) return set_err(HEFF_ENOCONV, "heff_svd_split: Jacobi did not converge in %d sweeps", kSvdMaxSweeps);

  if (timing) CK(cudaEventRecord(tev[2], s));
  // singular values = column norms of the final Xb (read back with the last sweep's scalars);
  // sort (descending, stable) and truncate on the host
  for (int64_t i = 0; i < ncols; ++i) order[i] = (int)i;
  std::stable_sort(order.begin(), order.begin() + ncols, [&](int a, int b) { return nrm[a] > nrm[b]; });
  std::vector<double> sv(kmin);
  for (int64_t i = 0; i < kmin; ++i) sv[i] = nrm[order[i]];
  double total = 0.0;
  for (int64_t i = kmin - 1; i >= 0; --i) total += sv[i] * sv[i];
  if (!(sv[0] > 0.0)) return set_err(HEFF_EZERO, "heff_svd_split: psi is zero");
  int64_t n = 0;
  double err = 0.0;
  truncate_rule(sv.data(), kmin, cutoff, maxdim, mindim, &n, &err);
  std::vector<double> sv_out(kmin);  // back to Psi's scale
  for (int64_t i = 0; i < kmin; ++i) sv_out[i] = sv[i] / pscale;
  CK(cudaMemcpyAsync(S, sv_out.data(), sizeof(double) * kmin, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_perm, order.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_skept, sv.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
  svd_sign_kernel<<<(unsigned)n, 256, 0, s>>>(Xb, R, d_perm, d_skept, d_scale, d_rowperm);
  dim3 gg((unsigned)std::min<int64_t>((R + 255) / 256, 1024), (unsigned)std::min<int64_t>(n, 65535));
  int nl = 0;
  int r = HEFF_OK;
  if (dir == 0) {
    svd_gather_t_kernel<<<gg, 256, 0, s>>>(Xb, R, d_perm, d_scale, d_Ut, d_rowperm, n);   // U^T [n][M]
    CKR(launch_transpose(d_Ut, Qout, n, M, s));                               // U [M][n]
    GemmOp g;  // C[n][N] = U^T[n][M] . Psi[M][N]
    g.M = n; g.N = N; g.K = M; g.A = d_Ut; g.lda = M; g.B = psi; g.ldb = N; g.b_kmajor = false; g.C = Cout; g.ldc = N;
    r = launch_gemm(g, 0, s, &nl, &t_svd_splitws());
  } else {
    svd_gather_t_kernel<<<gg, 256, 0, s>>>(Xb, R, d_perm, d_scale, Qout, d_rowperm, n);   // V^T [n][N]
    CK(cudaGetLastError());
    GemmOp g;  // C[M][n] = Psi[M][N] . (V^T)^T
    g.M = M; g.N = n; g.K = N; g.A = psi; g.lda = N; g.B = Qout; g.ldb = N; g.b_kmajor = true; g.C = Cout; g.ldc = n;
    r = launch_gemm(g, 0, s, &nl, &t_svd_splitws());
  }
  CK(cudaStreamSynchronize(s));
  if (r != HEFF_OK) return r;
  if (timing) {
    CK(cudaEventRecord(tev[3], s));
    CK(cudaEventSynchronize(tev[3]));
    float a = 0, b = 0, c = 0;
    cudaEventElapsedTime(&a, tev[0], tev[1]);
    cudaEventElapsedTime(&b, tev[1], tev[2]);
    cudaEventElapsedTime(&c, tev[2], tev[3]);
    fprintf(stderr, "heff_svd_split %lldx%lld dir %d: precondition %.2f ms, %d sweeps %.2f ms (%.2f ms/sweep), "
            "extract %.2f ms\n", (long long)M, (long long)N, dir, a, sweeps, b, b / std::max(1, sweeps), c);
    for (auto& e : tev) cudaEventDestroy(e);
  }
  *n_kept = n;
  *trunc_err = err;
  return HEFF_OK;
}

// --------------------------------------------------------------------------- U(1) split
// NEXT-2 x NEXT-3 (reading R24): Psi is block diagonal over the centre-bond charge; every
// block is split by heff_svd_split (dense Jacobi on the block), one truncation runs over the
// union of the blocks' spectra, the new bond is ordered by (charge, descending value).
// Process-lifetime pool of host worker threads (never joined: a leaked singleton) for the
// independent charge blocks of the U(1) split.  Each worker has its own CUDA stream and its
// own thread-local split arenas, so several blocks are split on the GPU at once.
static constexpr int kBlockWorkers = 4;
class BlockPool {
 public:
  struct Batch {
    std::mutex mu;
    std::condition_variable cv;
    int remaining = 0;
  };
  static BlockPool& get() {
    static BlockPool* pool = new BlockPool();
    return *pool;
  }
  // run every task on the workers; returns when all have finished
  // (on the calling thread's current device: each worker switches to it and uses its own
  // stream of that device)
  void run(std::vector<std::function<void(cudaStream_t)>>& tasks) {
    Batch b;
    b.remaining = (int)tasks.size();
    const int dev = cur_device();
    {
      std::lock_guard<std::mutex> lk(mu_);
      for (auto& t : tasks) q_.push_back({&t, &b, dev});
    }
    cv_.notify_all();
    std::unique_lock<std::mutex> lk(b.mu);
    b.cv.wait(lk, [&] { return b.remaining == 0; });
  }

 private:
  struct Item {
    std::function<void(cudaStream_t)>* fn;
    Batch* batch;
    int dev;
  };
  BlockPool() {
    for (int i = 0; i < kBlockWorkers; ++i) std::thread([this] { loop(); }).detach();
  }
  void loop() {
    std::vector<cudaStream_t> ws(kMaxDevices, nullptr);  // this worker's stream on each device
    for (;;) {
      Item it;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return !q_.empty(); });
        it = q_.front();
        q_.erase(q_.begin());
      }
      cudaSetDevice(it.dev);
      if (!ws[it.dev]) cudaStreamCreateWithFlags(&ws[it.dev], cudaStreamNonBlocking);
      (*it.fn)(ws[it.dev]);
      std::lock_guard<std::mutex> lk(it.batch->mu);
      if (--it.batch->remaining == 0) it.batch->cv.notify_all();
    }
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::vector<Item> q_;

 public:
  // one task on EVERY worker (thread-local cleanup): tasks park on a barrier until all
  // workers hold one, so no worker takes two
  void run_each_worker(std::vector<std::function<void(cudaStream_t)>>& tasks) {
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    const int W = (int)tasks.size();
    std::vector<std::function<void(cudaStream_t)>> wrapped;
    for (auto& t : tasks)
      wrapped.push_back([&, t](cudaStream_t ws) {
        t(ws);
        std::unique_lock<std::mutex> lk(m);
        if (++arrived == W) cv.notify_all();
        cv.wait(lk, [&] { return arrived >= W; });
      });
    run(wrapped);
  }
};

struct SvdQnArena {
  double* buf = nullptr;
  size_t bytes = 0;
};
static thread_local PerDev<SvdQnArena> t_svdqn_arena;

extern "C" int heff_svd_split_qn(int64_t M, int64_t N, const double* psi, const int* qrow, const int* qcol,
                                 const heff_trunc* trunc, int dir, double* Qout, double* S, double* Sk, int* qk,
                                 double* Cout, int64_t* n_kept, double* trunc_err, int* sweeps_out,
                                 heff_stream stream) {
  if (M < 1 || N < 1 || !psi || !qrow || !qcol || !Qout || !S || !Sk || !qk || !Cout || !n_kept || !trunc_err ||
      (dir != 0 && dir != 1))
    return set_err(HEFF_EINVAL, "heff_svd_split_qn: bad argument");
  const double cutoff = trunc ? trunc->cutoff : 0.0;
  const int64_t maxdim = trunc ? trunc->maxdim : 0;
  const int64_t mindim = trunc ? std::max<int64_t>(1, trunc->mindim) : 1;
  if (!(cutoff >= 0.0)) return set_err(HEFF_EINVAL, "heff_svd_split_qn: cutoff < 0");
  CKR(init_device_once());
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // sectors: charges present on both sides, ascending
  std::map<int, std::vector<int>> rows_of, cols_of;
  for (int64_t r = 0; r < M; ++r) rows_of[qrow[r]].push_back((int)r);
  for (int64_t c = 0; c < N; ++c) cols_of[qcol[c]].push_back((int)c);
  std::vector<int> sectors;
  for (auto& kv : rows_of)
    if (cols_of.count(kv.first)) sectors.push_back(kv.first);
  if (sectors.empty()) return set_err(HEFF_EZERO, "heff_svd_split_qn: no charge sector on both sides (psi = 0)");
  const int ns = (int)sectors.size();
  std::vector<int64_t> Mc(ns), Nc(ns), kc(ns), off_idx(ns), off_blk(ns), off_q(ns), off_c(ns), off_s(ns);
  std::vector<int> idx_host;
  int64_t tot_blk = 0, tot_q = 0, tot_c = 0, tot_s = 0;
  for (int si = 0; si < ns; ++si) {
    const auto& rw = rows_of[sectors[si]];
    const auto& cl = cols_of[sectors[si]];
    Mc[si] = (int64_t)rw.size();
    Nc[si] = (int64_t)cl.size();
    kc[si] = std::min(Mc[si], Nc[si]);
    off_idx[si] = (int64_t)idx_host.size();
    idx_host.insert(idx_host.end(), rw.begin(), rw.end());
    idx_host.insert(idx_host.end(), cl.begin(), cl.end());
    auto pad = [](int64_t x) { return (x + 31) / 32 * 32; };
    off_blk[si] = tot_blk; tot_blk += pad(Mc[si] * Nc[si]);
    off_q[si] = tot_q;     tot_q += pad(dir == 0 ? Mc[si] * kc[si] : kc[si] * Nc[si]);
    off_c[si] = tot_c;     tot_c += pad(dir == 0 ? kc[si] * Nc[si] : Mc[si] * kc[si]);
    off_s[si] = tot_s;     tot_s += pad(kc[si]);
  }
  const int64_t kmin = std::min(M, N);
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  const size_t need = al(sizeof(int) * idx_host.size()) + al(sizeof(int) * (M + N)) + al(sizeof(int)) +
                      al(sizeof(double) * (tot_blk + tot_q + tot_c + tot_s)) + al(sizeof(int2) * kmin);
  SvdQnArena& a = t_svdqn_arena();
  if (a.bytes < need) {
    cudaFree(a.buf);
    a.buf = nullptr;
    a.bytes = 0;
    CK(cudaMalloc(&a.buf, need));
    a.bytes = need;
  }
  unsigned char* w = reinterpret_cast<unsigned char*>(a.buf);
  int* d_idx = reinterpret_cast<int*>(w); w += al(sizeof(int) * idx_host.size());
  int* d_q = reinterpret_cast<int*>(w); w += al(sizeof(int) * (M + N));
  int* d_flag = reinterpret_cast<int*>(w); w += al(sizeof(int));
  double* d_blk = reinterpret_cast<double*>(w);
  double* d_qc = d_blk + tot_blk;
  double* d_cc = d_qc + tot_q;
  double* d_sc = d_cc + tot_c;
  w += al(sizeof(double) * (tot_blk + tot_q + tot_c + tot_s));
  int2* d_jk = reinterpret_cast<int2*>(w);
  CK(cudaMemcpyAsync(d_idx, idx_host.data(), sizeof(int) * idx_host.size(), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_q, qrow, sizeof(int) * M, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_q + M, qcol, sizeof(int) * N, cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(d_flag, 0, sizeof(int), s));
  svd_qn_check_kernel<<<ew_grid(M * N), 256, 0, s>>>(psi, M, N, d_q, d_q + M, d_flag);
  CK(cudaGetLastError());
  int h_flag = 0;
  CK(cudaMemcpyAsync(&h_flag, d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (h_flag) return set_err(HEFF_EINVAL, "heff_svd_split_qn: psi has entries outside its charge blocks");
  // one dense split per block (all values kept; numerical zeros per the block's own rank rule),
  // the blocks spread over the worker pool's streams, largest first
  std::vector<int64_t> nc(ns, 0);
  std::vector<double> sv_host(tot_s, 0.0);
  std::vector<int> rc(ns, HEFF_OK), swp(ns, 0);
  std::vector<std::string> msg(ns);
  int dev = 0;
  CK(cudaGetDevice(&dev));
  auto block_task = [&](int si, cudaStream_t ws) {
    cudaSetDevice(dev);
    const int* d_rows = d_idx + off_idx[si];
    const int* d_cols = d_rows + Mc[si];
    svd_qn_gather_kernel<<<ew_grid(Mc[si] * Nc[si]), 256, 0, ws>>>(psi, N, d_rows, d_cols, Mc[si], Nc[si],
                                                                   d_blk + off_blk[si]);
    int64_t nk = 0;
    double e = 0.0;
    int r = heff_svd_split(Mc[si], Nc[si], d_blk + off_blk[si], nullptr, dir, d_qc + off_q[si], d_sc + off_s[si],
                           d_cc + off_c[si], &nk, &e, &swp[si], ws);
    if (r == HEFF_OK) {
      nc[si] = nk;
      if (cudaMemcpyAsync(sv_host.data() + off_s[si], d_sc + off_s[si], sizeof(double) * kc[si],
                          cudaMemcpyDeviceToHost, ws) != cudaSuccess || cudaStreamSynchronize(ws) != cudaSuccess)
        r = set_err(HEFF_ECUDA, "heff_svd_split_qn: block copy failed");
    }
    if (r == HEFF_EZERO) r = HEFF_OK;  // an all-zero block contributes nothing
    rc[si] = r;
    if (r != HEFF_OK) msg[si] = heff_last_error();
  };
  std::vector<int> order(ns);
  for (int si = 0; si < ns; ++si) order[si] = si;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return Mc[x] * Nc[x] > Mc[y] * Nc[y]; });
  if (ns > 1 && getenv("HEFF_SVD_QN_SERIAL") == nullptr) {
    std::vector<std::function<void(cudaStream_t)>> tasks;
    for (int si : order) tasks.push_back([&, si](cudaStream_t ws) { block_task(si, ws); });
    BlockPool::get().run(tasks);
  } else {
    for (int si : order) block_task(si, s);
  }
  for (int si = 0; si < ns; ++si)
    if (rc[si] != HEFF_OK) return set_err(rc[si], "%s", msg[si].c_str());
  const int sweeps_max = *std::max_element(swp.begin(), swp.end());
  struct Cand { double v; int si; int j; };
  std::vector<Cand> cand;
  for (int si = 0; si < ns; ++si)
    if (nc[si] > 0)
      for (int64_t j = 0; j < kc[si]; ++j) cand.push_back({sv_host[off_s[si] + j], si, (int)j});
  if (cand.empty() || !(cand[0].v >= 0.0)) return set_err(HEFF_EZERO, "heff_svd_split_qn: psi is zero");
  std::stable_sort(cand.begin(), cand.end(), [](const Cand& x, const Cand& y) {
    if (x.v != y.v) return x.v > y.v;
    if (x.si != y.si) return x.si < y.si;
    return x.j < y.j;
  });
  std::vector<double> sall(kmin, 0.0);
  for (size_t i = 0; i < cand.size() && (int64_t)i < kmin; ++i) sall[i] = cand[i].v;
  if (!(sall[0] > 0.0)) return set_err(HEFF_EZERO, "heff_svd_split_qn: psi is zero");
  int64_t n = 0;
  double err = 0.0;
  truncate_rule(sall.data(), kmin, cutoff, maxdim, mindim, &n, &err);
  std::vector<Cand> kept(cand.begin(), cand.begin() + n);
  std::stable_sort(kept.begin(), kept.end(), [](const Cand& x, const Cand& y) {
    if (x.si != y.si) return x.si < y.si;
    if (x.v != y.v) return x.v > y.v;
    return x.j < y.j;
  });
  std::vector<double> sk(n);
  std::vector<int2> jk(n);
  for (int64_t k = 0; k < n; ++k) {
    if (kept[k].j >= nc[kept[k].si]) return set_err(HEFF_ECUDA, "heff_svd_split_qn: kept a numerical zero");
    sk[k] = kept[k].v;
    qk[k] = sectors[kept[k].si];
    jk[k] = make_int2(kept[k].j, (int)k);
  }
  CK(cudaMemcpyAsync(S, sall.data(), sizeof(double) * kmin, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(Sk, sk.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_jk, jk.data(), sizeof(int2) * n, cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(Qout, 0, sizeof(double) * (dir == 0 ? M * n : n * N), s));
  CK(cudaMemsetAsync(Cout, 0, sizeof(double) * (dir == 0 ? n * N : M * n), s));
  int64_t k0 = 0;
  for (int si = 0; si < ns && k0 < n; ++si) {
    int64_t k1 = k0;
    while (k1 < n && kept[k1].si == si) ++k1;
    if (k1 > k0) {
      const int* d_rows = d_idx + off_idx[si];
      const int* d_cols = d_rows + Mc[si];
      dim3 grid((unsigned)std::min<int64_t>((std::max(Mc[si], Nc[si]) + 255) / 256, 64),
                (unsigned)std::min<int64_t>(k1 - k0, 65535));
      svd_qn_scatter_kernel<<<grid, 256, 0, s>>>(d_qc + off_q[si], d_cc + off_c[si], d_jk + k0, d_rows, d_cols, Mc[si],
                                                Nc[si], nc[si], dir, Qout, Cout, M, N, n, (int)(k1 - k0));
      CK(cudaGetLastError());
    }
    k0 = k1;
  }
  CK(cudaStreamSynchronize(s));
  *n_kept = n;
  *trunc_err = err;
  if (sweeps_out) *sweeps_out = sweeps_max;
  return HEFF_OK;
}


// --------------------------------------------------------------------------- cache release
void split_release_thread_caches() {
  t_svd_splitws.each([](SplitWs& w) {
    cudaFree(w.ptr);
    cudaFree(w.sync);
    w = SplitWs();
  });
  t_svd_arena.each([](SvdArena& a) {
    cudaFree(a.buf);
    a = SvdArena();
  });
  t_svdqn_arena.each([](SvdQnArena& a) {
    cudaFree(a.buf);
    a = SvdQnArena();
  });
  t_small_info.each([](double*& p) {
    cudaFree(p);
    p = nullptr;
  });
}

int split_release_worker_caches(int dev) {
  std::vector<std::function<void(cudaStream_t)>> tasks;
  for (int i = 0; i < kBlockWorkers; ++i)
    tasks.push_back([dev](cudaStream_t) { cudaSetDevice(dev); release_thread_caches(); });
  BlockPool::get().run_each_worker(tasks);
  return HEFF_OK;
}
