// gemm.cuh -- FP64 tensor-core GEMMs for the two O(m^3 k d^2) steps of H_eff.psi.
//
//   C[M][N] = A[M][K] . B        B K-major ([N][K], "NT")  or N-major ([K][N], "NN")
//
// sm_100a has no FP64 tcgen05 kind; the FP64 tensor path is the warp-level
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4, 128 flop/clk/SM measured, profiles/r01_fp64_peaks.txt).
// The Blackwell parts are the memory pipeline: TMA (cp.async.bulk.tensor) with the
// 128-byte swizzle fills a STAGES-deep shared-memory ring guarded by mbarriers, one
// producer warp drives it, and 8 consumer warps run DMMA from ld.shared fragments.
// Persistent: grid = #SMs, static round-robin over output tiles in GROUP_M raster.
//
// k-permutation: inside each 16-wide k block, DMMA k-slice kk (0..3) lane t (0..3) uses
// k = 2t + (kk & 1) + 8 (kk >> 1), identically for A and B.  k is summed, so any
// consistent bijection is exact; this one lets a lane fetch its A/B values for two
// k-slices with one 16-byte ld.shared.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "ptx.cuh"

namespace heff {

constexpr int kGemmBK = 16;  // doubles per k block = one 128-byte swizzle row

__device__ __forceinline__ void tile_coords(int tile, int num_m, int num_n, int group_m, int& mb, int& nb) {
  const int per_group = group_m * num_n;
  const int group = tile / per_group;
  const int first_m = group * group_m;
  const int gm = min(group_m, num_m - first_m);
  const int local = tile - group * per_group;
  mb = first_m + local % gm;
  nb = local / gm;
}

template <int BM, int BN, int WM, int WN, int STAGES, bool B_KMAJOR>
struct TmaGemmCfg {
  static constexpr int kConsumerWarps = (BM / WM) * (BN / WN);
  // one extra warpgroup hosts the TMA producer (one lane works); setmaxnreg moves its
  // registers to the consumer warpgroups (the 64K-register file is split per SM sub-partition)
  static constexpr int kThreads = (kConsumerWarps + 4) * 32;
  static constexpr int kConsumerRegs = 232, kProducerRegs = 40;
  static_assert(kConsumerWarps % 4 == 0, "consumers must form whole warpgroups");
  static constexpr int kTileABytes = BM * 128;
  static constexpr int kTileBBytes = BN * 128;
  static constexpr int kStageBytes = kTileABytes + kTileBBytes;
  static constexpr int kSmemBytes = STAGES * kStageBytes + 2 * STAGES * 8 + 1024;  // + barriers + align slack
  static_assert(BM % WM == 0 && BN % WN == 0 && WM % 8 == 0 && WN % 16 == 0, "tile shape");
  static_assert(BM <= 256 && (B_KMAJOR ? BN <= 256 : BN % 16 == 0), "TMA box limits");
};

template <int BM, int BN, int WM, int WN, int STAGES, bool B_KMAJOR>
__global__ void __launch_bounds__(TmaGemmCfg<BM, BN, WM, WN, STAGES, B_KMAJOR>::kThreads, 1)
    gemm_dmma_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         double* __restrict__ C, int64_t ldc, int M, int N, int K, int group_m, int vec_store,
                         int splits, int64_t split_stride, int accumulate) {
  using Cfg = TmaGemmCfg<BM, BN, WM, WN, STAGES, B_KMAJOR>;
  constexpr int MI = WM / 8, NJ = WN / 8;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::kStageBytes);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_m = (M + BM - 1) / BM, num_n = (N + BN - 1) / BN;
  const int tiles = num_m * num_n;
  const int ktiles = (K + kGemmBK - 1) / kGemmBK;
  // split-K: work unit u = (tile, split); split s covers k blocks [s*kper, min((s+1)*kper, ktiles))
  // and writes its partial tile to C + s*split_stride (reduced by splitk_reduce_kernel).
  const int kper = (ktiles + splits - 1) / splits;
  const int units = tiles * splits;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp >= Cfg::kConsumerWarps) {
    // ---------------- producer warpgroup: one lane drives the TMA ring ----------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(Cfg::kProducerRegs));
    if (warp == Cfg::kConsumerWarps && lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int mb, nb;
        tile_coords(u / splits, num_m, num_n, group_m, mb, nb);
        const int kb0 = (u % splits) * kper, kb1 = min(ktiles, kb0 + kper);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          unsigned char* sA = smem + stage * Cfg::kStageBytes;
          unsigned char* sB = sA + Cfg::kTileABytes;
          mbar_arrive_expect_tx(&full[stage], Cfg::kStageBytes);
          tma_load_2d(sA, &tmA, &full[stage], kb * kGemmBK, mb * BM);
          if constexpr (B_KMAJOR) {
            tma_load_2d(sB, &tmB, &full[stage], kb * kGemmBK, nb * BN);
          } else {
#pragma unroll
            for (int q = 0; q < BN / 16; ++q)
              tma_load_2d(sB + q * 2048, &tmB, &full[stage], nb * BN + q * 16, kb * kGemmBK);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    return;
  }

  // ---------------- consumer warps: DMMA from swizzled shared memory ----------------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(Cfg::kConsumerRegs));
  const int g = lane >> 2, t = lane & 3;
  const int wm0 = (warp / (BN / WN)) * WM;
  const int wn0 = (warp % (BN / WN)) * WN;
  const uint32_t smem_base = smem_u32(smem);
  // A (and K-major B): row r, 16-byte chunk c lives at r*128 + ((c ^ (r&7)) << 4); r&7 == g here.
  const uint32_t offA0 = (wm0 + g) * 128 + ((t ^ g) << 4);
  const uint32_t offB0 = (wn0 + g) * 128 + ((t ^ g) << 4);

  int stage = 0;
  uint32_t phase = 0;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    int mb, nb;
    tile_coords(u / splits, num_m, num_n, group_m, mb, nb);
    const int kb0 = (u % splits) * kper, kb1 = min(ktiles, kb0 + kper);
    double* Cu = C + (int64_t)(u % splits) * split_stride;
    double acc[MI][NJ][2];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int kb = kb0; kb < kb1; ++kb) {
      mbar_wait(&full[stage], phase);
      const uint32_t sA = smem_base + stage * Cfg::kStageBytes;
      const uint32_t sB = sA + Cfg::kTileABytes;
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // h = 0: k-slices 0,1 (chunk t); h = 1: k-slices 2,3 (chunk t+4)
        double a[MI][2], b[NJ][2];
#pragma unroll
        for (int i = 0; i < MI; ++i) lds128(a[i][0], a[i][1], sA + ((offA0 + i * 1024) ^ (h * 64)));
        if constexpr (B_KMAJOR) {
#pragma unroll
          for (int j = 0; j < NJ; ++j) lds128(b[j][0], b[j][1], sB + ((offB0 + j * 1024) ^ (h * 64)));
        } else {
#pragma unroll
          for (int j = 0; j < NJ; ++j) {
            const int n = wn0 + 8 * j + g;          // column inside the CTA tile
            const int ni = n & 15;
            const uint32_t box = sB + (n >> 4) * 2048;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int k = 2 * t + q + 8 * h;      // k-slice kk = 2h + q
              b[j][q] = lds64(box + k * 128 + ((((ni >> 1) ^ (k & 7))) << 4) + ((ni & 1) << 3));
            }
          }
        }
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NJ; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i][q], b[j][q]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }

    // epilogue: fragments straight to global (row-major C)
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int row = mb * BM + wm0 + 8 * i + g;
      if (row >= M) continue;
      double* crow = Cu + (int64_t)row * ldc;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int col = nb * BN + wn0 + 8 * j + 2 * t;
        if (vec_store && col + 1 < N) {
          double2 v = make_double2(acc[i][j][0], acc[i][j][1]);
          if (accumulate) {
            const double2 o = *reinterpret_cast<const double2*>(crow + col);
            v.x += o.x;
            v.y += o.y;
          }
          *reinterpret_cast<double2*>(crow + col) = v;
        } else {
          if (col < N) crow[col] = acc[i][j][0] + (accumulate ? crow[col] : 0.0);
          if (col + 1 < N) crow[col + 1] = acc[i][j][1] + (accumulate ? crow[col + 1] : 0.0);
        }
      }
    }
  }
}

// C[r][c] (+)= sum_s W[s][r][c] over the split-K partial tiles, in fixed order (deterministic).
__global__ void splitk_reduce_kernel(const double* __restrict__ W, int splits, int64_t split_stride,
                                     double* __restrict__ C, int64_t ldc, int M, int N, int accumulate) {
  const int64_t total = (int64_t)M * N;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / N, c = i - r * N;
    const int64_t off = r * ldc + c;
    double acc = W[off];
    for (int s = 1; s < splits; ++s) acc += W[s * split_stride + off];
    C[off] = accumulate ? C[off] + acc : acc;
  }
}

// ------------------------------------------------------------------------------------
// Plain-load DMMA GEMM: any shape, any alignment (8 B).  Used for tiny / odd problems
// where the TMA stride rules (16-byte row pitch) do not hold.  64x64 tile, 4 warps.
// ------------------------------------------------------------------------------------
template <bool B_KMAJOR>
__global__ void __launch_bounds__(128) gemm_dmma_plain_kernel(const double* __restrict__ A, int64_t lda,
                                                               const double* __restrict__ B, int64_t ldb,
                                                               double* __restrict__ C, int64_t ldc, int M, int N,
                                                               int K, int accumulate) {
  constexpr int BM = 64, BN = 64, BK = 16, PITCH = BK + 1;
  __shared__ double sA[BM][PITCH];
  __shared__ double sB[BN][PITCH];  // stored [n][k]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm0 = (warp >> 1) * 32, wn0 = (warp & 1) * 32;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int k0 = 0; k0 < K; k0 += BK) {
    for (int e = threadIdx.x; e < BM * BK; e += 128) {
      const int r = e / BK, c = e % BK;
      const int gm = m0 + r, gk = k0 + c;
      sA[r][c] = (gm < M && gk < K) ? A[(int64_t)gm * lda + gk] : 0.0;
    }
    for (int e = threadIdx.x; e < BN * BK; e += 128) {
      if constexpr (B_KMAJOR) {
        const int r = e / BK, c = e % BK;
        const int gn = n0 + r, gk = k0 + c;
        sB[r][c] = (gn < N && gk < K) ? B[(int64_t)gn * ldb + gk] : 0.0;
      } else {
        const int c = e / BN, r = e % BN;  // coalesced along n
        const int gn = n0 + r, gk = k0 + c;
        sB[r][c] = (gn < N && gk < K) ? B[(int64_t)gk * ldb + gn] : 0.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sA[wm0 + 8 * i + g][4 * kk + t];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sB[wn0 + 8 * j + g][4 * kk + t];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + wm0 + 8 * i + g;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = n0 + wn0 + 8 * j + 2 * t;
      double* c = C + (int64_t)row * ldc + col;
      if (col < N) c[0] = acc[i][j][0] + (accumulate ? c[0] : 0.0);
      if (col + 1 < N) c[1] = acc[i][j][1] + (accumulate ? c[1] : 0.0);
    }
  }
}

}  // namespace heff
