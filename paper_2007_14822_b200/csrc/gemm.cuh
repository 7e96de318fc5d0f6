// gemm.cuh -- FP64 tensor-core GEMMs for the two O(m^3 k d^2) steps of H_eff.psi.
//
//   C[M][N] = A[M][K] . B        B K-major ([N][K], "NT")  or N-major ([K][N], "NN")
//
// sm_100a has no FP64 tcgen05 kind; the FP64 tensor path is the warp-level
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4, 128 flop/clk/SM measured, profiles/r01_fp64_peaks.txt).
// The Blackwell parts are the memory pipeline: TMA (cp.async.bulk.tensor) with the
// 128-byte swizzle fills a STAGES-deep shared-memory ring guarded by mbarriers, one
// producer warp drives it, and 8 consumer warps run DMMA from ld.shared fragments.
// Persistent: grid = #SMs, static round-robin over output tiles in GROUP_M raster, plus a
// stream-K tail; launched with programmatic dependent launch (pdl_wait after the prologue).
// Tiles: 128x128 (8 consumer warps of 64x32) and 64x64 (8 of 32x16) for sub-wave GEMMs.
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

__host__ __device__ __forceinline__ void tile_coords(int tile, int num_m, int num_n, int group_m, int& mb, int& nb) {
  const int per_group = group_m * num_n;
  const int group = tile / per_group;
  const int first_m = group * group_m;
  const int gm = (group_m < num_m - first_m) ? group_m : (num_m - first_m);
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

// Work assignment (hybrid data-parallel + stream-K).  Tiles [0, dp_tiles) are taken whole,
// round-robin (CTA b: b, b+G, ...), so concurrently running CTAs work on neighbouring
// tiles of the GROUP_M raster and share L2.  The remaining tiles' (tile, k-block)
// iterations are cut into G equal contiguous ranges, one per CTA, so the last wave is
// balanced to the k-block.  A tile whose k-range is split between CTAs is written as
// partial tiles (slot 2b for CTA b's first stream-K tile, 2b+1 for its last) and summed in
// CTA order (deterministic) -- inside the kernel by the tile's highest contributor
// (StreamKSync below), or by streamk_fixup_kernel.  dp_tiles == tiles: plain persistent.
struct WorkRange {
  int64_t it, it_end;  // stream-K iteration range (iterations counted from dp_tiles*ktiles)
  int tile;            // data-parallel cursor
  int dp_tiles, ktiles;
  // block-sparse mode (kb_list != null): tiles taken whole in `order` (CTA b: entries b,
  // b+G, ...; -1 = padding), each over the k-blocks kb_list[kb_ptr[t] .. kb_ptr[t+1])
  const int* order;
  const int* kb_ptr;
  __device__ WorkRange(int cta, int tiles, int dp_tiles_, int ktiles_, const int* order_, const int* kb_ptr_)
      : dp_tiles(dp_tiles_), ktiles(ktiles_), order(order_), kb_ptr(kb_ptr_) {
    const int64_t total = (int64_t)(tiles - dp_tiles_) * ktiles_;
    it = total * cta / gridDim.x;
    it_end = total * (cta + 1) / gridDim.x;
    tile = cta;
  }
  // next (tile, [i0, i1)) segment; i indexes k-blocks (dense) or kb_list (sparse)
  __device__ bool next(int& t, int& i0, int& i1) {
    while (tile < dp_tiles) {
      t = order ? __ldg(order + tile) : tile;
      tile += gridDim.x;
      if (t < 0) continue;  // padding of a per-CTA (LPT) block-sparse schedule
      if (kb_ptr) {
        i0 = __ldg(kb_ptr + t);
        i1 = __ldg(kb_ptr + t + 1);
      } else {
        i0 = 0;
        i1 = ktiles;
      }
      return true;
    }
    if (it >= it_end) return false;
    const int local = (int)(it / ktiles);
    t = dp_tiles + local;
    i0 = (int)(it - (int64_t)local * ktiles);
    i1 = (int)min((int64_t)ktiles, (int64_t)i0 + (it_end - it));
    it += i1 - i0;
    return true;
  }
};

// In-kernel stream-K fixup (replaces streamk_fixup_kernel when `sk` is non-null).  Every
// split tile is reduced by its HIGHEST contributing CTA after that CTA's own work: it waits
// (release/acquire flags, one per partial slot, tagged with the launch epoch) for the lower
// contributors' partial tiles, sums all slots in CTA order -- the fixup kernel's order, so
// results are bitwise identical -- and stores the tile.  CTA indices are tickets taken from
// a global counter at CTA start (not blockIdx), so every CTA a reducer waits for has already
// started: waits cannot deadlock whatever order the hardware dispatches CTAs in, or
// whatever else shares the GPU.  A wait that exceeds ~10 s traps (a reported launch error,
// never a hang).
struct StreamKSync {
  unsigned int* counter;  // ticket counter: 0 between launches (the last ticket holder resets it)
  int* flags;             // [2 * gridDim.x] slot flags
  int epoch;              // this launch's flag value (> 0, increasing)
};

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void consumers_bar(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// CTA owning stream-K iteration `it` when `total` iterations are cut into G equal ranges
__host__ __device__ __forceinline__ int sk_cta_of(int64_t it, int64_t total, int G) {
  int64_t b = (it * G) / total;
  while (b + 1 < G && total * (b + 1) / G <= it) ++b;
  while (b > 0 && total * b / G > it) --b;
  return (int)b;
}

// A operand split along K over up to kMaxShards tensor maps (NEXT-5 gather-fused GEMM_A):
// k-block kb is read from map (16 kb) / ksh at column 16 kb - shard * ksh.  The maps may
// address peer GPUs' memory (NCCL symmetric-window pointers over NVLink).
constexpr int kMaxShards = 8;
struct ShardedA {
  CUtensorMap map[kMaxShards];
  int nsh;
  int ksh;
};

template <int BM, int BN, int WM, int WN, int STAGES, bool B_KMAJOR, bool SHARDED_A>
__device__ __forceinline__ void gemm_dmma_tma_body(const CUtensorMap* tmA, const ShardedA* sa, const CUtensorMap* tmB,
                                                   double* __restrict__ C, int64_t ldc, int M, int N, int K,
                                                   int group_m, int vec_store, int dp_tiles,
                                                   double* __restrict__ partial_ws, int accumulate,
                                                   const int* __restrict__ tile_order, const int* __restrict__ kb_ptr,
                                                   const int* __restrict__ kb_list, const StreamKSync* sk) {
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

  __shared__ int s_cta;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::kConsumerWarps);
    }
    fence_barrier_init();
  }
  // launched with programmatic dependent launch: the prologue above overlaps the previous
  // kernel's tail; operands, C and the stream-K ticket counter are touched only after it
  pdl_wait();
  if (threadIdx.x == 0) {
    int c = (int)blockIdx.x;
    if (sk) {
      c = (int)atomicAdd(sk->counter, 1u);
      if (c == (int)gridDim.x - 1) atomicExch(sk->counter, 0u);  // every CTA holds its ticket
    }
    s_cta = c;
  }
  __syncthreads();
  const int cta = s_cta;

  if (warp >= Cfg::kConsumerWarps) {
    // ---------------- producer warpgroup: one lane drives the TMA ring ----------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(Cfg::kProducerRegs));
    if (warp == Cfg::kConsumerWarps && lane == 0) {
      if constexpr (SHARDED_A) {
        for (int q = 0; q < sa->nsh; ++q) tma_prefetch_desc(&sa->map[q]);
      } else {
        tma_prefetch_desc(tmA);
      }
      tma_prefetch_desc(tmB);
      int stage = 0;
      uint32_t phase = 0;
      WorkRange wr(cta, tiles, dp_tiles, ktiles, tile_order, kb_ptr);
      int tile, i0, i1;
      while (wr.next(tile, i0, i1)) {
        int mb, nb;
        tile_coords(tile, num_m, num_n, group_m, mb, nb);
        for (int idx = i0; idx < i1; ++idx) {
          const int kb = kb_list ? __ldg(kb_list + idx) : idx;
          mbar_wait(&empty[stage], phase ^ 1);
          unsigned char* sA = smem + stage * Cfg::kStageBytes;
          unsigned char* sB = sA + Cfg::kTileABytes;
          mbar_arrive_expect_tx(&full[stage], Cfg::kStageBytes);
          if constexpr (SHARDED_A) {
            const int k0 = kb * kGemmBK, sh = k0 / sa->ksh;
            tma_load_2d(sA, &sa->map[sh], &full[stage], k0 - sh * sa->ksh, mb * BM);
          } else {
            tma_load_2d(sA, tmA, &full[stage], kb * kGemmBK, mb * BM);
          }
          if constexpr (B_KMAJOR) {
            tma_load_2d(sB, tmB, &full[stage], kb * kGemmBK, nb * BN);
          } else {
#pragma unroll
            for (int q = 0; q < BN / 16; ++q)
              tma_load_2d(sB + q * 2048, tmB, &full[stage], nb * BN + q * 16, kb * kGemmBK);
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
  WorkRange wr(cta, tiles, dp_tiles, ktiles, tile_order, kb_ptr);
  int tile, kb0, kb1;
  bool first_seg = true;  // first stream-K segment of this CTA
  while (wr.next(tile, kb0, kb1)) {
    int mb, nb;
    tile_coords(tile, num_m, num_n, group_m, mb, nb);
    double acc[MI][NJ][2];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int idx = kb0; idx < kb1; ++idx) {  // the consumers only count k-blocks; the producer picks them
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
      // Release the stage.  The fragments were read by the generic proxy (ld.shared) and the
      // producer's next TMA write comes through the async proxy: without a proxy fence ptxas
      // may issue the arrive while the last ld.shared are still in flight and the refill
      // can overtake them (observed: stale rows 48-63 with short stream-K segments).
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }

    if (kb_list || (kb0 == 0 && kb1 == ktiles)) {
      // whole tile: fragments straight to global (row-major C)
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int row = mb * BM + wm0 + 8 * i + g;
        if (row >= M) continue;
        double* crow = C + (int64_t)row * ldc;
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
    } else {
      // stream-K partial tile -> workspace slot (full BM x BN, row-major)
      const int slot = cta * 2 + (first_seg ? 0 : 1);
      double* ws = partial_ws + (int64_t)slot * (BM * BN);
      first_seg = false;
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j)
          *reinterpret_cast<double2*>(ws + (wm0 + 8 * i + g) * BN + wn0 + 8 * j + 2 * t) =
              make_double2(acc[i][j][0], acc[i][j][1]);
      if (sk) {  // publish the slot: every writer fences, then one release store
        __threadfence();
        consumers_bar(Cfg::kConsumerWarps * 32);
        if (threadIdx.x == 0) st_release_gpu(sk->flags + slot, sk->epoch);
      }
    }
    if (tile >= dp_tiles) first_seg = false;
  }

  if (sk && !kb_list && dp_tiles < tiles) {
    // Reduce the split tile that holds this CTA's first stream-K iteration, if this CTA also
    // holds its last iteration (= the highest contributor) and the tile began in a lower CTA.
    const int64_t total = (int64_t)(tiles - dp_tiles) * ktiles;
    const int G = gridDim.x;
    const int64_t it0 = total * cta / G, it1 = total * (cta + 1) / G;
    if (it0 < it1 && it0 % ktiles != 0) {
      const int local = (int)(it0 / ktiles);
      if ((int64_t)(local + 1) * ktiles <= it1) {
        const int b0 = sk_cta_of((int64_t)local * ktiles, total, G);
        const int nthr = Cfg::kConsumerWarps * 32;
        if (threadIdx.x == 0) {
          long long t_start;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
          for (int b = b0; b < cta; ++b) {
            const int slot_b = 2 * b + ((int)((total * b / G) / ktiles) == local ? 0 : 1);
            while (ld_acquire_gpu(sk->flags + slot_b) != sk->epoch) {
              __nanosleep(64);
              long long t_now;
              asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_now));
              if (t_now - t_start > 10000000000ll) __trap();
            }
          }
        }
        consumers_bar(nthr);
        int mb, nb;
        tile_coords(dp_tiles + local, num_m, num_n, group_m, mb, nb);
        // each thread owns kPer double2 of the tile, taken kChunk at a time: for one chunk it
        // loads the slots in CTA order, kChunk independent L2 loads in flight per slot
        constexpr int kPer = BM * BN / (2 * Cfg::kConsumerWarps * 32);
        constexpr int kChunk = kPer < 16 ? kPer : 16;
        static_assert(kPer % kChunk == 0, "chunking");
#pragma unroll 1
        for (int i0 = 0; i0 < kPer; i0 += kChunk) {
          double2 a[kChunk];
#pragma unroll
          for (int i = 0; i < kChunk; ++i) a[i] = make_double2(0.0, 0.0);
          for (int b = b0; b <= cta; ++b) {
            const int slot_b = 2 * b + ((int)((total * b / G) / ktiles) == local ? 0 : 1);
            const double2* src = reinterpret_cast<const double2*>(partial_ws + (int64_t)slot_b * (BM * BN));
#pragma unroll
            for (int i = 0; i < kChunk; ++i) {
              const double2 v = __ldcg(src + threadIdx.x + (i0 + i) * nthr);
              a[i].x += v.x;
              a[i].y += v.y;
            }
          }
#pragma unroll
          for (int i = 0; i < kChunk; ++i) {
            const int e = 2 * (threadIdx.x + (i0 + i) * nthr);
            const int r = e / BN, c = e - r * BN;  // c even
            const int row = mb * BM + r, col = nb * BN + c;
            if (row >= M || col >= N) continue;
            double* cp = C + (int64_t)row * ldc + col;
            if (vec_store && col + 1 < N) {
              double2 v = a[i];
              if (accumulate) {
                const double2 o = *reinterpret_cast<const double2*>(cp);
                v.x += o.x;
                v.y += o.y;
              }
              *reinterpret_cast<double2*>(cp) = v;
            } else {
              cp[0] = accumulate ? cp[0] + a[i].x : a[i].x;
              if (col + 1 < N) cp[1] = accumulate ? cp[1] + a[i].y : a[i].y;
            }
          }
        }
      }
    }
  }
}

template <int BM, int BN, int WM, int WN, int STAGES, bool B_KMAJOR>
__global__ void __launch_bounds__(TmaGemmCfg<BM, BN, WM, WN, STAGES, B_KMAJOR>::kThreads, 1)
    gemm_dmma_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         double* __restrict__ C, int64_t ldc, int M, int N, int K, int group_m, int vec_store,
                         int dp_tiles, double* __restrict__ partial_ws, int accumulate,
                         const int* __restrict__ tile_order, const int* __restrict__ kb_ptr,
                         const int* __restrict__ kb_list, const __grid_constant__ StreamKSync sk, int use_sk) {
  gemm_dmma_tma_body<BM, BN, WM, WN, STAGES, B_KMAJOR, false>(&tmA, nullptr, &tmB, C, ldc, M, N, K, group_m, vec_store,
                                                              dp_tiles, partial_ws, accumulate, tile_order, kb_ptr,
                                                              kb_list, use_sk ? &sk : nullptr);
}

template <int BM, int BN, int WM, int WN, int STAGES, bool B_KMAJOR>
__global__ void __launch_bounds__(TmaGemmCfg<BM, BN, WM, WN, STAGES, B_KMAJOR>::kThreads, 1)
    gemm_dmma_tma_sharded_kernel(const __grid_constant__ ShardedA sa, const __grid_constant__ CUtensorMap tmB,
                                 double* __restrict__ C, int64_t ldc, int M, int N, int K, int group_m, int vec_store,
                                 int dp_tiles, double* __restrict__ partial_ws, int accumulate,
                                 const __grid_constant__ StreamKSync sk, int use_sk) {
  gemm_dmma_tma_body<BM, BN, WM, WN, STAGES, B_KMAJOR, true>(nullptr, &sa, &tmB, C, ldc, M, N, K, group_m, vec_store,
                                                             dp_tiles, partial_ws, accumulate, nullptr, nullptr,
                                                             nullptr, use_sk ? &sk : nullptr);
}

// Stream-K fixup: every stream-K tile whose k-range was split across CTAs is the sum, in
// CTA order, of their partial slots.  One block per stream-K tile; the slot list is
// computed once per block (no per-element integer division), then the tile is summed with
// 16-byte loads.
constexpr int kFixupMaxParts = 256;
constexpr int kFixupSplit = 16;  // blocks per tile (parallelism for small problems)

template <int BM, int BN>
__global__ void __launch_bounds__(256) streamk_fixup_kernel(const double* __restrict__ ws, double* __restrict__ C,
                                                            int64_t ldc, int M, int N, int ktiles, int group_m,
                                                            int grid, int dp_tiles, int accumulate) {
  __shared__ int s_slot[kFixupMaxParts];
  __shared__ int s_n;
  pdl_wait();
  const int num_m = (M + BM - 1) / BM, num_n = (N + BN - 1) / BN;
  const int local = blockIdx.x / kFixupSplit;  // stream-K tile index
  const int part = blockIdx.x % kFixupSplit;    // this block's 1/kFixupSplit of the tile
  const int tile = dp_tiles + local;
  if (threadIdx.x == 0) {
    const int64_t total = (int64_t)(num_m * num_n - dp_tiles) * ktiles;
    // CTA b owns stream-K iterations [total*b/grid, total*(b+1)/grid)
    auto cta_of = [&](int64_t it) { return sk_cta_of(it, total, grid); };
    const int64_t it_first = (int64_t)local * ktiles;
    const int b0 = cta_of(it_first), b1 = cta_of(it_first + ktiles - 1);
    int n = 0;
    if (b0 != b1)
      for (int b = b0; b <= b1 && n < kFixupMaxParts; ++b) {
        const int first_local_of_b = (int)((total * b / grid) / ktiles);
        s_slot[n++] = 2 * b + (first_local_of_b == local ? 0 : 1);
      }
    s_n = n;  // 0: the tile was written whole by one CTA
  }
  __syncthreads();
  const int n = s_n;
  if (n == 0) return;
  int mb, nb;
  tile_coords(tile, num_m, num_n, group_m, mb, nb);
  const bool vec = ((ldc & 1) == 0) && ((reinterpret_cast<uintptr_t>(C) & 15) == 0);
  constexpr int kPer = BM * BN / kFixupSplit;
  for (int e = part * kPer + threadIdx.x * 2; e < (part + 1) * kPer; e += blockDim.x * 2) {
    const int r = e / BN, c = e - r * BN;  // c even
    const int row = mb * BM + r, col = nb * BN + c;
    if (row >= M || col >= N) continue;
    double2 acc = make_double2(0.0, 0.0);
    for (int k = 0; k < n; ++k) {
      const double2 v = *reinterpret_cast<const double2*>(ws + (int64_t)s_slot[k] * (BM * BN) + e);
      acc.x += v.x;
      acc.y += v.y;
    }
    double* cp = C + (int64_t)row * ldc + col;
    if (vec && col + 1 < N) {
      if (accumulate) {
        const double2 o = *reinterpret_cast<const double2*>(cp);
        acc.x += o.x;
        acc.y += o.y;
      }
      *reinterpret_cast<double2*>(cp) = acc;
    } else {
      cp[0] = accumulate ? cp[0] + acc.x : acc.x;
      if (col + 1 < N) cp[1] = accumulate ? cp[1] + acc.y : acc.y;
    }
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
