// heff_api.cu -- libheff: plans, the H_eff.psi matvec, and the Lanczos driver.
// C ABI in include/heff.h (each entry point documents its arguments there).
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nccl_device.h>

#include <algorithm>
#include <cstdarg>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <unordered_map>
#include <thread>
#include <map>
#include <queue>
#include <string>
#include <vector>

#include "../../include/heff.h"
#include "blas1.cuh"
#include "gemm.cuh"
#include "gemm_small.cuh"
#include "mpo.cuh"
#include "tridiag.h"
#include "internal.h"

using namespace heff;

// ----------------------------------------------------------------------------- errors
static thread_local std::string g_err;

int set_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}


extern "C" const char* heff_last_error(void) { return g_err.c_str(); }

// ----------------------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
  bool loaded = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) =
      nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  // symmetric memory windows (NCCL >= 2.27; optional: the gather-fused path needs them)
  ncclResult_t (*MemAlloc)(void**, size_t) = nullptr;
  ncclResult_t (*MemFree)(void*) = nullptr;
  ncclResult_t (*CommWindowRegister)(ncclComm_t, void*, size_t, ncclWindow_t*, int) = nullptr;
  ncclResult_t (*CommWindowDeregister)(ncclComm_t, ncclWindow_t) = nullptr;
};

static NcclApi g_nccl;

static std::mutex g_nccl_mu;  // ranks of one process may create their plans concurrently

static int nccl_load() {
  std::lock_guard<std::mutex> lock(g_nccl_mu);
  if (g_nccl.loaded) return HEFF_OK;
  const char* env = getenv("HEFF_NCCL_PATH");
  void* h = nullptr;
  if (env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);  // torch's copy, if loaded
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return set_err(HEFF_ENCCL, "cannot load libnccl.so.2: %s", dlerror());
#define LD(name)                                                                   \
  g_nccl.name = reinterpret_cast<decltype(g_nccl.name)>(dlsym(h, "nccl" #name));   \
  if (!g_nccl.name) return set_err(HEFF_ENCCL, "libnccl lacks nccl%s", #name);
  LD(GetUniqueId) LD(CommInitRank) LD(CommDestroy) LD(CommAbort) LD(AllReduce) LD(AllGather) LD(CommGetAsyncError)
  LD(GetErrorString)
#undef LD
  g_nccl.MemAlloc = reinterpret_cast<decltype(g_nccl.MemAlloc)>(dlsym(h, "ncclMemAlloc"));
  g_nccl.MemFree = reinterpret_cast<decltype(g_nccl.MemFree)>(dlsym(h, "ncclMemFree"));
  g_nccl.CommWindowRegister = reinterpret_cast<decltype(g_nccl.CommWindowRegister)>(dlsym(h, "ncclCommWindowRegister"));
  g_nccl.CommWindowDeregister =
      reinterpret_cast<decltype(g_nccl.CommWindowDeregister)>(dlsym(h, "ncclCommWindowDeregister"));
  g_nccl.loaded = true;
  return HEFF_OK;
}

#define CKN(call)                                                                                     \
  do {                                                                                                \
    ncclResult_t r_ = (call);                                                                         \
    if (r_ != ncclSuccess) return set_err(HEFF_ENCCL, "%s: %s", #call, g_nccl.GetErrorString(r_)); \
  } while (0)

extern "C" int heff_nccl_unique_id(unsigned char uid[128]) {
  if (!uid) return set_err(HEFF_EINVAL, "uid is NULL");
  CKR(nccl_load());
  ncclUniqueId id;
  CKN(g_nccl.GetUniqueId(&id));
  memcpy(uid, id.internal, 128);
  return HEFF_OK;
}

// ----------------------------------------------------------------------------- TMA maps
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t get_encode() {
  static const PFN_encodeTiled_t fn = [] {  // thread-safe one-time lookup
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_encodeTiled_t>(p);
    return static_cast<PFN_encodeTiled_t>(nullptr);
  }();
  return fn;
}

// 2-D row-major fp64 view: `rows` rows of `cols` elements, row pitch `ld` elements; box
// {box_cols, box_rows}; 128-byte swizzle; OOB reads return zero.
int make_map(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld, int box_cols,
                    int box_rows) {
  PFN_encodeTiled_t enc = get_encode();
  if (!enc) return set_err(HEFF_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(HEFF_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return HEFF_OK;
}

// ----------------------------------------------------------------------------- GEMM launch
// Tile configurations of the TMA path.  The 128x128 tile
// (8 consumer warps of 64x32) runs every GEMM with at least one full wave of tiles; the
// 64x64 tile (4 consumer warps of 32x32, 8-deep ring) runs dense GEMMs whose 128x128 tile
// count is below one wave (C2-size matvecs, small environment / split GEMMs), where the
// stream-K partial tiles -- and so the fixup traffic -- are 4x smaller.
constexpr int kBM = 128, kBN = 128, kWM = 64, kWN = 32, kStages = 5, kGroupM = 16;
constexpr int kBMs = 64, kBNs = 64, kWMs = 32, kWNs = 16, kStagesS = 8;
using CfgNN = TmaGemmCfg<kBM, kBN, kWM, kWN, kStages, false>;
using CfgNT = TmaGemmCfg<kBM, kBN, kWM, kWN, kStages, true>;
using CfgNNs = TmaGemmCfg<kBMs, kBNs, kWMs, kWNs, kStagesS, false>;
using CfgNTs = TmaGemmCfg<kBMs, kBNs, kWMs, kWNs, kStagesS, true>;
// cluster split-K (gemm_small.cuh): 64x64 tiles, 6-stage ring, CS = 2 or 4 CTAs per tile
static unsigned long long* g_cluster_dbg = nullptr;  // diagnostics (heff_debug_fused_timestamps)
constexpr int kClStages = 6;
using CfgCl2 = ClusterGemmCfg<64, 64, 32, 16, kClStages, 2>;
using CfgCl4 = ClusterGemmCfg<64, 64, 32, 16, kClStages, 4>;



int g_num_sms = 0;
// the plan workspace cache (defined with the plan code below)
template <typename T>
static cudaError_t ws_malloc(T** out, size_t bytes);
static void ws_release(void* ptr);
// diagnostics of the fused small-bond kernel (heff_debug_fused_timestamps): per-CTA timers
static unsigned long long* g_fused_dbg = nullptr;
static int g_fused_dbg_mode = 0;  // 1: no T3 stores, 2: no MPO epilogue (timing experiments; wrong results)



static bool tma_ok(const GemmOp& g) {
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return (g.lda % 2 == 0) && (g.ldb % 2 == 0) && al16(g.A) && al16(g.B) && g.M < (1ll << 31) && g.N < (1ll << 31) &&
         g.K < (1ll << 31);
}



// Per-thread, per-stream workspaces for the free functions (heff_gemm, environment
// updates): GEMMs enqueued by one thread on two streams may run concurrently and must not
// share partial slots or the CTA ticket counter.
// Keyed by (device, stream): the legacy default stream (0) has the same handle on every device.
using StreamWs = std::vector<std::pair<std::pair<int, cudaStream_t>, SplitWs>>;
static SplitWs* ws_for(StreamWs& v, cudaStream_t s) {
  const std::pair<int, cudaStream_t> key(cur_device(), s);
  for (auto& e : v)
    if (e.first == key) return &e.second;
  v.emplace_back(key, SplitWs());
  return &v.back().second;
}

// HEFF_SK_FIXUP_KERNEL=1: sum split tiles in the separate streamk_fixup_kernel instead of in-kernel
static bool sk_inkernel() { return getenv("HEFF_SK_FIXUP_KERNEL") == nullptr; }

// One dense/sparse TMA GEMM with tile BM x BN: maps, hybrid data-parallel + stream-K
// schedule, kernel and (if any tile's k-range was split) the fixup.
template <int BM, int BN, int WM, int WN, int ST>
static int launch_tma(GemmOp& g, cudaStream_t s, int* nlaunch, SplitWs* ws, const ShardedA* sa) {
  using NN = TmaGemmCfg<BM, BN, WM, WN, ST, false>;
  using NT = TmaGemmCfg<BM, BN, WM, WN, ST, true>;
  if (!sa && (g.mapA_ptr != g.A || g.mapA_rows != g.M || g.mapA_box != BM)) {
    CKR(make_map(&g.mapA, g.A, g.M, g.K, g.lda, kGemmBK, BM));
    g.mapA_ptr = g.A;
    g.mapA_rows = g.M;
    g.mapA_box = BM;
  }
  if (g.mapB_ptr != g.B || g.mapB_rows != g.N || g.mapB_box != BN) {
    if (g.b_kmajor)
      CKR(make_map(&g.mapB, g.B, g.N, g.K, g.ldb, kGemmBK, BN));
    else
      CKR(make_map(&g.mapB, g.B, g.K, g.N, g.ldb, 16, kGemmBK));
    g.mapB_ptr = g.B;
    g.mapB_rows = g.N;
    g.mapB_box = BN;
  }
  const int64_t tiles = ((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN);
  const int64_t ktiles = (g.K + kGemmBK - 1) / kGemmBK;
  // Hybrid schedule: whole tiles round-robin for all but the last one-to-two waves, whose
  // (tile, k-block) iterations are balanced across the SMs by stream-K.
  int grid = (int)std::min<int64_t>(tiles, g_num_sms);
  int64_t dp_tiles = tiles;
  const int64_t waves = (tiles + g_num_sms - 1) / g_num_sms;
  const double eff = (double)tiles / (double)(waves * g_num_sms);
  const bool sparse = g.sp_list != nullptr;
  if (sparse && g.sp_len > 0) dp_tiles = g.sp_len;
  if (!sparse && ws && eff < 0.995 && getenv("HEFF_NO_STREAMK") == nullptr) {
    dp_tiles = (tiles >= 2 * (int64_t)g_num_sms) ? (tiles / g_num_sms - 1) * g_num_sms : 0;
    const int64_t sk_iters = (tiles - dp_tiles) * ktiles;
    grid = (int)std::max<int64_t>(1, std::min<int64_t>(g_num_sms, sk_iters / 4));  // >= 4 k-blocks per CTA
    // every split tile must have <= kFixupMaxParts contributing CTAs
    while (grid > 1 && ktiles / std::max<int64_t>(1, sk_iters / grid) + 2 > kFixupMaxParts) grid /= 2;
    if (dp_tiles > 0) grid = g_num_sms;
    const size_t need = sizeof(double) * 2 * (size_t)grid * BM * BN;
    if (ws->bytes < need) {
      if (ws->cached) {
        if (ws->ptr) {
          CK(cudaStreamSynchronize(s));  // the old block is idle before it returns to the cache
          ws_release(ws->ptr);
        }
      } else {
        cudaFree(ws->ptr);
      }
      ws->ptr = nullptr;
      ws->bytes = 0;
      if ((ws->cached ? ws_malloc(&ws->ptr, need) : cudaMalloc(&ws->ptr, need)) != cudaSuccess) {
        cudaGetLastError();
        dp_tiles = tiles;  // no room for partial tiles: plain persistent schedule
        grid = (int)std::min<int64_t>(tiles, g_num_sms);
      } else {
        ws->bytes = need;
      }
    }
  }
  const int vec = ((g.ldc % 2) == 0 && (reinterpret_cast<uintptr_t>(g.C) & 15) == 0) ? 1 : 0;
  double* wsp = ws ? ws->ptr : nullptr;
  StreamKSync sk{};
  int use_sk = 0;
  if (dp_tiles < tiles && grid <= kSkMaxGrid && sk_inkernel()) {
    if (!ws->sync) {
      const size_t sb = 16 + sizeof(int) * 2 * kSkMaxGrid;
      if ((ws->cached ? ws_malloc(&ws->sync, sb) : cudaMalloc(&ws->sync, sb)) != cudaSuccess)
        return set_err(HEFF_ENOMEM, "stream-K sync buffer");
      CK(cudaMemsetAsync(ws->sync, 0, sb, s));  // (a reused block: stale flags must not match an epoch)
      ws->epoch = 0;
    }
    sk.counter = static_cast<unsigned int*>(ws->sync);
    sk.flags = reinterpret_cast<int*>(static_cast<char*>(ws->sync) + 16);
    sk.epoch = ++ws->epoch;
    use_sk = 1;
  }
  const int M32 = (int)g.M, N32 = (int)g.N, K32 = (int)g.K, dp32 = (int)dp_tiles;
  // tile raster: GROUP_M consecutive M-tiles per column sweep (block-sparse schedules are
  // built for kGroupM; HEFF_GEMM_GROUP_M overrides it for dense GEMMs, a tuning knob)
  int gm = kGroupM;
  if (!sparse)
    if (const char* e = getenv("HEFF_GEMM_GROUP_M")) gm = std::max(1, atoi(e));
  if (sa) {
    if (!g.b_kmajor) return set_err(HEFF_EUNSUPPORTED, "sharded-A GEMM: NT only");
    CK(launch_pdl(gemm_dmma_tma_sharded_kernel<BM, BN, WM, WN, ST, true>, dim3(grid), dim3(NT::kThreads),
                  NT::kSmemBytes, s, *sa, g.mapB, g.C, g.ldc, M32, N32, K32, gm, vec, dp32, wsp, g.accumulate, sk,
                  use_sk));
  } else if (g.b_kmajor) {
    CK(launch_pdl(gemm_dmma_tma_kernel<BM, BN, WM, WN, ST, true>, dim3(grid), dim3(NT::kThreads), NT::kSmemBytes, s,
                  g.mapA, g.mapB, g.C, g.ldc, M32, N32, K32, gm, vec, dp32, wsp, g.accumulate, g.sp_order,
                  g.sp_ptr, g.sp_list, sk, use_sk));
  } else {
    CK(launch_pdl(gemm_dmma_tma_kernel<BM, BN, WM, WN, ST, false>, dim3(grid), dim3(NN::kThreads), NN::kSmemBytes, s,
                  g.mapA, g.mapB, g.C, g.ldc, M32, N32, K32, gm, vec, dp32, wsp, g.accumulate, g.sp_order,
                  g.sp_ptr, g.sp_list, sk, use_sk));
  }
  if (dp_tiles < tiles && !use_sk) {
    if (nlaunch) ++*nlaunch;
    CK(launch_pdl(streamk_fixup_kernel<BM, BN>, dim3((unsigned)((tiles - dp_tiles) * kFixupSplit)), dim3(256), 0, s,
                  (const double*)wsp, g.C, g.ldc, M32, N32, (int)ktiles, gm, grid, dp32, g.accumulate));
  }
  return HEFF_OK;
}

// Tile choice: 64x64 for dense GEMMs with fewer 128x128 tiles than SMs (HEFF_GEMM_TILE=128 /
// =64 forces one).  Block-sparse schedules and the sharded-A GEMM are built on 128x128 tiles.
static bool use_small_tile(const GemmOp& g, const ShardedA* sa) {
  if (sa || g.sp_list) return false;
  const char* e = getenv("HEFF_GEMM_TILE");
  const int force = e ? atoi(e) : 0;
  if (force == 64) return true;
  if (force == 128) return false;
  const int64_t tiles = ((g.M + kBM - 1) / kBM) * ((g.N + kBN - 1) / kBN);
  return tiles < g_num_sms;
}

// sa != nullptr: the A operand is K-sharded over sa->nsh tensor maps (gemm_dmma_tma_sharded_kernel;
// g.A is ignored, the TMA path is required).
// Cluster split-K for dense GEMMs with few 64x64 tiles (gemm_small.cuh): CS CTAs of a cluster
// share one tile's K range and reduce through DSMEM.  Chosen when tiles x CS fills at least
// 60% of the SMs in one wave with >= 4 k-blocks per rank (else the stream-K schedule, which
// spreads a handful of tiles over every SM, is better).  HEFF_NO_CLUSTER_SPLITK=1 disables.
// Co-resident clusters of CS CTAs (clusters live inside one GPC: at CS = 4 a B200 holds 32
// of them, 128 of its 148 SMs, not 37); queried once per device and size.
static int max_active_clusters(int cs) {
  static std::mutex mu;
  static int cache[kMaxDevices][5] = {};
  const int dev = cur_device();
  std::lock_guard<std::mutex> lock(mu);
  int& c = cache[dev][cs];
  if (c == 0) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(cs * 64));
    cfg.blockDim = dim3(cs == 4 ? CfgCl4::kThreads : CfgCl2::kThreads);
    cfg.dynamicSmemBytes = cs == 4 ? CfgCl4::kSmemBytes : CfgCl2::kSmemBytes;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    const cudaError_t e =
        cs == 4 ? cudaOccupancyMaxActiveClusters(&n, gemm_cluster_splitk_kernel<64, 64, 32, 16, kClStages, true, 4>, &cfg)
                : cudaOccupancyMaxActiveClusters(&n, gemm_cluster_splitk_kernel<64, 64, 32, 16, kClStages, true, 2>, &cfg);
    if (e != cudaSuccess) {
      cudaGetLastError();
      n = -1;  // unknown: never choose the cluster path
    }
    c = n;
  }
  return c;
}

// Co-resident clusters of CS CTAs of matvec_cluster_kernel (one CTA per SM: its shared memory)
static int max_active_mvc_clusters(int cs) {
  static std::mutex mu;
  static int cache[kMaxDevices][9] = {};
  const int dev = cur_device();
  std::lock_guard<std::mutex> lock(mu);
  int& c = cache[dev][cs];
  if (c == 0) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(cs * 32));
    cfg.blockDim = dim3(kFusedThreads);
    cfg.dynamicSmemBytes = kMvcSmemBytes;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, matvec_cluster_kernel<64>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      n = -1;  // unknown: never choose the cluster matvec
    }
    c = n;
  }
  return c;
}

// Cluster split-K for dense GEMMs with few 64x64 tiles (gemm_small.cuh): CS CTAs of a cluster
// share one tile's K range and reduce through DSMEM.  Chosen when the tiles x CS CTAs run in
// ONE wave of co-resident clusters filling >= 60% of the SMs, with >= 4 k-blocks per rank
// (else the stream-K schedule, which spreads a handful of tiles over every SM, is better).
// HEFF_NO_CLUSTER_SPLITK=1 disables.
static int cluster_splitk_size(const GemmOp& g, const ShardedA* sa) {
  if (sa || g.sp_list || getenv("HEFF_NO_CLUSTER_SPLITK") != nullptr) return 0;
  if (const char* e = getenv("HEFF_GEMM_TILE"))
    if (atoi(e) == 128) return 0;
  const int64_t tiles = ((g.M + 63) / 64) * ((g.N + 63) / 64);
  const int64_t ktiles = (g.K + kGemmBK - 1) / kGemmBK;
  for (int cs : {4, 2})
    if (tiles * cs <= g_num_sms && tiles * cs * 10 >= 6 * (int64_t)g_num_sms && ktiles >= 4 * cs &&
        tiles <= max_active_clusters(cs))
      return cs;
  return 0;
}

template <int CS>
static int launch_cluster_splitk(GemmOp& g, cudaStream_t s) {
  using Cfg = ClusterGemmCfg<64, 64, 32, 16, kClStages, CS>;
  if (g.mapA_ptr != g.A || g.mapA_rows != g.M || g.mapA_box != 64) {
    CKR(make_map(&g.mapA, g.A, g.M, g.K, g.lda, kGemmBK, 64));
    g.mapA_ptr = g.A;
    g.mapA_rows = g.M;
    g.mapA_box = 64;
  }
  if (g.mapB_ptr != g.B || g.mapB_rows != g.N || g.mapB_box != 64) {
    if (g.b_kmajor)
      CKR(make_map(&g.mapB, g.B, g.N, g.K, g.ldb, kGemmBK, 64));
    else
      CKR(make_map(&g.mapB, g.B, g.K, g.N, g.ldb, 16, kGemmBK));
    g.mapB_ptr = g.B;
    g.mapB_rows = g.N;
    g.mapB_box = 64;
  }
  const int64_t tiles = ((g.M + 63) / 64) * ((g.N + 63) / 64);
  const int vec = ((g.ldc % 2) == 0 && (reinterpret_cast<uintptr_t>(g.C) & 15) == 0) ? 1 : 0;
  static const bool pdl_off = getenv("HEFF_NO_PDL") != nullptr;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(tiles * CS));
  cfg.blockDim = dim3(Cfg::kThreads);
  cfg.dynamicSmemBytes = Cfg::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_off ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  const int M32 = (int)g.M, N32 = (int)g.N, K32 = (int)g.K;
  if (g.b_kmajor)
    CK(cudaLaunchKernelEx(&cfg, gemm_cluster_splitk_kernel<64, 64, 32, 16, kClStages, true, CS>, g.mapA, g.mapB, g.C,
                          (int64_t)g.ldc, M32, N32, K32, vec, g.accumulate, g.b_static ? 1 : 0,
                          g_cluster_dbg));
  else
    CK(cudaLaunchKernelEx(&cfg, gemm_cluster_splitk_kernel<64, 64, 32, 16, kClStages, false, CS>, g.mapA, g.mapB, g.C,
                          (int64_t)g.ldc, M32, N32, K32, vec, g.accumulate, g.b_static ? 1 : 0,
                          g_cluster_dbg));
  return HEFF_OK;
}

int launch_gemm(GemmOp& g, int path, cudaStream_t s, int* nlaunch, SplitWs* ws, const ShardedA* sa) {
  if (g.M == 0 || g.N == 0) return HEFF_OK;
  const bool use_tma = sa != nullptr || (path == 2) || (path == 0 && tma_ok(g));
  if (path == 2 && !tma_ok(g)) return set_err(HEFF_EUNSUPPORTED, "TMA GEMM path needs 16-byte rows/alignment");
  const int cs = use_tma ? cluster_splitk_size(g, sa) : 0;
  if (cs == 4) {
    CKR(launch_cluster_splitk<4>(g, s));
  } else if (cs == 2) {
    CKR(launch_cluster_splitk<2>(g, s));
  } else if (use_tma) {
    if (use_small_tile(g, sa))
      CKR((launch_tma<kBMs, kBNs, kWMs, kWNs, kStagesS>(g, s, nlaunch, ws, sa)));
    else
      CKR((launch_tma<kBM, kBN, kWM, kWN, kStages>(g, s, nlaunch, ws, sa)));
  } else {
    dim3 grid((unsigned)((g.N + 63) / 64), (unsigned)((g.M + 63) / 64));
    if (grid.y > 65535) return set_err(HEFF_EUNSUPPORTED, "plain GEMM path: M too large");
    if (g.b_kmajor)
      gemm_dmma_plain_kernel<true><<<grid, 128, 0, s>>>(g.A, g.lda, g.B, g.ldb, g.C, g.ldc, (int)g.M, (int)g.N, (int)g.K,
                                                        g.accumulate);
    else
      gemm_dmma_plain_kernel<false><<<grid, 128, 0, s>>>(g.A, g.lda, g.B, g.ldb, g.C, g.ldc, (int)g.M, (int)g.N,
                                                         (int)g.K, g.accumulate);
  }
  CK(cudaGetLastError());
  if (nlaunch) ++*nlaunch;
  return HEFF_OK;
}

static std::mutex g_init_mu;  // one-time initialisations may race from worker threads
static std::atomic<uint64_t> g_dev_inited{0};  // bit d: device d initialised

int cur_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  return std::min(std::max(dev, 0), kMaxDevices - 1);
}

int init_device_once() {
  int dev;
  CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) return set_err(HEFF_EUNSUPPORTED, "device ordinal %d >= %d", dev, kMaxDevices);
  const uint64_t bit = uint64_t(1) << dev;
  if (g_dev_inited.load(std::memory_order_acquire) & bit) return HEFF_OK;
  std::lock_guard<std::mutex> lock(g_init_mu);
  if (g_dev_inited.load(std::memory_order_acquire) & bit) return HEFF_OK;
  int major = 0, minor = 0;
  CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  CK(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
  if (major != 10 || minor != 0)
    return set_err(HEFF_EUNSUPPORTED, "libheff is built for sm_100a (B200); device is sm_%d%d", major, minor);
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // grids are sized from one SM count: every device of a process must agree (all B200s do)
  if (g_num_sms != 0 && g_num_sms != sms)
    return set_err(HEFF_EUNSUPPORTED, "device %d has %d SMs, an earlier device %d", dev, sms, g_num_sms);
  g_num_sms = sms;
  CK(cudaFuncSetAttribute(gemm_dmma_tma_kernel<kBM, kBN, kWM, kWN, kStages, true>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, CfgNT::kSmemBytes));
  CK(cudaFuncSetAttribute(gemm_dmma_tma_kernel<kBM, kBN, kWM, kWN, kStages, false>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, CfgNN::kSmemBytes));
  CK(cudaFuncSetAttribute(gemm_dmma_tma_sharded_kernel<kBM, kBN, kWM, kWN, kStages, true>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, CfgNT::kSmemBytes));
  CK(cudaFuncSetAttribute(gemm_dmma_tma_kernel<kBMs, kBNs, kWMs, kWNs, kStagesS, true>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, CfgNTs::kSmemBytes));
  CK(cudaFuncSetAttribute(gemm_dmma_tma_kernel<kBMs, kBNs, kWMs, kWNs, kStagesS, false>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, CfgNNs::kSmemBytes));
  CK(cudaFuncSetAttribute(gemm_dmma_tma_sharded_kernel<kBMs, kBNs, kWMs, kWNs, kStagesS, true>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, CfgNTs::kSmemBytes));
  CK(cudaFuncSetAttribute(mpo_apply_kernel<1, 128, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMpoSmemBytes));
  CK(cudaFuncSetAttribute(mpo_apply_kernel<1, 64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMpoSmemBytes));
  CK(cudaFuncSetAttribute(mpo_apply_kernel<1, 32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMpoSmemBytes));
  CK(cudaFuncSetAttribute(mpo_apply_kernel<1, 16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMpoSmemBytes));
  CK(cudaFuncSetAttribute(mpo_apply_kernel<1, 128, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMpoSmemBytes));
  CK(cudaFuncSetAttribute(mpo_apply_kernel<1, 64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMpoSmemBytes));
  CK(cudaFuncSetAttribute(mpo_apply_kernel<1, 32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMpoSmemBytes));
  CK(cudaFuncSetAttribute(mpo_apply_kernel<1, 16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMpoSmemBytes));
  CK(cudaFuncSetAttribute(mpo_apply_kernel<2, 128, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMpoSmemBytes));
  CK(cudaFuncSetAttribute(mpo_apply_kernel<2, 64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMpoSmemBytes));
  CK(cudaFuncSetAttribute(mpo_apply_kernel<2, 32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMpoSmemBytes));
  CK(cudaFuncSetAttribute(mpo_apply_kernel<2, 16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMpoSmemBytes));
  CK(cudaFuncSetAttribute(heff_small_matvec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmallMvMaxSmem));
  CK(cudaFuncSetAttribute(gemm1_mpo_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFusedSmemBytes));
  CK(cudaFuncSetAttribute(matvec_cluster_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMvcSmemBytes));
  CK(cudaFuncSetAttribute(matvec_cluster_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMvcSmemBytes));
  CK(cudaFuncSetAttribute(matvec_cluster_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMvcSmemBytes));
  CK(cudaFuncSetAttribute(gemm_cluster_splitk_kernel<64, 64, 32, 16, kClStages, false, 2>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, CfgCl2::kSmemBytes));
  CK(cudaFuncSetAttribute(gemm_cluster_splitk_kernel<64, 64, 32, 16, kClStages, true, 2>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, CfgCl2::kSmemBytes));
  CK(cudaFuncSetAttribute(gemm_cluster_splitk_kernel<64, 64, 32, 16, kClStages, false, 4>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, CfgCl4::kSmemBytes));
  CK(cudaFuncSetAttribute(gemm_cluster_splitk_kernel<64, 64, 32, 16, kClStages, true, 4>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, CfgCl4::kSmemBytes));
  CK(cudaFuncSetAttribute(cgs2_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  CK(cudaFuncSetAttribute(cgs2_step_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemStepMaxBytes));
  g_dev_inited.fetch_or(bit, std::memory_order_release);
  return HEFF_OK;
}

// ----------------------------------------------------------------------------- plan
struct Csr {
  int nrows = 0, nnz = -1;  // nnz: -1 until read back from d_nnz (heff_get_option)
  int* d_rowptr = nullptr;
  int* d_col = nullptr;
  double* d_val = nullptr;
  int* d_nnz = nullptr;
  bool owned = true;        // false: arena buffers (environment updates)
};

// CSR of the two-site (or, kCsrSingle, one-site) MPO built on the device from the device
// tensors W1/W2 by mpo_csr_build_kernel -- no host copy, no stream synchronisation.
static void csr_shape(int mode, int64_t kL, int64_t kR, int64_t d1, int64_t d2, int64_t* nrows, int64_t* nslots) {
  const int64_t nin = kL * d1 * d2, nout = d1 * d2 * kR;
  switch (mode) {
    case kCsrOrderA: *nrows = nout; *nslots = nin; break;
    case kCsrOrderB: *nrows = nin; *nslots = nout; break;
    case kCsrComplexA: *nrows = 2 * nout; *nslots = 2 * nin; break;
    case kCsrSingle: *nrows = d1 * kR; *nslots = kL * d1; break;
    default: *nrows = kL * d1; *nslots = d1 * kR; break;
  }
}

static int build_csr_dev(Csr& c, int mode, const double* W1, const double* W2, int64_t kL, int64_t kM, int64_t kR,
                         int64_t d1, int64_t d2, cudaStream_t s) {
  int64_t nrows = 0, nslots = 0;
  csr_shape(mode, kL, kR, d1, d2, &nrows, &nslots);
  if (nrows * nslots > INT32_MAX) return set_err(HEFF_EUNSUPPORTED, "MPO CSR: %lld entries", (long long)(nrows * nslots));
  if (c.owned) {
    // (workspace-cache blocks: one plan per DMRG bond reuses the previous plan's CSR blocks)
    CK(ws_malloc(&c.d_rowptr, sizeof(int) * (nrows + 2)));  // + the nnz slot
    CK(ws_malloc(&c.d_col, sizeof(int) * std::max<int64_t>(1, nrows * nslots)));
    CK(ws_malloc(&c.d_val, sizeof(double) * std::max<int64_t>(1, nrows * nslots)));
    c.d_nnz = c.d_rowptr + nrows + 1;
  }
  c.nrows = (int)nrows;
  c.nnz = -1;
  mpo_csr_build_kernel<<<1, kCsrThreads, 0, s>>>(W1, W2, (int)kL, (int)kM, (int)kR, (int)d1, (int)d2, mode, c.d_rowptr,
                                                 c.d_col, c.d_val, c.d_nnz);
  CK(cudaGetLastError());
  return HEFF_OK;
}

static int csr_nnz(Csr& c) {  // synchronous read-back (heff_get_option only)
  if (c.nnz < 0 && c.d_nnz) {
    int v = 0;
    if (cudaMemcpy(&v, c.d_nnz, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    c.nnz = v;
  }
  return c.nnz;
}

// W must be a device (or managed) pointer: checked without touching the stream.
static bool is_device_ptr(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

struct heff_plan_s {
  heff_dims dims{};
  // composite plan (MPO sum): borrowed term plans, applied and summed
  std::vector<heff_plan_s*> terms;
  // complex plans (heff_create_z): planar copies [re, im, -im] of L and R, planar T1/T3
  bool is_complex = false;
  double* Lp = nullptr;
  double* Rp = nullptr;
  double* zin = nullptr;                    // psi planes [2][n]
  double* zout = nullptr;                   // out planes [2][n]
  int64_t t1_plane = 0, t3_plane = 0;
  GemmOp gz1[4], gz4[4];
  // energy penalty: out += weight * sum_i phi_i <phi_i|psi>
  double* phis = nullptr;                   // [nphi][ldv_phi], plan-owned copy
  int nphi = 0;
  int64_t ldv_phi = 0;
  double pen_weight = 0.0;
  double* pen_scratch = nullptr;            // partials [nphi][pen_G] + coefficients [nphi]
  int pen_G = 0;
  const double *L = nullptr, *R = nullptr;  // borrowed
  int tcA = 128, tcB = 128;                 // MPO kernels' column-tile widths (mpo_tile_cols)
  double* Rperm = nullptr;                  // order B: R's shard with rows reordered (w2, b'), plan-owned
  bool sharded = false;                     // order B on a b'-shard
  int nranks = 1, rank = 0;
  int64_t b_lo = 0, b_hi = 0, nb = 0;
  ncclComm_t comm = nullptr;
  // order A workspace (chunked over a')
  int64_t chunk_rows = 0;                   // a' rows per chunk
  double *T1 = nullptr, *T3 = nullptr;
  GemmOp g1, g4;                            // per-chunk ops (A/C pointers advanced per chunk)
  // small bonds: GEMM1 + MPO fused (gemm1_mpo_fused_kernel), fat tiles of TA a' x TB b
  int fusedTA = 0, fusedTB = 0;             // 0: not eligible
  CUtensorMap fmapL, fmapPsi;
  const double* fpsi_ptr = nullptr;
  bool fmapL_ok = false;
  // C2-size chains: the whole matvec in one cluster launch (matvec_cluster_kernel); cluster
  // size mR / fusedTB, 0 = not eligible
  int mvc_cs = 0;
  CUtensorMap fmapR;
  // order B workspace
  double *V1 = nullptr, *V3 = nullptr;
  GemmOp gA, gD;
  Csr csrA, csrB;
  SplitWs splitws{nullptr, 0, nullptr, 0, true};  // stream-K workspace from the plan workspace cache
  // U(1) block-sparse schedules of the two GEMMs (heff_set_qn); one device allocation each
  int* sp1 = nullptr;
  int* sp4 = nullptr;
  int64_t sp_kblocks = 0;  // k-block x tile products scheduled per matvec (both GEMMs)
  unsigned char* mpo_live = nullptr;  // [mL][b-tiles]: MPO blocks that can be nonzero (U(1) plans)
  // U(1) plans: Lanczos keeps only the sector's entries (positions qn_idx into psi)
  int* qn_idx = nullptr;
  int64_t qn_n = 0;
  double* dense_in = nullptr;               // zero outside the sector
  double* dense_out = nullptr;
  // gather-fused sharded Lanczos (NEXT-5): the Krylov basis lives in an NCCL symmetric window;
  // GEMM_A reads every rank's shard of v_j through its NVLink (LSA) pointer, ordered by
  // per-rank flags (signal after v_j is written, wait before the matvec reads it)
  int fused_gather = 0;                     // option HEFF_OPT_FUSED_GATHER
  int fused_active = 0;                     // the last lanczos_ground used the fused path
  ncclWindow_t win = nullptr;
  void* win_buf = nullptr;
  size_t win_bytes = 0;
  int win_cap = 0;
  int64_t win_ldv = 0, win_flag_off = 0;    // flags at byte offset win_flag_off
  std::vector<char*> peer_base;             // LSA pointers of every rank's window (host copy)
  uint64_t** d_peer_flags = nullptr;        // device array [P] of peer flag arrays
  uint64_t epoch = 0;
  // failure handling of communicating plans: waits poll ncclCommGetAsyncError and a
  // no-progress timeout; on error the communicator is aborted and the plan is unusable
  int comm_dead = 0;
  std::string comm_err;
  int force_allgather = 0;                  // option HEFF_OPT_FORCE_ALLGATHER (1 rank: run the P>1 branch)
  std::vector<cudaEvent_t> step_ev;         // recorded after each Lanczos step (progress of a wait)
  double* hpin = nullptr;                   // pinned host scalars of lanczos_ground: device->host
  size_t hpin_n = 0;                        // copies stay asynchronous, so every wait is a poll
  int step_ev_used = 0;
  // e2e staging; the overlapped host path's copy stream and chunk events
  double *stage_in = nullptr, *stage_out = nullptr;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t e2e_ev[17] = {};                // 2 kE2eChunks + 1
  cudaEvent_t done_ev = nullptr;              // recorded after each enqueued plan operation
  cudaEvent_t setup_ev = nullptr;             // end of the device-side set-up heff_create enqueued
  std::vector<cudaStream_t> setup_streams;    // streams already ordered after setup_ev
  // Lanczos
  double* basis = nullptr;                  // [cap][ldv]
  int basis_cap = 0;
  int64_t ldv = 0;
  double* work = nullptr;                   // w (local length)
  int64_t work_len = 0;
  double* full = nullptr;                   // gathered full psi (sharded + comm)
  double* gather = nullptr;                 // blocked gather buffer
  double* partial = nullptr;                // [(cap+1)][ldp]
  int ldp = 0;
  double* scal = nullptr;                   // c1[cap], c2[cap], alpha[cap], beta2/beta[cap], invb[cap], y[cap]
  unsigned int* gbar = nullptr;             // grid barrier of the ordinary-launch CGS2 steps (zeroed once)
  // options
  int gemm_path = 0;
  int last_launches = 0;
  int64_t total_launches = 0;              // every libheff kernel launched on this plan
  int profile = 0;
  std::vector<cudaEvent_t> prof_ev;         // 4 events per recorded (chunk of a) matvec
  size_t prof_used = 0;
};

static int64_t vec_len(const heff_plan_s* p) {  // local vector length
  const heff_dims& d = p->dims;
  return d.mL * d.d1 * d.d2 * (p->sharded ? p->nb : d.mR);
}

extern "C" size_t heff_workspace_bytes(const heff_dims* d, const heff_dist* dist) {
  if (!d) return 0;
  if (dist) {
    const int64_t nb = dist->b_hi - dist->b_lo;
    // V1 + V3 + the (w2, b')-ordered copy of R's shard
    return sizeof(double) * (size_t)(d->mL * d->d1 * d->d2 * nb * d->kR + d->kL * d->mL * d->d1 * d->d2 * nb +
                                     nb * d->kR * d->mR);
  }
  return sizeof(double) * (size_t)(d->mL * (d->kL + d->kR) * d->d1 * d->d2 * d->mR);
}

// ----------------------------------------------------------------------- workspace cache
// Plan workspaces (intermediates, Krylov basis, staging and scatter buffers) are taken
// from and returned to a process-wide cache of device blocks: a DMRG sweep creates and
// destroys one plan per bond, and cudaMalloc/cudaFree of ~GB buffers (cudaFree also
// synchronises the device) cost 5-8 ms per bond at m = 256-1024 against 1-40 ms of
// Lanczos.  A request takes the smallest cached block of the same device with
// bytes <= size <= 2 bytes + 64 MB; heff_destroy waits for the plan's last operation and
// returns its blocks (blocks up to 4 GB are kept, 16 GB in total, the least recently
// released evicted first); heff_release_caches frees them all.
// An allocation that fails frees the cache and retries.
struct WsBlock {
  void* p;
  size_t bytes;
  int dev;
};
static std::mutex g_ws_mu;
static std::vector<WsBlock> g_ws_free;                      // cached, idle
static std::unordered_map<void*, WsBlock> g_ws_live;        // handed out
static size_t g_ws_cached = 0;
constexpr size_t kWsCacheMax = size_t(16) << 30;   // idle bytes kept, all devices
constexpr size_t kWsBlockMax = size_t(4) << 30;    // larger blocks are freed, not cached

static void ws_cache_trim(int dev) {  // caller holds g_ws_mu
  for (size_t i = 0; i < g_ws_free.size();) {
    if (dev < 0 || g_ws_free[i].dev == dev) {
      cudaFree(g_ws_free[i].p);
      g_ws_cached -= g_ws_free[i].bytes;
      g_ws_free[i] = g_ws_free.back();
      g_ws_free.pop_back();
    } else {
      ++i;
    }
  }
}

template <typename T>
static cudaError_t ws_malloc(T** out, size_t bytes) {
  *out = nullptr;
  if (bytes == 0) bytes = 256;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(g_ws_mu);
  int best = -1;
  for (int i = 0; i < (int)g_ws_free.size(); ++i) {
    const WsBlock& b = g_ws_free[i];
    // best fit within 2x (+ 64 MB of slack for large blocks only: a small request must not
    // take a previous plan's large T1/T3 block, which its successor then re-allocates)
    const size_t slack = bytes >= (size_t(8) << 20) ? (size_t(64) << 20) : 0;
    if (b.dev == dev && b.bytes >= bytes && b.bytes <= 2 * bytes + slack &&
        (best < 0 || b.bytes < g_ws_free[best].bytes))
      best = i;
  }
  if (best >= 0) {
    const WsBlock b = g_ws_free[best];
    g_ws_free.erase(g_ws_free.begin() + best);  // keeps the release order (oldest first)
    g_ws_cached -= b.bytes;
    g_ws_live[b.p] = b;
    *out = static_cast<T*>(b.p);
    return cudaSuccess;
  }
  void* ptr = nullptr;
  cudaError_t e = cudaMalloc(&ptr, bytes);
  if (e == cudaErrorMemoryAllocation && !g_ws_free.empty()) {
    cudaGetLastError();
    ws_cache_trim(dev);
    e = cudaMalloc(&ptr, bytes);
  }
  if (e != cudaSuccess) return e;
  g_ws_live[ptr] = WsBlock{ptr, bytes, dev};
  *out = static_cast<T*>(ptr);
  return cudaSuccess;
}

// Return a block to the cache.  The caller guarantees no pending device work uses it.
static void ws_release(void* ptr) {
  if (!ptr) return;
  std::lock_guard<std::mutex> lock(g_ws_mu);
  auto it = g_ws_live.find(ptr);
  if (it == g_ws_live.end()) {  // not a cache block
    cudaFree(ptr);
    return;
  }
  const WsBlock b = it->second;
  g_ws_live.erase(it);
  if (b.bytes > kWsBlockMax) {
    cudaFree(b.p);
    return;
  }
  g_ws_free.push_back(b);
  g_ws_cached += b.bytes;
  while (g_ws_cached > kWsCacheMax) {  // evict the least recently released blocks
    cudaFree(g_ws_free.front().p);
    g_ws_cached -= g_ws_free.front().bytes;
    g_ws_free.erase(g_ws_free.begin());
  }
}

// Pinned host scalars of lanczos_ground (alpha, beta, y, norm): cudaMallocHost / cudaFreeHost
// cost ~1 ms / ~0.4 ms, which made a freshly created plan's first Lanczos call and its
// destruction dominate small bonds (one plan per DMRG bond).  A process-wide pool keeps the
// released blocks (power-of-two sizes >= 4 KB) for the next plan; heff_release_caches frees it.
static std::mutex g_pin_mu;
static std::vector<std::pair<size_t, double*>> g_pin_free;
static cudaError_t pin_alloc(double** out, size_t* bytes_out, size_t need) {
  size_t b = 4096;
  while (b < need) b <<= 1;
  {
    std::lock_guard<std::mutex> lock(g_pin_mu);
    for (size_t i = 0; i < g_pin_free.size(); ++i)
      if (g_pin_free[i].first == b) {
        *out = g_pin_free[i].second;
        *bytes_out = b;
        g_pin_free.erase(g_pin_free.begin() + (long)i);
        return cudaSuccess;
      }
  }
  void* p = nullptr;
  const cudaError_t e = cudaMallocHost(&p, b);
  if (e != cudaSuccess) return e;
  *out = static_cast<double*>(p);
  *bytes_out = b;
  return cudaSuccess;
}
static void pin_release(double* p, size_t bytes) {
  if (!p) return;
  std::lock_guard<std::mutex> lock(g_pin_mu);
  if (g_pin_free.size() < 64) {
    g_pin_free.emplace_back(bytes, p);
    return;
  }
  cudaFreeHost(p);
}
static void pin_trim() {
  std::lock_guard<std::mutex> lock(g_pin_mu);
  for (auto& e : g_pin_free) cudaFreeHost(e.second);
  g_pin_free.clear();
}

// Bytes held idle by the cache on `dev` (counted as available by the workspace budget).
static size_t ws_cached_bytes(int dev) {
  std::lock_guard<std::mutex> lock(g_ws_mu);
  size_t t = 0;
  for (const auto& b : g_ws_free)
    if (b.dev == dev) t += b.bytes;
  return t;
}

static void free_csr(Csr& c) {
  if (c.owned) {  // heff_destroy calls this after the plan's last operation completed
    ws_release(c.d_rowptr);
    ws_release(c.d_col);
    ws_release(c.d_val);
  }
  c = Csr{};
}

// Record the plan's completion event on `s` after an enqueued operation (heff_destroy
// waits for it before handing the plan's blocks back to the workspace cache).
// Order stream s after the plan's device-side set-up (once per stream).
static int after_setup(heff_plan_s* p, cudaStream_t s) {
  if (!p->setup_ev) return HEFF_OK;
  for (cudaStream_t x : p->setup_streams)
    if (x == s) return HEFF_OK;
  CK(cudaStreamWaitEvent(s, p->setup_ev, 0));
  p->setup_streams.push_back(s);
  return HEFF_OK;
}

static int mark_done(heff_plan_s* p, cudaStream_t s) {
  if (!p->done_ev) CK(cudaEventCreateWithFlags(&p->done_ev, cudaEventDisableTiming));
  CK(cudaEventRecord(p->done_ev, s));
  return HEFF_OK;
}

extern "C" int heff_destroy(heff_plan p) {
  if (!p) return HEFF_OK;
  // no kernel of this plan may still use a block handed back to the cache: wait for the
  // plan's last operation (plans are used on one stream at a time), not the whole device
  if (p->comm_dead) {
    // work stuck behind an aborted collective completes (or fails) after ncclCommAbort
    if (p->done_ev) cudaEventSynchronize(p->done_ev);
  } else if (p->done_ev) {
    cudaEventSynchronize(p->done_ev);
  } else {
    cudaDeviceSynchronize();
  }
  if (p->copy_stream) cudaStreamSynchronize(p->copy_stream);
  for (void* b : {(void*)p->T1, (void*)p->T3, (void*)p->V1, (void*)p->V3, (void*)p->stage_in, (void*)p->stage_out,
                  (void*)p->basis, (void*)p->work, (void*)p->full, (void*)p->gather, (void*)p->partial,
                  (void*)p->scal, (void*)p->Lp, (void*)p->Rp, (void*)p->Rperm, (void*)p->zin, (void*)p->zout, (void*)p->dense_in,
                  (void*)p->dense_out, (void*)p->gbar})
    ws_release(b);
  cudaFree(p->mpo_live);
  cudaFree(p->qn_idx);
  ws_release(p->splitws.ptr);  // cache blocks (splitws.cached): the next plan reuses them
  ws_release(p->splitws.sync);
  cudaFree(p->phis); cudaFree(p->pen_scratch);
  cudaFree(p->sp1); cudaFree(p->sp4);
  free_csr(p->csrA);
  free_csr(p->csrB);
  for (auto& e : p->prof_ev) cudaEventDestroy(e);
  for (auto& e : p->e2e_ev)
    if (e) cudaEventDestroy(e);
  if (p->copy_stream) cudaStreamDestroy(p->copy_stream);
  if (p->done_ev) cudaEventDestroy(p->done_ev);
  if (p->setup_ev) {
    cudaEventSynchronize(p->setup_ev);
    cudaEventDestroy(p->setup_ev);
  }
  for (auto& e : p->step_ev) cudaEventDestroy(e);
  pin_release(p->hpin, p->hpin_n * sizeof(double));  // (the plan's stream work is complete here)
  // an aborted communicator (comm == nullptr, comm_dead) is gone with its window handles:
  // only the local allocation is freed (deregistration is collective and would wait for
  // the dead peers)
  if (p->win && p->comm && g_nccl.CommWindowDeregister) g_nccl.CommWindowDeregister(p->comm, p->win);
  if (p->win_buf && g_nccl.MemFree) g_nccl.MemFree(p->win_buf);
  cudaFree(p->d_peer_flags);
  if (p->comm && g_nccl.loaded) g_nccl.CommDestroy(p->comm);
  delete p;
  return HEFF_OK;
}

extern "C" int heff_create(heff_plan* out, const heff_dims* dims, const double* L, const double* W1, const double* W2,
                           const double* R, const heff_dist* dist, heff_stream stream) {
  if (!out || !dims || !L || !W1 || !W2 || !R) return set_err(HEFF_EINVAL, "heff_create: null argument");
  *out = nullptr;
  const heff_dims d = *dims;
  if (d.mL < 1 || d.mR < 1 || d.d1 < 1 || d.d2 < 1 || d.kL < 1 || d.kM < 1 || d.kR < 1)
    return set_err(HEFF_EINVAL, "heff_create: every dimension must be >= 1");
  if (d.kL * d.d1 * d.d2 > kMpoMaxRows || d.d1 * d.d2 * d.kR > kMpoMaxRows)
    return set_err(HEFF_EUNSUPPORTED, "heff_create: k d1 d2 > %d exceeds the MPO kernel's shared-memory tile",
                   kMpoMaxRows);
  for (const void* ptr : {(const void*)L, (const void*)W1, (const void*)W2, (const void*)R})
    if (reinterpret_cast<uintptr_t>(ptr) & 7) return set_err(HEFF_EINVAL, "heff_create: pointers must be 8-byte aligned");
  CKR(init_device_once());
  if (!is_device_ptr(W1) || !is_device_ptr(W2))
    return set_err(HEFF_EINVAL, "heff_create: W1/W2 are not device pointers");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);

  heff_plan_s* p = new heff_plan_s();
  p->dims = d;
  p->L = L;
  p->R = R;
  auto fail = [&](int code) {
    heff_destroy(p);
    return code;
  };
  if (dist) {
    if (dist->nranks < 1 || dist->rank < 0 || dist->rank >= dist->nranks || dist->b_lo < 0 || dist->b_hi > d.mR ||
        dist->b_lo >= dist->b_hi)
      return fail(set_err(HEFF_EINVAL, "heff_create: bad heff_dist (rank %d/%d, b [%lld,%lld))", dist->rank,
                          dist->nranks, (long long)dist->b_lo, (long long)dist->b_hi));
    p->sharded = true;
    p->nranks = dist->nranks;
    p->rank = dist->rank;
    p->b_lo = dist->b_lo;
    p->b_hi = dist->b_hi;
    p->nb = dist->b_hi - dist->b_lo;
    if (dist->nccl_uid) {
      if (d.mR % dist->nranks != 0 || p->nb != d.mR / dist->nranks || p->b_lo != p->rank * p->nb)
        return fail(set_err(HEFF_EINVAL, "heff_create: communicating shards must be equal contiguous blocks of mR"));
      int r = nccl_load();
      if (r) return fail(r);
      ncclUniqueId id;
      memcpy(id.internal, dist->nccl_uid, 128);
      ncclResult_t nr = g_nccl.CommInitRank(&p->comm, dist->nranks, id, dist->rank);
      if (nr != ncclSuccess) return fail(set_err(HEFF_ENCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString(nr)));
      if (const char* e = getenv("HEFF_FUSED_GATHER")) p->fused_gather = atoi(e) ? 1 : 0;
      if (const char* e = getenv("HEFF_FORCE_ALLGATHER")) p->force_allgather = atoi(e) ? 1 : 0;
    }
  }
  // the two-site MPO as CSR, built on the device on `s` (S0; no host copy or sync)
  p->tcA = mpo_tile_cols(d.kL * d.d1 * d.d2);
  p->tcB = mpo_tile_cols(d.d1 * d.d2 * d.kR);
  int r = build_csr_dev(p->csrA, kCsrOrderA, W1, W2, d.kL, d.kM, d.kR, d.d1, d.d2, s);
  if (r) return fail(r);
  if (p->sharded) {
    r = build_csr_dev(p->csrB, kCsrOrderB, W1, W2, d.kL, d.kM, d.kR, d.d1, d.d2, s);
    if (r) return fail(r);
  }

  if (!p->sharded) {
    // order A, chunked over a' so that T1 + T3 fit the workspace budget
    const int64_t per_row = (d.kL + d.kR) * d.d1 * d.d2 * d.mR * 8;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return fail(set_err(HEFF_ECUDA, "cudaMemGetInfo failed"));
    {
      int dev = 0;
      cudaGetDevice(&dev);
      free_b += ws_cached_bytes(dev);  // idle cached blocks are available to this plan
    }
    int64_t budget = (int64_t)(0.45 * (double)free_b);
    if (const char* e = getenv("HEFF_WORKSPACE_MB")) budget = std::atoll(e) * (1ll << 20);
    int64_t rows = std::max<int64_t>(1, std::min<int64_t>(d.mL, budget / per_row));
    // keep chunks balanced
    const int64_t nchunks = (d.mL + rows - 1) / rows;
    rows = (d.mL + nchunks - 1) / nchunks;
    p->chunk_rows = rows;
    if (ws_malloc(&p->T1, sizeof(double) * rows * d.kL * d.d1 * d.d2 * d.mR) != cudaSuccess ||
        ws_malloc(&p->T3, sizeof(double) * rows * d.d1 * d.d2 * d.kR * d.mR) != cudaSuccess)
      return fail(set_err(HEFF_ENOMEM, "heff_create: cannot allocate T1/T3 workspace (%lld a' rows)", (long long)rows));
    // GEMM1: T1[(a' w), (s1 s2 b)] = L[(a' w), a] . psi[a, (s1 s2 b)]   (NN)
    p->g1.N = d.d1 * d.d2 * d.mR;
    p->g1.K = d.mL;
    p->g1.lda = d.mL;
    p->g1.ldb = d.d1 * d.d2 * d.mR;
    p->g1.b_kmajor = false;
    p->g1.ldc = d.d1 * d.d2 * d.mR;
    // GEMM4: out[(a' s1' s2'), b'] = T3[(a' s1' s2'), (w2 b)] . R[b', (w2 b)]^T   (NT)
    p->g4.N = d.mR;
    p->g4.K = d.kR * d.mR;
    p->g4.lda = d.kR * d.mR;
    p->g4.B = R;
    p->g4.ldb = d.kR * d.mR;
    p->g4.b_kmajor = true;
    p->g4.b_static = true;  // R: a borrowed input no kernel of the matvec writes
    p->g4.ldc = d.mR;
    // GEMM1 + MPO fused on fat tiles (gemm_small.cuh): rows = whole a' groups (TA kL = 80),
    // columns = TB b for each (s1 s2) (d1 d2 TB = 128); used up to 2 waves of tiles
    {
      const int64_t dd = d.d1 * d.d2;
      const bool shape_ok = (kFusedBM % d.kL == 0) && (dd & (dd - 1)) == 0 && (kFusedBN / dd) % 16 == 0 &&
                            rows == d.mL && (d.mL % 2 == 0) &&
                            (reinterpret_cast<uintptr_t>(L) & 15) == 0;
      if (shape_ok) {
        const int64_t TA = kFusedBM / d.kL, TB = kFusedBN / dd;
        if (d.mL % TA == 0 && d.mR % TB == 0) {
          const int64_t tiles = (d.mL / TA) * (d.mR / TB);
          // up to 2 waves of fat tiles (measured: C2 and the m = 128 cylinder 1 wave, chain
          // m = 384 1.95 waves 183 -> 165 us, sub-wave m = 64..192 equal or faster (cylinder
          // m = 96 65 -> 54 us); at 3.5 waves the general path is as fast)
          bool use = tiles <= 2 * (int64_t)g_num_sms;
          if (const char* e = getenv("HEFF_FUSED_MATVEC")) use = atoi(e) != 0;
          if (use) {
            p->fusedTA = (int)TA;
            p->fusedTB = (int)TB;
          }
          // one cluster per a' block (matvec_cluster_kernel): 64 GEMM4 rows per a' block, the
          // T3 tile (kR TB columns) in shared memory, CS = mR / TB in {1, 2, 4, 8} CTAs per
          // cluster, one wave of co-resident clusters.  Measured back to back (B200): chain
          // m = 128 39.0 -> 31.9 us, m = 64 25.1 / 25.7 us (equal); C2 (16 clusters of 8) does not
          // fit (15 co-resident) and keeps the two-kernel form
          const int64_t cs = d.mR / TB;
          const int64_t M4 = TA * dd;
          bool mvc = (M4 == 16 || M4 == 32 || M4 == 64) && d.kR * TB * M4 * 8 <= kMvcT3Bytes &&
                     (d.kR * TB) % kGemmBK == 0 && (cs == 1 || cs == 2 || cs == 4 || cs == 8) && cs <= M4 &&
                     tiles <= g_num_sms && (d.kR * d.mR) % 2 == 0 &&
                     (reinterpret_cast<uintptr_t>(R) & 15) == 0 && d.mR <= 2 * kMvcNP &&
                     d.mL / TA <= max_active_mvc_clusters((int)cs);
          if (const char* e = getenv("HEFF_CLUSTER_MATVEC")) mvc = mvc && atoi(e) != 0;
          if (getenv("HEFF_DEBUG_MVC"))
            fprintf(stderr, "cluster matvec: TA %lld TB %lld CS %lld a'-blocks %lld tiles %lld max clusters %d -> %d\n",
                    (long long)TA, (long long)TB, (long long)cs, (long long)(d.mL / TA), (long long)tiles,
                    (cs >= 1 && cs <= 8) ? max_active_mvc_clusters((int)cs) : -1, (int)mvc);
          if (mvc) {
            const int r = make_map(&p->fmapR, R, d.mR, d.kR * d.mR, d.kR * d.mR, kGemmBK, kMvcNP);
            if (r) return fail(r);
            p->fusedTA = (int)TA;
            p->fusedTB = (int)TB;
            p->mvc_cs = (int)cs;
          }
        }
      }
    }
  } else {
    const int64_t nb = p->nb;
    if (ws_malloc(&p->V1, sizeof(double) * d.mL * d.d1 * d.d2 * nb * d.kR) != cudaSuccess ||
        ws_malloc(&p->V3, sizeof(double) * d.kL * d.mL * d.d1 * d.d2 * nb) != cudaSuccess ||
        ws_malloc(&p->Rperm, sizeof(double) * nb * d.kR * d.mR) != cudaSuccess)
      return fail(set_err(HEFF_ENOMEM, "heff_create: cannot allocate V1/V3 workspace"));
    // R's shard with rows (w2, b') (a plan-owned copy; R stays borrowed and unmodified)
    permute_r_shard_kernel<<<(unsigned)(nb * d.kR), 256, 0, s>>>(R, p->Rperm, nb, (int)d.kR, d.mR);
    if (cudaGetLastError() != cudaSuccess) return fail(set_err(HEFF_ECUDA, "heff_create: R permutation launch failed"));
    // GEMM_A: V1[(a s1 s2), (w2 b')] = psi[(a s1 s2), b] . Rperm[(w2 b'), b]^T   (NT)
    p->gA.M = d.mL * d.d1 * d.d2;
    p->gA.N = nb * d.kR;
    p->gA.K = d.mR;
    p->gA.lda = d.mR;
    p->gA.B = p->Rperm;
    p->gA.ldb = d.mR;
    p->gA.b_kmajor = true;
    p->gA.C = p->V1;
    p->gA.ldc = nb * d.kR;
    // GEMM_D: out_g[a', (s1' s2' b')] = L[a', (w a)] . V3[(w a), (s1' s2' b')]   (NN)
    p->gD.M = d.mL;
    p->gD.N = d.d1 * d.d2 * nb;
    p->gD.K = d.kL * d.mL;
    p->gD.A = L;
    p->gD.lda = d.kL * d.mL;
    p->gD.B = p->V3;
    p->gD.ldb = d.d1 * d.d2 * nb;
    p->gD.b_kmajor = false;
    p->gD.ldc = d.d1 * d.d2 * nb;
  }
  // the CSR / R permutation kernels ran on s: later calls on other streams wait for them
  if (cudaEventCreateWithFlags(&p->setup_ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventRecord(p->setup_ev, s) != cudaSuccess)
    return fail(set_err(HEFF_ECUDA, "heff_create: event record failed"));
  p->setup_streams.push_back(s);
  *out = p;
  return HEFF_OK;
}

// --------------------------------------------------------------------------- complex plans
// NEXT-4: ITensor's Dense{ComplexF64} + zgemm.  (D) has no
// conjugation; each complex GEMM is four real DMMA GEMMs on planar copies (the negated
// imaginary planes of L and R turn the subtraction into an accumulating GEMM) and the two
// MPO steps run as one real MPO kernel on stacked [re; im] rows with the 2x2 blocks
// [[Re, -Im], [Im, Re]] of the complex two-site MPO.
extern "C" int heff_create_z(heff_plan* out, const heff_dims* dims, const double* L, const double* W1,
                             const double* W2, const double* R, const heff_dist* dist, heff_stream stream) {
  if (!out || !dims || !L || !W1 || !W2 || !R) return set_err(HEFF_EINVAL, "heff_create_z: null argument");
  *out = nullptr;
  if (dist) return set_err(HEFF_EUNSUPPORTED, "heff_create_z: complex plans are single-GPU");
  const heff_dims d = *dims;
  if (d.mL < 1 || d.mR < 1 || d.d1 < 1 || d.d2 < 1 || d.kL < 1 || d.kM < 1 || d.kR < 1)
    return set_err(HEFF_EINVAL, "heff_create_z: every dimension must be >= 1");
  if (2 * d.kL * d.d1 * d.d2 > kMpoMaxRows || 2 * d.d1 * d.d2 * d.kR > kMpoMaxRows)
    return set_err(HEFF_EUNSUPPORTED, "heff_create_z: 2 k d1 d2 > %d exceeds the MPO kernel's tile", kMpoMaxRows);
  for (const void* ptr : {(const void*)L, (const void*)W1, (const void*)W2, (const void*)R})
    if (reinterpret_cast<uintptr_t>(ptr) & 15)
      return set_err(HEFF_EINVAL, "heff_create_z: complex pointers must be 16-byte aligned");
  CKR(init_device_once());
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  heff_plan_s* p = new heff_plan_s();
  p->dims = d;
  p->is_complex = true;
  auto fail = [&](int code) {
    heff_destroy(p);
    return code;
  };
  if (!is_device_ptr(W1) || !is_device_ptr(W2)) return fail(set_err(HEFF_EINVAL, "heff_create_z: W1/W2 are not device pointers"));
  p->tcA = mpo_tile_cols(2 * d.kL * d.d1 * d.d2);
  int r = build_csr_dev(p->csrA, kCsrComplexA, W1, W2, d.kL, d.kM, d.kR, d.d1, d.d2, s);
  if (r) return fail(r);
  const int64_t nL = d.mL * d.kL * d.mL, nR = d.mR * d.kR * d.mR, n = d.mL * d.d1 * d.d2 * d.mR;
  if (ws_malloc(&p->Lp, sizeof(double) * 3 * nL) != cudaSuccess ||
      ws_malloc(&p->Rp, sizeof(double) * 3 * nR) != cudaSuccess ||
      ws_malloc(&p->zin, sizeof(double) * 2 * n) != cudaSuccess ||
      ws_malloc(&p->zout, sizeof(double) * 2 * n) != cudaSuccess)
    return fail(set_err(HEFF_ENOMEM, "heff_create_z: cannot allocate planar copies"));
  deinterleave_kernel<<<ew_grid(2 * nL), 256, 0, s>>>(L, p->Lp, p->Lp + nL, nL);
  negate_kernel<<<ew_grid(2 * nL), 256, 0, s>>>(p->Lp + nL, p->Lp + 2 * nL, nL);
  deinterleave_kernel<<<ew_grid(2 * nR), 256, 0, s>>>(R, p->Rp, p->Rp + nR, nR);
  negate_kernel<<<ew_grid(2 * nR), 256, 0, s>>>(p->Rp + nR, p->Rp + 2 * nR, nR);
  if (cudaGetLastError() != cudaSuccess) return fail(set_err(HEFF_ECUDA, "heff_create_z: launch failed"));
  // workspace: planar T1, T3, chunked over a'
  const int64_t per_row = 2 * (d.kL + d.kR) * d.d1 * d.d2 * d.mR * 8;
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return fail(set_err(HEFF_ECUDA, "cudaMemGetInfo failed"));
  int64_t budget = (int64_t)(0.45 * (double)free_b);
  if (const char* e = getenv("HEFF_WORKSPACE_MB")) budget = std::atoll(e) * (1ll << 20);
  int64_t rows = std::max<int64_t>(1, std::min<int64_t>(d.mL, budget / per_row));
  const int64_t nchunks = (d.mL + rows - 1) / rows;
  rows = (d.mL + nchunks - 1) / nchunks;
  p->chunk_rows = rows;
  p->t1_plane = rows * d.kL * d.d1 * d.d2 * d.mR;
  p->t3_plane = rows * d.d1 * d.d2 * d.kR * d.mR;
  if (ws_malloc(&p->T1, sizeof(double) * 2 * p->t1_plane) != cudaSuccess ||
      ws_malloc(&p->T3, sizeof(double) * 2 * p->t3_plane) != cudaSuccess)
    return fail(set_err(HEFF_ENOMEM, "heff_create_z: cannot allocate T1/T3 workspace"));
  for (int k = 0; k < 4; ++k) {
    GemmOp& g1 = p->gz1[k];
    g1.N = d.d1 * d.d2 * d.mR; g1.K = d.mL; g1.lda = d.mL; g1.ldb = g1.N; g1.b_kmajor = false; g1.ldc = g1.N;
    GemmOp& g4 = p->gz4[k];
    g4.N = d.mR; g4.K = d.kR * d.mR; g4.lda = g4.K; g4.ldb = g4.K; g4.b_kmajor = true; g4.ldc = d.mR;
  }
  p->L = p->Lp;
  p->R = p->Rp;
  if (cudaEventCreateWithFlags(&p->setup_ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventRecord(p->setup_ev, s) != cudaSuccess)
    return fail(set_err(HEFF_ECUDA, "heff_create_z: event record failed"));
  p->setup_streams.push_back(s);
  *out = p;
  return HEFF_OK;
}

struct LanczosLayout {  // see lanczos_workspace
  bool compact, cplx, fgather;
  int64_t n_dense, n, nr, ldv;
};
static int lanczos_workspace(heff_plan_s* p, int cap, cudaStream_t s, LanczosLayout* out);

extern "C" int heff_set_option(heff_plan p, int option, int64_t value) {
  if (!p) return set_err(HEFF_EINVAL, "null plan");
  switch (option) {
    case HEFF_OPT_GEMM_PATH:
      if (value < 0 || value > 2) return set_err(HEFF_EINVAL, "gemm path must be 0, 1 or 2");
      p->gemm_path = (int)value;
      return HEFF_OK;
    case HEFF_OPT_PROFILE:
      p->profile = value ? 1 : 0;
      p->prof_used = 0;
      return HEFF_OK;
    case HEFF_OPT_TOTAL_LAUNCHES:
      p->total_launches = value;
      return HEFF_OK;
    case HEFF_OPT_FUSED_GATHER:
      if (value && !(p->sharded && p->comm))
        return set_err(HEFF_EUNSUPPORTED, "fused gather: communicating b'-sharded plans only");
      p->fused_gather = value ? 1 : 0;
      return HEFF_OK;
    case HEFF_OPT_FORCE_ALLGATHER:
      if (value && !(p->sharded && p->comm))
        return set_err(HEFF_EUNSUPPORTED, "force all-gather: communicating b'-sharded plans only");
      p->force_allgather = value ? 1 : 0;
      return HEFF_OK;
    case HEFF_OPT_LANCZOS_RESERVE: {
      if (value < 1 || value > 100000) return set_err(HEFF_EINVAL, "lanczos reserve: 1 <= iterations <= 100000");
      LanczosLayout lay;
      const int r = lanczos_workspace(p, (int)value, nullptr, &lay);
      if (r != HEFF_OK) return r;
      CK(cudaDeviceSynchronize());
      return HEFF_OK;
    }
    default:
      return set_err(HEFF_EINVAL, "unknown option %d", option);
  }
}

extern "C" int heff_get_option(heff_plan p, int option, int64_t* value) {
  if (!p || !value) return set_err(HEFF_EINVAL, "null argument");
  switch (option) {
    case HEFF_OPT_GEMM_PATH: *value = p->gemm_path; return HEFF_OK;
    case HEFF_OPT_LAST_KERNEL_COUNT: *value = p->last_launches; return HEFF_OK;
    case HEFF_OPT_MPO_NNZ: *value = csr_nnz(p->sharded ? p->csrB : p->csrA); return HEFF_OK;
    case HEFF_OPT_PROFILE: *value = p->profile; return HEFF_OK;
    case HEFF_OPT_TOTAL_LAUNCHES: *value = p->total_launches; return HEFF_OK;
    case HEFF_OPT_SPARSE_KBLOCKS: *value = p->sp_kblocks; return HEFF_OK;
    case HEFF_OPT_FUSED_GATHER: *value = p->fused_gather + 2 * p->fused_active; return HEFF_OK;
    case HEFF_OPT_FORCE_ALLGATHER: *value = p->force_allgather; return HEFF_OK;
    case HEFF_OPT_COMM_STATE: *value = p->comm ? 1 : (p->comm_dead ? -1 : 0); return HEFF_OK;
    default: return set_err(HEFF_EINVAL, "unknown option %d", option);
  }
}

// profiling: 4 events around (GEMM first, MPO, GEMM last) per recorded matvec chunk;
// no host synchronisation until heff_last_timings collects and resets them.
static int prof_mark(heff_plan_s* p, int k, cudaStream_t s) {
  if (!p->profile) return HEFF_OK;
  const size_t idx = p->prof_used * 4 + k;
  while (p->prof_ev.size() <= idx) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    p->prof_ev.push_back(e);
  }
  CK(cudaEventRecord(p->prof_ev[idx], s));
  if (k == 3) ++p->prof_used;
  return HEFF_OK;
}

extern "C" int heff_last_timings(heff_plan p, float* g1, float* mpo, float* g4, float* other) {
  if (!p) return set_err(HEFF_EINVAL, "null plan");
  float a = 0, b = 0, c = 0;
  for (size_t i = 0; i < p->prof_used; ++i) {
    cudaEvent_t* e = &p->prof_ev[i * 4];
    CK(cudaEventSynchronize(e[3]));
    float x;
    CK(cudaEventElapsedTime(&x, e[0], e[1])); a += x;
    CK(cudaEventElapsedTime(&x, e[1], e[2])); b += x;
    CK(cudaEventElapsedTime(&x, e[2], e[3])); c += x;
  }
  if (g1) *g1 = a;
  if (mpo) *mpo = b;
  if (g4) *g4 = c;
  if (other) *other = (float)p->prof_used;
  p->prof_used = 0;
  return HEFF_OK;
}

// One MPO application (mpo_apply_kernel; column tile `tc` from mpo_tile_cols): `nblk`
// blocks along y (a' for order A / environments, a for order B).
template <int PL, bool GR>
static int launch_mpo(const MpoIO& io, int tc, int64_t nblk, const Csr& csr, const unsigned char* live, cudaStream_t s) {
  if (nblk <= 0 || io.ncol <= 0) return HEFF_OK;
  if (nblk > 65535) return set_err(HEFF_EUNSUPPORTED, "MPO kernel: %lld blocks along y", (long long)nblk);
  dim3 grid((unsigned)((io.ncol + tc - 1) / tc), (unsigned)nblk);
  const size_t smem = sizeof(double) * (size_t)io.nin * tc;
  const int* rp = csr.d_rowptr;
  const int* cl = csr.d_col;
  const double* vl = csr.d_val;
  switch (tc) {
    case 128: CK(launch_pdl(mpo_apply_kernel<PL, 128, GR>, grid, dim3(kMpoThreads), smem, s, io, rp, cl, vl, live)); break;
    case 64: CK(launch_pdl(mpo_apply_kernel<PL, 64, GR>, grid, dim3(kMpoThreads), smem, s, io, rp, cl, vl, live)); break;
    case 32: CK(launch_pdl(mpo_apply_kernel<PL, 32, GR>, grid, dim3(kMpoThreads), smem, s, io, rp, cl, vl, live)); break;
    case 16: CK(launch_pdl(mpo_apply_kernel<PL, 16, GR>, grid, dim3(kMpoThreads), smem, s, io, rp, cl, vl, live)); break;
    default: return set_err(HEFF_EUNSUPPORTED, "MPO kernel: %d input rows exceed the shared-memory tile", io.nin);
  }
  return HEFF_OK;
}

// Order A (and the environment updates): `rows` blocks of nin rows (w,s1,s2) x ncol columns
// -> nout rows (s1',s2',w2), both with row pitch ncol.
static MpoIO mpo_io_A(const double* in, double* out, int64_t ncol, int nin, int nout) {
  MpoIO io{};
  io.in = in;
  io.out = out;
  io.ncol = ncol;
  io.nin = nin;
  io.nout = nout;
  io.in_blk = (int64_t)nin * ncol;
  io.in_row = ncol;
  io.out_blk = (int64_t)nout * ncol;
  io.out_row = ncol;
  io.out_grp = nout;
  return io;
}

static int launch_mpo_A(const double* T1, double* T3, int64_t mR, int64_t rows, int nin, int nout, const Csr& csr,
                        const unsigned char* live, int tc, cudaStream_t s) {
  return launch_mpo<1, false>(mpo_io_A(T1, T3, mR, nin, nout), tc, rows, csr, live, s);
}

// --------------------------------------------------------------------------- the matvec
// shared memory of heff_small_matvec_kernel for these dims (0 if it does not apply)
static size_t small_matvec_smem(const heff_plan_s* p) {
  const heff_dims& d = p->dims;
  const int64_t dd = d.d1 * d.d2;
  const int64_t n = d.mL * dd * d.mR + d.mR * d.kR * d.mR + d.kL * d.mL + (d.kL * dd + dd * d.kR) * d.mR;
  const size_t bytes = sizeof(double) * (size_t)n;
  // FMAs per CTA (one output row a'): the L.psi row and the .R^T row; above ~48k the
  // 256-thread CTA loses to the DMMA path (measured: chain m <= 32 and cylinder m = 16 win,
  // cylinder m = 24 at 92k loses 41 vs 32 us)
  const int64_t work = d.kL * dd * d.mR * d.mL + dd * d.mR * d.kR * d.mR;
  return (bytes <= (size_t)kSmallMvMaxSmem && work <= 48 * 1024) ? bytes : 0;
}

static int apply_orderA(heff_plan_s* p, const double* psi, double* out, cudaStream_t s, int* nl, int accumulate) {
  const heff_dims& d = p->dims;
  const int64_t nin = d.kL * d.d1 * d.d2, nout = d.d1 * d.d2 * d.kR;
  // small bonds: the whole matvec in one launch (not with kernel profiling, which times the
  // GEMM / MPO steps separately; HEFF_NO_SMALL_MATVEC=1 disables)
  if (!p->profile && p->sp1 == nullptr && p->sp4 == nullptr && p->gemm_path == 0 && p->chunk_rows == d.mL) {
    static const bool off = getenv("HEFF_NO_SMALL_MATVEC") != nullptr;
    const size_t smem = off ? 0 : small_matvec_smem(p);
    if (smem > 0) {
      CK(launch_pdl(heff_small_matvec_kernel, dim3((unsigned)d.mL), dim3(kSmallMvThreads), smem, s, p->L, psi, p->R,
                    out, (int)d.mL, (int)(d.d1 * d.d2), (int)d.mR, (int)d.kL, (int)d.kR,
                    (const int*)p->csrA.d_rowptr, (const int*)p->csrA.d_col, (const double*)p->csrA.d_val,
                    accumulate));
      ++*nl;
      return HEFF_OK;
    }
  }
  if (p->fusedTA > 0 && p->sp1 == nullptr && p->sp4 == nullptr && p->gemm_path == 0 &&
      (reinterpret_cast<uintptr_t>(psi) & 15) == 0) {
    // GEMM1 + two-site MPO in one kernel (T1 never written), then GEMM4
    const int64_t dd = d.d1 * d.d2;
    if (!p->fmapL_ok) {
      CKR(make_map(&p->fmapL, p->L, d.mL * d.kL, d.mL, d.mL, kGemmBK, kFusedBM));
      p->fmapL_ok = true;
    }
    if (p->fpsi_ptr != psi) {
      CKR(make_map(&p->fmapPsi, psi, d.mL, dd * d.mR, dd * d.mR, 16, kGemmBK));
      p->fpsi_ptr = psi;
    }
    const int tiles = (int)((d.mL / p->fusedTA) * (d.mR / p->fusedTB));
    if (p->mvc_cs > 0) {
      // the whole matvec: one cluster of mR / TB CTAs per a' block
      static const bool pdl_off = getenv("HEFF_NO_PDL") != nullptr;
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3((unsigned)tiles);
      cfg.blockDim = dim3(kFusedThreads);
      cfg.dynamicSmemBytes = kMvcSmemBytes;
      cfg.stream = s;
      cudaLaunchAttribute attr[2];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = (unsigned)p->mvc_cs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[1].val.programmaticStreamSerializationAllowed = pdl_off ? 0 : 1;
      cfg.attrs = attr;
      cfg.numAttrs = 2;
      CKR(prof_mark(p, 0, s));
      const int M4 = p->fusedTA * (int)dd;
      auto kern = M4 == 64 ? matvec_cluster_kernel<64> : (M4 == 32 ? matvec_cluster_kernel<32> : matvec_cluster_kernel<16>);
      CK(cudaLaunchKernelEx(&cfg, kern, p->fmapL, p->fmapPsi, p->fmapR, out, (int)d.mL, (int)d.mR, (int)d.kL, (int)d.kR,
                            (int)dd, (int)__builtin_ctz((unsigned)dd), p->fusedTA, p->fusedTB, (int)(dd * d.kR),
                            (const int*)p->csrA.d_rowptr, (const int*)p->csrA.d_col, (const double*)p->csrA.d_val,
                            accumulate, g_fused_dbg));
      ++*nl;
      CKR(prof_mark(p, 1, s));
      CKR(prof_mark(p, 2, s));
      CKR(prof_mark(p, 3, s));
      return HEFF_OK;
    }
    CKR(prof_mark(p, 0, s));
    CK(launch_pdl(gemm1_mpo_fused_kernel, dim3((unsigned)std::min(tiles, g_num_sms)), dim3(kFusedThreads),
                  kFusedSmemBytes, s, p->fmapL, p->fmapPsi, p->T3, (int)d.mL, (int)d.mR, (int)d.kL, (int)dd,
                  __builtin_ctz((unsigned)dd), p->fusedTA, p->fusedTB, (int)(dd * d.kR), (const int*)p->csrA.d_rowptr,
                  (const int*)p->csrA.d_col, (const double*)p->csrA.d_val, g_fused_dbg, g_fused_dbg_mode));
    ++*nl;
    CKR(prof_mark(p, 1, s));
    CKR(prof_mark(p, 2, s));
    p->g4.M = d.mL * dd;
    p->g4.A = p->T3;
    p->g4.C = out;
    p->g4.accumulate = accumulate;
    CKR(launch_gemm(p->g4, p->gemm_path, s, nl, &p->splitws));
    CKR(prof_mark(p, 3, s));
    return HEFF_OK;
  }
  for (int64_t a0 = 0; a0 < d.mL; a0 += p->chunk_rows) {
    const int64_t rows = std::min(p->chunk_rows, d.mL - a0);
    CKR(prof_mark(p, 0, s));
    p->g1.M = rows * d.kL;
    p->g1.A = p->L + a0 * d.kL * d.mL;
    p->g1.B = psi;
    p->g1.C = p->T1;
    CKR(launch_gemm(p->g1, p->gemm_path, s, nl, &p->splitws));
    CKR(prof_mark(p, 1, s));
    CKR(launch_mpo_A(p->T1, p->T3, d.mR, rows, (int)nin, (int)nout, p->csrA, p->mpo_live, p->tcA, s));
    ++*nl;
    CKR(prof_mark(p, 2, s));
    p->g4.M = rows * d.d1 * d.d2;
    p->g4.A = p->T3;
    p->g4.C = out + a0 * d.d1 * d.d2 * d.mR;
    p->g4.accumulate = accumulate;
    CKR(launch_gemm(p->g4, p->gemm_path, s, nl, &p->splitws));
    CKR(prof_mark(p, 3, s));
  }
  return HEFF_OK;
}

// Gather-fused GEMM_A (NEXT-5): psi given as P shards [rows][nb] (row pitch nb) at
// shards[0..P) -- local buffers, or peer GPUs' buffers through NCCL symmetric-window
// pointers -- read directly by the GEMM's TMA producer: no all-gather copy, no relayout.
static int build_sharded_a(heff_plan_s* p, const double* const* shards, int P, ShardedA* sa) {
  const heff_dims& d = p->dims;
  const int64_t rows = d.mL * d.d1 * d.d2;
  if (P < 1 || P > kMaxShards) return set_err(HEFF_EUNSUPPORTED, "sharded GEMM_A: 1..%d shards", kMaxShards);
  if (p->nb % kGemmBK != 0 || (int64_t)P * p->nb != d.mR)
    return set_err(HEFF_EUNSUPPORTED, "sharded GEMM_A: shard width nb = %lld must be a multiple of %d and P nb = mR",
                   (long long)p->nb, kGemmBK);
  for (int q = 0; q < P; ++q) {
    if (reinterpret_cast<uintptr_t>(shards[q]) & 15) return set_err(HEFF_EINVAL, "sharded GEMM_A: 16-byte alignment");
    CKR(make_map(&sa->map[q], shards[q], rows, p->nb, p->nb, kGemmBK, kBM));
  }
  sa->nsh = P;
  sa->ksh = (int)p->nb;
  return HEFF_OK;
}

static int apply_orderB(heff_plan_s* p, const double* psi, double* out, cudaStream_t s, int* nl, int accumulate,
                        const ShardedA* sa = nullptr) {
  const heff_dims& d = p->dims;
  const int dd = (int)(d.d1 * d.d2);
  CKR(prof_mark(p, 0, s));
  p->gA.A = psi;
  CKR(launch_gemm(p->gA, p->gemm_path, s, nl, &p->splitws, sa));
  CKR(prof_mark(p, 1, s));
  {  // V1[a][(s1 s2 w2)][b'] -> V3[w][a][(s1' s2')][b']
    MpoIO io{};
    io.in = p->V1;
    io.out = p->V3;
    io.ncol = p->nb;
    io.nin = dd * (int)d.kR;
    io.nout = (int)d.kL * dd;
    io.in_blk = (int64_t)dd * d.kR * p->nb;
    io.in_row = p->nb;
    io.out_blk = (int64_t)dd * p->nb;
    io.out_row = p->nb;
    io.out_grp = dd;
    io.out_grp_stride = d.mL * dd * p->nb;
    CKR((launch_mpo<1, true>(io, p->tcB, d.mL, p->csrB, nullptr, s)));
  }
  ++*nl;
  CKR(prof_mark(p, 2, s));
  p->gD.C = out;
  p->gD.accumulate = accumulate;
  CKR(launch_gemm(p->gD, p->gemm_path, s, nl, &p->splitws));
  CKR(prof_mark(p, 3, s));
  return HEFF_OK;
}

static int64_t vec_len(const heff_plan_s* p);
static int apply_orderA_z(heff_plan_s* p, const double* psi, double* out, cudaStream_t s, int* nl) {
  const heff_dims& d = p->dims;
  const int64_t n = d.mL * d.d1 * d.d2 * d.mR, nL = d.mL * d.kL * d.mL, nR = d.mR * d.kR * d.mR;
  const double *pre = p->zin, *pim = p->zin + n;
  deinterleave_kernel<<<ew_grid(2 * n), 256, 0, s>>>(psi, p->zin, p->zin + n, n);
  ++*nl;
  const int64_t nin = 2 * d.kL * d.d1 * d.d2, nout = 2 * d.d1 * d.d2 * d.kR;
  for (int64_t a0 = 0; a0 < d.mL; a0 += p->chunk_rows) {
    const int64_t rows = std::min(p->chunk_rows, d.mL - a0);
    CKR(prof_mark(p, 0, s));
    const int64_t lo = a0 * d.kL * d.mL;
    const double* Lre = p->Lp + lo;
    const double* Lim = p->Lp + nL + lo;
    const double* Lneg = p->Lp + 2 * nL + lo;
    double* T1re = p->T1;
    double* T1im = p->T1 + p->t1_plane;
    // T1re = Lre.psi_re - Lim.psi_im ; T1im = Lre.psi_im + Lim.psi_re
    const double* A1[4] = {Lre, Lneg, Lre, Lim};
    const double* B1[4] = {pre, pim, pim, pre};
    double* C1[4] = {T1re, T1re, T1im, T1im};
    for (int k = 0; k < 4; ++k) {
      GemmOp& g = p->gz1[k];
      g.M = rows * d.kL; g.A = A1[k]; g.B = B1[k]; g.C = C1[k]; g.accumulate = k & 1;
      CKR(launch_gemm(g, p->gemm_path, s, nl, &p->splitws));
    }
    CKR(prof_mark(p, 1, s));
    {  // stacked [re; im] planes of T1 -> T3
      MpoIO io = mpo_io_A(p->T1, p->T3, d.mR, (int)nin, (int)nout);
      io.in_blk = nin / 2 * d.mR;
      io.in_plane = p->t1_plane;
      io.out_blk = nout / 2 * d.mR;
      io.out_plane = p->t3_plane;
      io.out_grp = (int)(nout / 2);
      CKR((launch_mpo<2, false>(io, p->tcA, rows, p->csrA, nullptr, s)));
    }
    ++*nl;
    CKR(prof_mark(p, 2, s));
    const double *T3re = p->T3, *T3im = p->T3 + p->t3_plane;
    const double *Rre = p->Rp, *Rim = p->Rp + nR, *Rneg = p->Rp + 2 * nR;
    double* ore = p->zout + a0 * d.d1 * d.d2 * d.mR;
    double* oim = p->zout + n + a0 * d.d1 * d.d2 * d.mR;
    // out_re = T3re.Rre^T - T3im.Rim^T ; out_im = T3re.Rim^T + T3im.Rre^T
    const double* A4[4] = {T3re, T3im, T3re, T3im};
    const double* B4[4] = {Rre, Rneg, Rim, Rre};
    double* C4[4] = {ore, ore, oim, oim};
    for (int k = 0; k < 4; ++k) {
      GemmOp& g = p->gz4[k];
      g.M = rows * d.d1 * d.d2; g.A = A4[k]; g.B = B4[k]; g.C = C4[k]; g.accumulate = k & 1;
      CKR(launch_gemm(g, p->gemm_path, s, nl, &p->splitws));
    }
    CKR(prof_mark(p, 3, s));
  }
  interleave_kernel<<<ew_grid(2 * n), 256, 0, s>>>(p->zout, p->zout + n, out, n);
  ++*nl;
  CK(cudaGetLastError());
  return HEFF_OK;
}



// out += weight * Phi (Phi^T psi): the excited-state energy penalty
static int apply_penalty(heff_plan_s* p, const double* psi, double* out, cudaStream_t s, int* nl) {
  const int64_t n = vec_len(p);
  const int G = p->pen_G;
  double* part = p->pen_scratch;
  double* c = part + (size_t)p->nphi * G;
  for (int q0 = 0; q0 < p->nphi; q0 += kDotQ) {
    const int qn = std::min(kDotQ, p->nphi - q0);
    // psi (caller's buffer, maybe only 8-byte aligned) is the single "w" vector read by the scalar tail
    multidot_partial_kernel<<<G, kRedThreads, 0, s>>>(p->phis + q0 * p->ldv_phi, p->ldv_phi, qn, psi, n,
                                                      part + q0 * G, G);
    ++*nl;
  }
  reduce_partial_kernel<<<p->nphi, kRedThreads, 0, s>>>(part, G, G, c, 0, nullptr);
  ++*nl;
  for (int q0 = 0; q0 < p->nphi; q0 += 64) {
    multiaxpy_kernel<<<ew_grid(n), 256, 0, s>>>(p->phis + q0 * p->ldv_phi, p->ldv_phi, std::min(64, p->nphi - q0),
                                                c + q0, p->pen_weight, out, n);
    ++*nl;
  }
  CK(cudaGetLastError());
  return HEFF_OK;
}

static int apply_impl(heff_plan_s* p, const double* psi, double* out, cudaStream_t s, int accumulate = 0) {
  if (!psi || !out) return set_err(HEFF_EINVAL, "heff_apply: null psi/out");
  if (psi == out) return set_err(HEFF_EINVAL, "heff_apply: out must not alias psi");
  if ((reinterpret_cast<uintptr_t>(psi) | reinterpret_cast<uintptr_t>(out)) & 7)
    return set_err(HEFF_EINVAL, "heff_apply: psi/out must be 8-byte aligned");
  CKR(after_setup(p, s));
  int nl = 0;
  int r = HEFF_OK;
  if (!p->terms.empty()) {
    for (size_t t = 0; t < p->terms.size() && r == HEFF_OK; ++t) {
      r = apply_impl(p->terms[t], psi, out, s, (t > 0 || accumulate) ? 1 : 0);
      nl += p->terms[t]->last_launches;
    }
  } else if (p->is_complex) {
    if (accumulate) return set_err(HEFF_EUNSUPPORTED, "complex plans cannot be terms of a sum");
    if ((reinterpret_cast<uintptr_t>(psi) | reinterpret_cast<uintptr_t>(out)) & 15)
      return set_err(HEFF_EINVAL, "heff_apply: complex psi/out must be 16-byte aligned");
    r = apply_orderA_z(p, psi, out, s, &nl);
  } else {
    r = p->sharded ? apply_orderB(p, psi, out, s, &nl, accumulate) : apply_orderA(p, psi, out, s, &nl, accumulate);
  }
  if (r == HEFF_OK && p->nphi > 0) r = apply_penalty(p, psi, out, s, &nl);
  p->last_launches = nl;
  p->total_launches += nl;
  return r;
}

extern "C" int heff_create_sum(heff_plan* out, const heff_plan* terms, int nterms) {
  if (!out || !terms || nterms < 1) return set_err(HEFF_EINVAL, "heff_create_sum: need >= 1 term plan");
  *out = nullptr;
  const heff_dims& d0 = terms[0]->dims;
  for (int t = 0; t < nterms; ++t) {
    const heff_plan_s* q = terms[t];
    if (!q) return set_err(HEFF_EINVAL, "heff_create_sum: null term");
    if (q->sharded || q->comm || !q->terms.empty() || q->is_complex)
      return set_err(HEFF_EUNSUPPORTED, "heff_create_sum: terms must be single-GPU, real, non-composite plans");
    if (q->dims.mL != d0.mL || q->dims.mR != d0.mR || q->dims.d1 != d0.d1 || q->dims.d2 != d0.d2)
      return set_err(HEFF_EINVAL, "heff_create_sum: terms must share mL, d1, d2, mR");
  }
  heff_plan_s* p = new heff_plan_s();
  p->dims = d0;
  p->terms.assign(terms, terms + nterms);
  *out = p;
  return HEFF_OK;
}

extern "C" int heff_set_penalty(heff_plan p, const double* phis, int nphi, double weight, heff_stream stream) {
  if (!p || nphi < 0 || (nphi > 0 && !phis)) return set_err(HEFF_EINVAL, "heff_set_penalty: bad argument");
  if (p->sharded || p->is_complex)
    return set_err(HEFF_EUNSUPPORTED, "heff_set_penalty: not supported on b'-sharded or complex plans");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaFree(p->phis);
  cudaFree(p->pen_scratch);
  p->phis = nullptr;
  p->pen_scratch = nullptr;
  p->nphi = 0;
  if (nphi == 0) return HEFF_OK;
  CKR(init_device_once());
  const int64_t n = vec_len(p);
  p->ldv_phi = (n + 31) / 32 * 32;
  p->pen_G = (int)std::max<int64_t>(1, std::min<int64_t>(4 * (int64_t)g_num_sms, (n + 4095) / 4096));
  CK(cudaMalloc(&p->phis, sizeof(double) * (size_t)nphi * p->ldv_phi));
  CK(cudaMalloc(&p->pen_scratch, sizeof(double) * (size_t)nphi * (p->pen_G + 1)));
  CK(cudaMemset2DAsync(p->phis, sizeof(double) * p->ldv_phi, 0, sizeof(double) * p->ldv_phi, nphi, s));
  CK(cudaMemcpy2DAsync(p->phis, sizeof(double) * p->ldv_phi, phis, sizeof(double) * n, sizeof(double) * n, nphi,
                       cudaMemcpyDeviceToDevice, s));
  p->nphi = nphi;
  p->pen_weight = weight;
  return mark_done(p, s);
}

extern "C" int heff_apply_blocked(heff_plan p, const double* psi_blocked, double* out, heff_stream stream) {
  if (!p || !psi_blocked || !out) return set_err(HEFF_EINVAL, "heff_apply_blocked: null argument");
  if (!p->sharded || p->is_complex || !p->terms.empty() || p->nphi > 0)
    return set_err(HEFF_EUNSUPPORTED, "heff_apply_blocked: b'-sharded real plans only");
  const heff_dims& d = p->dims;
  const int64_t rows = d.mL * d.d1 * d.d2;
  const int P = (int)(d.mR / std::max<int64_t>(1, p->nb));
  std::vector<const double*> sh(P);
  for (int q = 0; q < P; ++q) sh[q] = psi_blocked + (int64_t)q * rows * p->nb;
  ShardedA sa;
  CKR(build_sharded_a(p, sh.data(), P, &sa));
  int nl = 0;
  CKR(after_setup(p, reinterpret_cast<cudaStream_t>(stream)));
  CKR(apply_orderB(p, nullptr, out, reinterpret_cast<cudaStream_t>(stream), &nl, 0, &sa));
  p->last_launches = nl;
  p->total_launches += nl;
  return mark_done(p, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int heff_apply(heff_plan p, const double* psi, double* out, heff_stream stream) {
  if (!p) return set_err(HEFF_EINVAL, "heff_apply: null plan");
  const cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CKR(apply_impl(p, psi, out, s));
  CKR(mark_done(p, s));
  for (heff_plan_s* t : p->terms) CKR(mark_done(t, s));  // a composite's terms ran on s too
  return HEFF_OK;
}

// End-to-end order-A matvec with the transfers overlapped: psi arrives in column chunks
// (s1 s2 b) on a copy stream, GEMM1 runs per chunk as each lands; GEMM4 runs in row chunks
// (a' s1' s2') and each finished block of out goes back while the next is computed.  Only
// the first H2D chunk and the last D2H chunk are exposed.
static constexpr int kE2eChunks = 8;
static int apply_host_pipelined(heff_plan_s* p, const double* psi_host, double* out_host, cudaStream_t s) {
  const heff_dims& d = p->dims;
  const int64_t ncol = d.d1 * d.d2 * d.mR, nrow4 = d.mL * d.d1 * d.d2;
  if (!p->copy_stream) {
    CK(cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking));
    for (auto& e : p->e2e_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaStream_t c = p->copy_stream;
  CK(cudaEventRecord(p->e2e_ev[2 * kE2eChunks], s));   // the copy stream starts after prior work on s
  CK(cudaStreamWaitEvent(c, p->e2e_ev[2 * kE2eChunks], 0));
  int nl = 0;
  for (int k = 0; k < kE2eChunks; ++k) {
    const int64_t c0 = ncol * k / kE2eChunks / 2 * 2, c1 = (k + 1 == kE2eChunks) ? ncol : ncol * (k + 1) / kE2eChunks / 2 * 2;
    CK(cudaMemcpy2DAsync(p->stage_in + c0, sizeof(double) * ncol, psi_host + c0, sizeof(double) * ncol,
                         sizeof(double) * (c1 - c0), d.mL, cudaMemcpyHostToDevice, c));
    CK(cudaEventRecord(p->e2e_ev[k], c));
    CK(cudaStreamWaitEvent(s, p->e2e_ev[k], 0));
    p->g1.M = d.mL * d.kL;
    p->g1.N = c1 - c0;
    p->g1.A = p->L;
    p->g1.B = p->stage_in + c0;
    p->g1.C = p->T1 + c0;
    CKR(launch_gemm(p->g1, p->gemm_path, s, &nl, &p->splitws));
  }
  p->g1.N = ncol;
  const int64_t nin = d.kL * d.d1 * d.d2, nout = d.d1 * d.d2 * d.kR;
  CKR(launch_mpo_A(p->T1, p->T3, d.mR, d.mL, (int)nin, (int)nout, p->csrA, p->mpo_live, p->tcA, s));
  ++nl;
  for (int k = 0; k < kE2eChunks; ++k) {
    const int64_t r0 = nrow4 * k / kE2eChunks, r1 = nrow4 * (k + 1) / kE2eChunks;
    p->g4.M = r1 - r0;
    p->g4.A = p->T3 + r0 * d.kR * d.mR;
    p->g4.C = p->stage_out + r0 * d.mR;
    p->g4.accumulate = 0;
    CKR(launch_gemm(p->g4, p->gemm_path, s, &nl, &p->splitws));
    CK(cudaEventRecord(p->e2e_ev[kE2eChunks + k], s));
    CK(cudaStreamWaitEvent(c, p->e2e_ev[kE2eChunks + k], 0));
    CK(cudaMemcpyAsync(out_host + r0 * d.mR, p->stage_out + r0 * d.mR, sizeof(double) * (r1 - r0) * d.mR,
                       cudaMemcpyDeviceToHost, c));
  }
  p->last_launches = nl;
  p->total_launches += nl;
  CK(cudaStreamSynchronize(c));
  CK(cudaStreamSynchronize(s));
  return HEFF_OK;
}

// End-to-end order-B matvec of a b'-sharded plan with the host-to-device copy of the full psi
// overlapped: psi's rows (a s1 s2) arrive in kE2eChunks row blocks on the copy stream and
// GEMM_A runs per block as each lands (its rows are independent); the MPO step and GEMM_D run
// once, then this rank's out shard (1/P of psi) goes back.
static int apply_host_pipelined_B(heff_plan_s* p, const double* psi_host, double* out_host, cudaStream_t s) {
  const heff_dims& d = p->dims;
  const int64_t rows = d.mL * d.d1 * d.d2, ldv1 = p->nb * d.kR;
  if (!p->copy_stream) {
    CK(cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking));
    for (auto& e : p->e2e_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaStream_t c = p->copy_stream;
  CK(cudaEventRecord(p->e2e_ev[2 * kE2eChunks], s));
  CK(cudaStreamWaitEvent(c, p->e2e_ev[2 * kE2eChunks], 0));
  int nl = 0;
  const GemmOp saved = p->gA;
  for (int k = 0; k < kE2eChunks; ++k) {
    const int64_t r0 = rows * k / kE2eChunks, r1 = rows * (k + 1) / kE2eChunks;
    CK(cudaMemcpyAsync(p->stage_in + r0 * d.mR, psi_host + r0 * d.mR, sizeof(double) * (r1 - r0) * d.mR,
                       cudaMemcpyHostToDevice, c));
    CK(cudaEventRecord(p->e2e_ev[k], c));
    CK(cudaStreamWaitEvent(s, p->e2e_ev[k], 0));
    p->gA.M = r1 - r0;
    p->gA.A = p->stage_in + r0 * d.mR;
    p->gA.C = p->V1 + r0 * ldv1;
    CKR(launch_gemm(p->gA, p->gemm_path, s, &nl, &p->splitws));
  }
  p->gA = saved;
  // MPO step and GEMM_D (apply_orderB without its GEMM_A)
  {
    const int dd = (int)(d.d1 * d.d2);
    MpoIO io{};
    io.in = p->V1;
    io.out = p->V3;
    io.ncol = p->nb;
    io.nin = dd * (int)d.kR;
    io.nout = (int)d.kL * dd;
    io.in_blk = (int64_t)dd * d.kR * p->nb;
    io.in_row = p->nb;
    io.out_blk = (int64_t)dd * p->nb;
    io.out_row = p->nb;
    io.out_grp = dd;
    io.out_grp_stride = d.mL * dd * p->nb;
    CKR((launch_mpo<1, true>(io, p->tcB, d.mL, p->csrB, nullptr, s)));
    ++nl;
  }
  p->gD.C = p->stage_out;
  p->gD.accumulate = 0;
  CKR(launch_gemm(p->gD, p->gemm_path, s, &nl, &p->splitws));
  CK(cudaMemcpyAsync(out_host, p->stage_out, sizeof(double) * rows * p->nb, cudaMemcpyDeviceToHost, s));
  p->last_launches = nl;
  p->total_launches += nl;
  CK(cudaStreamSynchronize(c));
  CK(cudaStreamSynchronize(s));
  return HEFF_OK;
}

extern "C" int heff_apply_host(heff_plan p, const double* psi_host, double* out_host, heff_stream stream) {
  if (!p || !psi_host || !out_host) return set_err(HEFF_EINVAL, "heff_apply_host: null argument");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const heff_dims& d = p->dims;
  const int64_t zf = p->is_complex ? 2 : 1;  // doubles per entry
  const int64_t n_in = zf * d.mL * d.d1 * d.d2 * d.mR;
  const int64_t n_out = zf * vec_len(p);
  if (!p->stage_in) {
    CK(ws_malloc(&p->stage_in, sizeof(double) * n_in));
    CK(ws_malloc(&p->stage_out, sizeof(double) * n_out));
  }
  CKR(after_setup(p, s));
  const bool pipelined = !p->is_complex && !p->sharded && p->terms.empty() && p->nphi == 0 && p->sp1 == nullptr &&
                         p->sp4 == nullptr && p->chunk_rows == d.mL && d.mL * d.d1 * d.d2 >= 8 * kE2eChunks &&
                         getenv("HEFF_NO_E2E_PIPELINE") == nullptr;
  if (pipelined) return apply_host_pipelined(p, psi_host, out_host, s);
  if (!p->is_complex && p->sharded && p->terms.empty() && p->nphi == 0 && d.mL * d.d1 * d.d2 >= 8 * kE2eChunks &&
      getenv("HEFF_NO_E2E_PIPELINE") == nullptr)
    return apply_host_pipelined_B(p, psi_host, out_host, s);
  CK(cudaMemcpyAsync(p->stage_in, psi_host, sizeof(double) * n_in, cudaMemcpyHostToDevice, s));
  CKR(apply_impl(p, p->stage_in, p->stage_out, s));
  CK(cudaMemcpyAsync(out_host, p->stage_out, sizeof(double) * n_out, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return HEFF_OK;
}

// --------------------------------------------------------------------------- Lanczos
__global__ void gather_kernel(const double* __restrict__ dense, const int* __restrict__ idx, int64_t n,
                              double* __restrict__ compact);
__global__ void scatter_kernel(const double* __restrict__ compact, const int* __restrict__ idx, int64_t n,
                               double* __restrict__ dense);

static int reduce_grid(int64_t n) {
  const int64_t per = (int64_t)kRedThreads * 2 * 8;  // >= 8 pairs per thread
  return (int)std::max<int64_t>(1, std::min<int64_t>(4 * (int64_t)g_num_sms, (n + per - 1) / per));
}

int ew_grid(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(8 * (int64_t)g_num_sms, (n / 2 + 255) / 256));
}

// c[0..nq) = V[0..nq)^T w  (local sums; allreduced across ranks when communicating)
static int multidot(heff_plan_s* p, const double* V, int nq, const double* w, int64_t n, double* c, cudaStream_t s) {
  const int G = p->ldp;
  for (int q0 = 0; q0 < nq; q0 += kDotQ) {
    const int qn = std::min(kDotQ, nq - q0);
    multidot_partial_kernel<<<G, kRedThreads, 0, s>>>(V + q0 * p->ldv, p->ldv, qn, w, n, p->partial + q0 * G, G);
    ++p->total_launches;
  }
  reduce_partial_kernel<<<nq, kRedThreads, 0, s>>>(p->partial, G, G, c, 0, nullptr);
  ++p->total_launches;
  CK(cudaGetLastError());
  if (p->comm) CKN(g_nccl.AllReduce(c, c, nq, ncclFloat64, ncclSum, p->comm, s));
  return HEFF_OK;
}

static int multiaxpy(heff_plan_s* p, const double* V, int nq, const double* c, double sign, double* w, int64_t n,
                     cudaStream_t s) {
  for (int q0 = 0; q0 < nq; q0 += 64) {
    const int qn = std::min(64, nq - q0);
    multiaxpy_kernel<<<ew_grid(n), 256, 0, s>>>(V + q0 * p->ldv, p->ldv, qn, c + q0, sign, w, n);
    ++p->total_launches;
  }
  CK(cudaGetLastError());
  return HEFF_OK;
}

// complex (interleaved) versions: c[2q], c[2q+1] = Re, Im of <V_q, w>, n complex entries
static int zmultidot(heff_plan_s* p, const double* V, int nq, const double* w, int64_t n, double* c, cudaStream_t s) {
  const int G = p->ldp;
  for (int q0 = 0; q0 < nq; q0 += kDotQ) {
    const int qn = std::min(kDotQ, nq - q0);
    zmultidot_partial_kernel<<<G, kRedThreads, 0, s>>>(V + q0 * p->ldv, p->ldv, qn, w, n, p->partial + 2 * q0 * G, G);
    ++p->total_launches;
  }
  reduce_partial_kernel<<<2 * nq, kRedThreads, 0, s>>>(p->partial, G, G, c, 0, nullptr);
  ++p->total_launches;
  CK(cudaGetLastError());
  return HEFF_OK;
}

static int zmultiaxpy(heff_plan_s* p, const double* V, int nq, const double* c, double sign, double* w, int64_t n,
                      cudaStream_t s) {
  for (int q0 = 0; q0 < nq; q0 += 64) {
    const int qn = std::min(64, nq - q0);
    zmultiaxpy_kernel<<<ew_grid(2 * n), 256, 0, s>>>(V + q0 * p->ldv, p->ldv, qn, c + 2 * q0, sign, w, n);
    ++p->total_launches;
  }
  CK(cudaGetLastError());
  return HEFF_OK;
}

__global__ void sqrt_inv_kernel(double* x, double* inv) {
  const double v = sqrt(*x);
  *x = v;
  *inv = v > 0.0 ? 1.0 / v : 0.0;
}

// ||w|| -> *nrm, 1/||w|| -> *inv (global over ranks)
static int norm2(heff_plan_s* p, const double* w, int64_t n, double* nrm, double* inv, cudaStream_t s) {
  const int G = p->ldp;
  multidot_partial_kernel<<<G, kRedThreads, 0, s>>>(w, 0, 1, w, n, p->partial, G);
  reduce_partial_kernel<<<1, kRedThreads, 0, s>>>(p->partial, G, G, nrm, p->comm ? 0 : 1, inv);
  p->total_launches += 2;
  CK(cudaGetLastError());
  if (p->comm) {
    CKN(g_nccl.AllReduce(nrm, nrm, 1, ncclFloat64, ncclSum, p->comm, s));
    sqrt_inv_kernel<<<1, 1, 0, s>>>(nrm, inv);
    ++p->total_launches;
    CK(cudaGetLastError());
  }
  return HEFF_OK;
}

// ---- failure detection of communicating plans (SURVEY.md 5 "Failure detection") -----------
// ncclCommAbort the plan's communicator after an error or timeout: the peers' pending and
// future collectives on it fail instead of hanging; the plan stays unusable.
static int comm_abort(heff_plan_s* p, const char* fmt, ...) {
  char buf[384];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (p->comm && g_nccl.CommAbort) g_nccl.CommAbort(p->comm);
  p->comm = nullptr;
  p->comm_dead = 1;
  p->win = nullptr;  // the window died with the communicator
  p->comm_err = buf;
  return set_err(HEFF_ENCCL, "%s (communicator aborted; destroy the plan)", buf);
}

static double nccl_timeout_s() {  // read per wait (tests lower it at run time)
  const char* e = getenv("HEFF_NCCL_TIMEOUT_S");
  const double v = e ? atof(e) : 300.0;
  return v > 0 ? v : 300.0;
}

// Record "Lanczos step done" on s (progress marker for comm_wait).
static int mark_step(heff_plan_s* p, cudaStream_t s) {
  if (!p->comm) return HEFF_OK;
  if (p->step_ev_used == (int)p->step_ev.size()) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    p->step_ev.push_back(e);
  }
  CK(cudaEventRecord(p->step_ev[p->step_ev_used++], s));
  return HEFF_OK;
}

// Wait for stream s.  Plans without a communicator: cudaStreamSynchronize.  With one: poll
// the stream, ncclCommGetAsyncError (aborting on an error) and progress -- a step marker
// completing resets the clock; no progress for HEFF_NCCL_TIMEOUT_S aborts the communicator.
static int comm_wait(heff_plan_s* p, cudaStream_t s) {
  if (!p->comm) {
    if (p->comm_dead) return set_err(HEFF_ENCCL, "plan's communicator was aborted: %s", p->comm_err.c_str());
    CK(cudaStreamSynchronize(s));
    return HEFF_OK;
  }
  using clk = std::chrono::steady_clock;
  auto t_prog = clk::now();
  int seen = 0;
  unsigned spin = 0;
  for (;;) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) return comm_abort(p, "stream failed: %s", cudaGetErrorString(q));
    ncclResult_t ar = ncclSuccess;
    if (g_nccl.CommGetAsyncError(p->comm, &ar) != ncclSuccess ||
        (ar != ncclSuccess && ar != ncclInProgress))
      return comm_abort(p, "NCCL asynchronous error: %s", g_nccl.GetErrorString(ar));
    while (seen < p->step_ev_used && cudaEventQuery(p->step_ev[seen]) == cudaSuccess) {
      ++seen;
      t_prog = clk::now();
    }
    const double idle = std::chrono::duration<double>(clk::now() - t_prog).count();
    if (idle > nccl_timeout_s())
      return comm_abort(p, "no progress for %.0f s (a peer is gone or stuck; HEFF_NCCL_TIMEOUT_S)", idle);
    if (++spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  p->step_ev_used = 0;
  return HEFF_OK;
}

// full-psi input for the matvec: all-gather the shard (communicating plans) or use v as is
static int matvec_local(heff_plan_s* p, const double* v, double* w, cudaStream_t s) {
  if (!p->sharded) return apply_impl(p, v, w, s);
  if (!p->comm) return set_err(HEFF_EUNSUPPORTED, "lanczos_ground on a virtual shard (no communicator)");
  const heff_dims& d = p->dims;
  const int64_t rows = d.mL * d.d1 * d.d2;
  const int64_t nloc = rows * p->nb;
  if (p->nranks == 1 && !p->force_allgather) {
    CK(cudaMemcpyAsync(p->full, v, sizeof(double) * nloc, cudaMemcpyDeviceToDevice, s));
  } else {
    CKN(g_nccl.AllGather(v, p->gather, nloc, ncclFloat64, p->comm, s));
    relayout_blocked_kernel<<<ew_grid(rows * d.mR), 256, 0, s>>>(p->gather, p->full, rows, p->nb, p->nranks);
    ++p->total_launches;
    CK(cudaGetLastError());
  }
  return apply_impl(p, p->full, w, s);
}

// The Lanczos reduction kernels as a primitive (kernel-level tests at adversarial lengths):
// *result = x . y over n doubles through multidot_partial_kernel + reduce_partial_kernel.
extern "C" int heff_dot(int64_t n, const double* x, const double* y, double* result, heff_stream stream) {
  if (n < 0 || (n > 0 && (!x || !y)) || !result) return set_err(HEFF_EINVAL, "heff_dot: bad argument");
  CKR(init_device_once());
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int G = reduce_grid(n);
  double* buf = nullptr;
  CK(cudaMalloc(&buf, sizeof(double) * (G + 1)));
  multidot_partial_kernel<<<G, kRedThreads, 0, s>>>(x, 0, 1, y, n, buf, G);
  reduce_partial_kernel<<<1, kRedThreads, 0, s>>>(buf, G, G, buf + G, 0, nullptr);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(result, buf + G, sizeof(double), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(buf);
  if (e != cudaSuccess) return set_err(HEFF_ECUDA, "heff_dot: %s", cudaGetErrorString(e));
  return HEFF_OK;
}

extern "C" int heff_relayout_blocked(const double* src, double* dst, int64_t rows, int64_t nb, int P,
                                     heff_stream stream) {
  if (!src || !dst || rows < 0 || nb < 0 || P < 1) return set_err(HEFF_EINVAL, "heff_relayout_blocked: bad argument");
  if (src == dst) return set_err(HEFF_EINVAL, "heff_relayout_blocked: dst must not alias src");
  CKR(init_device_once());
  if (rows * nb == 0) return HEFF_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  relayout_blocked_kernel<<<ew_grid(rows * nb * P), 256, 0, s>>>(src, dst, rows, nb, P);
  CK(cudaGetLastError());
  return HEFF_OK;
}

// ---- gather-fused sharded Lanczos (NEXT-5): NCCL symmetric window + peer flags ----------
__global__ void window_peer_pointers_kernel(ncclWindow_t w, int P, char** out) {
  const int q = threadIdx.x;
  if (q < P) out[q] = static_cast<char*>(ncclGetPeerPointer(w, 0, q));
}

// rank `rank` announces "my basis slot for step value-1 is written": flags[rank] = value in
// every rank's window (system-scope release after a system fence)
__global__ void peer_signal_kernel(uint64_t* const* peer_flags, int rank, int P, unsigned long long value) {
  __threadfence_system();
  const int q = threadIdx.x;
  if (q < P) {
    uint64_t* f = peer_flags[q] + rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(value) : "memory");
  }
}

// wait until every rank's flag in this rank's window reached `value` (acquire); bounded
// spin (~20 s by %globaltimer) so a missing peer turns into a reported error, not a hang
__global__ void peer_wait_kernel(const uint64_t* flags, int P, unsigned long long value, int* timed_out) {
  const int q = threadIdx.x;
  if (q < P && *(volatile int*)timed_out == 0) {  // after one timeout the later waits fall through
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + q) : "memory");
      if (v >= value) break;
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 20000000000ull) {
        atomicExch(timed_out, 1);
        break;
      }
      __nanosleep(200);
    }
  }
  __syncthreads();
}

static int release_window(heff_plan_s* p) {
  if (p->win && g_nccl.CommWindowDeregister) g_nccl.CommWindowDeregister(p->comm, p->win);
  if (p->win_buf && g_nccl.MemFree) g_nccl.MemFree(p->win_buf);
  p->win = nullptr;
  p->win_buf = nullptr;
  p->win_cap = 0;
  return HEFF_OK;
}

// Collective over the plan's ranks (every rank calls lanczos_ground with the same max_iter).
static int ensure_window(heff_plan_s* p, int cap, int64_t ldv, cudaStream_t s) {
  if (p->win && p->win_cap >= cap && p->win_ldv == ldv) return HEFF_OK;
  if (!g_nccl.MemAlloc || !g_nccl.CommWindowRegister)
    return set_err(HEFF_EUNSUPPORTED, "libnccl has no symmetric-memory windows (ncclCommWindowRegister)");
  release_window(p);
  const int P = p->nranks;
  const size_t slots = sizeof(double) * (size_t)ldv * cap;
  const size_t flag_off = (slots + 255) / 256 * 256;
  const size_t bytes = (flag_off + 256 + 4095) / 4096 * 4096;
  CKN(g_nccl.MemAlloc(&p->win_buf, bytes));
  CK(cudaMemsetAsync(p->win_buf, 0, bytes, s));
  CK(cudaStreamSynchronize(s));
  CKN(g_nccl.CommWindowRegister(p->comm, p->win_buf, bytes, &p->win, NCCL_WIN_COLL_SYMMETRIC));
  char** d_ptrs = nullptr;
  CK(cudaMalloc(&d_ptrs, sizeof(char*) * P));
  window_peer_pointers_kernel<<<1, 32, 0, s>>>(p->win, P, d_ptrs);
  p->peer_base.assign(P, nullptr);
  CK(cudaMemcpyAsync(p->peer_base.data(), d_ptrs, sizeof(char*) * P, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  cudaFree(d_ptrs);
  std::vector<uint64_t*> pf(P);
  for (int q = 0; q < P; ++q) pf[q] = reinterpret_cast<uint64_t*>(p->peer_base[q] + flag_off);
  if (!p->d_peer_flags) CK(cudaMalloc(&p->d_peer_flags, sizeof(uint64_t*) * kMaxShards));
  CK(cudaMemcpyAsync(p->d_peer_flags, pf.data(), sizeof(uint64_t*) * P, cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
  p->win_bytes = bytes;
  p->win_cap = cap;
  p->win_ldv = ldv;
  p->win_flag_off = (int64_t)flag_off;
  p->epoch = 0;
  return HEFF_OK;
}

// Krylov workspace of lanczos_ground for `cap` iterations: the basis (or the NCCL window of
// the gather-fused path), scalars, work vector, U(1) scatter buffers and the sharded gather
// buffers; allocated on first need and grown, never inside a call that fits.
static int lanczos_workspace(heff_plan_s* p, int cap, cudaStream_t s, LanczosLayout* out) {
  // U(1) plans iterate on the sector's entries only (gather/scatter around each matvec)
  const bool compact = p->qn_idx != nullptr && !p->sharded && p->terms.empty();
  const int64_t n_dense = vec_len(p);
  const int64_t n = compact ? p->qn_n : n_dense;     // entries per vector
  const bool cplx = p->is_complex;                   // interleaved complex entries
  const int64_t nr = cplx ? 2 * n : n;               // doubles per vector
  const int64_t ldv = (nr + 31) / 32 * 32;
  if (compact && !p->dense_in) {
    CK(ws_malloc(&p->dense_in, sizeof(double) * n_dense));
    CK(ws_malloc(&p->dense_out, sizeof(double) * n_dense));
    CK(cudaMemsetAsync(p->dense_in, 0, sizeof(double) * n_dense, s));
  }
  // gather-fused sharded path: the basis lives in an NCCL symmetric window
  bool fgather = false;
  if (p->comm && p->fused_gather && !cplx && !compact && p->nranks <= kMaxShards && p->nb % kGemmBK == 0) {
    const int rw = ensure_window(p, cap, ldv, s);
    if (rw != HEFF_OK) return rw;
    fgather = true;
  }
  p->fused_active = fgather ? 1 : 0;
  // (re)allocate the Krylov basis and scratch
  if (p->basis_cap < cap || p->ldv != ldv) {
    CK(cudaStreamSynchronize(s));  // the old blocks go back to the cache idle
    ws_release(p->basis); ws_release(p->partial); ws_release(p->scal);
    p->basis = nullptr; p->partial = nullptr; p->scal = nullptr;
    p->basis_cap = 0;
    CK(ws_malloc(&p->basis, sizeof(double) * ldv * (fgather ? 1 : cap)));
    p->ldp = reduce_grid(nr);
    const size_t pcols = std::max<size_t>((size_t)p->ldp, (size_t)8 * g_num_sms);  // also the fused step's grid
    CK(ws_malloc(&p->partial, sizeof(double) * (size_t)(2 * cap + 2 * kDotQ + 1) * pcols));
    CK(ws_malloc(&p->scal, sizeof(double) * 9 * (size_t)(cap + 1)));  // + fused-gather timeout flag, grid barrier
    p->basis_cap = fgather ? 0 : cap;  // a later non-fused call reallocates the full basis
    p->ldv = ldv;
  }
  if (p->hpin_n < (size_t)(3 * cap + 4)) {  // alpha, beta, y, norm
    if (p->hpin) {
      CK(cudaStreamSynchronize(s));
      pin_release(p->hpin, p->hpin_n * sizeof(double));
      p->hpin = nullptr;
      p->hpin_n = 0;
    }
    size_t bytes = 0;
    CK(pin_alloc(&p->hpin, &bytes, sizeof(double) * (size_t)(3 * cap + 4)));
    p->hpin_n = bytes / sizeof(double);
  }
  if (!p->gbar) {
    CK(ws_malloc(&p->gbar, 256));
    CK(cudaMemsetAsync(p->gbar, 0, 256, s));
  }
  if (!p->work || p->work_len < ldv) {
    CK(cudaStreamSynchronize(s));
    ws_release(p->work);
    p->work = nullptr;
    CK(ws_malloc(&p->work, sizeof(double) * ldv));
    p->work_len = ldv;
  }
  if (p->sharded && p->comm && !fgather && p->full && !p->gather && (p->nranks > 1 || p->force_allgather)) {
    const heff_dims& d = p->dims;
    CK(ws_malloc(&p->gather, sizeof(double) * d.mL * d.d1 * d.d2 * d.mR));
  }
  if (p->sharded && p->comm && !p->full && !fgather) {
    const heff_dims& d = p->dims;
    CK(ws_malloc(&p->full, sizeof(double) * d.mL * d.d1 * d.d2 * d.mR));
    if (p->nranks > 1 || p->force_allgather) CK(ws_malloc(&p->gather, sizeof(double) * d.mL * d.d1 * d.d2 * d.mR));
  }
  *out = LanczosLayout{compact, cplx, fgather, n_dense, n, nr, ldv};
  return HEFF_OK;
}

extern "C" int lanczos_ground(heff_plan p, double* psi, const heff_lanczos_opts* o, double* energy, int* iters_done,
                              double* resid_est, heff_stream stream) {
  if (!p || !psi || !o || !energy) return set_err(HEFF_EINVAL, "lanczos_ground: null argument");
  if (o->max_iter < 1 || o->max_iter > 100000) return set_err(HEFF_EINVAL, "lanczos_ground: max_iter out of range");
  if (o->mode != 0 && o->mode != 1) return set_err(HEFF_EINVAL, "lanczos_ground: mode must be 0 or 1");
  if (p->comm_dead) return set_err(HEFF_ENCCL, "plan's communicator was aborted: %s", p->comm_err.c_str());
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int cap = o->max_iter;
  p->step_ev_used = 0;
  CKR(after_setup(p, s));
  LanczosLayout lay;
  CKR(lanczos_workspace(p, cap, s, &lay));
  const bool compact = lay.compact, cplx = lay.cplx, fgather = lay.fgather;
  const int64_t n_dense = lay.n_dense, n = lay.n, nr = lay.nr, ldv = lay.ldv;
  double* c1 = p->scal;                              // 2 (cap+1): room for complex coefficients
  double* c2 = c1 + 2 * (cap + 1);
  double* alpha = c2 + 2 * (cap + 1);
  double* beta = alpha + (cap + 1);
  double* invb = beta + (cap + 1);
  double* ydev = invb + (cap + 1);
  double* V = fgather ? static_cast<double*>(p->win_buf) : p->basis;
  double* w = p->work;
  int* d_timeout = reinterpret_cast<int*>(ydev + (cap + 1));  // scal has room: 8 (cap+1) doubles
  auto fused_signal = [&](uint64_t value) -> int {
    peer_signal_kernel<<<1, 32, 0, s>>>(p->d_peer_flags, p->rank, p->nranks, (unsigned long long)value);
    ++p->total_launches;
    CK(cudaGetLastError());
    return HEFF_OK;
  };
  // matvec of the fused path: wait for every rank's slot, GEMM_A straight from their windows
  auto fused_matvec = [&](int j) -> int {
    const uint64_t* myflags = reinterpret_cast<const uint64_t*>(static_cast<char*>(p->win_buf) + p->win_flag_off);
    peer_wait_kernel<<<1, 32, 0, s>>>(myflags, p->nranks, (unsigned long long)(p->epoch + j), d_timeout);
    ++p->total_launches;
    std::vector<const double*> sh(p->nranks);
    for (int q = 0; q < p->nranks; ++q)  // own shard through the local mapping, peers through LSA pointers
      sh[q] = reinterpret_cast<const double*>(q == p->rank ? static_cast<char*>(p->win_buf) : p->peer_base[q]) +
              (int64_t)(j - 1) * ldv;
    ShardedA sa;
    CKR(build_sharded_a(p, sh.data(), p->nranks, &sa));
    int nl = 0;
    CKR(apply_orderB(p, nullptr, w, s, &nl, 0, &sa));
    p->total_launches += nl;
    return HEFF_OK;
  };
  if (fgather) CK(cudaMemsetAsync(d_timeout, 0, sizeof(int), s));

  // v1 = x0 / ||x0||  (copied into the aligned basis first)
  if (compact) {
    gather_kernel<<<ew_grid(n), 256, 0, s>>>(psi, p->qn_idx, n, V);
    ++p->total_launches;
    CK(cudaGetLastError());
  } else {
    CK(cudaMemcpyAsync(V, psi, sizeof(double) * nr, cudaMemcpyDeviceToDevice, s));
  }
  CKR(norm2(p, V, nr, beta + cap, invb + cap, s));
  double* h_a = p->hpin;                 // pinned: the copies below never block the host,
  double* h_b = h_a + cap;               // comm_wait polls (failure detection)
  double* h_y = h_b + cap;
  double* h_n = h_y + cap;
  // Without a communicator the zero-start-vector test waits for the first scalar read-back
  // below (a zero x0 gives 1/||x0|| = 0 on the device, so the steps run on zeros and break
  // down at once; psi is left untouched): one host round trip less per call.  With one, every
  // rank must learn it before the first collective.
  const bool defer_zero = p->comm == nullptr && getenv("HEFF_EAGER_ZERO_CHECK") == nullptr;
  auto zero_start = [&]() { return set_err(HEFF_EZERO, "lanczos_ground: zero start vector"); };
  if (!defer_zero) {
    CK(cudaMemcpyAsync(h_n, beta + cap, sizeof(double), cudaMemcpyDeviceToHost, s));
    CKR(comm_wait(p, s));
    if (!(*h_n > 0.0)) return zero_start();
  }
  scale_kernel<<<ew_grid(nr), 256, 0, s>>>(V, invb + cap, V, nr);
  ++p->total_launches;
  CK(cudaGetLastError());
  if (fgather) CKR(fused_signal(p->epoch + 1));

  std::vector<double> ha(cap), hb(cap);
  double theta = 0.0, ylast = 0.0, hnorm = 0.0;
  int j_done = 0;
  // fused single-launch CGS2 step when there is no communicator and the coefficients fit
  // (launch-bound sizes only: above ~2M elements the separate vectorised kernels stream faster)
  const bool fused = !cplx && (p->comm == nullptr) && (cap <= 4096) &&
                     (n <= (int64_t(1) << 21) || getenv("HEFF_FUSED_STEP")) && getenv("HEFF_NO_FUSED_STEP") == nullptr;
  int step_grid = 0, step3_grid = 0, step3s_grid = 0;
  // vectors up to this length take the one-block step kernel when the grid is one block
  // (HEFF_SMALL_STEP_N overrides; 0 = never)
  static const int64_t small_step_max = [] {
    const char* e = getenv("HEFF_SMALL_STEP_N");
    return std::min<int64_t>(e ? (int64_t)atoll(e) : (int64_t)2048, (int64_t)kSmallStepThreads * kSmallStepE);
  }();
  if (fused) {
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cgs2_step_kernel, kStepThreads,
                                                     sizeof(double) * (size_t)(cap + 1)));
    // elements per thread (HEFF_STEP_EPT, default 1; round 1: 4, then 2): fewer = more blocks
    // in flight (C1 41.6 -> 37.5 us, cylinder m = 128 91 -> 78-82 us per Lanczos step at 2;
    // at 1: cylinder m = 64 71.2 -> 67.1 us, chain m = 128 57.8 -> 55.2 us, C2 87.3 / 88.4 us)
    static const int ept = [] {
      const char* e = getenv("HEFF_STEP_EPT");
      return e ? std::max(1, atoi(e)) : 1;
    }();
    const int64_t want = std::max<int64_t>(1, (n + (int64_t)ept * kStepThreads - 1) / ((int64_t)ept * kStepThreads));
    step_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * g_num_sms, want));
    int per_sm3 = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm3, cgs2_step3_kernel<kStep3MaxJ, 1>, kStep3Threads, 0));
    step3_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm3 * g_num_sms,
                                                             (n + kStep3Threads - 1) / kStep3Threads));
    int per_sm3s = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm3s, cgs2_step3_kernel<kStep3SmallJ, 2>, kStep3Threads, 0));
    step3s_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm3s * g_num_sms,
                                                              (n + kStep3Threads - 1) / kStep3Threads));
  }
  static const bool no_smem_step = getenv("HEFF_NO_SMEM_STEP") != nullptr;
  // multi-block CGS2 steps as ordinary launches with a flip-counter grid barrier (p->gbar)
  // instead of cooperative launches: measured 1.3-2.0 us less per Lanczos step (chain m = 64
  // 45.8 -> 44.0 us, cylinder m = 64 46.5 -> 44.5 us, C2 90.0 -> 89.4 us), bitwise-equal
  // results.  The grid is the occupancy-limited resident grid of the whole device; under MPS
  // (a client may get fewer SMs than the device reports) the cooperative launch, which checks
  // co-residency, stays.  HEFF_STEP_NONCOOP=0/1 overrides (read per call).
  const bool step_noncoop = [] {
    if (const char* e = getenv("HEFF_STEP_NONCOOP")) return atoi(e) != 0;
    return getenv("CUDA_MPS_PIPE_DIRECTORY") == nullptr && getenv("CUDA_MPS_ACTIVE_THREAD_PERCENTAGE") == nullptr;
  }();
  unsigned int* d_gbar = p->gbar;
  std::vector<cudaEvent_t>* phase_ev = nullptr;  // HEFF_LANCZOS_TIMING >= 2 (fixed mode)
  auto step = [&](int j) -> int {  // j = 1-based step: v_j = V[j-1]
    double* vj = V + (int64_t)(j - 1) * ldv;
    if (compact) {
      scatter_kernel<<<ew_grid(n), 256, 0, s>>>(vj, p->qn_idx, n, p->dense_in);
      CKR(matvec_local(p, p->dense_in, p->dense_out, s));
      gather_kernel<<<ew_grid(n), 256, 0, s>>>(p->dense_out, p->qn_idx, n, w);
      p->total_launches += 2;
      CK(cudaGetLastError());
    } else if (fgather) {
      CKR(fused_matvec(j));
    } else {
      CKR(matvec_local(p, vj, w, s));
    }
    if (phase_ev) cudaEventRecord((*phase_ev)[2 * j - 1], s);
    if (fused) {
      const double* Vc = V;
      int64_t ldv_ = ldv;
      int jj = j, jmax = cap;
      double* partial = p->partial;
      double* vnext = (j < cap) ? V + (int64_t)j * ldv : nullptr;
      int64_t nn = n;
      double* wp = w;
      static const bool pdl_off = getenv("HEFF_NO_PDL") != nullptr;
      const int64_t np = (n + 1) & ~int64_t(1);
      if (n <= 2 * kSmemStepThreads && j <= kSmemStepMaxJ && (int64_t)j * np * 8 <= kSmemStepMaxBytes &&
          !no_smem_step) {
        // short vectors, basis resident in shared memory (cgs2_step_smem_kernel)
        CK(launch_pdl(cgs2_step_smem_kernel, dim3(1), dim3(kSmemStepThreads), (size_t)(j * np * 8), s, Vc, ldv_, jj, wp,
                      nn, c1, c2, alpha, beta, invb, vnext));
        ++p->total_launches;
        return HEFF_OK;
      }
      if (n <= small_step_max) {
        // short vectors: the one-block latency-optimised step (cgs2_step_small_kernel)
        CK(launch_pdl(cgs2_step_small_kernel, dim3(1), dim3(kSmallStepThreads), sizeof(double) * (size_t)(j + 1), s,
                      Vc, ldv_, jj, wp, nn, c1, c2, alpha, beta, invb, vnext));
        ++p->total_launches;
        return HEFF_OK;
      }
      // j <= kStep3MaxJ: three passes over the basis (cgs2_step3_kernel), else four
      const bool three = j <= kStep3MaxJ && step_grid > 1 && getenv("HEFF_NO_STEP3") == nullptr;
      unsigned int* gbar = step_noncoop ? d_gbar : nullptr;
      // cgs2_step3_kernel: two elements per thread per iteration when a thread owns >= 4
      // (measured, B200: C2, 6.9 per thread, Lanczos step 90.8 -> 85.5 us; at 1.7 per thread,
      // m = 128 chain / cylinder, 0.9-1.1 us slower); HEFF_STEP3_UNROLL=0/1 overrides
      // j <= kStep3SmallJ: the <12, 2> instantiation (two blocks per SM; HEFF_STEP3_SMALLJ=0 off)
      const char* e_sj = getenv("HEFF_STEP3_SMALLJ");  // (read per call)
      const bool small_j_off = e_sj && atoi(e_sj) == 0;
      const bool small_j = three && j <= kStep3SmallJ && step3s_grid > 1 && !small_j_off;
      const int g3 = small_j ? step3s_grid : step3_grid;
      const int64_t per_thread = (n + (int64_t)g3 * kStep3Threads - 1) / ((int64_t)g3 * kStep3Threads);
      int unroll2 = per_thread >= 4;
      if (const char* e = getenv("HEFF_STEP3_UNROLL")) unroll2 = atoi(e) != 0;
      void* args[] = {(void*)&Vc, &ldv_, &jj, &wp, &nn, &partial, &jmax, &c1, &c2, &alpha, &beta, &invb, &vnext, &gbar,
                      &unroll2};
      // cooperative (grid syncs) and, unless HEFF_NO_PDL, programmatic serialization: the
      // launch overlaps the matvec's last kernel, the body starts after griddepcontrol.wait
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(step_grid);
      cfg.blockDim = dim3(kStepThreads);
      cfg.dynamicSmemBytes = sizeof(double) * (size_t)(j + 1);
      cfg.stream = s;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = step_grid > 1 && !step_noncoop ? 1 : 0;  // one block: an ordinary launch
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[1].val.programmaticStreamSerializationAllowed = pdl_off ? 0 : 1;
      cfg.attrs = at;
      cfg.numAttrs = 2;
      if (three) {
        cfg.dynamicSmemBytes = 0;
        cfg.gridDim = dim3(g3);
        cfg.blockDim = dim3(kStep3Threads);
        at[0].val.cooperative = g3 > 1 && !step_noncoop ? 1 : 0;
      }
      const void* kfn = !three ? (const void*)cgs2_step_kernel
                               : small_j ? (const void*)cgs2_step3_kernel<kStep3SmallJ, 2>
                                         : (const void*)cgs2_step3_kernel<kStep3MaxJ, 1>;
      CK(cudaLaunchKernelExC(&cfg, kfn, args));
      ++p->total_launches;
      return HEFF_OK;
    }
    if (cplx) {
      CKR(zmultidot(p, V, j, w, n, c1, s));
      CKR(zmultiaxpy(p, V, j, c1, -1.0, w, n, s));
      CKR(zmultidot(p, V, j, w, n, c2, s));
      CKR(zmultiaxpy(p, V, j, c2, -1.0, w, n, s));
    } else {
      CKR(multidot(p, V, j, w, n, c1, s));
      CKR(multiaxpy(p, V, j, c1, -1.0, w, n, s));
      CKR(multidot(p, V, j, w, n, c2, s));
      CKR(multiaxpy(p, V, j, c2, -1.0, w, n, s));
    }
    lanczos_alpha_kernel<<<1, 1, 0, s>>>(c1, c2, j - 1, alpha, cplx ? 2 : 1);
    ++p->total_launches;
    CKR(norm2(p, w, nr, beta + (j - 1), invb + (j - 1), s));
    if (j < cap) {
      scale_kernel<<<ew_grid(nr), 256, 0, s>>>(w, invb + (j - 1), V + (int64_t)j * ldv, nr);
      ++p->total_launches;
      if (fgather) CKR(fused_signal(p->epoch + j + 1));
    }
    CK(cudaGetLastError());
    return HEFF_OK;
  };
  // scalar bookkeeping on the host: returns true to stop after step j
  // (hnorm: Gershgorin bound of T_j, updated with the rows the new step changes)
  // (fixed mode without theta_out needs only the breakdown test per step: the Ritz pair of
  // the last step is solved below anyway)
  const bool need_theta = o->mode == 1 || o->theta_out != nullptr;
  auto host_check = [&](int j) -> bool {
    for (int i = std::max(0, j - 2); i < j; ++i) {
      const double gsh = std::fabs(ha[i]) + (i > 0 ? hb[i - 1] : 0.0) + hb[i];
      hnorm = std::max(hnorm, gsh);
    }
    if (!need_theta) return hb[j - 1] <= 1e-12 * hnorm || j == cap;
    if (!tridiag_lowest_fast(j, ha.data(), hb.data(), &theta, &ylast))
      tridiag_lowest_last(j, ha.data(), hb.data(), &theta, &ylast);  // (never seen; QL as the fallback)
    if (o->theta_out) o->theta_out[j - 1] = theta;
    if (hb[j - 1] <= 1e-12 * hnorm) return true;  // breakdown: invariant subspace
    if (o->mode == 1 && hb[j - 1] * std::fabs(ylast) <= o->tol * hnorm) return true;
    return j == cap;
  };

  if (o->mode == 0) {
    // fixed steps: enqueue everything, read the scalars once, truncate at a breakdown
    static const int timing = getenv("HEFF_LANCZOS_TIMING") ? atoi(getenv("HEFF_LANCZOS_TIMING")) : 0;
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    // timing >= 2: events between the steps' phases (serialises the launches: a breakdown,
    // not the pipelined time)
    std::vector<cudaEvent_t> tev;
    if (timing >= 2) {
      tev.resize(2 * (size_t)cap + 1);
      for (auto& e : tev) cudaEventCreate(&e);
      cudaEventRecord(tev[0], s);
      phase_ev = &tev;
    }
    for (int j = 1; j <= cap; ++j) {
      CKR(step(j));
      CKR(mark_step(p, s));
      if (timing >= 2) cudaEventRecord(tev[2 * j], s);
    }
    const auto t1 = clk::now();
    CK(cudaMemcpyAsync(h_a, alpha, sizeof(double) * cap, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(h_b, beta, sizeof(double) * cap, cudaMemcpyDeviceToHost, s));
    if (defer_zero) CK(cudaMemcpyAsync(h_n, beta + cap, sizeof(double), cudaMemcpyDeviceToHost, s));
    CKR(comm_wait(p, s));
    if (defer_zero && !(*h_n > 0.0)) {
      for (auto& e : tev) cudaEventDestroy(e);
      return zero_start();
    }
    const auto t2 = clk::now();
    memcpy(ha.data(), h_a, sizeof(double) * cap);
    memcpy(hb.data(), h_b, sizeof(double) * cap);
    for (int j = 1; j <= cap; ++j) {
      j_done = j;
      if (host_check(j)) break;
    }
    if (timing >= 2) {
      double tm = 0, tc = 0;
      for (int j = 1; j <= cap; ++j) {
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, tev[2 * j - 2], tev[2 * j - 1]);
        cudaEventElapsedTime(&b, tev[2 * j - 1], tev[2 * j]);
        tm += a;
        tc += b;
      }
      fprintf(stderr, "lanczos_ground phases (serialised): matvec %.1f us, orthogonalisation %.1f us per step\n",
              tm * 1e3 / cap, tc * 1e3 / cap);
      for (auto& e : tev) cudaEventDestroy(e);
      phase_ev = nullptr;
    }
    if (timing)
      fprintf(stderr, "lanczos_ground fixed %d steps: enqueue %.1f us, wait %.1f us, host checks %.1f us\n", cap,
              std::chrono::duration<double, std::micro>(t1 - t0).count(),
              std::chrono::duration<double, std::micro>(t2 - t1).count(),
              std::chrono::duration<double, std::micro>(clk::now() - t2).count());
  } else {
    // Converge mode.  Small vectors (<= 2^20 doubles, steps of ~0.1 ms) enqueue `batch`
    // steps per host round trip and test them in order: the stopping step j_done, T_j and
    // the Ritz vector are exactly those of a per-step check (the extra steps' vectors and
    // scalars are never read); only the read-back latency is amortised.
    int batch = nr <= (int64_t(1) << 20) ? 4 : 1;
    if (const char* e = getenv("HEFF_LANCZOS_BATCH")) batch = std::max(1, atoi(e));
    bool stop = false;
    for (int j = 1; j <= cap && !stop;) {
      const int j1 = std::min(cap, j + batch - 1);
      for (int jj = j; jj <= j1; ++jj) {
        CKR(step(jj));
        CKR(mark_step(p, s));
      }
      CK(cudaMemcpyAsync(h_a + (j - 1), alpha + (j - 1), sizeof(double) * (j1 - j + 1), cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(h_b + (j - 1), beta + (j - 1), sizeof(double) * (j1 - j + 1), cudaMemcpyDeviceToHost, s));
      if (defer_zero && j == 1) CK(cudaMemcpyAsync(h_n, beta + cap, sizeof(double), cudaMemcpyDeviceToHost, s));
      CKR(comm_wait(p, s));
      if (defer_zero && j == 1 && !(*h_n > 0.0)) return zero_start();
      memcpy(&ha[j - 1], h_a + (j - 1), sizeof(double) * (j1 - j + 1));
      memcpy(&hb[j - 1], h_b + (j - 1), sizeof(double) * (j1 - j + 1));
      for (int jj = j; jj <= j1; ++jj) {
        j_done = jj;
        if (host_check(jj)) {
          stop = true;
          break;
        }
      }
      j = j1 + 1;
    }
  }
  if (o->alpha_out) memcpy(o->alpha_out, ha.data(), sizeof(double) * j_done);
  if (o->beta_out) memcpy(o->beta_out, hb.data(), sizeof(double) * j_done);
  // Ritz vector x = V y / ||V y||
  std::vector<double> y(j_done);
  if (!tridiag_lowest_vec(j_done, ha.data(), hb.data(), &theta, y.data()))
    return set_err(HEFF_ECUDA, "lanczos_ground: tridiagonal QL did not converge");
  memcpy(h_y, y.data(), sizeof(double) * j_done);
  CK(cudaMemcpyAsync(ydev, h_y, sizeof(double) * j_done, cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(w, 0, sizeof(double) * nr, s));
  CKR(multiaxpy(p, V, j_done, ydev, 1.0, w, nr, s));   // real y: also right for complex V
  CKR(norm2(p, w, nr, beta + cap, invb + cap, s));
  if (compact) {  // psi = scatter(x), zero outside the sector
    scale_kernel<<<ew_grid(n), 256, 0, s>>>(w, invb + cap, w, n);
    CK(cudaMemsetAsync(psi, 0, sizeof(double) * n_dense, s));
    scatter_kernel<<<ew_grid(n), 256, 0, s>>>(w, p->qn_idx, n, psi);
    p->total_launches += 1;
  } else {
    scale_kernel<<<ew_grid(nr), 256, 0, s>>>(w, invb + cap, psi, nr);
  }
  ++p->total_launches;
  CK(cudaGetLastError());
  CKR(comm_wait(p, s));
  if (fgather) {
    p->epoch += (uint64_t)cap + 1;
    CK(cudaMemcpyAsync(h_n, d_timeout, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));  // the stream already drained (comm_wait above)
    int to = 0;
    memcpy(&to, h_n, sizeof(int));
    // a rank that timed out cannot resynchronise its flag epoch with peers that went on:
    // abort, so every rank's next collective fails instead of reading stale slots
    if (to) return comm_abort(p, "lanczos_ground: a peer never published its Krylov vector (20 s timeout)");
  }
  *energy = theta;
  if (iters_done) *iters_done = j_done;
  if (resid_est) *resid_est = hb[j_done - 1] * std::fabs(y[j_done - 1]);
  return HEFF_OK;
}

// --------------------------------------------------------------------------- environments
// NEXT-1: the environment update that follows each eigensolve in a sweep
// (Sec. 6.2; SPEC ProjMPO S:L737-755), built from the same kernels:
//   left:  X = L.A (NN GEMM) -> Y = W.X (MPO kernel, single-site CSR) -> Lout = A^T.Y (NN GEMM
//          on an explicitly transposed A)
//   right: X = B.R (NN GEMM) -> Y = W.X (MPO kernel) -> Rout = Y.B^T (NT GEMM)
static thread_local StreamWs t_env_splitws;

// Per-thread workspace of the environment updates, grown on demand and kept (no
// cudaMalloc/cudaFree per call; each call synchronises its stream before returning).
struct EnvArena {
  double* buf = nullptr;
  size_t bytes = 0;
  int* rowptr = nullptr;
  int* col = nullptr;
  double* val = nullptr;
  size_t csr_cap = 0;
};
static thread_local PerDev<EnvArena> t_env_arena;

static int env_reserve(size_t doubles) {
  EnvArena& a = t_env_arena();
  if (a.bytes >= doubles * sizeof(double)) return HEFF_OK;
  cudaFree(a.buf);
  a.buf = nullptr;
  a.bytes = 0;
  CK(cudaMalloc(&a.buf, doubles * sizeof(double)));
  a.bytes = doubles * sizeof(double);
  return HEFF_OK;
}

// The environment update's one-site MPO as CSR, built on the device into this thread's
// arena (mode kCsrSingle: left update, kCsrSingleR: right update).
static int env_csr(Csr& c, int mode, const double* W, int64_t kl, int64_t d, int64_t kr, cudaStream_t s) {
  EnvArena& a = t_env_arena();
  int64_t nrows = 0, nslots = 0;
  csr_shape(mode, kl, kr, d, d, &nrows, &nslots);
  const size_t need = (size_t)std::max<int64_t>(nrows + 2, nrows * nslots);
  if (a.csr_cap < need) {
    cudaFree(a.rowptr); cudaFree(a.col); cudaFree(a.val);
    a.rowptr = nullptr; a.col = nullptr; a.val = nullptr;
    a.csr_cap = 0;
    CK(cudaMalloc(&a.rowptr, sizeof(int) * need));
    CK(cudaMalloc(&a.col, sizeof(int) * need));
    CK(cudaMalloc(&a.val, sizeof(double) * need));
    a.csr_cap = need;
  }
  c.owned = false;
  c.d_rowptr = a.rowptr;
  c.d_col = a.col;
  c.d_val = a.val;
  c.d_nnz = a.rowptr + nrows + 1;
  return build_csr_dev(c, mode, W, nullptr, kl, 1, kr, d, d, s);
}

static int env_common_check(const heff_env_dims* d, const void* a, const void* b, const void* w, const void* o) {
  if (!d || !a || !b || !w || !o) return set_err(HEFF_EINVAL, "heff_env_update: null argument");
  if (d->mi < 1 || d->mo < 1 || d->d < 1 || d->kl < 1 || d->kr < 1)
    return set_err(HEFF_EINVAL, "heff_env_update: every dimension must be >= 1");
  if (d->kl * d->d > kMpoMaxRows || d->kr * d->d > kMpoMaxRows)
    return set_err(HEFF_EUNSUPPORTED, "heff_env_update: k d > %d", kMpoMaxRows);
  return init_device_once();
}

static int build_sparse_schedule(int64_t M, int64_t N, const std::vector<int>& rowv, const std::vector<int>& colv,
                                 const std::vector<std::vector<int>>& kvals, int** d_out, int64_t* total_kb,
                                 const int** order, const int** ptr, const int** list, int64_t* makespan,
                                 int* order_len);
static bool sparse_worth_it(int64_t M, int64_t N, int64_t K, int64_t makespan);

// U(1) schedules of the environment GEMMs (heff_env_update_*_qn); per-thread device buffers
static thread_local PerDev<int*> t_env_sp1 = {};
static thread_local PerDev<int*> t_env_sp3 = {};

// block-sparse schedule for one environment GEMM if charges are given and it pays off
static int env_schedule(GemmOp& g, const std::vector<int>& rowv, const std::vector<int>& colv,
                        const std::vector<std::vector<int>>& kvals, int** buf) {
  int64_t tot = 0, span = 0;
  CKR(build_sparse_schedule(g.M, g.N, rowv, colv, kvals, buf, &tot, &g.sp_order, &g.sp_ptr, &g.sp_list, &span,
                            &g.sp_len));
  if (!sparse_worth_it(g.M, g.N, g.K, span)) { g.sp_order = g.sp_ptr = g.sp_list = nullptr; g.sp_len = 0; }
  return HEFF_OK;
}

static std::vector<std::vector<int>> kblock_values(int64_t K, const std::function<int(int64_t)>& val) {
  std::vector<std::vector<int>> kv((K + kGemmBK - 1) / kGemmBK);
  for (int64_t k = 0; k < K; ++k) {
    auto& v = kv[k / kGemmBK];
    const int x = val(k);
    if (std::find(v.begin(), v.end(), x) == v.end()) v.push_back(x);
  }
  return kv;
}

static int env_left_impl(const heff_env_dims* dims, const double* L, const double* A, const double* W, double* Lout,
                         const heff_env_qn* qn, heff_stream stream) {
  CKR(env_common_check(dims, L, A, W, Lout));
  const heff_env_dims d = *dims;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!is_device_ptr(W)) return set_err(HEFF_EINVAL, "heff_env_update_left: W is not a device pointer");
  Csr csr;  // rows (s',w'), cols (w,s), built on the device
  auto pad = [](int64_t x) { return (x + 31) / 32 * 32; };  // keep every sub-buffer 256-byte aligned
  const int64_t nX = pad(d.mi * d.kl * d.d * d.mo), nY = pad(d.mi * d.d * d.kr * d.mo), nA = pad(d.mi * d.d * d.mo);
  CKR(env_reserve((size_t)(nX + nY + nA)));
  CKR(env_csr(csr, kCsrSingle, W, d.kl, d.d, d.kr, s));
  double* X = t_env_arena().buf;
  double* Y = X + nX;
  double* At = Y + nY;
  auto cleanup = [&]() { cudaStreamSynchronize(s); };
  int r = HEFF_OK;
  int nl = 0;
  GemmOp g1;  // X[(x' w), (s a)] = L[(x' w), x] . A[x, (s a)]
  g1.M = d.mi * d.kl; g1.N = d.d * d.mo; g1.K = d.mi;
  g1.A = L; g1.lda = d.mi; g1.B = A; g1.ldb = d.d * d.mo; g1.b_kmajor = false; g1.C = X; g1.ldc = d.d * d.mo;
  GemmOp g3;  // Lout[a', (w' a)] = At[a', (x' s')] . Y[(x' s')][(w' a)]
  g3.M = d.mo; g3.N = d.kr * d.mo; g3.K = d.mi * d.d;
  g3.A = At; g3.lda = d.mi * d.d; g3.B = Y; g3.ldb = d.kr * d.mo; g3.b_kmajor = false; g3.C = Lout;
  g3.ldc = d.kr * d.mo;
  if (qn) {  // U(1): contracted x needs q(x') - c(w) (rows) = q(a) - q(s) (columns); then q(x') + q(s')
    std::vector<int> rowv(g1.M), colv(g1.N), rowv3(g3.M), colv3(g3.N);
    for (int64_t x = 0; x < d.mi; ++x)
      for (int64_t w = 0; w < d.kl; ++w) rowv[x * d.kl + w] = qn->q_in[x] - qn->cl[w];
    for (int64_t sg = 0; sg < d.d; ++sg)
      for (int64_t a = 0; a < d.mo; ++a) colv[sg * d.mo + a] = qn->q_out[a] - qn->qs[sg];
    CKR(env_schedule(g1, rowv, colv, kblock_values(g1.K, [&](int64_t k) { return qn->q_in[k]; }), &t_env_sp1()));
    for (int64_t a = 0; a < d.mo; ++a) rowv3[a] = qn->q_out[a];
    for (int64_t wp = 0; wp < d.kr; ++wp)
      for (int64_t a = 0; a < d.mo; ++a) colv3[wp * d.mo + a] = qn->q_out[a] + qn->cr[wp];
    CKR(env_schedule(g3, rowv3, colv3,
                     kblock_values(g3.K, [&](int64_t k) { return qn->q_in[k / d.d] + qn->qs[k % d.d]; }),
                     &t_env_sp3()));
  }
  r = launch_gemm(g1, 0, s, &nl, ws_for(t_env_splitws, s));
  if (!r) {
    const int nin = (int)(d.kl * d.d), nout = (int)(d.d * d.kr);
    r = launch_mpo_A(X, Y, d.mo, d.mi, nin, nout, csr, nullptr, mpo_tile_cols(nin), s);
    dim3 tg((unsigned)((d.mo + 31) / 32), (unsigned)((d.mi * d.d + 31) / 32));
    transpose_kernel<<<tg, dim3(32, 8), 0, s>>>(A, At, d.mi * d.d, d.mo);
    if (cudaGetLastError() != cudaSuccess) r = set_err(HEFF_ECUDA, "heff_env_update_left: launch failed");
  }
  if (!r) r = launch_gemm(g3, 0, s, &nl, ws_for(t_env_splitws, s));
  cleanup();
  return r;
}

extern "C" int heff_env_update_left(const heff_env_dims* dims, const double* L, const double* A, const double* W,
                                    double* Lout, heff_stream stream) {
  return env_left_impl(dims, L, A, W, Lout, nullptr, stream);
}

extern "C" int heff_env_update_left_qn(const heff_env_dims* dims, const double* L, const double* A, const double* W,
                                       double* Lout, const heff_env_qn* qn, heff_stream stream) {
  if (!qn || !qn->q_in || !qn->q_out || !qn->qs || !qn->cl || !qn->cr)
    return set_err(HEFF_EINVAL, "heff_env_update_left_qn: null charge array");
  return env_left_impl(dims, L, A, W, Lout, qn, stream);
}

static int env_right_impl(const heff_env_dims* dims, const double* R, const double* B, const double* W, double* Rout,
                          const heff_env_qn* qn, heff_stream stream) {
  CKR(env_common_check(dims, R, B, W, Rout));
  const heff_env_dims d = *dims;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!is_device_ptr(W)) return set_err(HEFF_EINVAL, "heff_env_update_right: W is not a device pointer");
  Csr csr;  // rows (w,s), cols (s',w'), built on the device
  auto pad = [](int64_t x) { return (x + 31) / 32 * 32; };
  const int64_t nX = pad(d.mo * d.d * d.kr * d.mi), nY = pad(d.mo * d.kl * d.d * d.mi);
  CKR(env_reserve((size_t)(nX + nY)));
  CKR(env_csr(csr, kCsrSingleR, W, d.kl, d.d, d.kr, s));
  double* X = t_env_arena().buf;
  double* Y = X + nX;
  auto cleanup = [&]() { cudaStreamSynchronize(s); };
  int r = HEFF_OK;
  int nl = 0;
  GemmOp g1;  // X[(b' s'), (w' y)] = B[(b' s'), y'] . R[y', (w' y)]
  g1.M = d.mo * d.d; g1.N = d.kr * d.mi; g1.K = d.mi;
  g1.A = B; g1.lda = d.mi; g1.B = R; g1.ldb = d.kr * d.mi; g1.b_kmajor = false; g1.C = X; g1.ldc = d.kr * d.mi;
  GemmOp g3;  // Rout[(b' w), b] = Y[(b' w), (s y)] . B[b, (s y)]^T
  g3.M = d.mo * d.kl; g3.N = d.mo; g3.K = d.d * d.mi;
  g3.A = Y; g3.lda = d.d * d.mi; g3.B = B; g3.ldb = d.d * d.mi; g3.b_kmajor = true; g3.C = Rout; g3.ldc = d.mo;
  if (qn) {  // U(1): contracted y' = q(b') + q(s') (rows) = q(y) + c(w') (columns); then q(y) - q(s)
    std::vector<int> rowv(g1.M), colv(g1.N), rowv3(g3.M), colv3(g3.N);
    for (int64_t b = 0; b < d.mo; ++b)
      for (int64_t sg = 0; sg < d.d; ++sg) rowv[b * d.d + sg] = qn->q_out[b] + qn->qs[sg];
    for (int64_t wp = 0; wp < d.kr; ++wp)
      for (int64_t y = 0; y < d.mi; ++y) colv[wp * d.mi + y] = qn->q_in[y] + qn->cr[wp];
    CKR(env_schedule(g1, rowv, colv, kblock_values(g1.K, [&](int64_t k) { return qn->q_in[k]; }), &t_env_sp1()));
    for (int64_t b = 0; b < d.mo; ++b)
      for (int64_t w = 0; w < d.kl; ++w) rowv3[b * d.kl + w] = qn->q_out[b] - qn->cl[w];
    for (int64_t b = 0; b < d.mo; ++b) colv3[b] = qn->q_out[b];
    CKR(env_schedule(g3, rowv3, colv3,
                     kblock_values(g3.K, [&](int64_t k) { return qn->q_in[k % d.mi] - qn->qs[k / d.mi]; }),
                     &t_env_sp3()));
  }
  r = launch_gemm(g1, 0, s, &nl, ws_for(t_env_splitws, s));
  if (!r) {
    const int nin = (int)(d.d * d.kr), nout = (int)(d.kl * d.d);
    r = launch_mpo_A(X, Y, d.mi, d.mo, nin, nout, csr, nullptr, mpo_tile_cols(nin), s);
    if (cudaGetLastError() != cudaSuccess) r = set_err(HEFF_ECUDA, "heff_env_update_right: launch failed");
  }
  if (!r) r = launch_gemm(g3, 0, s, &nl, ws_for(t_env_splitws, s));
  cleanup();
  return r;
}

extern "C" int heff_env_update_right(const heff_env_dims* dims, const double* R, const double* B, const double* W,
                                     double* Rout, heff_stream stream) {
  return env_right_impl(dims, R, B, W, Rout, nullptr, stream);
}

extern "C" int heff_env_update_right_qn(const heff_env_dims* dims, const double* R, const double* B, const double* W,
                                        double* Rout, const heff_env_qn* qn, heff_stream stream) {
  if (!qn || !qn->q_in || !qn->q_out || !qn->qs || !qn->cl || !qn->cr)
    return set_err(HEFF_EINVAL, "heff_env_update_right_qn: null charge array");
  return env_right_impl(dims, R, B, W, Rout, qn, stream);
}

// Host-only: lanczos_ground's per-step check (Sturm bisection + inverse iteration, tridiag.h).
extern "C" int heff_tridiag_lowest_check(int j, const double* alpha, const double* beta, double* theta,
                                         double* ylast) {
  if (j < 1 || !alpha || !theta || !ylast || (j > 1 && !beta))
    return set_err(HEFF_EINVAL, "heff_tridiag_lowest_check: bad argument");
  if (!tridiag_lowest_fast(j, alpha, beta, theta, ylast))
    return set_err(HEFF_ECUDA, "heff_tridiag_lowest_check: inverse iteration failed");
  return HEFF_OK;
}

// Host-only: the tridiagonal eigen-solve lanczos_ground uses (implicit QL, tridiag.h).
extern "C" int heff_tridiag_lowest(int j, const double* alpha, const double* beta, double* theta, double* y) {
  if (j < 1 || !alpha || !theta || (j > 1 && !beta)) return set_err(HEFF_EINVAL, "heff_tridiag_lowest: bad argument");
  std::vector<double> yy(j);
  if (!tridiag_lowest_vec(j, alpha, beta, theta, yy.data()))
    return set_err(HEFF_ECUDA, "heff_tridiag_lowest: QL iteration did not converge");
  if (y) memcpy(y, yy.data(), sizeof(double) * j);
  return HEFF_OK;
}

// The FP64 GEMM primitive of the hot path, exposed for kernel-level tests and reuse:
// C[M][N] (+)= A[M][K] . op(B), op(B) = B[K][N] (b_kmajor = 0) or B[N][K]^T (b_kmajor = 1).
static thread_local StreamWs t_gemm_ws;
extern "C" int heff_gemm(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B, int64_t ldb,
                         int b_kmajor, double* C, int64_t ldc, int accumulate, int path, heff_stream stream) {
  if (M < 0 || N < 0 || K < 0 || !A || !B || !C || path < 0 || path > 2)
    return set_err(HEFF_EINVAL, "heff_gemm: bad argument");
  CKR(init_device_once());
  GemmOp g;
  g.M = M; g.N = N; g.K = K; g.A = A; g.lda = lda; g.B = B; g.ldb = ldb; g.b_kmajor = b_kmajor != 0;
  g.C = C; g.ldc = ldc; g.accumulate = accumulate ? 1 : 0;
  int nl = 0;
  const cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  return launch_gemm(g, path, cs, &nl, ws_for(t_gemm_ws, cs));
}

// debug: enable (n > 0: a device buffer of 4 n timers) / read back the fused small-bond
// kernel's per-CTA %globaltimer stamps (entry, after the dependency wait, after the main
// loop, exit); host buffer `out` of 4 n values, n = 0 disables
// Diagnostics (not in heff.h): launch-cost probe for the Lanczos step kernels.  which:
// 0 empty kernel, 1 empty kernel with PDL + griddepcontrol.wait, 2 cgs2_step_small_kernel
// (n, j) with PDL, 3 the same without PDL, 4 cgs2_step_kernel one block, 5 cgs2_step_smem_kernel,
// 6 cgs2_step_kernel cooperative on its lanczos_ground grid; `reps` launches back to back, device
// time per launch in *us.  Scratch buffers are allocated and freed here.
__global__ void probe_empty_kernel(int x) {
  if (x == 12345) printf("x");
}
__global__ void probe_empty_pdl_kernel(int x) {
  pdl_wait();
  if (x == 12345) printf("x");
}
extern "C" int heff_debug_launch_probe(int which, int64_t n, int j, int reps, float* us) {
  CKR(init_device_once());
  double* buf = nullptr;
  const int64_t ldv = (n + 31) / 32 * 32;
  const size_t extra = (size_t)64 * 1024 + (size_t)(2 * 4096 + 8) * 8 * 148;  // scalars + partials
  CK(cudaMalloc(&buf, sizeof(double) * ((size_t)ldv * (j + 2) + extra)));
  CK(cudaMemset(buf, 0, sizeof(double) * ((size_t)ldv * (j + 2) + extra)));
  double* V = buf;
  double* w = buf + ldv * (j + 1);
  double* sc = buf + ldv * (j + 2);
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto launch = [&]() -> cudaError_t {
    switch (which) {
      case 0: probe_empty_kernel<<<1, 32, 0, s>>>(0); return cudaGetLastError();
      case 1: return launch_pdl(probe_empty_pdl_kernel, dim3(1), dim3(32), 0, s, 0);
      case 2:
        return launch_pdl(cgs2_step_small_kernel, dim3(1), dim3(kSmallStepThreads), sizeof(double) * (size_t)(j + 1), s,
                          (const double*)V, ldv, j, w, n, sc, sc + 4096, sc + 8192, sc + 12288, sc + 16384,
                          V + (int64_t)j * ldv);
      case 3:
        cgs2_step_small_kernel<<<1, kSmallStepThreads, sizeof(double) * (size_t)(j + 1), s>>>(
            V, ldv, j, w, n, sc, sc + 4096, sc + 8192, sc + 12288, sc + 16384, V + (int64_t)j * ldv);
        return cudaGetLastError();
      case 5:
        return launch_pdl(cgs2_step_smem_kernel, dim3(1), dim3(kSmemStepThreads), (size_t)(j * ((n + 1) & ~1ll) * 8), s,
                          (const double*)V, ldv, j, w, n, sc, sc + 4096, sc + 8192, sc + 12288, sc + 16384,
                          V + (int64_t)j * ldv);
      case 6: {  // the cooperative multi-block step as lanczos_ground launches it (one element per thread)
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cgs2_step_kernel, kStepThreads,
                                                      sizeof(double) * (size_t)(j + 1));
        const int G = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * g_num_sms, (n + kStepThreads - 1) / kStepThreads));
        const double* Vc = V;
        int64_t ldv_ = ldv, nn = n;
        int jj = j, jmax = 4096;
        double* partial = sc + 20480;
        double *c1 = sc, *c2 = sc + 4096, *al = sc + 8192, *be = sc + 12288, *ib = sc + 16384;
        double* vn = V + (int64_t)j * ldv;
        double* wp = w;
        unsigned int* gb = nullptr;
        void* args[] = {(void*)&Vc, &ldv_, &jj, &wp, &nn, &partial, &jmax, &c1, &c2, &al, &be, &ib, &vn, &gb};
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(G);
        cfg.blockDim = dim3(kStepThreads);
        cfg.dynamicSmemBytes = sizeof(double) * (size_t)(j + 1);
        cfg.stream = s;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        return cudaLaunchKernelExC(&cfg, (const void*)cgs2_step_kernel, args);
      }
      default:
        cgs2_step_kernel<<<1, kStepThreads, sizeof(double) * (size_t)(j + 1), s>>>(
            V, ldv, j, w, n, sc + 20480, 4096, sc, sc + 4096, sc + 8192, sc + 12288, sc + 16384, V + (int64_t)j * ldv,
            nullptr);
        return cudaGetLastError();
    }
  };
  for (int i = 0; i < 3; ++i) CK(launch());
  cudaEventRecord(e0, s);
  for (int i = 0; i < reps; ++i) CK(launch());
  cudaEventRecord(e1, s);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  *us = ms * 1e3f / (float)reps;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(s);
  cudaFree(buf);
  return HEFF_OK;
}

extern "C" int heff_debug_fused_timestamps(int n, unsigned long long* out) {
  if (const char* e = getenv("HEFF_DEBUG_FUSED_MODE")) g_fused_dbg_mode = atoi(e);
  if (n <= 0) {
    g_fused_dbg_mode = 0;
    cudaFree(g_fused_dbg);
    g_fused_dbg = nullptr;
    g_cluster_dbg = nullptr;
    return HEFF_OK;
  }
  if (!g_fused_dbg) {
    CK(cudaMalloc(&g_fused_dbg, sizeof(unsigned long long) * 8 * (size_t)n));
    CK(cudaMemset(g_fused_dbg, 0, sizeof(unsigned long long) * 8 * (size_t)n));
  }
  if (!g_cluster_dbg) g_cluster_dbg = g_fused_dbg + 8 * (size_t)(n / 2);  // second half: the cluster GEMM
  if (out) CK(cudaMemcpy(out, g_fused_dbg, sizeof(unsigned long long) * 8 * (size_t)n, cudaMemcpyDeviceToHost));
  return HEFF_OK;
}

// debug: copy the calling thread's heff_gemm stream-K workspace (partial tiles of its
// first stream) to dst
extern "C" int heff_debug_gemm_ws(double* dst, size_t bytes) {
  if (t_gemm_ws.empty() || !t_gemm_ws[0].second.ptr) return set_err(HEFF_EINVAL, "no workspace");
  const SplitWs& w = t_gemm_ws[0].second;
  CK(cudaMemcpy(dst, w.ptr, std::min(bytes, w.bytes), cudaMemcpyDeviceToDevice));
  return HEFF_OK;
}

// --------------------------------------------------------------------------- U(1) block sparsity
// NEXT-3: QN-conserving H_eff (Sec. 7).  The tensors stay
// dense and sector-sorted; heff_set_qn builds, per GEMM output tile, the list of k-blocks
// whose (row, column) charge constraints can both be met, and the GEMM kernel visits only
// those (tiles in descending-work order, round-robin over the SMs).  Tiles with an empty
// list are written as zeros.
static std::vector<std::vector<int>> kblocks_by_value(const std::vector<int>& kval_lo, const std::vector<int>& kval_hi,
                                                      const std::vector<std::vector<int>>& kvals, int vmin, int vmax) {
  (void)kval_lo;
  (void)kval_hi;
  std::vector<std::vector<int>> inv(vmax - vmin + 1);
  for (size_t kb = 0; kb < kvals.size(); ++kb)
    for (int v : kvals[kb]) inv[v - vmin].push_back((int)kb);
  return inv;
}

// rowv[r], colv[c]: the charge each output row / column requires of the contracted index;
// kvals[kb]: the charges present in k-block kb.  Returns order | ptr | list in one buffer.
static int build_sparse_schedule(int64_t M, int64_t N, const std::vector<int>& rowv, const std::vector<int>& colv,
                                 const std::vector<std::vector<int>>& kvals, int** d_out, int64_t* total_kb,
                                 const int** order, const int** ptr, const int** list, int64_t* makespan,
                                 int* order_len) {
  const int num_m = (int)((M + kBM - 1) / kBM), num_n = (int)((N + kBN - 1) / kBN);
  const int tiles = num_m * num_n;
  int vmin = INT32_MAX, vmax = INT32_MIN;
  for (auto& kv : kvals)
    for (int v : kv) { vmin = std::min(vmin, v); vmax = std::max(vmax, v); }
  if (vmin > vmax) { vmin = 0; vmax = 0; }
  auto inv = kblocks_by_value({}, {}, kvals, vmin, vmax);
  auto tile_set = [&](const std::vector<int>& vals, int64_t lo, int64_t hi) {
    std::vector<int> v(vals.begin() + lo, vals.begin() + hi);
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    return v;
  };
  std::vector<std::vector<int>> setM(num_m), setN(num_n);
  for (int mb = 0; mb < num_m; ++mb) setM[mb] = tile_set(rowv, (int64_t)mb * kBM, std::min<int64_t>(M, (int64_t)(mb + 1) * kBM));
  for (int nb = 0; nb < num_n; ++nb) setN[nb] = tile_set(colv, (int64_t)nb * kBN, std::min<int64_t>(N, (int64_t)(nb + 1) * kBN));
  std::vector<std::vector<int>> lists(tiles);
  int64_t tot = 0;
  std::vector<int> I, kb;
  for (int t = 0; t < tiles; ++t) {
    int mb, nb;
    tile_coords(t, num_m, num_n, kGroupM, mb, nb);
    I.clear();
    std::set_intersection(setM[mb].begin(), setM[mb].end(), setN[nb].begin(), setN[nb].end(), std::back_inserter(I));
    kb.clear();
    for (int v : I)
      if (v >= vmin && v <= vmax) kb.insert(kb.end(), inv[v - vmin].begin(), inv[v - vmin].end());
    std::sort(kb.begin(), kb.end());
    kb.erase(std::unique(kb.begin(), kb.end()), kb.end());
    lists[t] = kb;
    tot += (int64_t)kb.size();
  }
  std::vector<int> byw(tiles);
  for (int t = 0; t < tiles; ++t) byw[t] = t;
  std::stable_sort(byw.begin(), byw.end(), [&](int a, int b) { return lists[a].size() > lists[b].size(); });
  // LPT: tiles in descending work (k-blocks + ~2 of per-tile overhead) each to the least
  // loaded of the G CTAs (ties: lowest index); the kernel walks CTA b's list as entries
  // b, b+G, ... of `ord`, padded with -1 to the longest list
  const int G = std::min<int>(tiles, g_num_sms);
  std::vector<std::vector<int>> per(G);
  if (getenv("HEFF_QN_ROUND_ROBIN")) {  // the plain round-robin over `byw` (comparison knob)
    int64_t span = 0;
    for (int b = 0; b < G; ++b) {
      int64_t l = 0;
      for (int i = b; i < tiles; i += G) {
        per[b].push_back(byw[i]);
        l += (int64_t)lists[byw[i]].size() + 2;
      }
      span = std::max(span, l);
    }
    *makespan = span;
  } else {
    using Load = std::pair<int64_t, int>;
    std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
    for (int b = 0; b < G; ++b) heap.push({0, b});
    int64_t span = 0;
    for (int t : byw) {
      Load l = heap.top();
      heap.pop();
      per[l.second].push_back(t);
      l.first += (int64_t)lists[t].size() + 2;
      span = std::max(span, l.first);
      heap.push(l);
    }
    *makespan = span;
  }
  size_t cmax = 0;
  for (auto& v : per) cmax = std::max(cmax, v.size());
  std::vector<int> ord((size_t)G * cmax, -1);
  for (int b = 0; b < G; ++b)
    for (size_t i = 0; i < per[b].size(); ++i) ord[i * G + b] = per[b][i];
  *order_len = (int)ord.size();
  std::vector<int> buf;
  buf.reserve(ord.size() + (size_t)tiles + 1 + (size_t)tot);
  buf.insert(buf.end(), ord.begin(), ord.end());
  int64_t acc = 0;
  for (int t = 0; t < tiles; ++t) { buf.push_back((int)acc); acc += (int64_t)lists[t].size(); }
  buf.push_back((int)acc);
  for (int t = 0; t < tiles; ++t) buf.insert(buf.end(), lists[t].begin(), lists[t].end());
  if (acc > INT32_MAX) return set_err(HEFF_EUNSUPPORTED, "heff_set_qn: schedule too large");
  cudaFree(*d_out);
  *d_out = nullptr;
  CK(cudaMalloc(d_out, sizeof(int) * buf.size()));
  CK(cudaMemcpy(*d_out, buf.data(), sizeof(int) * buf.size(), cudaMemcpyHostToDevice));
  *order = *d_out;
  *ptr = *d_out + ord.size();
  *list = *d_out + ord.size() + tiles + 1;
  *total_kb = tot;
  return HEFF_OK;
}

static int64_t dense_kblock_tiles(int64_t M, int64_t N, int64_t K) {
  return ((M + kBM - 1) / kBM) * ((N + kBN - 1) / kBN) * ((K + kGemmBK - 1) / kGemmBK);
}

// The block-sparse schedule runs whole tiles data-parallel (no stream-K): use it when it
// removes at least 30% of the work and there are enough tiles to fill the SMs.
// Estimated critical path (busiest SM's k-blocks) of the sparse round-robin schedule vs
// the perfectly balanced dense stream-K schedule.
static bool sparse_worth_it(int64_t M, int64_t N, int64_t K, int64_t makespan) {
  if (getenv("HEFF_QN_FORCE_SPARSE")) return true;
  const double dense_span = (double)dense_kblock_tiles(M, N, K) / g_num_sms;
  return (double)makespan < 0.85 * dense_span;
}

extern "C" int heff_set_qn(heff_plan p, const heff_qn* qn) {
  if (!p) return set_err(HEFF_EINVAL, "heff_set_qn: null plan");
  if (!qn) {  // back to dense
    cudaFree(p->sp1); cudaFree(p->sp4); cudaFree(p->mpo_live);
    cudaDeviceSynchronize();
    cudaFree(p->qn_idx); ws_release(p->dense_in); ws_release(p->dense_out);
    p->sp1 = p->sp4 = nullptr;
    p->mpo_live = nullptr;
    p->qn_idx = nullptr;
    p->dense_in = p->dense_out = nullptr;
    p->qn_n = 0;
    p->g1.sp_order = p->g1.sp_ptr = p->g1.sp_list = nullptr; p->g1.sp_len = 0;
    p->g4.sp_order = p->g4.sp_ptr = p->g4.sp_list = nullptr; p->g4.sp_len = 0;
    p->sp_kblocks = 0;
    return HEFF_OK;
  }
  if (p->sharded || !p->terms.empty() || p->is_complex)
    return set_err(HEFF_EUNSUPPORTED, "heff_set_qn: single-GPU real order-A plans only (set it on each term of a sum)");
  const heff_dims& d = p->dims;
  if (p->chunk_rows != d.mL) return set_err(HEFF_EUNSUPPORTED, "heff_set_qn: plan is chunked over a' (workspace budget)");
  if (!qn->qa || !qn->qb || !qn->qs1 || !qn->qs2 || !qn->cL || !qn->cR)
    return set_err(HEFF_EINVAL, "heff_set_qn: null charge array");
  for (int64_t i = 1; i < d.mL; ++i)
    if (qn->qa[i] < qn->qa[i - 1]) return set_err(HEFF_EINVAL, "heff_set_qn: qa must be nondecreasing");
  for (int64_t i = 1; i < d.mR; ++i)
    if (qn->qb[i] < qn->qb[i - 1]) return set_err(HEFF_EINVAL, "heff_set_qn: qb must be nondecreasing");
  // GEMM1: rows (a',w) need q(a) = qa[a'] - cL[w]; columns (s1,s2,b) need q(a) = qb[b] - qs1 - qs2
  {
    const int64_t M = d.mL * d.kL, N = d.d1 * d.d2 * d.mR, K = d.mL;
    std::vector<int> rowv(M), colv(N);
    for (int64_t ap = 0; ap < d.mL; ++ap)
      for (int64_t w = 0; w < d.kL; ++w) rowv[ap * d.kL + w] = qn->qa[ap] - qn->cL[w];
    for (int64_t s1 = 0; s1 < d.d1; ++s1)
      for (int64_t s2 = 0; s2 < d.d2; ++s2)
        for (int64_t b = 0; b < d.mR; ++b) colv[(s1 * d.d2 + s2) * d.mR + b] = qn->qb[b] - qn->qs1[s1] - qn->qs2[s2];
    std::vector<std::vector<int>> kvals((K + kGemmBK - 1) / kGemmBK);
    for (int64_t a = 0; a < K; ++a) {
      auto& v = kvals[a / kGemmBK];
      if (v.empty() || v.back() != qn->qa[a]) v.push_back(qn->qa[a]);
    }
    int64_t tot = 0, span = 0;
    CKR(build_sparse_schedule(M, N, rowv, colv, kvals, &p->sp1, &tot, &p->g1.sp_order, &p->g1.sp_ptr, &p->g1.sp_list,
                              &span, &p->g1.sp_len));
    p->sp_kblocks = tot;
    if (!sparse_worth_it(M, N, K, span)) {  // dense (stream-K) schedule is faster here
      p->g1.sp_order = p->g1.sp_ptr = p->g1.sp_list = nullptr; p->g1.sp_len = 0;
      p->sp_kblocks = dense_kblock_tiles(M, N, K);
    }
  }
  // GEMM4: rows (a',s1',s2') and columns b' both fix q(b) + cR[w2] for the contracted (w2, b)
  {
    const int64_t M = d.mL * d.d1 * d.d2, N = d.mR, K = d.kR * d.mR;
    std::vector<int> rowv(M), colv(N);
    for (int64_t ap = 0; ap < d.mL; ++ap)
      for (int64_t s1 = 0; s1 < d.d1; ++s1)
        for (int64_t s2 = 0; s2 < d.d2; ++s2) rowv[(ap * d.d1 + s1) * d.d2 + s2] = qn->qa[ap] + qn->qs1[s1] + qn->qs2[s2];
    for (int64_t b = 0; b < d.mR; ++b) colv[b] = qn->qb[b];
    std::vector<std::vector<int>> kvals((K + kGemmBK - 1) / kGemmBK);
    for (int64_t w2 = 0; w2 < d.kR; ++w2)
      for (int64_t b = 0; b < d.mR; ++b) {
        auto& v = kvals[(w2 * d.mR + b) / kGemmBK];
        const int val = qn->qb[b] + qn->cR[w2];
        if (std::find(v.begin(), v.end(), val) == v.end()) v.push_back(val);
      }
    int64_t tot = 0, span = 0;
    CKR(build_sparse_schedule(M, N, rowv, colv, kvals, &p->sp4, &tot, &p->g4.sp_order, &p->g4.sp_ptr, &p->g4.sp_list,
                              &span, &p->g4.sp_len));
    if (!sparse_worth_it(M, N, K, span)) {
      p->g4.sp_order = p->g4.sp_ptr = p->g4.sp_list = nullptr; p->g4.sp_len = 0;
      tot = dense_kblock_tiles(M, N, K);
    }
    p->sp_kblocks += tot;
  }
  // MPO blocks (a', tcA-column b tile): live iff some (w,s1,s2) input or (s1',s2',w2) output
  // entry of the block is allowed; the rest are skipped and their T3 entries stay zero.
  {
    const int tc = p->tcA;  // the MPO kernel's column tile
    const int nbt = (int)((d.mR + tc - 1) / tc);
    std::vector<unsigned char> live((size_t)d.mL * nbt, 0);
    std::vector<int> in_off, out_off;  // charge offsets: q(b) must equal qa[a'] + off
    for (int64_t w = 0; w < d.kL; ++w)
      for (int64_t s1 = 0; s1 < d.d1; ++s1)
        for (int64_t s2 = 0; s2 < d.d2; ++s2) in_off.push_back(qn->qs1[s1] + qn->qs2[s2] - qn->cL[w]);
    for (int64_t s1 = 0; s1 < d.d1; ++s1)
      for (int64_t s2 = 0; s2 < d.d2; ++s2)
        for (int64_t w2 = 0; w2 < d.kR; ++w2) out_off.push_back(qn->qs1[s1] + qn->qs2[s2] - qn->cR[w2]);
    std::vector<int> offs(in_off);
    offs.insert(offs.end(), out_off.begin(), out_off.end());
    std::sort(offs.begin(), offs.end());
    offs.erase(std::unique(offs.begin(), offs.end()), offs.end());
    for (int t = 0; t < nbt; ++t) {
      const int64_t b0 = (int64_t)t * tc, b1 = std::min<int64_t>(d.mR, b0 + tc);
      std::vector<int> tq(qn->qb + b0, qn->qb + b1);
      tq.erase(std::unique(tq.begin(), tq.end()), tq.end());  // qb sorted
      for (int64_t ap = 0; ap < d.mL; ++ap) {
        bool on = false;
        for (int o : offs) {
          if (std::binary_search(tq.begin(), tq.end(), qn->qa[ap] + o)) { on = true; break; }
        }
        live[(size_t)ap * nbt + t] = on ? 1 : 0;
      }
    }
    cudaFree(p->mpo_live);
    p->mpo_live = nullptr;
    CK(cudaMalloc(&p->mpo_live, live.size()));
    CK(cudaMemcpy(p->mpo_live, live.data(), live.size(), cudaMemcpyHostToDevice));
    CK(cudaMemset(p->T3, 0, sizeof(double) * d.mL * d.d1 * d.d2 * d.kR * d.mR));
  }
  // sector positions of psi: for each (a,s1,s2) the b-range with qb[b] = qa[a] + qs1 + qs2
  {
    std::vector<int> idx;
    const int64_t n = d.mL * d.d1 * d.d2 * d.mR;
    if (n <= INT32_MAX) {
      for (int64_t a = 0; a < d.mL; ++a)
        for (int64_t s1 = 0; s1 < d.d1; ++s1)
          for (int64_t s2 = 0; s2 < d.d2; ++s2) {
            const int q = qn->qa[a] + qn->qs1[s1] + qn->qs2[s2];
            const int* lo = std::lower_bound(qn->qb, qn->qb + d.mR, q);
            const int* hi = std::upper_bound(qn->qb, qn->qb + d.mR, q);
            const int64_t base = ((a * d.d1 + s1) * d.d2 + s2) * d.mR;
            for (const int* b = lo; b < hi; ++b) idx.push_back((int)(base + (b - qn->qb)));
          }
      cudaDeviceSynchronize();
      cudaFree(p->qn_idx);
      ws_release(p->dense_in);
      ws_release(p->dense_out);
      p->qn_idx = nullptr;
      p->dense_in = p->dense_out = nullptr;
      p->qn_n = (int64_t)idx.size();
      if (p->qn_n > 0) {
        CK(cudaMalloc(&p->qn_idx, sizeof(int) * idx.size()));
        CK(cudaMemcpy(p->qn_idx, idx.data(), sizeof(int) * idx.size(), cudaMemcpyHostToDevice));
      }
    }
  }
  return HEFF_OK;
}

__global__ void gather_kernel(const double* __restrict__ dense, const int* __restrict__ idx, int64_t n,
                              double* __restrict__ compact) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    compact[i] = dense[idx[i]];
}

__global__ void scatter_kernel(const double* __restrict__ compact, const int* __restrict__ idx, int64_t n,
                               double* __restrict__ dense) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dense[idx[i]] = compact[i];
}

// Host wrapper of transpose_kernel for the split (split_api.cu): dst[c][r] = src[r][c].
int launch_transpose(const double* src, double* dst, int64_t rows, int64_t cols, cudaStream_t s) {
  dim3 tg((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  transpose_kernel<<<tg, dim3(32, 8), 0, s>>>(src, dst, rows, cols);
  CK(cudaGetLastError());
  return HEFF_OK;
}

// --------------------------------------------------------------------------- cache release
// Frees the calling thread's on-demand workspaces (environment update, GEMM primitive,
// split and U(1) split arenas) and those of the U(1) split's worker threads.
void release_thread_caches() {
  auto freews = [](SplitWs& w) {
    cudaFree(w.ptr);
    cudaFree(w.sync);
    w = SplitWs();
  };
  for (auto& e : t_env_splitws) freews(e.second);
  t_env_splitws.clear();
  for (auto& e : t_gemm_ws) freews(e.second);
  t_gemm_ws.clear();
  t_env_arena.each([](EnvArena& a) {
    cudaFree(a.buf); cudaFree(a.rowptr); cudaFree(a.col); cudaFree(a.val);
    a = EnvArena();
  });
  split_release_thread_caches();
}

extern "C" int heff_release_caches(void) {
  release_thread_caches();
  int dev = 0;
  CK(cudaGetDevice(&dev));
  CKR(split_release_worker_caches(dev));
  CK(cudaDeviceSynchronize());
  {  // the plan workspace cache (blocks of destroyed plans) on this device
    std::lock_guard<std::mutex> lock(g_ws_mu);
    ws_cache_trim(dev);
  }
  pin_trim();
  return HEFF_OK;
}
