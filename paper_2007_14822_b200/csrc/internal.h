// internal.h -- host-side declarations shared by libheff's translation units
// (heff_api.cu: plans, matvec, Lanczos, environments, U(1) schedules, GEMM launch;
// split_api.cu: the two-site split and its U(1) version).  Not part of the C ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <utility>

#include "../../include/heff.h"
#include "gemm.cuh"

using namespace heff;

// errors: the thread-local message of heff_last_error
int set_err(int code, const char* fmt, ...);

#define CK(call)                                                                                 \
  do {                                                                                           \
    cudaError_t e_ = (call);                                                                     \
    if (e_ != cudaSuccess)                                                                       \
      return set_err(e_ == cudaErrorMemoryAllocation ? HEFF_ENOMEM : HEFF_ECUDA, "%s: %s (%s:%d)", \
                     #call, cudaGetErrorString(e_), __FILE__, __LINE__);                         \
  } while (0)

#define CKR(call)                 \
  do {                            \
    int r_ = (call);              \
    if (r_ != HEFF_OK) return r_; \
  } while (0)

extern int g_num_sms;
// One-time per-DEVICE initialisation (sm_100 check, SM count, >48 KB shared-memory
// attributes -- function attributes belong to a device context).  Every entry point calls
// it for the calling thread's current device; cheap after the first call per device.
int init_device_once();
constexpr int kMaxDevices = 64;
int cur_device();  // cudaGetDevice(), clamped to [0, kMaxDevices)

// Per-thread, per-device state (workspace arenas): one T per device, selected by the
// calling thread's current device, so a thread that switches devices (torchrun ranks after
// set_device, the U(1) split's workers) never uses another device's buffers.
template <typename T>
struct PerDev {
  T v[kMaxDevices];
  T& operator()() { return v[cur_device()]; }
  template <typename F>
  void each(F&& f) {
    for (int d = 0; d < kMaxDevices; ++d) f(v[d]);
  }
};
int ew_grid(int64_t n);
// 2-D row-major fp64 tensor map: `rows` x `cols`, row pitch `ld`; box {box_cols, box_rows};
// 128-byte swizzle; OOB reads return zero
int make_map(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld, int box_cols, int box_rows);
int launch_transpose(const double* src, double* dst, int64_t rows, int64_t cols, cudaStream_t s);

struct GemmOp {
  int64_t M = 0, N = 0, K = 0;
  const double* A = nullptr;
  int64_t lda = 0;
  const double* B = nullptr;
  int64_t ldb = 0;
  bool b_kmajor = false;
  double* C = nullptr;
  int64_t ldc = 0;
  int accumulate = 0;  // C += A.B instead of C = A.B
  bool b_static = false;  // B is never written by the kernel before this GEMM (it may be prefetched early)
  // block-sparse schedule (heff_set_qn): tile order + per-tile k-block lists, device arrays
  const int* sp_order = nullptr;
  const int* sp_ptr = nullptr;
  const int* sp_list = nullptr;
  int sp_len = 0;  // length of sp_order (per-CTA LPT lists interleaved, -1 padded); 0: #tiles
  // cached TMA maps (rebuilt when A/B pointers or the tile box change)
  CUtensorMap mapA, mapB;
  const double* mapA_ptr = nullptr;
  const double* mapB_ptr = nullptr;
  int64_t mapA_rows = -1, mapB_rows = -1;
  int mapA_box = 0, mapB_box = 0;
};

struct SplitWs {  // stream-K partial-tile workspace, grown on demand
  double* ptr = nullptr;
  size_t bytes = 0;
  // in-kernel fixup state (StreamKSync): [0] ticket counter, then int flags[2 * kSkMaxGrid]
  void* sync = nullptr;
  int epoch = 0;
  bool cached = false;  // blocks from the plan workspace cache (ws_malloc / ws_release): plans'
                        // own stream-K workspaces, reused by the next plan of a DMRG sweep
};
constexpr int kSkMaxGrid = 1024;

// The FP64 DMMA GEMM of libheff (TMA path with 64x64 / 128x128 tiles, stream-K, PDL; the
// plain-load path for unaligned operands).  sa != nullptr: A is K-sharded over tensor maps.
int launch_gemm(GemmOp& g, int path, cudaStream_t s, int* nlaunch, SplitWs* ws, const ShardedA* sa = nullptr);

// Launch with programmatic dependent launch allowed (the kernel calls pdl_wait before it
// touches memory the previous kernel in the stream writes or reads): the next kernel's
// launch and prologue overlap this one's tail.  HEFF_NO_PDL=1 launches normally.
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  static const bool off = getenv("HEFF_NO_PDL") != nullptr;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = off ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// cache release across translation units
void release_thread_caches();                  // heff_api.cu: this thread's workspaces (all TUs)
void split_release_thread_caches();            // split_api.cu: this thread's split arenas
int split_release_worker_caches(int dev);      // split_api.cu: the U(1) split's worker threads
