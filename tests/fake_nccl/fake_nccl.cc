// Test double of the NCCL calls libheff makes (tests/test_gpu_fake_nccl.py) -- TEST
// INFRASTRUCTURE, never part of the product path.
//
// The communicating b'-sharded path needs P GPUs to run with real
// NCCL.  This library lets P host threads of ONE process, each owning one rank's libheff
// plan on the same GPU, execute that path's orchestration end to end (ncclAllGather of the
// Krylov shard + the blocked re-layout, ncclAllReduce of the CGS2 dot products and norms,
// the failure-detection polling) by exporting the same symbols with host-side semantics:
//   * every collective first synchronises the caller's stream (NCCL is stream-ordered),
//   * the ranks meet at a host barrier (std::condition_variable), exchange device
//     pointers, copy / sum with blocking driver-API copies, and meet again before return.
// No kernel ever waits for another rank: all waiting happens on the host, so the ranks'
// kernels never need to be co-resident on the GPU (B200_PROFILING.md, "kernels that wait
// on one another").  Sums are formed on the host in rank order (deterministic).  The
// symmetric-window calls (ncclMemAlloc, ncclCommWindowRegister) are deliberately absent:
// the gather-fused path's peer flag spin must not run on one GPU.
//
// Loaded by libheff through HEFF_NCCL_PATH (heff_api.cu nccl_load).  Types come from the
// real nccl.h so that the ABI (ncclUniqueId, enums) matches what libheff was compiled with.
#include <cuda.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

namespace {

struct World {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool aborted = false;
  int refs = 0;
  std::vector<const void*> send;
};

std::mutex g_mu;
std::map<std::string, World*> g_worlds;
uint64_t g_uid_counter = 0;

int timeout_s() {  // FAKE_NCCL_TIMEOUT_S (default 120): how long a rank waits for its peers
  static const int t = [] {
    const char* e = getenv("FAKE_NCCL_TIMEOUT_S");
    return e ? atoi(e) : 120;
  }();
  return t;
}

// all n ranks arrive; false on abort or a timeout (a peer that never arrives)
bool barrier(World* w) {
  std::unique_lock<std::mutex> lk(w->m);
  if (w->aborted) return false;
  const uint64_t g = w->gen;
  if (++w->arrived == w->n) {
    w->arrived = 0;
    ++w->gen;
    w->cv.notify_all();
    return true;
  }
  w->cv.wait_for(lk, std::chrono::seconds(timeout_s()), [&] { return w->gen != g || w->aborted; });
  return w->gen != g && !w->aborted;
}

}  // namespace

struct ncclComm {
  World* w;
  int rank;
  ncclResult_t async_err;
};

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  std::lock_guard<std::mutex> lk(g_mu);
  memset(id->internal, 0, sizeof id->internal);
  snprintf(id->internal, sizeof id->internal, "fake-nccl-%llu", (unsigned long long)++g_uid_counter);
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) return ncclInvalidArgument;
  World* w;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    const std::string key(id.internal, strnlen(id.internal, sizeof id.internal));
    auto it = g_worlds.find(key);
    if (it == g_worlds.end()) {
      w = new World();
      w->n = nranks;
      w->send.assign(nranks, nullptr);
      g_worlds[key] = w;
    } else {
      w = it->second;
    }
    if (w->n != nranks) return ncclInvalidArgument;
    ++w->refs;
  }
  *comm = new ncclComm{w, rank, ncclSuccess};
  return barrier(w) ? ncclSuccess : ncclSystemError;  // every rank joined
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  delete comm;  // the world stays registered: its key is never reused
  return ncclSuccess;
}

ncclResult_t ncclCommAbort(ncclComm_t comm) {
  {
    std::lock_guard<std::mutex> lk(comm->w->m);
    comm->w->aborted = true;
    comm->w->cv.notify_all();
  }
  delete comm;
  return ncclSuccess;
}

ncclResult_t ncclCommGetAsyncError(ncclComm_t comm, ncclResult_t* err) {
  *err = comm->async_err;
  return ncclSuccess;
}

const char* ncclGetErrorString(ncclResult_t r) {
  switch (r) {
    case ncclSuccess: return "fake nccl: success";
    case ncclInvalidArgument: return "fake nccl: invalid argument (only ncclFloat64 / ncclSum are implemented)";
    case ncclSystemError: return "fake nccl: a peer aborted or never arrived";
    default: return "fake nccl: error";
  }
}

ncclResult_t ncclAllGather(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t dt, ncclComm_t comm,
                           cudaStream_t stream) {
  if (dt != ncclFloat64) return ncclInvalidArgument;
  const size_t bytes = count * sizeof(double);
  World* w = comm->w;
  if (cuStreamSynchronize(reinterpret_cast<CUstream>(stream)) != CUDA_SUCCESS) return ncclUnhandledCudaError;
  w->send[comm->rank] = sendbuff;
  if (!barrier(w)) return ncclSystemError;
  char* recv = static_cast<char*>(recvbuff);
  for (int q = 0; q < w->n; ++q) {
    char* dst = recv + (size_t)q * bytes;
    if (dst == w->send[q] && q == comm->rank) continue;  // in place
    if (cuMemcpyDtoD(reinterpret_cast<CUdeviceptr>(dst), reinterpret_cast<CUdeviceptr>(w->send[q]), bytes) !=
        CUDA_SUCCESS)
      return ncclUnhandledCudaError;
  }
  return barrier(w) ? ncclSuccess : ncclSystemError;  // nobody reuses its send buffer early
}

ncclResult_t ncclAllReduce(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t dt, ncclRedOp_t op,
                           ncclComm_t comm, cudaStream_t stream) {
  if (dt != ncclFloat64 || op != ncclSum) return ncclInvalidArgument;
  World* w = comm->w;
  if (cuStreamSynchronize(reinterpret_cast<CUstream>(stream)) != CUDA_SUCCESS) return ncclUnhandledCudaError;
  w->send[comm->rank] = sendbuff;
  if (!barrier(w)) return ncclSystemError;
  std::vector<double> acc(count, 0.0), part(count);
  for (int q = 0; q < w->n; ++q) {  // rank order: every rank forms the same sums
    if (count && cuMemcpyDtoH(part.data(), reinterpret_cast<CUdeviceptr>(w->send[q]), count * sizeof(double)) !=
                     CUDA_SUCCESS)
      return ncclUnhandledCudaError;
    for (size_t i = 0; i < count; ++i) acc[i] += part[i];
  }
  if (!barrier(w)) return ncclSystemError;  // every rank has read every send buffer
  if (count && cuMemcpyHtoD(reinterpret_cast<CUdeviceptr>(recvbuff), acc.data(), count * sizeof(double)) !=
                   CUDA_SUCCESS)
    return ncclUnhandledCudaError;
  return ncclSuccess;
}

}  // extern "C"
