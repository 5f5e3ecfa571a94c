#include "dp.hpp"

#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

namespace mimose_rt {

namespace {
// the subset of nccl.h used here (ABI-stable since NCCL 2.0)
using ncclComm_t = void*;
using ncclResult_t = int;
struct UniqueId {
  char internal[128];
};
enum { kNcclFloat32 = 7, kNcclBfloat16 = 9 };  // ncclFloat32, ncclBfloat16
enum { kNcclSum = 0, kNcclMax = 2 };
}  // namespace

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*get_unique_id)(UniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, UniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

namespace {
const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    const char* env = std::getenv("MIMOSE_NCCL_LIB");
    const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      if (n == nullptr || *n == 0) continue;
      a.handle = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (a.handle) break;
    }
    if (!a.handle) return a;
    auto sym = [&](const char* s) { return dlsym(a.handle, s); };
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(sym("ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(sym("ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(sym("ncclCommDestroy"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(sym("ncclAllReduce"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(sym("ncclGetErrorString"));
    return a;
  }();
  if (!api.handle || !api.get_unique_id || !api.comm_init_rank || !api.all_reduce)
    throw std::runtime_error("NCCL not available (dlopen libnccl.so.2 failed; set MIMOSE_NCCL_LIB)");
  return api;
}

void nck(const NcclApi& a, ncclResult_t r, const char* what) {
  if (r != 0)
    throw std::runtime_error(std::string(what) + ": " +
                             (a.error_string ? a.error_string(r) : std::to_string(r)));
}

void cck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace

void DataParallel::unique_id(void* out128) {
  const NcclApi& a = nccl();
  UniqueId id;
  nck(a, a.get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
}

DataParallel::DataParallel(int device, const void* uid, int rank, int world)
    : api_(&nccl()), rank_(rank), world_(world), device_(device) {
  if (world < 1 || rank < 0 || rank >= world) throw std::runtime_error("bad rank / world");
  cck(cudaSetDevice(device), "cudaSetDevice");
  UniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  size_t free0 = 0, free1 = 0, total = 0;
  cck(cudaDeviceSynchronize(), "sync");
  cck(cudaMemGetInfo(&free0, &total), "cudaMemGetInfo");
  nck(*api_, api_->comm_init_rank(&comm_, world, id, rank), "ncclCommInitRank");
  init_streams();
  // first collective: NCCL sets up its channel / proxy buffers lazily
  float* probe = nullptr;
  cck(cudaMalloc(&probe, 4096), "cudaMalloc");
  cck(cudaMemsetAsync(probe, 0, 4096, stream_), "memset");
  allreduce(probe, 1024, 0, 0, stream_);
  cck(cudaStreamSynchronize(stream_), "sync");
  cck(cudaFree(probe), "cudaFree");
  cck(cudaMemGetInfo(&free1, &total), "cudaMemGetInfo");
  device_bytes_ = free0 > free1 ? static_cast<int64_t>(free0 - free1) : 0;
}

DataParallel::DataParallel(int device, int rank, int world, ReduceFn fn, void* user)
    : fn_(fn), user_(user), rank_(rank), world_(world), device_(device) {
  if (world < 1 || rank < 0 || rank >= world) throw std::runtime_error("bad rank / world");
  if (fn == nullptr) throw std::runtime_error("null reduce callback");
  cck(cudaSetDevice(device), "cudaSetDevice");
  init_streams();
}

void DataParallel::init_streams() {
  int lo = 0, hi = 0;
  cck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
  cck(cudaStreamCreateWithPriority(&stream_, cudaStreamNonBlocking, hi), "comm stream");
  cck(cudaEventCreateWithFlags(&ready_, cudaEventDisableTiming), "event");
  cck(cudaEventCreateWithFlags(&done_, cudaEventDisableTiming), "event");
}

DataParallel::~DataParallel() {
  if (stream_) cudaStreamSynchronize(stream_);
  if (comm_ && api_ && api_->comm_destroy) api_->comm_destroy(comm_);
  if (ready_) cudaEventDestroy(ready_);
  if (done_) cudaEventDestroy(done_);
  if (stream_) cudaStreamDestroy(stream_);
}

void DataParallel::allreduce(void* buf, int64_t n, int dtype, int op, cudaStream_t s) {
  if (n <= 0) return;
  if (fn_ != nullptr) {
    if (fn_(user_, buf, n, dtype, op, s) != 0) throw std::runtime_error("reduce callback failed");
    return;
  }
  const int dt = dtype == 1 ? kNcclBfloat16 : kNcclFloat32;
  nck(*api_, api_->all_reduce(buf, buf, static_cast<size_t>(n), dt, op == 1 ? kNcclMax : kNcclSum,
                              comm_, s),
      "ncclAllReduce");
}

void DataParallel::allreduce_after(float* buf, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  cck(cudaEventRecord(ready_, s), "event");
  cck(cudaStreamWaitEvent(stream_, ready_, 0), "wait");
  allreduce(buf, n, 0, 0, stream_);
  pending_ = true;
}

void DataParallel::join(cudaStream_t s) {
  if (!pending_) return;
  cck(cudaEventRecord(done_, stream_), "event");
  cck(cudaStreamWaitEvent(s, done_, 0), "wait");
  pending_ = false;
}

std::vector<Bucket> plan_buckets(const std::vector<int64_t>& off, int64_t bucket_elems) {
  std::vector<Bucket> out;
  const int U = static_cast<int>(off.size()) - 1;
  if (U < 1) return out;
  int64_t end = off[U];
  for (int u = U - 1; u >= 0; --u) {
    if (end - off[u] >= bucket_elems || u == 0) {
      if (end > off[u]) out.push_back({u, off[u], end});
      end = off[u];
    }
  }
  return out;
}

}  // namespace mimose_rt
