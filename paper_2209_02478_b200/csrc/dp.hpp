// Native data-parallel gradient exchange (SURVEY §8(e), §8(b2) mimose_dp_*):
// one NCCL communicator per rank, gradients all-reduced in buckets on a
// dedicated high-priority stream while the backward of earlier layers is
// still running. NCCL is resolved at run time (dlopen of libnccl.so.2: the
// copy torch already loaded in this process, else the system one), so the
// library has no link-time NCCL dependency.
//
// The transport is injectable: instead of NCCL a caller-supplied reduce
// callback receives every (bucket, stream) the schedule issues - after the
// comm stream has been ordered behind the backward work that produced the
// bucket - and must leave the sum across ranks in place. Tests use it to
// run two ranks' trainers on ONE GPU (in one process with a pairing
// reducer, or in two processes over gloo) through the same bucket schedule
// and stream ordering the NCCL path uses.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace mimose_rt {

struct NcclApi;
// returns 0 on success; buf is a device pointer, stream the comm stream
using ReduceFn = int (*)(void* user, void* buf, int64_t n, int dtype, int op, void* stream);

class DataParallel {
 public:
  DataParallel(int device, const void* unique_id, int rank, int world);
  // custom transport (no NCCL communicator)
  DataParallel(int device, int rank, int world, ReduceFn fn, void* user);
  ~DataParallel();
  static void unique_id(void* out128);

  // in-place sum (dtype 0 fp32, 1 bf16) or max (op 1) on `stream`
  void allreduce(void* buf, int64_t n, int dtype, int op, cudaStream_t stream);
  // bucketed: comm stream waits for `ready` work on `s`, then reduces [off, off+n) fp32
  void allreduce_after(float* buf, int64_t n, cudaStream_t s);
  // the compute stream waits for every reduction issued so far
  void join(cudaStream_t s);

  int rank() const { return rank_; }
  // device bytes the NCCL communicator holds outside any arena (measured with
  // cudaMemGetInfo around init and a first collective; 0 for custom transports)
  int64_t device_bytes() const { return device_bytes_; }
  int world() const { return world_; }
  cudaStream_t stream() const { return stream_; }

 private:
  void init_streams();
  const NcclApi* api_ = nullptr;
  void* comm_ = nullptr;
  ReduceFn fn_ = nullptr;
  void* user_ = nullptr;
  int64_t device_bytes_ = 0;
  int rank_ = 0, world_ = 1, device_ = 0;
  cudaStream_t stream_ = nullptr;
  cudaEvent_t ready_ = nullptr, done_ = nullptr;
  bool pending_ = false;
};

// Bucket schedule over contiguous gradient units that complete in reverse
// order (unit U-1 first, unit 0 last): after unit u completes, emit
// [off[u], pending_end) once it holds >= bucket_elems (always at u = 0).
// Returns {after_unit, begin, end} triples.
struct Bucket {
  int after_unit;
  int64_t begin, end;
};
std::vector<Bucket> plan_buckets(const std::vector<int64_t>& unit_off, int64_t bucket_elems);

}  // namespace mimose_rt
