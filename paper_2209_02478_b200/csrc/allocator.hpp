// Budget-enforcing caching device allocator.
//
// One device arena of exactly `budget` bytes is reserved up front; every
// device tensor of the training run (parameters, gradients, optimizer state,
// activations, transients) is carved out of it. An allocation that cannot be
// satisfied inside the arena FAILS (it never falls through to cudaMalloc), so
// "never exceeds the budget" holds by construction and is observable from the
// peak counters.
//
// Counters realise the reference's `resident` bookkeeping
// (reference simulator.hpp:113-155): `requested` is the byte-exact sum of
// live request sizes (what the collector feeds to the estimator, see
// collector.hpp:138-150), `reserved` adds the 256 B rounding, and both keep
// running peaks. Per-tag counters attribute bytes to parameter / activation /
// transient classes.
//
// The book-keeping core (ArenaBook) is plain host C++ so it is unit-testable
// without a GPU; DeviceArena binds it to one cudaMalloc'd region. Frees are
// ordered on the step's compute stream: a block freed after its last use there
// may be handed out again immediately. The arena does not track streams, so
// the two other streams follow one rule each (trainer.cpp):
//   - keep-bit side stream: its block is taken on the host before the side
//     stream waits on an event recorded on the compute stream (every earlier
//     use of those bytes has finished), and the compute stream waits on the
//     side stream's completion event before the block is read or dropped;
//   - NCCL comm stream (dp.cpp): it only touches the gradient buffers, which
//     live for the whole run, and is joined before the optimizer and hooks.
#pragma once

#include <cstddef>
#include <cstdint>
#include <map>
#include <set>
#include <string>
#include <utility>

namespace mimose_rt {

constexpr int kNumTags = 8;
enum Tag : int {
  kTagParam = 0,     // bf16 weights, fp32 master weights
  kTagGrad = 1,      // fp32 gradients
  kTagOptim = 2,     // AdamW moments
  kTagAct = 3,       // saved activations (the planner-managed bytes)
  kTagBoundary = 4,  // retained layer outputs of dropped layers
  kTagTransient = 5, // scratch freed inside one layer step
  kTagInput = 6,     // per-step inputs (token ids, labels, sort tables)
  kTagOther = 7,
};

struct MemStats {
  int64_t budget = 0;
  int64_t reserved = 0;       // live bytes incl. rounding
  int64_t peak_reserved = 0;
  int64_t requested = 0;      // live bytes as requested
  int64_t peak_requested = 0;
  int64_t largest_free = 0;
  int64_t n_live = 0;
  int64_t n_allocs = 0;
  int64_t n_failures = 0;
  int64_t tag_requested[kNumTags] = {};
  int64_t tag_peak[kNumTags] = {};
};

class ArenaBook {
 public:
  static constexpr int64_t kAlign = 256;

  explicit ArenaBook(int64_t capacity = 0) { reset(capacity); }

  void reset(int64_t capacity);
  // Returns the offset or -1 when the arena cannot satisfy the request.
  int64_t allocate(int64_t bytes, int tag);
  // Returns false for an unknown offset (double free / foreign pointer).
  bool release(int64_t offset);
  void reset_peak();
  const MemStats& stats() const { return stats_; }
  int64_t block_size(int64_t offset) const;
  int64_t capacity() const { return capacity_; }

 private:
  struct Block {
    int64_t size = 0;
    int64_t requested = 0;
    int tag = 0;
    bool free = true;
  };
  void insert_free(int64_t off, int64_t size) { free_.insert({size, off}); }
  void erase_free(int64_t off, int64_t size) { free_.erase({size, off}); }
  void refresh_largest();

  int64_t capacity_ = 0;
  std::map<int64_t, Block> blocks_;           // offset -> block (covers the arena)
  std::set<std::pair<int64_t, int64_t>> free_;  // (size, offset) best-fit index
  MemStats stats_;
};

class DeviceArena {
 public:
  DeviceArena() = default;
  ~DeviceArena();
  DeviceArena(const DeviceArena&) = delete;
  DeviceArena& operator=(const DeviceArena&) = delete;

  // Reserves `budget` bytes on the current device. Returns an error string
  // (empty on success).
  std::string init(int64_t budget);
  void* alloc(int64_t bytes, int tag);  // nullptr on budget breach
  bool free(void* p);
  const MemStats& stats() const { return book_.stats(); }
  void reset_peak() { book_.reset_peak(); }
  char* base() const { return base_; }

 private:
  char* base_ = nullptr;
  ArenaBook book_;
};

}  // namespace mimose_rt
