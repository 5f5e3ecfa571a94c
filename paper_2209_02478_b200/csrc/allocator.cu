// Budget-enforcing arena allocator; see allocator.hpp.
#include <cuda_runtime.h>

#include <algorithm>

#include "allocator.hpp"

namespace mimose_rt {

void ArenaBook::reset(int64_t capacity) {
  capacity_ = capacity - capacity % kAlign;
  blocks_.clear();
  free_.clear();
  stats_ = MemStats{};
  stats_.budget = capacity;
  if (capacity_ > 0) {
    blocks_[0] = Block{capacity_, 0, 0, true};
    insert_free(0, capacity_);
  }
  refresh_largest();
}

void ArenaBook::refresh_largest() {
  stats_.largest_free = free_.empty() ? 0 : free_.rbegin()->first;
}

int64_t ArenaBook::allocate(int64_t bytes, int tag) {
  if (bytes <= 0) bytes = 1;
  if (tag < 0 || tag >= kNumTags) tag = kTagOther;
  const int64_t need = (bytes + kAlign - 1) / kAlign * kAlign;
  auto it = free_.lower_bound({need, -1});  // best fit: smallest block >= need
  if (it == free_.end()) {
    stats_.n_failures += 1;
    return -1;
  }
  const int64_t off = it->second;
  const int64_t size = it->first;
  free_.erase(it);
  Block& b = blocks_[off];
  if (size - need >= kAlign) {
    blocks_[off + need] = Block{size - need, 0, 0, true};
    insert_free(off + need, size - need);
    b.size = need;
  }
  b.free = false;
  b.requested = bytes;
  b.tag = tag;

  stats_.reserved += b.size;
  stats_.requested += bytes;
  stats_.peak_reserved = std::max(stats_.peak_reserved, stats_.reserved);
  stats_.peak_requested = std::max(stats_.peak_requested, stats_.requested);
  stats_.tag_requested[tag] += bytes;
  stats_.tag_peak[tag] = std::max(stats_.tag_peak[tag], stats_.tag_requested[tag]);
  stats_.n_live += 1;
  stats_.n_allocs += 1;
  refresh_largest();
  return off;
}

bool ArenaBook::release(int64_t offset) {
  auto it = blocks_.find(offset);
  if (it == blocks_.end() || it->second.free) return false;
  Block& b = it->second;
  stats_.reserved -= b.size;
  stats_.requested -= b.requested;
  stats_.tag_requested[b.tag] -= b.requested;
  stats_.n_live -= 1;
  b.free = true;
  b.requested = 0;

  // Coalesce with the following block.
  auto next = std::next(it);
  if (next != blocks_.end() && next->second.free) {
    erase_free(next->first, next->second.size);
    b.size += next->second.size;
    blocks_.erase(next);
  }
  // Coalesce with the preceding block.
  if (it != blocks_.begin()) {
    auto prev = std::prev(it);
    if (prev->second.free) {
      erase_free(prev->first, prev->second.size);
      prev->second.size += b.size;
      blocks_.erase(it);
      it = prev;
    }
  }
  insert_free(it->first, it->second.size);
  refresh_largest();
  return true;
}

void ArenaBook::reset_peak() {
  stats_.peak_reserved = stats_.reserved;
  stats_.peak_requested = stats_.requested;
  for (int t = 0; t < kNumTags; ++t) stats_.tag_peak[t] = stats_.tag_requested[t];
}

int64_t ArenaBook::block_size(int64_t offset) const {
  auto it = blocks_.find(offset);
  return it == blocks_.end() ? -1 : it->second.size;
}

DeviceArena::~DeviceArena() {
  if (base_ != nullptr) cudaFree(base_);
}

std::string DeviceArena::init(int64_t budget) {
  if (base_ != nullptr) return "arena already initialised";
  if (budget <= 0) return "budget must be positive";
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, static_cast<size_t>(budget));
  if (e != cudaSuccess) return std::string("cudaMalloc(budget) failed: ") + cudaGetErrorString(e);
  base_ = static_cast<char*>(p);
  book_.reset(budget);
  return {};
}

void* DeviceArena::alloc(int64_t bytes, int tag) {
  const int64_t off = book_.allocate(bytes, tag);
  return off < 0 ? nullptr : base_ + off;
}

bool DeviceArena::free(void* p) {
  if (p == nullptr) return true;
  return book_.release(static_cast<char*>(p) - base_);
}

}  // namespace mimose_rt
