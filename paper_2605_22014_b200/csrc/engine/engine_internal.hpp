// Internal helpers shared by the engine's translation units (engine.cpp,
// engine_staged.cpp, engine_host.cpp).  Not part of any public interface.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "engine.hpp"

namespace rsb {
namespace detail {

constexpr std::size_t kAlign = 256;
constexpr std::size_t kFlagBytes = 1 << 20;  // ring flags per slot (131072 u64)
constexpr std::size_t kSyncFlagBytes = 256;   // tail of a slot's flag area: the strict-layer done flag
constexpr std::uint64_t kRingSlotDefault = 128u << 10;  // default ring slot cap (rs_engine_options.ring_slot_kib)
constexpr std::uint64_t kRingSlotStreamDefault = 64u << 10;  // same, stream lanes
constexpr std::uint64_t kSpinLimit = 200000000ull;

inline std::uint64_t key(int rank, std::uint32_t ti) {
  return (static_cast<std::uint64_t>(ti) << 32) | static_cast<std::uint32_t>(rank);
}

inline std::size_t align_up(std::size_t x, std::size_t a) { return (x + a - 1) / a * a; }

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

inline std::string escape_msg(const char* who, const reshard::ShardView& b, const reshard::ShardView& owner) {
  return std::string(who) + ": bounds " + b.to_string() + " escape owner view " + owner.to_string();
}

inline std::string no_buffer(int rank, std::uint32_t ti) {
  return "shard store: no buffer for rank " + std::to_string(rank) + " tensor " + std::to_string(ti);
}

inline std::uint64_t addr(const char* p) { return reinterpret_cast<std::uint64_t>(p); }


// Pointer of an entry that local work must touch.
inline char* need_ptr(const Entry* e, const char* what) {
  if (!e->ptr)
    throw DomainError(std::string(what) + " shard rank " + std::to_string(e->rank) + " tensor " +
                      std::to_string(e->ti) + " on slot " + std::to_string(e->slot) +
                      " is not mapped in this process (rs_arena_import)");
  return e->ptr;
}

// Address of the entry's view origin: shard buffers are addressed row-major
// over the view; a flat-bucket shard's buffer starts flat_off bytes in.
inline std::uint64_t view_base(const Entry* e, const char* what) {
  return addr(need_ptr(e, what)) - static_cast<std::uint64_t>(e->flat_off);
}

// Does the entry's buffer hold every element of `box`?  (Inside the view,
// and for a flat-bucket shard its first and last elements -- row-major --
// inside the held range.)
inline bool holds(const Entry* e, const reshard::ShardView& box) {
  if (!e->view.contains(box)) return false;
  if (!e->flat) return true;
  std::int64_t first = 0, last = 0;
  for (std::size_t k = 0; k < box.ndims(); ++k) {
    const std::int64_t len = e->view.dim(k).length();
    first = first * len + (box.dim(k).lo - e->view.dim(k).lo);
    last = last * len + (box.dim(k).hi - 1 - e->view.dim(k).lo);
  }
  return first >= e->flat_lo && last < e->flat_lo + e->flat_elems;
}

}  // namespace detail
}  // namespace rsb
