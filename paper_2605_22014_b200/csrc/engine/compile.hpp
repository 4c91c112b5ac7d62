// Descriptor compiler: plan geometry -> device work descriptors.
#pragma once
#include <cstdint>
#include <vector>

#include "desc.h"
#include "reshard_b200/reshard.hpp"

namespace rsb {

// Contiguous runs longer than this are cut into sub-rows of kSubRowBytes so a
// warp-per-row schedule load-balances multi-MB runs.
constexpr std::uint64_t kSubRowBytes = 8192;

// Append the copy of `region` from a row-major buffer laid out as `src_owner`
// at address src_base into one laid out as `dst_owner` at dst_base.  Passing
// dst_owner == region packs (slice_local); src_owner == region unpacks
// (scatter_local).  Emits one or two descriptors (main + run tail).
void append_copy(std::vector<rs_copy_desc>& out, std::uint64_t src_base,
                 const reshard::ShardView& src_owner, std::uint64_t dst_base,
                 const reshard::ShardView& dst_owner, const reshard::ShardView& region,
                 std::int64_t elem_bytes, std::uint32_t tag, bool cut_runs = true);

// Assign work items (rows_per_item from item_bytes) and return item0 prefix
// sums for descs[first..]; returns the total item count after the range.
std::uint64_t assign_items(std::vector<rs_copy_desc>& descs, std::size_t first,
                           std::uint64_t item_base, std::uint64_t item_bytes);

// Pattern descriptors for one shard buffer (view of tensor `t`).
void append_pattern(std::vector<rs_pattern_desc>& out, std::uint64_t ptr,
                    const reshard::TensorSpec& t, const reshard::ShardView& view,
                    std::int64_t elem_bytes, std::uint32_t tensor_index, std::uint32_t entry,
                    std::uint64_t item_bytes);

std::uint64_t bytes_of(const rs_copy_desc& d);

}  // namespace rsb
