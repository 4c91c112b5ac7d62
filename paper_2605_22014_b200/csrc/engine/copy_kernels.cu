// Copy kernels of the reshard engine: the batched strided->strided byte copy
// over rs_copy_desc work lists (pack / unpack / relayout / carryover;
// proj/src/executor.cpp:23-93 + :142-166 on the device).  The default is the
// non-persistent TMA bulk copy (rs_copy_tma_np_kernel, one 1-warp CTA per
// 16 KB item); the LDG warp engine serves unaligned plans and peer stores;
// the persistent / ring variants are kept as measured alternatives.
#include <cuda_runtime.h>

#include <atomic>
#include <stdint.h>

#include "desc.h"
#include "device_common.cuh"
#include "kernels.h"

namespace {

template <int U, bool kStream = false, int kLd = 0>
__global__ void __launch_bounds__(256) rs_copy_kernel(const rs_copy_desc* __restrict__ descs,
                                                      const uint64_t* __restrict__ item0,
                                                      uint32_t ndesc, uint64_t item_begin,
                                                      uint64_t item_end) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t item = item_begin + warp; item < item_end; item += nwarps) {
    const uint32_t di = find_desc(item0, ndesc, item);
    warp_copy_item<true, U, kStream, kLd>(descs[di], item - descs[di].item0, lane);
  }
}

// CTA-cooperative variant: an item belongs to a whole CTA and its rows are
// dealt to the CTA's warps, so the grid keeps 8x fewer item streams open at a
// time (DRAM page locality) with the same bytes in flight per warp.
template <int U>
__global__ void __launch_bounds__(256) rs_copy_cta_kernel(const rs_copy_desc* __restrict__ descs,
                                                          const uint64_t* __restrict__ item0,
                                                          uint32_t ndesc, uint64_t item_begin,
                                                          uint64_t item_end) {
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (uint64_t item = item_begin + blockIdx.x; item < item_end; item += gridDim.x) {
    const uint32_t di = find_desc(item0, ndesc, item);
    const rs_copy_desc& D = descs[di];
    const uint64_t r0 = (item - D.item0) * D.rows_per_item;
    const uint64_t r1 = min(r0 + D.rows_per_item, D.rows);
    const char* src = reinterpret_cast<const char*>(D.src);
    char* dst = reinterpret_cast<char*>(D.dst);
    for (uint64_t r = r0 + w; r < r1; r += nw) {
      int64_t so, dof;
      row_offsets(D, static_cast<uint32_t>(r), so, dof);
      warp_copy_any<true, U>(src + so, dst + dof, D.row_bytes, D.vec_log2, lane);
    }
  }
}

// ------------------------------------------------------ TMA bulk-copy ring
//
// One elected thread per CTA streams rows through a ring of kStages shared
// memory stages with the Blackwell bulk-copy engine (cp.async.bulk, SASS
// UBLKCP): global -> smem completes on a per-stage mbarrier (complete_tx),
// smem -> global is a bulk_group store.  Loads run kLag stages ahead of
// stores; a stage is refilled only after `cp.async.bulk.wait_group.read`
// proves its previous store has read it.  Requires 16 B aligned rows
// (descriptors with vec_log2 < 4 go to the LDG kernel).

constexpr int kBulkStages = 8;
constexpr int kBulkLag = 5;
constexpr uint32_t kBulkStageBytes = 24576;
constexpr int kBulkMaxPieces = 32;

struct BulkPiece {
  uint64_t src, dst;
  uint32_t off, bytes;
};

__global__ void __launch_bounds__(32, 1) rs_copy_bulk_kernel(const rs_copy_desc* __restrict__ descs,
                                                             const uint64_t* __restrict__ item0,
                                                             uint32_t ndesc, uint64_t item_begin,
                                                             uint64_t item_end) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t bars[kBulkStages];
  __shared__ BulkPiece pieces[kBulkStages][kBulkMaxPieces];
  __shared__ int npieces[kBulkStages];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kBulkStages; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");

  uint64_t chunk = 0;   // stages filled so far
  uint64_t drained = 0; // stages whose stores were issued
  int s = 0, n = 0;
  uint32_t fill = 0;

  auto drain_one = [&]() {
    const int ds = static_cast<int>(drained % kBulkStages);
    mbar_wait(&bars[ds], static_cast<uint32_t>((drained / kBulkStages) & 1));
    for (int k = 0; k < npieces[ds]; ++k) {
      const BulkPiece& p = pieces[ds][k];
      bulk_store(reinterpret_cast<void*>(p.dst), ring + ds * kBulkStageBytes + p.off, p.bytes);
    }
    bulk_commit();
    ++drained;
  };
  auto issue = [&]() {  // launch the loads of the stage being filled
    npieces[s] = n;
    mbar_expect_tx(&bars[s], fill);
    for (int k = 0; k < n; ++k) {
      const BulkPiece& p = pieces[s][k];
      bulk_load(ring + s * kBulkStageBytes + p.off, reinterpret_cast<const void*>(p.src), p.bytes, &bars[s]);
    }
    ++chunk;
    if (chunk > static_cast<uint64_t>(kBulkLag)) drain_one();
    s = static_cast<int>(chunk % kBulkStages);
    n = 0;
    fill = 0;
    // the next stage to fill was last stored by chunk - kStages: make sure that
    // store finished reading smem (groups committed after it: stages-lag-1)
    if (chunk >= static_cast<uint64_t>(kBulkStages)) bulk_wait_read<kBulkStages - kBulkLag - 1>();
  };

  const uint64_t per = gridDim.x;
  for (uint64_t item = item_begin + blockIdx.x; item < item_end; item += per) {
    const uint32_t di = find_desc(item0, ndesc, item);
    const rs_copy_desc& D = descs[di];
    const uint64_t r0 = (item - D.item0) * D.rows_per_item;
    const uint64_t r1 = min(r0 + D.rows_per_item, D.rows);
    for (uint64_t r = r0; r < r1; ++r) {
      int64_t so, dof;
      row_offsets(D, static_cast<uint32_t>(r), so, dof);
      uint64_t src = D.src + so, dst = D.dst + dof, left = D.row_bytes;
      while (left) {
        uint32_t room = kBulkStageBytes - fill;
        if (room == 0 || n == kBulkMaxPieces) {
          issue();
          room = kBulkStageBytes;
        }
        const uint32_t b = static_cast<uint32_t>(left < room ? left : static_cast<uint64_t>(room));
        pieces[s][n++] = BulkPiece{src, dst, fill, b};
        fill += b;
        src += b;
        dst += b;
        left -= b;
      }
    }
  }
  if (n) issue();
  while (drained < chunk) drain_one();
  bulk_wait_all();
}

// Multi-issuer TMA bulk ring: every warp's elected lane runs an independent
// kMwStages-deep ring of kMwStageBytes stages over its own work items (the
// warp-granular item schedule of rs_copy_kernel), so an SM keeps
// kMwWarps x kMwLag stages of bulk loads in flight instead of one issuer's.
constexpr int kMwPieces = 16;

template <int kMwWarps, int kMwStages, int kMwLag, uint32_t kMwStageBytes>
__global__ void __launch_bounds__(kMwWarps * 32, 1) rs_copy_bulk_mw_kernel(const rs_copy_desc* __restrict__ descs,
                                                                           const uint64_t* __restrict__ item0,
                                                                           uint32_t ndesc, uint64_t item_begin,
                                                                           uint64_t item_end) {
  extern __shared__ __align__(128) unsigned char ring_all[];
  __shared__ __align__(8) uint64_t bars_all[kMwWarps][kMwStages];
  __shared__ BulkPiece pieces_all[kMwWarps][kMwStages][kMwPieces];
  __shared__ int npieces_all[kMwWarps][kMwStages];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) != 0) return;
  unsigned char* ring = ring_all + w * kMwStages * kMwStageBytes;
  uint64_t* bars = bars_all[w];
  auto& pieces = pieces_all[w];
  int* npieces = npieces_all[w];
  for (int s = 0; s < kMwStages; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");

  uint64_t chunk = 0, drained = 0;
  int s = 0, n = 0;
  uint32_t fill = 0;
  auto drain_one = [&]() {
    const int ds = static_cast<int>(drained % kMwStages);
    mbar_wait(&bars[ds], static_cast<uint32_t>((drained / kMwStages) & 1));
    for (int k = 0; k < npieces[ds]; ++k) {
      const BulkPiece& p = pieces[ds][k];
      bulk_store(reinterpret_cast<void*>(p.dst), ring + ds * kMwStageBytes + p.off, p.bytes);
    }
    bulk_commit();
    ++drained;
  };
  auto issue = [&]() {
    npieces[s] = n;
    mbar_expect_tx(&bars[s], fill);
    for (int k = 0; k < n; ++k) {
      const BulkPiece& p = pieces[s][k];
      bulk_load(ring + s * kMwStageBytes + p.off, reinterpret_cast<const void*>(p.src), p.bytes, &bars[s]);
    }
    ++chunk;
    if (chunk > static_cast<uint64_t>(kMwLag)) drain_one();
    s = static_cast<int>(chunk % kMwStages);
    n = 0;
    fill = 0;
    if (chunk >= static_cast<uint64_t>(kMwStages)) bulk_wait_read<kMwStages - kMwLag - 1>();
  };

  const uint64_t worker = static_cast<uint64_t>(blockIdx.x) * kMwWarps + w;
  const uint64_t workers = static_cast<uint64_t>(gridDim.x) * kMwWarps;
  for (uint64_t item = item_begin + worker; item < item_end; item += workers) {
    const uint32_t di = find_desc(item0, ndesc, item);
    const rs_copy_desc& D = descs[di];
    const uint64_t r0 = (item - D.item0) * D.rows_per_item;
    const uint64_t r1 = min(r0 + D.rows_per_item, D.rows);
    for (uint64_t r = r0; r < r1; ++r) {
      int64_t so, dof;
      row_offsets(D, static_cast<uint32_t>(r), so, dof);
      uint64_t src = D.src + so, dst = D.dst + dof, left = D.row_bytes;
      while (left) {
        uint32_t room = kMwStageBytes - fill;
        if (room == 0 || n == kMwPieces) {
          issue();
          room = kMwStageBytes;
        }
        const uint32_t b = static_cast<uint32_t>(left < room ? left : static_cast<uint64_t>(room));
        pieces[s][n++] = BulkPiece{src, dst, fill, b};
        fill += b;
        src += b;
        dst += b;
        left -= b;
      }
    }
  }
  if (n) issue();
  while (drained < chunk) drain_one();
  bulk_wait_all();
}

// Non-persistent TMA bulk copy: one 1-warp CTA per work item (<= the dynamic
// shared memory of the launch: 16 or 32 KB of 16 B aligned rows).  The elected lane bulk-loads every row piece of the
// item into shared memory on one mbarrier (complete_tx), waits, bulk-stores
// them back out and waits for the stores to have read shared memory before the
// CTA retires.  ~14 such CTAs fit an SM (16 KB of smem each), so an SM keeps
// ~14 items of loads in flight with one issuing thread per item.
constexpr uint32_t kNpTmaBytes = 16384;

__global__ void __launch_bounds__(32) rs_copy_tma_np_kernel(const rs_copy_desc* __restrict__ descs,
                                                            const uint64_t* __restrict__ item0,
                                                            uint32_t ndesc, uint64_t item_begin,
                                                            uint64_t item_end) {
  extern __shared__ __align__(128) unsigned char buf[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x != 0) return;
  const uint64_t item = item_begin + blockIdx.x;
  if (item >= item_end) return;
  const uint32_t di = find_desc(item0, ndesc, item);
  const rs_copy_desc& D = descs[di];
  const uint64_t r0 = (item - D.item0) * D.rows_per_item;
  const uint64_t r1 = min(r0 + D.rows_per_item, D.rows);
  mbar_init(&bar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint32_t total = static_cast<uint32_t>((r1 - r0) * D.row_bytes);
  mbar_expect_tx(&bar, total);
  uint32_t off = 0;
  for (uint64_t r = r0; r < r1; ++r) {
    int64_t so, dof;
    row_offsets(D, static_cast<uint32_t>(r), so, dof);
    bulk_load(buf + off, reinterpret_cast<const void*>(D.src + so), static_cast<uint32_t>(D.row_bytes), &bar);
    off += static_cast<uint32_t>(D.row_bytes);
  }
  mbar_wait(&bar, 0);
  off = 0;
  for (uint64_t r = r0; r < r1; ++r) {
    int64_t so, dof;
    row_offsets(D, static_cast<uint32_t>(r), so, dof);
    bulk_store(reinterpret_cast<void*>(D.dst + dof), buf + off, static_cast<uint32_t>(D.row_bytes));
    // DP broadcast: the second destination from the same shared-memory copy
    if (D.dst2_delta)
      bulk_store(reinterpret_cast<void*>(D.dst + dof + D.dst2_delta), buf + off, static_cast<uint32_t>(D.row_bytes));
    off += static_cast<uint32_t>(D.row_bytes);
  }
  bulk_commit();
  bulk_wait_all();
}

// The dynamic shared-memory opt-in is a per-device function attribute: one
// bit per device ordinal records where it has been set, so a process driving
// several GPUs opts in on each of them (not just the first one launched on).
template <class K>
cudaError_t opt_in_smem(K* kernel, int smem, std::atomic<uint64_t>& configured) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (configured.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) configured.fetch_or(bit, std::memory_order_release);
  return e;
}

template <int W, int S, int L, uint32_t T>
cudaError_t launch_bulk_mw(const rs_copy_desc* descs, const uint64_t* item0, uint32_t ndesc, uint64_t item_begin,
                           uint64_t item_end, int grid, cudaStream_t stream) {
  static std::atomic<uint64_t> configured{0};
  const int smem = W * S * static_cast<int>(T);
  cudaError_t e = opt_in_smem(rs_copy_bulk_mw_kernel<W, S, L, T>, smem, configured);
  if (e != cudaSuccess) return e;
  rs_copy_bulk_mw_kernel<W, S, L, T><<<grid, W * 32, smem, stream>>>(descs, item0, ndesc, item_begin, item_end);
  return cudaGetLastError();
}

}  // namespace

extern "C" {

cudaError_t rs_launch_copy(const rs_copy_desc* descs, const uint64_t* item0, uint32_t ndesc,
                           uint64_t item_begin, uint64_t item_end, int grid, int variant,
                           cudaStream_t stream) {
  if (item_end <= item_begin || ndesc == 0) return cudaSuccess;
  switch (variant) {
    case 2:
      rs_copy_kernel<8><<<grid, 256, 0, stream>>>(descs, item0, ndesc, item_begin, item_end);
      break;
    case 4:
      rs_copy_kernel<4, true><<<grid, 256, 0, stream>>>(descs, item0, ndesc, item_begin, item_end);
      break;
    case 5:
      rs_copy_kernel<8, true><<<grid, 256, 0, stream>>>(descs, item0, ndesc, item_begin, item_end);
      break;
    case 6:
      rs_copy_kernel<16><<<grid, 256, 0, stream>>>(descs, item0, ndesc, item_begin, item_end);
      break;
    case 7:
      rs_copy_cta_kernel<8><<<grid, 256, 0, stream>>>(descs, item0, ndesc, item_begin, item_end);
      break;
    case 13:
      rs_copy_kernel<8, false, 1><<<grid, 256, 0, stream>>>(descs, item0, ndesc, item_begin, item_end);
      break;
    case 17:    // non-persistent TMA bulk copy: one 1-warp CTA per <= 16 KB item
    case 18: {  // same with <= 32 KB items
      const uint64_t ctas = item_end - item_begin;
      const uint32_t smem = variant == 18 ? 2 * kNpTmaBytes : kNpTmaBytes;
      rs_copy_tma_np_kernel<<<static_cast<unsigned>(ctas), 32, smem, stream>>>(descs, item0, ndesc, item_begin,
                                                                              item_end);
      break;
    }
    case 15: {  // non-persistent: one item per warp, the block scheduler deals CTAs
      const uint64_t ctas = (item_end - item_begin + 7) / 8;
      rs_copy_kernel<8><<<static_cast<unsigned>(ctas), 256, 0, stream>>>(descs, item0, ndesc, item_begin, item_end);
      break;
    }
    case 14:
      rs_copy_kernel<8, false, 2><<<grid, 256, 0, stream>>>(descs, item0, ndesc, item_begin, item_end);
      break;
    case 8: return launch_bulk_mw<4, 6, 4, 8192>(descs, item0, ndesc, item_begin, item_end, grid, stream);
    case 9: return launch_bulk_mw<8, 3, 2, 8192>(descs, item0, ndesc, item_begin, item_end, grid, stream);
    case 10: return launch_bulk_mw<4, 3, 2, 16384>(descs, item0, ndesc, item_begin, item_end, grid, stream);
    case 11: return launch_bulk_mw<8, 6, 4, 4096>(descs, item0, ndesc, item_begin, item_end, grid, stream);
    case 12: return launch_bulk_mw<16, 3, 2, 4096>(descs, item0, ndesc, item_begin, item_end, grid, stream);
    case 3: {
      static std::atomic<uint64_t> configured{0};
      const int smem = kBulkStages * static_cast<int>(kBulkStageBytes);
      cudaError_t e = opt_in_smem(rs_copy_bulk_kernel, smem, configured);
      if (e != cudaSuccess) return e;
      rs_copy_bulk_kernel<<<grid, 32, smem, stream>>>(descs, item0, ndesc, item_begin, item_end);
      break;
    }
    default:
      rs_copy_kernel<4><<<grid, 256, 0, stream>>>(descs, item0, ndesc, item_begin, item_end);
  }
  return cudaGetLastError();
}

// occupancy of the copy kernels (rs_kernel_max_blocks_per_sm dispatches here)
int copy_max_blocks_per_sm(int which) {
  int n = 0;
  if (which == 0) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rs_copy_kernel<4>, 256, 0);
  else if (which == 3) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rs_copy_kernel<8>, 256, 0);
  else if (which == 5) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rs_copy_kernel<16>, 256, 0);
  else if (which == 6) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rs_copy_cta_kernel<8>, 256, 0);
  else if (which == 4) n = 1;  // bulk ring: one CTA (one issuer, ~200 KB smem) per SM
  return n;
}

int rs_kernel_max_blocks_per_sm(int which) {
  if (which == 1) return pattern_max_blocks_per_sm();
  if (which == 2 || (which >= 7 && which <= 12)) return exchange_max_blocks_per_sm(which);
  return copy_max_blocks_per_sm(which);
}

}  // extern "C"
