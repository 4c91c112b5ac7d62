// sm_100a kernels of the reshard engine.
//
//   rs_copy_kernel     batched strided->strided byte copy over rs_copy_desc
//                      work lists (pack / unpack / relayout / carryover;
//                      proj/src/executor.cpp:23-93 + :142-166 on the device).
//                      Warp-granular persistent loop, 16 B vector accesses,
//                      U independent loads in flight per lane.
//   rs_pattern_kernel  synthetic state fill / verify against the reference
//                      pattern (proj/src/shard_store.cpp:12-85), one hash per
//                      element, 16 B stores / compares.
//   rs_exchange_kernel ring-staged transfer: sender warps pack frames into the
//                      receiver's staging slots (peer stores over NVLink when
//                      the receiver is another GPU), publish with a .sys
//                      release flag; receiver warps acquire, unpack, return a
//                      credit (bounded staging, proj/src/executor.cpp:183-206).
//
// Everything is integer/byte movement: no floating point touches the data.
#include <cuda_runtime.h>
#include <stdint.h>

#include "desc.h"
#include "kernels.h"

namespace {

constexpr int kUnroll = 4;

// ---------------------------------------------------------------- accesses

// Read-only path (L1 no-allocate): for shard buffers that nothing writes
// during the launch.
template <typename T, bool kReadOnly>
__device__ __forceinline__ T load(const T* p);

template <>
__device__ __forceinline__ uint4 load<uint4, true>(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
// Coherent-at-L2 path: staging slots written by another SM / GPU.
template <>
__device__ __forceinline__ uint4 load<uint4, false>(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
template <>
__device__ __forceinline__ uint2 load<uint2, true>(const uint2* p) { return __ldg(p); }
template <>
__device__ __forceinline__ uint2 load<uint2, false>(const uint2* p) { return __ldcg(p); }
template <>
__device__ __forceinline__ uint32_t load<uint32_t, true>(const uint32_t* p) { return __ldg(p); }
template <>
__device__ __forceinline__ uint32_t load<uint32_t, false>(const uint32_t* p) { return __ldcg(p); }
template <>
__device__ __forceinline__ uint16_t load<uint16_t, true>(const uint16_t* p) { return __ldg(p); }
template <>
__device__ __forceinline__ uint16_t load<uint16_t, false>(const uint16_t* p) { return __ldcg(p); }
template <>
__device__ __forceinline__ uint8_t load<uint8_t, true>(const uint8_t* p) { return __ldg(p); }
template <>
__device__ __forceinline__ uint8_t load<uint8_t, false>(const uint8_t* p) { return __ldcg(p); }

template <typename T>
__device__ __forceinline__ void store(T* p, const T& v) { *p = v; }
template <>
__device__ __forceinline__ void store<uint4>(uint4* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// Streaming store (evict-first in L2): the destination is not re-read.
__device__ __forceinline__ void store_cs(uint4* p, const uint4& v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// Read-only 16 B load flavours of the copy engine (RS_COPY_LDG8_PF / _EF):
// 1 = L2 256 B sector prefetch hint, 2 = evict-first L2 policy.
template <int kLd>
__device__ __forceinline__ uint4 load16(const uint4* p, uint64_t pol) {
  uint4 r;
  if constexpr (kLd == 1)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
  return r;
}

// One warp copies one contiguous run: lanes stride T-sized vectors, U loads
// issued before their stores.
template <typename T, bool kReadOnly, int U = kUnroll, bool kStream = false, int kLd = 0>
__device__ __forceinline__ void warp_copy_run(const char* src, char* dst, uint64_t nbytes,
                                              int lane) {
  const T* s = reinterpret_cast<const T*>(src);
  T* d = reinterpret_cast<T*>(dst);
  const uint64_t n = nbytes / sizeof(T);
  uint64_t i = static_cast<uint64_t>(lane);
  uint64_t pol = 0;
  if constexpr (kLd == 2) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  for (; i + 32 * (U - 1) < n; i += 32 * U) {
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if constexpr (kLd != 0 && kReadOnly && sizeof(T) == 16)
        v[u] = load16<kLd>(reinterpret_cast<const uint4*>(s + i + 32 * u), pol);
      else
        v[u] = load<T, kReadOnly>(s + i + 32 * u);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if constexpr (kStream && sizeof(T) == 16) store_cs(reinterpret_cast<uint4*>(d + i + 32 * u), v[u]);
      else store<T>(d + i + 32 * u, v[u]);
    }
  }
  for (; i < n; i += 32) store<T>(d + i, load<T, kReadOnly>(s + i));
}

template <bool kReadOnly, int U = kUnroll, bool kStream = false, int kLd = 0>
__device__ __forceinline__ void warp_copy_any(const char* src, char* dst, uint64_t nbytes,
                                              uint32_t vec_log2, int lane) {
  switch (vec_log2) {
    case 4: warp_copy_run<uint4, kReadOnly, U, kStream, kLd>(src, dst, nbytes, lane); break;
    case 3: warp_copy_run<uint2, kReadOnly>(src, dst, nbytes, lane); break;
    case 2: warp_copy_run<uint32_t, kReadOnly>(src, dst, nbytes, lane); break;
    case 1: warp_copy_run<uint16_t, kReadOnly>(src, dst, nbytes, lane); break;
    default: warp_copy_run<uint8_t, kReadOnly>(src, dst, nbytes, lane); break;
  }
}

// Largest i with item0[i] <= item (item0 ascending, item0[0] == 0).
__device__ __forceinline__ uint32_t find_desc(const uint64_t* __restrict__ item0, uint32_t n,
                                              uint64_t item) {
  uint32_t lo = 0, hi = n;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(item0 + mid) <= item) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Byte offsets of row r: decompose r over the outer extents (32-bit: the
// compiler guarantees every extent and row count fits, see compile.cpp).
__device__ __forceinline__ void row_offsets(const rs_copy_desc& D, uint32_t r, int64_t& so,
                                            int64_t& dof) {
  so = 0;
  dof = 0;
  for (uint32_t k = 0; k < D.nouter; ++k) {
    const uint32_t e = static_cast<uint32_t>(D.ext[k]);
    const uint32_t q = r / e;
    const uint32_t i = r - q * e;
    so += static_cast<int64_t>(i) * D.sstr[k];
    dof += static_cast<int64_t>(i) * D.dstr[k];
    r = q;
  }
}

template <bool kReadOnly, int U = kUnroll, bool kStream = false, int kLd = 0>
__device__ __forceinline__ void warp_copy_item(const rs_copy_desc& D, uint64_t local_item,
                                               int lane) {
  const uint64_t r0 = local_item * D.rows_per_item;
  const uint64_t r1 = min(r0 + D.rows_per_item, D.rows);
  const char* src = reinterpret_cast<const char*>(D.src);
  char* dst = reinterpret_cast<char*>(D.dst);
  for (uint64_t r = r0; r < r1; ++r) {
    int64_t so, dof;
    row_offsets(D, static_cast<uint32_t>(r), so, dof);
    warp_copy_any<kReadOnly, U, kStream, kLd>(src + so, dst + dof, D.row_bytes, D.vec_log2, lane);
  }
}

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

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(done)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return done != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_store(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_addr(smem_src)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void bulk_load_hint(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                               uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void bulk_store_hint(void* gdst, const void* smem_src, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
               "r"(smem_addr(smem_src)), "r"(bytes), "l"(pol)
               : "memory");
}

// Order generic-proxy global accesses against async-proxy (TMA) ones.
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

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
    off += static_cast<uint32_t>(D.row_bytes);
  }
  bulk_commit();
  bulk_wait_all();
}

// ------------------------------------------------------------- pattern

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// 16 bytes of pattern starting at element g (elements of EB bytes, EB | 16).
template <int EB>
__device__ __forceinline__ uint4 pattern16(uint64_t base, int64_t g) {
  uint32_t w[4];
  if constexpr (EB == 8) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint64_t h = splitmix64(base ^ static_cast<uint64_t>(g + k));
      w[2 * k] = static_cast<uint32_t>(h);
      w[2 * k + 1] = static_cast<uint32_t>(h >> 32);
    }
  } else if constexpr (EB == 4) {
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] = static_cast<uint32_t>(splitmix64(base ^ static_cast<uint64_t>(g + k)));
  } else if constexpr (EB == 2) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t a = static_cast<uint32_t>(splitmix64(base ^ static_cast<uint64_t>(g + 2 * k))) & 0xffffu;
      const uint32_t b = static_cast<uint32_t>(splitmix64(base ^ static_cast<uint64_t>(g + 2 * k + 1))) & 0xffffu;
      w[k] = a | (b << 16);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t v = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        v |= (static_cast<uint32_t>(splitmix64(base ^ static_cast<uint64_t>(g + 4 * k + j))) & 0xffu) << (8 * j);
      w[k] = v;
    }
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}


template <int EB>
__device__ __forceinline__ uint32_t mismatch_count16(const uint4& have, const uint4& want) {
  const uint32_t hv[4] = {have.x, have.y, have.z, have.w};
  const uint32_t wv[4] = {want.x, want.y, want.z, want.w};
  uint32_t bad = 0;
  if constexpr (EB == 8) {
    bad += (hv[0] != wv[0]) | (hv[1] != wv[1]);
    bad += (hv[2] != wv[2]) | (hv[3] != wv[3]);
  } else if constexpr (EB == 4) {
#pragma unroll
    for (int k = 0; k < 4; ++k) bad += hv[k] != wv[k];
  } else if constexpr (EB == 2) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t x = hv[k] ^ wv[k];
      bad += ((x & 0xffffu) != 0) + ((x >> 16) != 0);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t x = hv[k] ^ wv[k];
#pragma unroll
      for (int j = 0; j < 4; ++j) bad += ((x >> (8 * j)) & 0xffu) != 0;
    }
  }
  return bad;
}

// One row of a pattern descriptor: g = global element index of the row start.
template <int EB, bool kVerify>
__device__ __forceinline__ uint32_t pattern_row_vec(char* row, uint64_t n_elems, uint64_t base,
                                                    int64_t g, int lane) {
  constexpr int kPer = 16 / EB;
  const uint64_t nvec = n_elems / kPer;
  uint4* p = reinterpret_cast<uint4*>(row);
  uint32_t bad = 0;
  for (uint64_t i = lane; i < nvec; i += 32) {
    const uint4 want = pattern16<EB>(base, g + static_cast<int64_t>(i) * kPer);
    if constexpr (kVerify) bad += mismatch_count16<EB>(__ldcg(p + i), want);
    else p[i] = want;
  }
  // tail elements
  for (uint64_t e = nvec * kPer + lane; e < n_elems; e += 32) {
    const uint64_t h = splitmix64(base ^ static_cast<uint64_t>(g + static_cast<int64_t>(e)));
    uint8_t* q = reinterpret_cast<uint8_t*>(row) + e * EB;
    bool ok = true;
#pragma unroll
    for (int b = 0; b < EB; ++b) {
      const uint8_t v = static_cast<uint8_t>(h >> ((b % 8) * 8));
      if constexpr (kVerify) ok &= q[b] == v;
      else q[b] = v;
    }
    if constexpr (kVerify) bad += !ok;
  }
  return bad;
}

template <bool kVerify>
__device__ __forceinline__ uint32_t pattern_row_any(char* row, uint64_t n_elems, uint32_t eb,
                                                    bool aligned, uint64_t base, int64_t g,
                                                    int lane) {
  if (aligned) {
    switch (eb) {
      case 1: return pattern_row_vec<1, kVerify>(row, n_elems, base, g, lane);
      case 2: return pattern_row_vec<2, kVerify>(row, n_elems, base, g, lane);
      case 4: return pattern_row_vec<4, kVerify>(row, n_elems, base, g, lane);
      case 8: return pattern_row_vec<8, kVerify>(row, n_elems, base, g, lane);
      default: break;
    }
  }
  uint32_t bad = 0;
  for (uint64_t e = lane; e < n_elems; e += 32) {
    const uint64_t h = splitmix64(base ^ static_cast<uint64_t>(g + static_cast<int64_t>(e)));
    uint8_t* q = reinterpret_cast<uint8_t*>(row) + e * eb;
    bool ok = true;
    for (uint32_t b = 0; b < eb; ++b) {
      const uint8_t v = static_cast<uint8_t>(h >> ((b % 8) * 8));
      if constexpr (kVerify) ok &= q[b] == v;
      else q[b] = v;
    }
    if constexpr (kVerify) bad += !ok;
  }
  return bad;
}

template <bool kVerify>
__global__ void __launch_bounds__(256) rs_pattern_kernel(const rs_pattern_desc* __restrict__ descs,
                                                         const uint64_t* __restrict__ item0,
                                                         uint32_t ndesc, uint64_t nitems,
                                                         uint64_t seed,
                                                         unsigned long long* mismatches,
                                                         unsigned long long* first_bad) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t item = warp; item < nitems; item += nwarps) {
    const uint32_t di = find_desc(item0, ndesc, item);
    const rs_pattern_desc& D = descs[di];
    const uint64_t base = seed ^ (0x1000003ULL * D.tensor_index);
    const uint64_t r0 = (item - D.item0) * D.rows_per_item;
    const uint64_t r1 = min(r0 + D.rows_per_item, D.rows);
    const uint64_t row_bytes = D.row_elems * D.elem_bytes;
    uint32_t bad = 0;
    for (uint64_t r = r0; r < r1; ++r) {
      int64_t g = D.g0;
      uint32_t rr = static_cast<uint32_t>(r);
      for (uint32_t k = 0; k < D.nouter; ++k) {
        const uint32_t e = static_cast<uint32_t>(D.ext[k]);
        const uint32_t q = rr / e;
        g += static_cast<int64_t>(rr - q * e) * D.gstr[k];
        rr = q;
      }
      char* row = reinterpret_cast<char*>(D.ptr) + r * row_bytes;
      const bool aligned = ((D.ptr | row_bytes) & 15u) == 0;
      bad += pattern_row_any<kVerify>(row, D.row_elems, D.elem_bytes, aligned, base, g, lane);
    }
    if constexpr (kVerify) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
      if (lane == 0 && bad) {
        atomicAdd(mismatches, static_cast<unsigned long long>(bad));
        atomicMin(first_bad, static_cast<unsigned long long>(D.entry));
      }
    }
  }
}

// ------------------------------------------------- L2 eviction-priority hints
//
// Ring staging wants the opposite of plain streaming: the slot a sender just
// packed should survive in L2 until the receiver unpacks it, while the source
// and destination shards stream through once.  createpolicy gives 64-bit L2
// cache policies; .L2::cache_hint loads / stores carry them.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
template <bool kReadOnly>
__device__ __forceinline__ uint4 load_hint(const uint4* p, uint64_t pol) {
  uint4 r;
  if constexpr (kReadOnly)
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
  else
    asm volatile("ld.global.cg.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ void store_hint(uint4* p, const uint4& v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w), "l"(pol)
               : "memory");
}

// warp_copy_item with L2 policies on the 16 B path (other widths unhinted).
template <bool kReadOnly, int U>
__device__ __forceinline__ void warp_copy_item_hint(const rs_copy_desc& D, uint64_t local_item, int lane,
                                                    uint64_t lpol, uint64_t spol) {
  if (D.vec_log2 != 4) {
    warp_copy_item<kReadOnly, U>(D, local_item, lane);
    return;
  }
  const uint64_t r0 = local_item * D.rows_per_item;
  const uint64_t r1 = min(r0 + D.rows_per_item, D.rows);
  for (uint64_t r = r0; r < r1; ++r) {
    int64_t so, dof;
    row_offsets(D, static_cast<uint32_t>(r), so, dof);
    const uint4* s = reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(D.src) + so);
    uint4* d = reinterpret_cast<uint4*>(reinterpret_cast<char*>(D.dst) + dof);
    const uint64_t n = D.row_bytes / 16;
    uint64_t i = static_cast<uint64_t>(lane);
    for (; i + 32 * (U - 1) < n; i += 32 * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = load_hint<kReadOnly>(s + i + 32 * u, lpol);
#pragma unroll
      for (int u = 0; u < U; ++u) store_hint(d + i + 32 * u, v[u], spol);
    }
    for (; i < n; i += 32) store_hint(d + i, load_hint<kReadOnly>(s + i, lpol), spol);
  }
}

// ------------------------------------------------------------- exchange

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Same-device lanes (sender and receiver CTAs on one GPU, one process) only
// need GPU scope: cheaper fences and flag accesses than .sys.
__device__ __forceinline__ uint64_t ld_acquire_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_gpu(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Publish everything this CTA wrote (after a __syncthreads) with one release.
__device__ __forceinline__ void publish(uint64_t* flag, uint64_t v, bool peer) {
  if (peer) {
    __threadfence_system();
    st_release_sys(flag, v);
  } else {
    __threadfence();
    st_release_gpu(flag, v);
  }
}

// Spin with a bounded budget; on expiry raise the error flag (no hangs on a
// protocol bug: the host reports failed_layer instead).
__device__ __forceinline__ bool wait_geq(const uint64_t* flag, uint64_t want,
                                         unsigned int* error_flag, uint64_t spin_limit, bool peer) {
  uint64_t spins = 0;
  while ((peer ? ld_acquire_sys(flag) : ld_acquire_gpu(flag)) < want) {
    if (*reinterpret_cast<volatile unsigned int*>(error_flag)) return false;
    if (++spins > spin_limit) {
      atomicExch(error_flag, 1u);
      return false;
    }
    __nanosleep(64);
  }
  return true;
}

// Drop one 128 B line from L2 without writing it back (its value becomes
// undefined).  A drained ring slot is rewritten by the next batch, so its
// dirty lines never need to reach HBM: with slots small enough to stay
// L2-resident the staging traffic never leaves the L2.
__device__ __forceinline__ void discard_l2_line(uint64_t a) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
}

// Frame of batch-relative item `it`: largest f with frames[f].item0 <= it.
__device__ __forceinline__ uint32_t find_frame(const rs_copy_desc* __restrict__ frames, uint32_t n, uint32_t it) {
  uint32_t lo = 0, hi = n;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (frames[mid].item0 <= it) lo = mid;
    else hi = mid;
  }
  return lo;
}

// One work item through the copy warp's shared-memory buffer with TMA (the
// elected lane issues everything): bulk-load the item's rows on the warp's
// mbarrier, wait, bulk-store them, and wait until the stores have read the
// buffer.  Returns false (nothing done) when the item does not fit the buffer
// or is not 16 B aligned -- the caller copies it with the warp instead.
constexpr uint32_t kLaneTmaBytes = 16384;

__device__ __forceinline__ bool tma_copy_item(const rs_copy_desc& D, uint64_t local_item, unsigned char* buf,
                                              uint64_t* bar, uint32_t& phase, uint64_t lpol, uint64_t spol,
                                              int lane) {
  const uint64_t r0 = local_item * D.rows_per_item;
  const uint64_t r1 = min(r0 + D.rows_per_item, D.rows);
  const uint64_t total = (r1 - r0) * D.row_bytes;
  if (D.vec_log2 != 4 || total > kLaneTmaBytes) return false;
  if (lane == 0) {
    mbar_expect_tx(bar, static_cast<uint32_t>(total));
    uint32_t off = 0;
    for (uint64_t r = r0; r < r1; ++r) {
      int64_t so, dof;
      row_offsets(D, static_cast<uint32_t>(r), so, dof);
      bulk_load_hint(buf + off, reinterpret_cast<const void*>(D.src + so), static_cast<uint32_t>(D.row_bytes), bar,
                     lpol);
      off += static_cast<uint32_t>(D.row_bytes);
    }
    mbar_wait(bar, phase);
    off = 0;
    for (uint64_t r = r0; r < r1; ++r) {
      int64_t so, dof;
      row_offsets(D, static_cast<uint32_t>(r), so, dof);
      bulk_store_hint(reinterpret_cast<void*>(D.dst + dof), buf + off, static_cast<uint32_t>(D.row_bytes), spol);
      off += static_cast<uint32_t>(D.row_bytes);
    }
    bulk_commit();
    bulk_wait_read<0>();
  }
  phase ^= 1;
  __syncwarp();
  return true;
}

// flags of rs_launch_exchange
constexpr int kExFaultRx = 1;   // test hook: ring receivers drop out (peer failure)
constexpr int kExDiscard = 2;   // receivers discard drained slot lines from L2
constexpr int kExHints = 4;     // L2 policies: shards evict-first, ring slots evict-last
constexpr int kExWarpSpec = 8;  // warp-specialised lanes: a control warp runs the handshakes
constexpr int kExLaneTma = 16;  // (with kExWarpSpec) copy warps move items with TMA bulk copies

// Block roles: blocks [0, ntx) send lanes_tx[b], [ntx, ntx + nrx) receive
// lanes_rx[b - ntx], the rest run the local (DIRECT) copy list.  The launch
// never exceeds the co-resident CTA capacity, so every waiting role has its
// counterpart running (same device) or launched on its own device (peers).
template <int kThreads>
__global__ void __launch_bounds__(kThreads) rs_exchange_kernel(
    const rs_lane_desc* __restrict__ lanes_tx, uint32_t ntx, const rs_lane_desc* __restrict__ lanes_rx,
    uint32_t nrx, const rs_batch_desc* __restrict__ batches,
    const rs_copy_desc* __restrict__ frames, const rs_copy_desc* __restrict__ local_descs,
    const uint64_t* __restrict__ local_item0, uint32_t nlocal, uint64_t local_items, uint64_t epoch,
    unsigned int* error_flag, uint64_t spin_limit, int flags) {
  const int lane_id = threadIdx.x & 31;
  const int warp_in_block = threadIdx.x >> 5;
  const int warps_per_block = blockDim.x >> 5;
  __shared__ int ok_shared;

  if (blockIdx.x < ntx + nrx) {
    const bool sender = blockIdx.x < ntx;
    if ((flags & kExFaultRx) && !sender) return;  // test hook: the receiving peer is gone
    const rs_lane_desc L = sender ? lanes_tx[blockIdx.x] : lanes_rx[blockIdx.x - ntx];
    const bool peer = (L.flags & RS_LANE_PEER) != 0;
    const uint64_t pol_first = (flags & kExHints) ? policy_evict_first() : 0;
    const uint64_t pol_last = (flags & kExHints) ? policy_evict_last() : 0;
    if (flags & kExWarpSpec) {
      // Warp-specialised lane: warp 0 polls flags, publishes and discards;
      // warps 1.. copy.  Two mbarrier pairs hand batches over: go[b % 2]
      // (control -> copy: slot free / data ready) and done[b % 2] (copy ->
      // control: batch copied), so the copy warps work on batch b while the
      // control warp fences and publishes batch b - 1 and polls for b + 1.
      __shared__ __align__(8) uint64_t go_bar[2], done_bar[2];
      __shared__ int abort_shared;
      const int ncopy = warps_per_block - 1;
      if (threadIdx.x == 0) {
        mbar_init(&go_bar[0], 1);
        mbar_init(&go_bar[1], 1);
        mbar_init(&done_bar[0], static_cast<uint32_t>(ncopy));
        mbar_init(&done_bar[1], static_cast<uint32_t>(ncopy));
        abort_shared = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
      __syncthreads();
      if (warp_in_block == 0) {
        // Event loop, the whole warp in lockstep (lane 0 polls, shuffles the
        // verdicts): hand batch g to the copy warps as soon as its flag is up
        // (ready for receivers, the credit of batch g - K for senders) and
        // publish batch f as soon as its copy is done -- neither waits behind
        // the other, so no circular wait between the two ends even at K = 2.
        // go(g) needs done(g - 2) consumed (mbarrier phase reuse): g <= f + 1.
        uint32_t g = 0, f = 0;
        uint64_t idle = 0;
        while (f < L.nbatches) {
          bool progress = false;
          if (g < L.nbatches && g <= f + 1) {
            int up = 0;
            if (lane_id == 0) {
              if (sender) {
                up = g < L.slots ||
                     (peer ? ld_acquire_sys(reinterpret_cast<const uint64_t*>(L.credit_flags_tx) + g % L.slots)
                           : ld_acquire_gpu(reinterpret_cast<const uint64_t*>(L.credit_flags_tx) + g % L.slots)) >=
                         epoch + g - L.slots + 1;
              } else {
                up = (peer ? ld_acquire_sys(reinterpret_cast<const uint64_t*>(L.ready_flags_rx) + g % L.slots)
                           : ld_acquire_gpu(reinterpret_cast<const uint64_t*>(L.ready_flags_rx) + g % L.slots)) >=
                     epoch + g + 1;
              }
              if (up) mbar_arrive(&go_bar[g & 1]);
            }
            if (__shfl_sync(0xffffffffu, up, 0)) {
              ++g;
              progress = true;
            }
          }
          if (f < g && mbar_test(&done_bar[f & 1], (f >> 1) & 1)) {
            const rs_batch_desc Bc = batches[L.batch0 + f];
            const uint32_t sc = f % L.slots;
            if (!sender && (flags & kExDiscard) && Bc.extent && ((L.slot_base_rx | L.slot_bytes) & 127) == 0) {
              const uint64_t base = L.slot_base_rx + static_cast<uint64_t>(sc) * L.slot_bytes;
              const uint64_t lines = (Bc.extent + 127) >> 7;
              for (uint64_t i = lane_id; i < lines; i += 32) discard_l2_line(base + (i << 7));
            }
            __syncwarp();
            if (lane_id == 0)
              publish(reinterpret_cast<uint64_t*>(sender ? L.ready_flags : L.credit_flags) + sc, epoch + f + 1, peer);
            ++f;
            progress = true;
          }
          if (progress) {
            idle = 0;
            continue;
          }
          int stop = 0;
          if (lane_id == 0) {
            if (*reinterpret_cast<volatile unsigned int*>(error_flag)) stop = 1;
            else if (++idle > spin_limit) {
              atomicExch(error_flag, 1u);
              stop = 1;
            }
            if (stop && g < L.nbatches) {  // wake the copy warps waiting for batch g: they see the abort
              abort_shared = 1;
              mbar_arrive(&go_bar[g & 1]);
            }
            if (!stop) __nanosleep(64);
          }
          if (__shfl_sync(0xffffffffu, stop, 0)) return;
        }
      } else {
        const int cw = warp_in_block - 1;
        extern __shared__ __align__(128) unsigned char lane_smem[];
        const bool tma = (flags & kExLaneTma) != 0;
        __shared__ __align__(8) uint64_t tma_bar[32];
        unsigned char* buf = lane_smem + static_cast<size_t>(cw) * kLaneTmaBytes;
        uint32_t phase = 0;
        if (tma && lane_id == 0) {
          mbar_init(&tma_bar[cw], 1);
          asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        const uint64_t tpol_first = policy_evict_first(), tpol_last = policy_evict_last();
        for (uint32_t b = 0; b < L.nbatches; ++b) {
          mbar_wait(&go_bar[b & 1], (b >> 1) & 1);
          if (*reinterpret_cast<volatile int*>(&abort_shared)) return;
          const rs_batch_desc B = batches[L.batch0 + b];
          // receivers: the slot bytes were published through the generic proxy
          if (tma && !sender && lane_id == 0) fence_proxy_async_global();
          __syncwarp();
          if (sender) {
            for (uint32_t it = cw; it < B.pack_items; it += ncopy) {
              const rs_copy_desc& D = frames[B.pack0 + find_frame(frames + B.pack0, B.npack, it)];
              if (tma && tma_copy_item(D, it - D.item0, buf, &tma_bar[cw], phase, tpol_first, tpol_last, lane_id))
                continue;
              if (flags & kExHints) warp_copy_item_hint<true, 8>(D, it - D.item0, lane_id, pol_first, pol_last);
              else warp_copy_item<true, 8>(D, it - D.item0, lane_id);
            }
          } else {
            for (uint32_t it = cw; it < B.unpack_items; it += ncopy) {
              const rs_copy_desc& D = frames[B.unpack0 + find_frame(frames + B.unpack0, B.nunpack, it)];
              if (tma && tma_copy_item(D, it - D.item0, buf, &tma_bar[cw], phase, tpol_first, tpol_first, lane_id))
                continue;
              if (flags & kExHints) warp_copy_item_hint<false, 8>(D, it - D.item0, lane_id, pol_first, pol_first);
              else warp_copy_item<false, 8>(D, it - D.item0, lane_id);
            }
          }
          // senders: the slot writes of the async proxy complete and become
          // ordered before the control warp's release
          if (tma && lane_id == 0) {
            bulk_wait_all();
            fence_proxy_async_global();
          }
          __syncwarp();
          if (lane_id == 0) mbar_arrive(&done_bar[b & 1]);
        }
      }
      return;
    }
    for (uint32_t b = 0; b < L.nbatches; ++b) {
      const rs_batch_desc B = batches[L.batch0 + b];
      const uint32_t slot = b % L.slots;
      const uint64_t seq = epoch + b + 1;           // value published for batch b
      if (threadIdx.x == 0) {
        bool ok;
        if (sender) {
          // slot reuse: the receiver must have drained batch b - slots
          ok = b < L.slots ||
               wait_geq(reinterpret_cast<const uint64_t*>(L.credit_flags_tx) + slot,
                        epoch + b - L.slots + 1, error_flag, spin_limit, peer);
        } else {
          ok = wait_geq(reinterpret_cast<const uint64_t*>(L.ready_flags_rx) + slot, seq, error_flag,
                        spin_limit, peer);
        }
        ok_shared = ok;
      }
      __syncthreads();
      if (!ok_shared) return;
      if (sender) {
        // pack: the batch's frames copy their source boxes into the slot
        // (remote stores); one flat item space over the frames, dealt to warps
        for (uint32_t it = warp_in_block; it < B.pack_items; it += warps_per_block) {
          const rs_copy_desc& D = frames[B.pack0 + find_frame(frames + B.pack0, B.npack, it)];
          if (flags & kExHints) warp_copy_item_hint<true, 8>(D, it - D.item0, lane_id, pol_first, pol_last);
          else warp_copy_item<true, 8>(D, it - D.item0, lane_id);
        }
        __syncthreads();
        if (threadIdx.x == 0) publish(reinterpret_cast<uint64_t*>(L.ready_flags) + slot, seq, peer);
      } else {
        for (uint32_t it = warp_in_block; it < B.unpack_items; it += warps_per_block) {
          const rs_copy_desc& D = frames[B.unpack0 + find_frame(frames + B.unpack0, B.nunpack, it)];
          if (flags & kExHints) warp_copy_item_hint<false, 8>(D, it - D.item0, lane_id, pol_first, pol_first);
          else warp_copy_item<false, 8>(D, it - D.item0, lane_id);
        }
        if ((flags & kExDiscard) && B.extent && ((L.slot_base_rx | L.slot_bytes) & 127) == 0) {
          // every load of the slot has completed (its data was stored); the
          // discards are ordered before the credit like writes (bar + fence)
          __syncthreads();
          const uint64_t base = L.slot_base_rx + static_cast<uint64_t>(slot) * L.slot_bytes;
          const uint64_t lines = (B.extent + 127) >> 7;
          for (uint64_t i = threadIdx.x; i < lines; i += blockDim.x) discard_l2_line(base + (i << 7));
        }
        __syncthreads();
        if (threadIdx.x == 0) publish(reinterpret_cast<uint64_t*>(L.credit_flags) + slot, seq, peer);
      }
    }
    return;
  }

  // local copy role
  const uint64_t warp = (static_cast<uint64_t>(blockIdx.x - ntx - nrx) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x - ntx - nrx) * blockDim.x) >> 5;
  for (uint64_t item = warp; item < local_items; item += nwarps) {
    const uint32_t di = find_desc(local_item0, nlocal, item);
    warp_copy_item<true, 8>(local_descs[di], item - local_descs[di].item0, lane_id);
  }
}

template <int W, int S, int L, uint32_t T>
cudaError_t launch_bulk_mw(const rs_copy_desc* descs, const uint64_t* item0, uint32_t ndesc, uint64_t item_begin,
                           uint64_t item_end, int grid, cudaStream_t stream) {
  static bool configured = false;
  const int smem = W * S * static_cast<int>(T);
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(rs_copy_bulk_mw_kernel<W, S, L, T>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
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
      static bool configured = false;
      const int smem = kBulkStages * static_cast<int>(kBulkStageBytes);
      if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(rs_copy_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        configured = true;
      }
      rs_copy_bulk_kernel<<<grid, 32, smem, stream>>>(descs, item0, ndesc, item_begin, item_end);
      break;
    }
    default:
      rs_copy_kernel<4><<<grid, 256, 0, stream>>>(descs, item0, ndesc, item_begin, item_end);
  }
  return cudaGetLastError();
}

cudaError_t rs_launch_pattern(const rs_pattern_desc* descs, const uint64_t* item0, uint32_t ndesc,
                              uint64_t nitems, uint64_t seed, int verify,
                              unsigned long long* mismatches, unsigned long long* first_bad,
                              int grid, cudaStream_t stream) {
  if (nitems == 0 || ndesc == 0) return cudaSuccess;
  if (verify)
    rs_pattern_kernel<true><<<grid, 256, 0, stream>>>(descs, item0, ndesc, nitems, seed, mismatches, first_bad);
  else
    rs_pattern_kernel<false><<<grid, 256, 0, stream>>>(descs, item0, ndesc, nitems, seed, mismatches, first_bad);
  return cudaGetLastError();
}

cudaError_t rs_launch_exchange(const rs_lane_desc* lanes_tx, uint32_t ntx, const rs_lane_desc* lanes_rx,
                               uint32_t nrx, const rs_batch_desc* batches, const rs_copy_desc* frames,
                               const rs_copy_desc* local_descs, const uint64_t* local_item0,
                               uint32_t nlocal, uint64_t local_items, uint64_t epoch,
                               unsigned int* error_flag, uint64_t spin_limit, int flags,
                               int local_blocks, int threads, cudaStream_t stream) {
  const int grid = static_cast<int>(ntx + nrx) + (local_items ? local_blocks : 0);
  if (grid == 0) return cudaSuccess;
  const int smem = (flags & kExLaneTma) ? (threads / 32 - 1) * static_cast<int>(kLaneTmaBytes) : 0;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaSuccess;
    if (threads == 1024) e = cudaFuncSetAttribute(rs_exchange_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    else if (threads == 512) e = cudaFuncSetAttribute(rs_exchange_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    else e = cudaFuncSetAttribute(rs_exchange_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
#define RS_EXCHANGE_LAUNCH(T)                                                                                 \
  rs_exchange_kernel<T><<<grid, T, smem, stream>>>(lanes_tx, ntx, lanes_rx, nrx, batches, frames, local_descs,  \
                                                   local_item0, nlocal, local_items, epoch, error_flag, spin_limit, \
                                                   flags)
  if (threads == 1024) RS_EXCHANGE_LAUNCH(1024);
  else if (threads == 512) RS_EXCHANGE_LAUNCH(512);
  else RS_EXCHANGE_LAUNCH(256);
#undef RS_EXCHANGE_LAUNCH
  return cudaGetLastError();
}

int rs_kernel_max_blocks_per_sm(int which) {
  int n = 0;
  if (which == 0) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rs_copy_kernel<4>, 256, 0);
  else if (which == 3) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rs_copy_kernel<8>, 256, 0);
  else if (which == 5) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rs_copy_kernel<16>, 256, 0);
  else if (which == 6) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rs_copy_cta_kernel<8>, 256, 0);
  else if (which == 4) n = 1;  // bulk ring: one CTA (one issuer, ~200 KB smem) per SM
  else if (which == 1) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rs_pattern_kernel<false>, 256, 0);
  else if (which == 9) {
    const int smem = 7 * static_cast<int>(kLaneTmaBytes);
    cudaFuncSetAttribute(rs_exchange_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rs_exchange_kernel<256>, 256, smem);
  } else if (which == 7) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rs_exchange_kernel<512>, 512, 0);
  else if (which == 8) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rs_exchange_kernel<1024>, 1024, 0);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rs_exchange_kernel<256>, 256, 0);
  return n;
}

}  // extern "C"
