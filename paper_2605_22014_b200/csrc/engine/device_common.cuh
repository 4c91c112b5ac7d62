// Device helpers shared by the engine's kernels (copy_kernels.cu,
// pattern_kernel.cu, exchange_kernel.cu): vector loads / stores, the warp
// copy engine over rs_copy_desc work items, mbarrier and TMA bulk-copy
// wrappers, L2 eviction-priority policies.  Internal header: every kernel TU
// gets its own copies (anonymous namespace, no relocatable device code).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "desc.h"

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
                                              int lane, int64_t dst2 = 0) {
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
    if (dst2) {  // DP broadcast: the same registers to the second destination
      T* d2 = reinterpret_cast<T*>(dst + dst2);
#pragma unroll
      for (int u = 0; u < U; ++u) store<T>(d2 + i + 32 * u, v[u]);
    }
  }
  for (; i < n; i += 32) {
    const T v = load<T, kReadOnly>(s + i);
    store<T>(d + i, v);
    if (dst2) store<T>(reinterpret_cast<T*>(dst + dst2) + i, v);
  }
}

template <bool kReadOnly, int U = kUnroll, bool kStream = false, int kLd = 0>
__device__ __forceinline__ void warp_copy_any(const char* src, char* dst, uint64_t nbytes,
                                              uint32_t vec_log2, int lane, int64_t dst2 = 0) {
  switch (vec_log2) {
    case 4: warp_copy_run<uint4, kReadOnly, U, kStream, kLd>(src, dst, nbytes, lane, dst2); break;
    case 3: warp_copy_run<uint2, kReadOnly>(src, dst, nbytes, lane, dst2); break;
    case 2: warp_copy_run<uint32_t, kReadOnly>(src, dst, nbytes, lane, dst2); break;
    case 1: warp_copy_run<uint16_t, kReadOnly>(src, dst, nbytes, lane, dst2); break;
    default: warp_copy_run<uint8_t, kReadOnly>(src, dst, nbytes, lane, dst2); break;
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
  // unrolled over the fixed capacity (constant indices: a descriptor held by
  // value stays in registers)
#pragma unroll
  for (uint32_t k = 0; k < RS_MAX_OUTER; ++k) {
    if (k < D.nouter) {
      const uint32_t e = static_cast<uint32_t>(D.ext[k]);
      const uint32_t q = r / e;
      const uint32_t i = r - q * e;
      so += static_cast<int64_t>(i) * D.sstr[k];
      dof += static_cast<int64_t>(i) * D.dstr[k];
      r = q;
    }
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
    warp_copy_any<kReadOnly, U, kStream, kLd>(src + so, dst + dof, D.row_bytes, D.vec_log2, lane, D.dst2_delta);
  }
}

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

}  // namespace
