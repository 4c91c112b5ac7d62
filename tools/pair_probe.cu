// Ring-lane shape probe (measurement tool, not product code): what one GPU
// sustains when every CTA runs a sender (HBM -> L2-resident slot) next to a
// receiver (slot -> HBM), with no handshakes -- the transfer shapes of a
// STAGED lane pair, to compare receiver designs before building one.
//   mode 0: both halves are TMA warps with 2 x 16 KB stages each (64 KB smem/CTA)
//   mode 1: TMA sender warp (2 x 16 KB stages) + register receiver warp
//           (LDG.128 x U from the slot, STG.128 to HBM; no shared memory)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC tools/pair_probe.cu -o tools/_pair_probe.so
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

constexpr uint32_t kStage = 16384;

__device__ __forceinline__ uint32_t smem(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void tma_warp(const char* src, uint64_t src_bytes, char* dst, uint64_t dst_bytes,
                                         uint64_t items, uint64_t first, uint64_t stride, unsigned char* st,
                                         uint64_t* bar) {
  if ((threadIdx.x & 31) != 0) return;
  uint64_t n = 0;
  for (uint64_t it = first; it < items; it += stride, ++n) {
    const uint32_t s = static_cast<uint32_t>(n & 1);
    if (n >= 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem(&bar[s])), "r"(kStage) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem(st + s * kStage)),
                 "l"(src + (it * kStage) % src_bytes), "r"(kStage), "r"(smem(&bar[s]))
                 : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(smem(&bar[s])), "r"(static_cast<uint32_t>((n >> 1) & 1))
                   : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + (it * kStage) % dst_bytes),
                 "r"(smem(st + s * kStage)), "r"(kStage)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int U>
__device__ __forceinline__ void reg_warp(const char* src, uint64_t src_bytes, char* dst, uint64_t dst_bytes,
                                         uint64_t items, uint64_t first, uint64_t stride) {
  const int lane = threadIdx.x & 31;
  for (uint64_t it = first; it < items; it += stride) {
    const uint4* s = reinterpret_cast<const uint4*>(src + (it * kStage) % src_bytes);
    uint4* d = reinterpret_cast<uint4*>(dst + (it * kStage) % dst_bytes);
    for (uint32_t i = lane; i < kStage / 16; i += 32 * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldcg(s + i + 32 * u);
#pragma unroll
      for (int u = 0; u < U; ++u) __stcs(d + i + 32 * u, v[u]);
    }
  }
}

// warp 0: sender (big src -> small slot buffer); warp 1: receiver (small slot buffer -> big dst)
template <int kMode>
__global__ void __launch_bounds__(64) pair_kernel(const char* hbm_src, uint64_t hbm_src_bytes, char* slots,
                                                  uint64_t slot_bytes, char* hbm_dst, uint64_t hbm_dst_bytes,
                                                  uint64_t items) {
  extern __shared__ __align__(128) unsigned char st[];
  __shared__ __align__(8) uint64_t bar[4];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    tma_warp(hbm_src, hbm_src_bytes, slots, slot_bytes, items, blockIdx.x, gridDim.x, st, bar);
  } else if (kMode == 0) {
    tma_warp(slots, slot_bytes, hbm_dst, hbm_dst_bytes, items, blockIdx.x, gridDim.x, st + 2 * kStage, bar + 2);
  } else {
    reg_warp<8>(slots, slot_bytes, hbm_dst, hbm_dst_bytes, items, blockIdx.x, gridDim.x);
  }
}

}  // namespace

extern "C" int pair_probe(int mode, const void* src, uint64_t src_bytes, void* slots, uint64_t slot_bytes, void* dst,
                          uint64_t dst_bytes, uint64_t items, int grid, float* ms) {
  const int smem = mode == 0 ? 4 * kStage : 2 * kStage;
  auto k = mode == 0 ? pair_kernel<0> : pair_kernel<1>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<<<grid, 64, smem>>>(static_cast<const char*>(src), src_bytes, static_cast<char*>(slots), slot_bytes,
                        static_cast<char*>(dst), dst_bytes, items);
  cudaEventRecord(a);
  k<<<grid, 64, smem>>>(static_cast<const char*>(src), src_bytes, static_cast<char*>(slots), slot_bytes,
                        static_cast<char*>(dst), dst_bytes, items);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pair_probe_occupancy(int mode) {
  const int smem = mode == 0 ? 4 * kStage : 2 * kStage;
  auto k = mode == 0 ? pair_kernel<0> : pair_kernel<1>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, 64, smem);
  return n;
}
