// L2 / HBM copy-throughput probe (measurement tool, not product code).
//
// The STAGED ring lanes are TMA bulk copies through shared memory whose slot
// traffic should stay in L2.  This probe measures what the memory system
// sustains for the same access shape: 1-warp CTAs, two 16 KB shared-memory
// stages each, bulk global->smem loads (mbarrier complete_tx) and smem->global
// bulk stores, with the source / destination working sets chosen small
// (L2-resident) or large (HBM).  Bytes counted: read + written.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC tools/l2_probe.cu -o tools/_l2_probe.so
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

constexpr uint32_t kStage = 16384;

__device__ __forceinline__ uint32_t smem(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(32) probe_kernel(const char* src, uint64_t src_bytes, char* dst, uint64_t dst_bytes,
                                                   uint64_t items) {
  extern __shared__ __align__(128) unsigned char st[];
  __shared__ __align__(8) uint64_t bar[2];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint64_t n = 0;  // items this CTA has issued
  for (uint64_t it = blockIdx.x; it < items; it += gridDim.x, ++n) {
    const uint32_t s = static_cast<uint32_t>(n & 1);
    if (threadIdx.x == 0) {
      if (n >= 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // stage s free again
      const char* g = src + (it * kStage) % src_bytes;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem(&bar[s])), "r"(kStage) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem(st + s * kStage)),
                   "l"(g), "r"(kStage), "r"(smem(&bar[s]))
                   : "memory");
      const uint32_t parity = static_cast<uint32_t>((n >> 1) & 1);
      uint32_t done = 0;
      while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem(&bar[s])), "r"(parity)
            : "memory");
      char* d = dst + (it * kStage) % dst_bytes;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d), "r"(smem(st + s * kStage)),
                   "r"(kStage)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace

extern "C" int l2_probe(const void* src, uint64_t src_bytes, void* dst, uint64_t dst_bytes, uint64_t items, int grid,
                        float* ms) {
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kStage);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  probe_kernel<<<grid, 32, 2 * kStage>>>(static_cast<const char*>(src), src_bytes, static_cast<char*>(dst), dst_bytes,
                                         items);  // warm-up
  cudaEventRecord(a);
  probe_kernel<<<grid, 32, 2 * kStage>>>(static_cast<const char*>(src), src_bytes, static_cast<char*>(dst), dst_bytes,
                                         items);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return static_cast<int>(cudaGetLastError());
}
