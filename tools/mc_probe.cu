// NVSwitch multicast / VMM capability probe (standalone binary, not product code).
//
// Prints the device attributes the multicast DP-broadcast path needs, then
// tries the whole chain on the one visible GPU: cuMemCreate physical memory,
// cuMulticastCreate (1 device), cuMulticastAddDevice, cuMulticastBindMem, map
// the multicast VA, store through it with multimem.st, read the bytes back
// through the unicast mapping; plus fabric / POSIX-FD handle export.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/mc_probe.cu -lcuda -o /tmp/mc_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    CUresult r_ = (x);                                                                 \
    if (r_ != CUDA_SUCCESS) {                                                          \
      const char* s_ = nullptr;                                                        \
      cuGetErrorName(r_, &s_);                                                         \
      std::printf("{\"step\": \"%s\", \"ok\": false, \"err\": \"%s\"}\n", #x, s_ ? s_ : "?"); \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)

__global__ void mc_store(uint4* mc, const uint4* src, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = src[i];
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + i), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
  }
}

int main() {
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUcontext ctx;
  CK(cuDevicePrimaryCtxRetain(&ctx, dev));
  CK(cuCtxSetCurrent(ctx));
  const struct { const char* name; CUdevice_attribute a; } attrs[] = {
      {"vmm", CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED},
      {"posix_fd", CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED},
      {"fabric", CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED},
      {"multicast", CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED},
  };
  int mc_supported = 0;
  for (auto& x : attrs) {
    int v = -1;
    cuDeviceGetAttribute(&v, x.a, dev);
    std::printf("{\"attr\": \"%s\", \"value\": %d}\n", x.name, v);
    if (x.a == CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED) mc_supported = v;
  }
  int count = 0;
  cuDeviceGetCount(&count);
  std::printf("{\"visible_devices\": %d}\n", count);

  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = 0;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  CK(cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  std::printf("{\"vmm_granularity\": %zu}\n", gran);

  // handle export: POSIX fd and fabric
  {
    CUmemGenericAllocationHandle h;
    CK(cuMemCreate(&h, gran, &prop, 0));
    int fd = -1;
    CUresult r = cuMemExportToShareableHandle(&fd, h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    std::printf("{\"export_posix_fd\": %d}\n", r == CUDA_SUCCESS);
    cuMemRelease(h);
    CUmemAllocationProp fp = prop;
    fp.requestedHandleTypes = CU_MEM_HANDLE_TYPE_FABRIC;
    r = cuMemCreate(&h, gran, &fp, 0);
    if (r == CUDA_SUCCESS) {
      CUmemFabricHandle fh;
      CUresult r2 = cuMemExportToShareableHandle(&fh, h, CU_MEM_HANDLE_TYPE_FABRIC, 0);
      const char* s = nullptr;
      cuGetErrorName(r2, &s);
      std::printf("{\"export_fabric\": %d, \"err\": \"%s\"}\n", r2 == CUDA_SUCCESS, s ? s : "");
      cuMemRelease(h);
    } else {
      const char* s = nullptr;
      cuGetErrorName(r, &s);
      std::printf("{\"create_fabric\": 0, \"err\": \"%s\"}\n", s ? s : "");
    }
  }
  if (!mc_supported) {
    std::printf("{\"multicast\": \"unsupported on this device\"}\n");
    return 0;
  }

  CUmulticastObjectProp mp{};
  mp.numDevices = 1;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t mc_min = 0, mc_rec = 0;
  mp.size = gran;
  CK(cuMulticastGetGranularity(&mc_min, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  CK(cuMulticastGetGranularity(&mc_rec, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  std::printf("{\"mc_granularity_min\": %zu, \"mc_granularity_recommended\": %zu}\n", mc_min, mc_rec);
  const size_t bytes = ((size_t(64) << 20) + mc_rec - 1) / mc_rec * mc_rec;
  mp.size = bytes;
  CUmemGenericAllocationHandle mc;
  // which object shapes does the driver accept with one visible GPU?
  for (unsigned nd : {1u, 2u, 8u})
    for (int ht : {0, (int)CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, (int)CU_MEM_HANDLE_TYPE_FABRIC}) {
      CUmulticastObjectProp t = mp;
      t.numDevices = nd;
      t.handleTypes = static_cast<unsigned long long>(ht);
      CUmemGenericAllocationHandle h;
      CUresult r = cuMulticastCreate(&h, &t);
      const char* s = nullptr;
      cuGetErrorName(r, &s);
      std::printf("{\"mc_create\": {\"numDevices\": %u, \"handleTypes\": %d}, \"result\": \"%s\"}\n", nd, ht, s ? s : "?");
      if (r == CUDA_SUCCESS) {
        CUresult a = cuMulticastAddDevice(h, dev);
        cuGetErrorName(a, &s);
        std::printf("{\"mc_add_device\": \"%s\"}\n", s ? s : "?");
        cuMemRelease(h);
      }
    }
  mp.handleTypes = 0;
  CK(cuMulticastCreate(&mc, &mp));
  CK(cuMulticastAddDevice(mc, dev));
  CUmemGenericAllocationHandle phys;
  CK(cuMemCreate(&phys, bytes, &prop, 0));
  CK(cuMulticastBindMem(mc, 0, phys, 0, bytes, 0));
  CUdeviceptr uc = 0, mcva = 0;
  CK(cuMemAddressReserve(&uc, bytes, mc_rec, 0, 0));
  CK(cuMemMap(uc, bytes, 0, phys, 0));
  CK(cuMemAddressReserve(&mcva, bytes, mc_rec, 0, 0));
  CK(cuMemMap(mcva, bytes, 0, mc, 0));
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = 0;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc, bytes, &acc, 1));
  CK(cuMemSetAccess(mcva, bytes, &acc, 1));
  // random bytes incl. NaN encodings through a .f32 multimem store
  std::vector<uint32_t> host(bytes / 4);
  uint64_t x = 0x9E3779B97F4A7C15ull;
  for (auto& w : host) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    w = static_cast<uint32_t>(x);
  }
  for (size_t i = 0; i < host.size(); i += 97) host[i] = 0x7fc00001u + (uint32_t)(i & 0xff);  // NaN payloads
  void* src = nullptr;
  cudaMalloc(&src, bytes);
  cudaMemcpy(src, host.data(), bytes, cudaMemcpyHostToDevice);
  CK(cuMemsetD8(uc, 0, bytes));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  mc_store<<<148 * 8, 256>>>(reinterpret_cast<uint4*>(mcva), static_cast<const uint4*>(src), bytes / 16);
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i)
    mc_store<<<148 * 8, 256>>>(reinterpret_cast<uint4*>(mcva), static_cast<const uint4*>(src), bytes / 16);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  std::vector<uint32_t> back(bytes / 4);
  cudaMemcpy(back.data(), reinterpret_cast<void*>(uc), bytes, cudaMemcpyDeviceToHost);
  size_t bad = 0;
  for (size_t i = 0; i < back.size(); ++i) bad += back[i] != host[i];
  std::printf("{\"multimem_st\": \"%s\", \"bytes\": %zu, \"mismatched_words\": %zu, \"GBps_read_plus_write\": %.1f}\n",
              cudaGetErrorName(e), bytes, bad, 2.0 * bytes * 10 / (ms / 1e3) / 1e9);
  return 0;
}
