// Synthetic-state kernels (test infrastructure): fill / verify shard buffers
// against the reference pattern (proj/src/shard_store.cpp:12-85), one hash
// per element, 16 B stores / compares.
#include <cuda_runtime.h>
#include <stdint.h>

#include "desc.h"
#include "device_common.cuh"
#include "kernels.h"

namespace {

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

}  // namespace

extern "C" {

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

int pattern_max_blocks_per_sm() {
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rs_pattern_kernel<false>, 256, 0);
  return n;
}

}  // extern "C"
