// Ring-staged transfer kernel (STAGED mode): sender CTAs pack frames into the
// receiver's staging slots (peer stores over NVLink when the receiver is
// another GPU), publish with a release flag; receiver CTAs acquire, unpack,
// return a credit (bounded staging, proj/src/executor.cpp:183-206); spare
// CTAs run the local copies.  Integer / byte movement only.
#include <cuda_runtime.h>
#include <stdint.h>

#include "desc.h"
#include "device_common.cuh"
#include "kernels.h"

namespace {

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

// Strict layer barrier `li`: the whole CTA calls it after its
// layer-li work.  Arrivals are cumulative over the launch (a CTA cannot pass
// barrier li before every CTA arrived at it), so one counter serves every
// layer.  The GPU's last arriver publishes the slot's layer-done flag, waits
// for every slot's (peer-mapped, system scope) and releases its GPU.
// Bounded like every ring wait: false = abort (error flag raised).
__device__ __noinline__ bool layer_barrier(const rs_layer_sync& S, uint32_t li, uint64_t epoch,
                                           unsigned int* error_flag, uint64_t spin_limit) {
  __shared__ int passed;
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t want = epoch + li + 1;
    bool ok = true;
    __threadfence_system();  // this CTA's layer-li stores (peer rings / shards) before its arrival
    const unsigned long long n = atomicAdd(S.arrive, 1ull) + 1ull;
    if (n == static_cast<unsigned long long>(li + 1) * gridDim.x) {
      if (S.nslots) {
        st_release_sys(S.done_self, want);
        for (uint32_t s = 0; ok && s < S.nslots; ++s) ok = wait_geq(S.done_all[s], want, error_flag, spin_limit, true);
      }
      if (ok) st_release_gpu(S.release, want);
    } else {
      ok = wait_geq(S.release, want, error_flag, spin_limit, false);
    }
    passed = ok;
  }
  __syncthreads();
  return passed != 0;
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
constexpr uint32_t kLaneTmaBytes = 8192;

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

__device__ __forceinline__ void record_batch(rs_trace_record* trace, const rs_lane_desc& L, const rs_batch_desc& B,
                                             uint32_t b, uint32_t role, uint64_t t_begin) {
  uint64_t t_end;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
  rs_trace_record r;
  r.lane = L.batch0;
  r.batch = b;
  r.layer = B.layer;
  r.role = role;
  r.bytes = B.bytes;
  r.t_begin = t_begin;
  r.t_end = t_end;
  trace[2ull * (L.batch0 + b) + role] = r;
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
// 3 x 256-thread CTAs per SM: up to 85 registers, so the lane copy loops do
// not spill (the 64-register build spilled and ran STAGED 8-16 % slower,
// profiles/r1/lane_share_sweep.jsonl)
template <int kThreads, bool kWs>
__global__ void __launch_bounds__(kThreads, 768 / kThreads) rs_exchange_kernel(
    const rs_lane_desc* __restrict__ lanes_tx, uint32_t ntx, const rs_lane_desc* __restrict__ lanes_rx,
    uint32_t nrx, const rs_batch_desc* __restrict__ batches,
    const rs_copy_desc* __restrict__ frames, const rs_copy_desc* __restrict__ local_descs,
    const uint64_t* __restrict__ local_item0, uint32_t nlocal, uint64_t local_items, uint64_t epoch,
    unsigned int* error_flag, uint64_t spin_limit, int flags, rs_trace_record* __restrict__ trace,
    const rs_layer_sync sync) {
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
    if constexpr (kWs) {
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
    } else {
    uint32_t li = 0;  // strict: layer barriers passed so far
    for (uint32_t b = 0; b < L.nbatches; ++b) {
      const rs_batch_desc B = batches[L.batch0 + b];
      // strict: batches never span layers; meet the barriers of the layers before this batch's
      for (; li < sync.nlayers && li < B.layer_idx; ++li)
        if (!layer_barrier(sync, li, epoch, error_flag, spin_limit)) return;
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
      uint64_t t_begin = 0;
      if (trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
      if (sender) {
        // pack: the batch's frames copy their source boxes into the slot
        // (remote stores); one flat item space over the frames, dealt to warps
        for (uint32_t it = warp_in_block; it < B.pack_items; it += warps_per_block) {
          const rs_copy_desc& D = frames[B.pack0 + find_frame(frames + B.pack0, B.npack, it)];
          if (flags & kExHints) warp_copy_item_hint<true, 8>(D, it - D.item0, lane_id, pol_first, pol_last);
          else warp_copy_item<true, 8>(D, it - D.item0, lane_id);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          publish(reinterpret_cast<uint64_t*>(L.ready_flags) + slot, seq, peer);
          if (trace) record_batch(trace, L, B, b, 0, t_begin);
        }
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
        if (threadIdx.x == 0) {
          publish(reinterpret_cast<uint64_t*>(L.credit_flags) + slot, seq, peer);
          if (trace) record_batch(trace, L, B, b, 1, t_begin);
        }
      }
    }
    for (; li < sync.nlayers; ++li)
      if (!layer_barrier(sync, li, epoch, error_flag, spin_limit)) return;
    return;
    }  // classic lanes
  }

  // local copy role
  const uint64_t warp = (static_cast<uint64_t>(blockIdx.x - ntx - nrx) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x - ntx - nrx) * blockDim.x) >> 5;
  if (sync.nlayers) {  // strict: layer by layer, a barrier after each
    uint64_t begin = 0;
    for (uint32_t li = 0; li < sync.nlayers; ++li) {
      const uint64_t end = sync.local_layer_end[li];
      for (uint64_t item = begin + warp; item < end; item += nwarps) {
        const uint32_t di = find_desc(local_item0, nlocal, item);
        warp_copy_item<true, 8>(local_descs[di], item - local_descs[di].item0, lane_id);
      }
      begin = end;
      if (!layer_barrier(sync, li, epoch, error_flag, spin_limit)) return;
    }
    return;
  }
  for (uint64_t item = warp; item < local_items; item += nwarps) {
    const uint32_t di = find_desc(local_item0, nlocal, item);
    warp_copy_item<true, 8>(local_descs[di], item - local_descs[di].item0, lane_id);
  }
}

}  // namespace

extern "C" {

cudaError_t rs_launch_exchange(const rs_lane_desc* lanes_tx, uint32_t ntx, const rs_lane_desc* lanes_rx,
                               uint32_t nrx, const rs_batch_desc* batches, const rs_copy_desc* frames,
                               const rs_copy_desc* local_descs, const uint64_t* local_item0,
                               uint32_t nlocal, uint64_t local_items, uint64_t epoch,
                               unsigned int* error_flag, uint64_t spin_limit, int flags,
                               int local_blocks, int threads, rs_trace_record* trace,
                               const rs_layer_sync* sync_in, cudaStream_t stream) {
  rs_layer_sync sync{};
  if (sync_in) sync = *sync_in;
  int grid = static_cast<int>(ntx + nrx) + (local_items ? local_blocks : 0);
  // strict: a slot with no work of its own still meets every layer barrier
  if (grid == 0 && sync.nlayers) grid = 1;
  if (grid == 0) return cudaSuccess;
  if (sync.nlayers && (flags & kExWarpSpec)) return cudaErrorInvalidValue;  // classic lanes only
  const int smem = (flags & kExLaneTma) ? (threads / 32 - 1) * static_cast<int>(kLaneTmaBytes) : 0;
  const bool ws = (flags & kExWarpSpec) != 0;
  if (smem > 48 * 1024) {  // TMA lanes: 256-thread warp-specialised kernel only
    cudaError_t e = cudaFuncSetAttribute(rs_exchange_kernel<256, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
#define RS_EXCHANGE_LAUNCH(T, W)                                                                                 \
  rs_exchange_kernel<T, W><<<grid, T, smem, stream>>>(lanes_tx, ntx, lanes_rx, nrx, batches, frames, local_descs,  \
                                                      local_item0, nlocal, local_items, epoch, error_flag,         \
                                                      spin_limit, flags, trace, sync)
  if (threads == 1024) {
    if (ws) RS_EXCHANGE_LAUNCH(1024, true); else RS_EXCHANGE_LAUNCH(1024, false);
  } else if (threads == 512) {
    if (ws) RS_EXCHANGE_LAUNCH(512, true); else RS_EXCHANGE_LAUNCH(512, false);
  } else {
    if (ws) RS_EXCHANGE_LAUNCH(256, true); else RS_EXCHANGE_LAUNCH(256, false);
  }
#undef RS_EXCHANGE_LAUNCH
  return cudaGetLastError();
}

int exchange_max_blocks_per_sm(int which) {
  // 2 / 7 / 8: classic lanes, 256 / 512 / 1024 threads; 9: warp-specialised
  // 256-thread lanes with TMA copy warps (112 KB of shared memory); 10 / 11 /
  // 12: warp-specialised lanes, 256 / 512 / 1024 threads
  int n = 0;
  if (which == 9) {
    const int smem = 7 * static_cast<int>(kLaneTmaBytes);
    cudaFuncSetAttribute(rs_exchange_kernel<256, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rs_exchange_kernel<256, true>, 256, smem);
  } else if (which == 7) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rs_exchange_kernel<512, false>, 512, 0);
  else if (which == 8) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rs_exchange_kernel<1024, false>, 1024, 0);
  else if (which == 10) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rs_exchange_kernel<256, true>, 256, 0);
  else if (which == 11) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rs_exchange_kernel<512, true>, 512, 0);
  else if (which == 12) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rs_exchange_kernel<1024, true>, 1024, 0);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rs_exchange_kernel<256, false>, 256, 0);
  return n;
}

}  // extern "C"
