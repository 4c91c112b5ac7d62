// Ring-staged transfer kernel (STAGED mode): sender CTAs pack frames into the
// receiver's staging slots (peer stores over NVLink when the receiver is
// another GPU), publish with a release flag; receiver CTAs acquire, unpack,
// return a credit (bounded staging, proj/src/executor.cpp:183-206); spare
// CTAs run the local copies.  Integer / byte movement only.
#include <cuda_runtime.h>

#include <algorithm>
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

// Stream lanes: one release store, no separate fence.  The lane's writes
// are ordered before it by __syncwarp (the warp's other lanes) and, for bulk
// copies, by cp.async.bulk.wait_group + fence.proxy.async; st.release is
// cumulative over what the publishing lane has observed.  (__threadfence
// before it costs a second MEMBAR + L1 invalidate per batch: profiles/r2.)
__device__ __forceinline__ void publish_release(uint64_t* flag, uint64_t v, bool peer) {
  if (peer) st_release_sys(flag, v);
  else st_release_gpu(flag, v);
}

__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p, bool peer) {
  uint64_t v;
  if (peer) asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Poll a ring flag: relaxed loads while it is short of `want` (no L1
// invalidate per poll), one acquire load of the same flag once it is there
// (synchronises with the publisher's release).
__device__ __forceinline__ bool flag_reached(const uint64_t* p, uint64_t want, bool peer) {
  if (ld_relaxed(p, peer) < want) return false;
  return (peer ? ld_acquire_sys(p) : ld_acquire_gpu(p)) >= want;
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
//
// Layer-scoped roles (S.expect): barrier li has its own counter and completes
// at expect[li] arrivals; `wait` = false arrives without waiting (a role's
// last barrier -- it exits and frees its CTA slot).  The GPU's last arriver
// always completes the barrier (cross-slot flags, release) itself.
__device__ __noinline__ bool layer_barrier(const rs_layer_sync& S, uint32_t li, uint64_t epoch,
                                           unsigned int* error_flag, uint64_t spin_limit, bool wait = true) {
  __shared__ int passed;
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t want = epoch + li + 1;
    bool ok = true;
    __threadfence_system();  // this CTA's layer-li stores (peer rings / shards) before its arrival
    const unsigned long long n = atomicAdd(S.expect ? S.arrive + li : S.arrive, 1ull) + 1ull;
    const unsigned long long full =
        S.expect ? static_cast<unsigned long long>(S.expect[li]) : static_cast<unsigned long long>(li + 1) * gridDim.x;
    if (n == full) {
      if (S.nslots) {
        st_release_sys(S.done_self, want);
        for (uint32_t s = 0; ok && s < S.nslots; ++s) ok = wait_geq(S.done_all[s], want, error_flag, spin_limit, true);
      }
      if (ok) st_release_gpu(S.release, want);
    } else if (wait) {
      ok = wait_geq(S.release, want, error_flag, spin_limit, false);
    }
    passed = ok;
  }
  __syncthreads();
  return passed != 0;
}

// Wait (without arriving) until barrier li has completed: a layer-scoped
// role's entry into its first layer li + 1.  A role resident early may wait
// through many layers, so the spin budget restarts whenever a barrier
// completes (bounded per layer, like every other wait, not per handoff).
__device__ __noinline__ bool layer_wait(const rs_layer_sync& S, uint32_t li, uint64_t epoch,
                                        unsigned int* error_flag, uint64_t spin_limit) {
  __shared__ int passed;
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t want = epoch + li + 1;
    uint64_t seen = 0, spins = 0;
    int ok = 1;
    for (uint64_t v; (v = ld_acquire_gpu(S.release)) < want;) {
      if (v != seen) {
        seen = v;
        spins = 0;
      }
      if (*reinterpret_cast<volatile unsigned int*>(error_flag) || ++spins > spin_limit) {
        atomicExch(error_flag, 1u);
        ok = 0;
        break;
      }
      __nanosleep(64);
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

// ------------------------------------------------------------ stream lanes
//
// TMA-pipelined ring lanes (RS_RING_STREAM).  One 1-warp CTA per lane end.
// The classic lanes move a batch through registers, 32 KB in flight per CTA,
// and a 9.6 us pack of a 128 KiB slot is latency-bound (profiles/r1
// trace_capacity.jsonl: ~10 GB/s per lane).  Here the warp streams the
// lane's items through kStages x 16 KB shared-memory stages with bulk copies:
// loads run up to kStages items ahead of the stores and across batch
// boundaries (a sender prefetches the next batch's source rows before its
// credit arrives; a receiver returns the credit as soon as a batch's slot
// bytes have landed in shared memory, before its destination stores finish),
// so ~kStages x 16 KB are in flight per lane without registers.  Rows are
// dealt to the 32 lanes, each issuing its own bulk copies; the slot side of an
// item is contiguous and moves as one bulk copy.  Flags / credits / epochs are
// the classic lanes' protocol (bounded waits, .sys scope across GPUs).
constexpr uint32_t kStreamStageBytes = 16384;

// wait until at most n of this thread's bulk groups are still reading smem
__device__ __forceinline__ void bulk_wait_read_dyn(uint32_t n) {
  switch (n) {
    case 0: bulk_wait_read<0>(); break;
    case 1: bulk_wait_read<1>(); break;
    case 2: bulk_wait_read<2>(); break;
    case 3: bulk_wait_read<3>(); break;
    case 4: bulk_wait_read<4>(); break;
    case 5: bulk_wait_read<5>(); break;
    case 6: bulk_wait_read<6>(); break;
    case 7: bulk_wait_read<7>(); break;
    case 8: bulk_wait_read<8>(); break;
    case 9: bulk_wait_read<9>(); break;
    case 10: bulk_wait_read<10>(); break;
    case 11: bulk_wait_read<11>(); break;
    case 12: bulk_wait_read<12>(); break;
    case 13: bulk_wait_read<13>(); break;
    default: bulk_wait_read<14>(); break;
  }
}

// Is the descriptor's source (src_side) / destination run sequence one
// contiguous span?  (A packed ring-slot frame is.)
__device__ __forceinline__ bool side_contiguous(const rs_copy_desc& D, bool src_side) {
  uint64_t span = D.row_bytes;
  bool contiguous = true;
#pragma unroll
  for (uint32_t k = 0; k < RS_MAX_OUTER; ++k) {
    if (k < D.nouter) {
      const int64_t st = src_side ? D.sstr[k] : D.dstr[k];
      contiguous = contiguous && st == static_cast<int64_t>(span);
      span *= D.ext[k];
    }
  }
  return contiguous;
}

// A lane end's descriptors, staged into shared memory by bulk copies.  The
// frames of one role are contiguous in batch order (compile_staged), and so
// are the lane's batch descriptors: both are read through small rings of
// chunks (kNB buffers, one mbarrier each) that the load cursor fills one chunk
// ahead.  The descriptor tables are far larger than L2; demand-fetching them
// with generic loads stalled the warp at every frame / batch boundary and
// kept loads outstanding under every release fence (profiles/r2).
template <int kStages>
struct DescRing {
  static constexpr uint32_t kNB = 3;                             // buffers per table
  static constexpr uint32_t kCF = kStages > 6 ? kStages : 6;     // frames per chunk (>= the cursors' lag)
  static constexpr uint32_t kCB = kStages > 8 ? kStages : 8;     // batch descriptors per chunk
  rs_copy_desc* fbuf;   // kNB x kCF
  rs_batch_desc* bbuf;  // kNB x kCB
  uint64_t* fbar;       // kNB
  uint64_t* bbar;       // kNB
  const rs_copy_desc* frames;
  const rs_batch_desc* batches;
  uint32_t f0, nf;  // this role's frames in the global table
  uint32_t b0, nb;  // the lane's batches
  bool whole_cta;   // the calling warp is the whole CTA (one-warp lanes): order with bar.sync

  // every lane's earlier generic reads of a buffer before the bulk write that
  // refills it: a barrier over the readers (the CTA is the lane's one warp),
  // then a generic -> async proxy fence
  __device__ __forceinline__ void before_refill() const {
    if (whole_cta) __syncthreads();
    else __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }

  // (warp-uniform calls)
  __device__ __forceinline__ void load_frames(uint32_t j, int lane) const {
    if (j * kCF >= nf) return;
    before_refill();
    if (lane != 0) return;
    const uint32_t n = min(kCF, nf - j * kCF);
    const uint32_t buf = j % kNB;
    mbar_expect_tx(&fbar[buf], n * static_cast<uint32_t>(sizeof(rs_copy_desc)));
    bulk_load(fbuf + buf * kCF, frames + f0 + j * kCF, n * static_cast<uint32_t>(sizeof(rs_copy_desc)), &fbar[buf]);
  }
  __device__ __forceinline__ void load_batches(uint32_t j, int lane) const {
    if (j * kCB >= nb) return;
    before_refill();
    if (lane != 0) return;
    const uint32_t n = min(kCB, nb - j * kCB);
    const uint32_t buf = j % kNB;
    mbar_expect_tx(&bbar[buf], n * static_cast<uint32_t>(sizeof(rs_batch_desc)));
    bulk_load(bbuf + buf * kCB, batches + b0 + j * kCB, n * static_cast<uint32_t>(sizeof(rs_batch_desc)), &bbar[buf]);
  }
  __device__ __forceinline__ void wait_frames(uint32_t j) const { mbar_wait(&fbar[j % kNB], (j / kNB) & 1); }
  __device__ __forceinline__ void wait_batches(uint32_t j) const { mbar_wait(&bbar[j % kNB], (j / kNB) & 1); }
  __device__ __forceinline__ const rs_copy_desc& frame(uint32_t i) const {  // i: role-relative frame
    return fbuf[((i / kCF) % kNB) * kCF + i % kCF];
  }
  __device__ __forceinline__ const rs_batch_desc& batch(uint32_t b) const {  // b: lane-relative batch
    return bbuf[((b / kCB) % kNB) * kCB + b % kCB];
  }
};

// Walks a lane end's work items in order: batch b, frame i (role-relative),
// item k of nk.  The leading (load) cursor waits for descriptor chunks and
// issues the next ones; the store cursor trails it by <= kStages items and
// reads chunks the leader has already waited for.
struct ItemCursor {
  uint32_t b = 0;     // batch of the item at the cursor (lane-relative)
  uint32_t i = 0;     // frame of the item at the cursor (role-relative)
  uint32_t left = 0;  // frames of batch b after i
  uint64_t k = 0, nk = 0;
  uint64_t extent = 0;  // slot bytes in use by batch b
  bool first_of_batch = true;  // the item at the cursor opens batch b
  bool src_contig = false, dst_contig = false;
  rs_copy_desc D;
};

__device__ __forceinline__ uint32_t role_frames(const rs_batch_desc& B, bool sender) {
  return sender ? B.npack : B.nunpack;
}

template <int kStages>
__device__ __forceinline__ void cursor_install(ItemCursor& c, const DescRing<kStages>& R) {
  c.D = R.frame(c.i);
  c.nk = (c.D.rows + c.D.rows_per_item - 1) / c.D.rows_per_item;
  c.src_contig = side_contiguous(c.D, true);
  c.dst_contig = side_contiguous(c.D, false);
}

// position the cursor on the lane's first item (the leader also primes the rings)
template <int kStages>
__device__ __forceinline__ void cursor_start(ItemCursor& c, const DescRing<kStages>& R, bool sender, bool leader,
                                             int lane) {
  c.b = 0;
  c.i = 0;
  c.k = 0;
  c.first_of_batch = true;
  if (R.nb == 0) return;
  if (leader) {
    R.load_batches(0, lane);
    R.load_batches(1, lane);
    R.load_frames(0, lane);
    R.load_frames(1, lane);
  }
  R.wait_batches(0);  // (a trailing warp observes the chunk's completion itself)
  R.wait_frames(0);
  const rs_batch_desc& B0 = R.batch(0);
  c.left = role_frames(B0, sender) - 1;  // (an empty batch is never emitted by compile_staged)
  c.extent = B0.extent;
  cursor_install(c, R);
}

// advance one item; returns true when the item just passed was its batch's last
template <int kStages>
__device__ __forceinline__ bool cursor_next(ItemCursor& c, const DescRing<kStages>& R, bool sender, bool leader,
                                            int lane) {
  using DR = DescRing<kStages>;
  c.first_of_batch = false;
  if (++c.k < c.nk) return false;
  c.k = 0;
  const bool batch_end = c.left == 0;
  if (batch_end) {
    if (++c.b >= R.nb) return true;
    if (c.b % DR::kCB == 0) {  // entering batch chunk j: wait for it (the leader then fetches j + 1)
      R.wait_batches(c.b / DR::kCB);
      if (leader) R.load_batches(c.b / DR::kCB + 1, lane);
    }
    const rs_batch_desc& B = R.batch(c.b);
    c.left = role_frames(B, sender) - 1;
    c.extent = B.extent;
    c.first_of_batch = true;
  } else {
    --c.left;
  }
  ++c.i;
  if (c.i % DR::kCF == 0) {
    R.wait_frames(c.i / DR::kCF);
    if (leader) R.load_frames(c.i / DR::kCF + 1, lane);
  }
  cursor_install(c, R);
  return batch_end;
}

// Issue the loads of item (D, k) into `stage` (lanes split the rows; the
// slot side, when contiguous, is one copy by lane 0).  Lane 0 has armed the
// stage's mbarrier with the item's bytes.
__device__ __forceinline__ void stream_item_load(const rs_copy_desc& D, bool contiguous, uint64_t k,
                                                 unsigned char* stage, uint64_t* bar, uint64_t pol, int lane) {
  const uint64_t r0 = k * D.rows_per_item;
  const uint64_t r1 = min(r0 + D.rows_per_item, D.rows);
  if (contiguous) {
    if (lane == 0) {
      int64_t so, dof;
      row_offsets(D, static_cast<uint32_t>(r0), so, dof);
      bulk_load_hint(stage, reinterpret_cast<const void*>(D.src + so), static_cast<uint32_t>((r1 - r0) * D.row_bytes),
                     bar, pol);
    }
    return;
  }
  for (uint64_t r = r0 + lane; r < r1; r += 32) {
    int64_t so, dof;
    row_offsets(D, static_cast<uint32_t>(r), so, dof);
    bulk_load_hint(stage + (r - r0) * D.row_bytes, reinterpret_cast<const void*>(D.src + so),
                   static_cast<uint32_t>(D.row_bytes), bar, pol);
  }
}

// fwd: relay forwarder (a receiver whose batches continue to the next hop's
// ring): the item's slot-side bytes -- already in `stage` -- are also stored
// at the same offsets of the next ring (slot address + fwd_delta), in the same
// bulk group, so stage reuse and the batch's publish cover both stores.
__device__ __forceinline__ void stream_item_store(const rs_copy_desc& D, bool contiguous, uint64_t k,
                                                  const unsigned char* stage, uint64_t pol, int lane,
                                                  bool fwd = false, bool src_contig = false, int64_t fwd_delta = 0,
                                                  uint64_t fwd_pol = 0) {
  const uint64_t r0 = k * D.rows_per_item;
  const uint64_t r1 = min(r0 + D.rows_per_item, D.rows);
  if (fwd) {
    if (src_contig) {
      if (lane == 0) {
        int64_t so, dof;
        row_offsets(D, static_cast<uint32_t>(r0), so, dof);
        bulk_store_hint(reinterpret_cast<void*>(D.src + so + fwd_delta), stage,
                        static_cast<uint32_t>((r1 - r0) * D.row_bytes), fwd_pol);
      }
    } else {
      for (uint64_t r = r0 + lane; r < r1; r += 32) {
        int64_t so, dof;
        row_offsets(D, static_cast<uint32_t>(r), so, dof);
        bulk_store_hint(reinterpret_cast<void*>(D.src + so + fwd_delta), stage + (r - r0) * D.row_bytes,
                        static_cast<uint32_t>(D.row_bytes), fwd_pol);
      }
    }
  }
  if (contiguous) {
    if (lane == 0) {
      int64_t so, dof;
      row_offsets(D, static_cast<uint32_t>(r0), so, dof);
      bulk_store_hint(reinterpret_cast<void*>(D.dst + dof), stage, static_cast<uint32_t>((r1 - r0) * D.row_bytes), pol);
    }
  } else {
    for (uint64_t r = r0 + lane; r < r1; r += 32) {
      int64_t so, dof;
      row_offsets(D, static_cast<uint32_t>(r), so, dof);
      bulk_store_hint(reinterpret_cast<void*>(D.dst + dof), stage + (r - r0) * D.row_bytes,
                      static_cast<uint32_t>(D.row_bytes), pol);
    }
  }
  bulk_commit();  // one group per item on every lane (possibly empty): stage reuse counts groups
}

// Same as stream_item_store, through registers: the warp reads the stage
// (ld.shared) and writes the rows with 16 B stores, so the stage is free as
// soon as the loop ends (no bulk-store read-out to wait for).
__device__ __forceinline__ void stream_item_store_regs(const rs_copy_desc& D, uint64_t k, const unsigned char* stage,
                                                       uint64_t pol, int lane) {
  const uint64_t r0 = k * D.rows_per_item;
  const uint64_t r1 = min(r0 + D.rows_per_item, D.rows);
  const uint64_t rb = D.row_bytes;
  for (uint64_t r = r0; r < r1; ++r) {
    int64_t so, dof;
    row_offsets(D, static_cast<uint32_t>(r), so, dof);
    const uint4* src = reinterpret_cast<const uint4*>(stage + (r - r0) * rb);
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<char*>(D.dst) + dof);
    const uint32_t n = static_cast<uint32_t>(rb >> 4);
    uint32_t i = static_cast<uint32_t>(lane);
    for (; i + 96 < n; i += 128) {
      const uint4 a = src[i], b = src[i + 32], c = src[i + 64], d = src[i + 96];
      store_hint(dst + i, a, pol);
      store_hint(dst + i + 32, b, pol);
      store_hint(dst + i + 64, c, pol);
      store_hint(dst + i + 96, d, pol);
    }
    for (; i < n; i += 32) store_hint(dst + i, src[i], pol);
  }
  // the stage's next bulk load (async proxy) is ordered after these reads
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

constexpr int kExStreamRegStore = 64;  // stream lanes: stores from the stage through registers

template <int kStages>
__global__ void __launch_bounds__(32) rs_stream_lane_kernel(
    const rs_lane_desc* __restrict__ lanes_tx, uint32_t ntx, const rs_lane_desc* __restrict__ lanes_rx,
    uint32_t nrx, const rs_batch_desc* __restrict__ batches, const rs_copy_desc* __restrict__ frames,
    uint64_t epoch, unsigned int* error_flag, uint64_t spin_limit, int flags, rs_trace_record* __restrict__ trace,
    unsigned long long* __restrict__ prof, const rs_copy_desc* __restrict__ local_descs,
    const uint64_t* __restrict__ local_item0, uint32_t nlocal, rs_layer_sync sync) {
  extern __shared__ __align__(128) unsigned char stages[];
  __shared__ __align__(8) uint64_t bar[kStages];
  using DR = DescRing<kStages>;
  __shared__ __align__(128) rs_copy_desc desc_frames[DR::kNB * DR::kCF];
  __shared__ __align__(128) rs_batch_desc desc_batches[DR::kNB * DR::kCB];
  __shared__ __align__(8) uint64_t desc_bar[2 * DR::kNB];
  const int lane = threadIdx.x;
  uint32_t vb = blockIdx.x;  // the CTA's role: sender lane, receiver lane or local-copy CTA
  if (sync.roles) {          // strict, layer-scoped roles: dealt by ticket in first-layer order
    __shared__ uint32_t role;
    if (lane == 0) role = sync.roles[atomicAdd(sync.tickets, 1ull)];
    __syncwarp();
    vb = role;
  }
  const bool sender = vb < ntx;
  if (vb >= ntx + nrx) {
    // Strict layers (sync.nlayers > 0): the launch's local-copy roles copy
    // the local tasks + carryovers layer by layer through the shared-memory
    // stages and meet the barriers of their layers with the lanes.
    if (!sync.nlayers) return;
    if (lane == 0) {
      for (int i = 0; i < kStages; ++i) mbar_init(&bar[i], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const uint64_t pol = policy_evict_first();
    uint64_t wid = vb - ntx - nrx;
    // layer-scoped local roles (sync.local_n): layer li's items are shared by
    // local_n[li] CTAs; this role is share `wid` in every layer of its run
    // [l0, l1] and meets only those barriers
    uint32_t l0 = 0, l1 = sync.nlayers - 1;
    if (sync.local_n) {
      const uint32_t q = static_cast<uint32_t>(wid);
      wid = sync.local_roles[2 * q];
      l0 = sync.local_roles[2 * q + 1] & 0xffffu;
      l1 = sync.local_roles[2 * q + 1] >> 16;
      if (l0 && !layer_wait(sync, l0 - 1, epoch, error_flag, spin_limit)) return;
    }
    uint64_t n = 0, begin = l0 ? sync.local_layer_end[l0 - 1] : 0;
    for (uint32_t li = l0; li <= l1; ++li) {
      const uint64_t end = sync.local_layer_end[li];
      const uint64_t nw = sync.local_n ? sync.local_n[li] : gridDim.x - ntx - nrx;
      for (uint64_t item = begin + wid; item < end && wid < nw; item += nw, ++n) {
        const uint32_t s = static_cast<uint32_t>(n % kStages);
        if (n >= static_cast<uint64_t>(kStages)) bulk_wait_read_dyn(kStages - 1);  // item n - kStages left stage s
        __syncwarp();
        const rs_copy_desc D = local_descs[find_desc(local_item0, nlocal, item)];
        const uint64_t k = item - D.item0;
        const uint64_t r0 = k * D.rows_per_item;
        const uint32_t bytes = static_cast<uint32_t>((min(r0 + D.rows_per_item, D.rows) - r0) * D.row_bytes);
        unsigned char* stage = stages + static_cast<size_t>(s) * kStreamStageBytes;
        if (lane == 0) mbar_expect_tx(&bar[s], bytes);
        __syncwarp();
        stream_item_load(D, side_contiguous(D, true), k, stage, &bar[s], pol, lane);
        mbar_wait(&bar[s], static_cast<uint32_t>((n / kStages) & 1));
        stream_item_store(D, side_contiguous(D, false), k, stage, pol, lane);
      }
      begin = end;
      bulk_wait_all();  // this layer's stores are written before the barrier's release
      fence_proxy_async_global();
      __syncwarp();
      if (!layer_barrier(sync, li, epoch, error_flag, spin_limit, !(sync.local_n && li == l1))) return;
    }
    return;
  }
  if ((flags & kExFaultRx) && !sender) return;  // test hook: the receiving peer is gone
  const rs_lane_desc L = sender ? lanes_tx[vb] : lanes_rx[vb - ntx];
  const bool peer = (L.flags & RS_LANE_PEER) != 0;
  const bool fwd = !sender && L.fwd_slot_base != 0;  // relay forwarder
  const bool fpeer = (L.fwd_flags & RS_LANE_PEER) != 0;
  const int64_t fwd_delta = static_cast<int64_t>(L.fwd_slot_base - L.slot_base_rx);
  const bool scoped = sync.nlayers && sync.expect;  // meets only its own layers' barriers
  if (scoped && !L.nbatches) return;                // never counted in expect
  if (lane == 0) {
    for (int i = 0; i < 2 * static_cast<int>(DR::kNB); ++i) mbar_init(&desc_bar[i], 1);
    for (int i = 0; i < kStages; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();
  // sender: shard rows in evict-first, slot out evict-last; receiver: slot in
  // evict-first (it is discarded next), shard out evict-first
  const uint64_t ld_pol = pol_first, st_pol = sender ? pol_last : pol_first;

  const DR ring{desc_frames, desc_batches, desc_bar, desc_bar + DR::kNB, frames, batches,
                sender ? L.tx_frame0 : L.rx_frame0, sender ? L.tx_nframes : L.rx_nframes, L.batch0, L.nbatches,
                true};
  ItemCursor ld, st;
  cursor_start(ld, ring, sender, true, lane);
  cursor_start(st, ring, sender, false, lane);
  // strict layers: barriers passed so far; a lane end meets barrier l as soon
  // as its own layer-<=l batches are done (before that, at its first batch,
  // the barriers of the layers it has no part in)
  // (layer-scoped: a lane end enters at its first batch's layer once the
  // barrier before it completed, arrives at every barrier up to its last
  // batch's layer, and arrives at that last one without waiting)
  uint32_t barriers = 0;
  auto pass_to = [&](uint32_t target, bool final_arrive) -> bool {
    for (; barriers < target; ++barriers)
      if (!layer_barrier(sync, barriers, epoch, error_flag, spin_limit, !(final_arrive && barriers + 1 == target)))
        return false;
    return true;
  };
  if (scoped) {
    barriers = ring.batch(0).layer_idx;
    if (barriers && !layer_wait(sync, barriers - 1, epoch, error_flag, spin_limit)) return;
  } else if (sync.nlayers && !pass_to(L.nbatches ? ring.batch(0).layer_idx : sync.nlayers, false)) {
    return;
  }
  uint64_t g_ld = 0, g_st = 0;       // items loaded (issued) / stored (issued)
  uint32_t ready_b = 0xffffffffu;    // receiver: batch whose ready flag was acquired last
  uint32_t credit_b = 0xffffffffu;   // sender: batch whose slot credit was acquired last
  uint64_t idle = 0;
  // register stores: 64 both roles, 128 receivers only, 256 senders only
  const bool reg_store =
      !fwd && ((flags & kExStreamRegStore) || ((flags & 128) && !sender) || ((flags & 256) && sender));
  uint64_t prof_reuse = 0, prof_store = 0, prof_pub = 0, prof_idle = 0, prof_items = 0;
  const uint64_t prof_t0 = clock64();
  __shared__ uint64_t t_open[kStages];  // trace: flag-acquire time of each open batch (<= kStages open)
  __shared__ uint64_t t_issue[kStages];  // diagnostic: load issue time per stage
  uint64_t prof_land = 0, prof_loadloop = 0;

  // sender: slot credit of its ring; forwarder (store side): slot credit of
  // the next hop's ring; receiver (load side): ready flag of its ring
  auto flag_up = [&](uint32_t b, bool credit) -> bool {  // lane 0 polls, the warp agrees
    int up = 0;
    if (lane == 0) {
      if (credit) {
        const uint64_t* f = reinterpret_cast<const uint64_t*>(sender ? L.credit_flags_tx : L.fwd_credit_flags) +
                            b % L.slots;
        up = b < L.slots || flag_reached(f, epoch + b - L.slots + 1, sender ? peer : fpeer);
      } else {
        up = flag_reached(reinterpret_cast<const uint64_t*>(L.ready_flags_rx) + b % L.slots, epoch + b + 1, peer);
      }
    }
    return __shfl_sync(0xffffffffu, up, 0) != 0;
  };

  while (st.b < L.nbatches) {
    bool progress = false;
    // ---- loads: up to kStages items ahead of the stores
    const uint64_t tl0 = prof ? clock64() : 0;
    while (ld.b < L.nbatches && g_ld - g_st < static_cast<uint64_t>(kStages)) {
      if (!sender && ld.first_of_batch && ready_b != ld.b) {
        if (!flag_up(ld.b, false)) break;
        ready_b = ld.b;
        if (trace && lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_open[ld.b % kStages]));
        fence_proxy_async_global();  // the slot bytes were published through the generic proxy
      }
      const uint32_t s = static_cast<uint32_t>(g_ld % kStages);
      if (g_ld >= static_cast<uint64_t>(kStages) && !reg_store) {  // the stage's previous item must have been read out
        const uint64_t t0 = prof ? clock64() : 0;
        bulk_wait_read_dyn(static_cast<uint32_t>(g_st - 1 - (g_ld - kStages)));
        if (prof && lane == 0) prof_reuse += clock64() - t0;
      }
      const uint64_t r0 = ld.k * ld.D.rows_per_item;
      const uint32_t bytes = static_cast<uint32_t>((min(r0 + ld.D.rows_per_item, ld.D.rows) - r0) * ld.D.row_bytes);
      if (lane == 0) mbar_expect_tx(&bar[s], bytes);
      if (prof && lane == 0) t_issue[s] = clock64();
      __syncwarp();
      stream_item_load(ld.D, ld.src_contig, ld.k, stages + static_cast<size_t>(s) * kStreamStageBytes, &bar[s], ld_pol,
                       lane);
      cursor_next(ld, ring, sender, true, lane);
      ++g_ld;
      progress = true;
    }
    if (prof && lane == 0) prof_loadloop += clock64() - tl0;
    // ---- stores of landed items, in order
    while (g_st < g_ld) {
      const uint32_t s = static_cast<uint32_t>(g_st % kStages);
      const uint32_t parity = static_cast<uint32_t>((g_st / kStages) & 1);
      // lane 0 tests, the warp agrees; every lane then observes the completed
      // phase itself (acquire of the bulk-loaded bytes it is about to store)
      const int landed = lane == 0 ? mbar_test(&bar[s], parity) : 0;
      if (!__shfl_sync(0xffffffffu, landed, 0)) break;
      mbar_wait(&bar[s], parity);
      if (prof && lane == 0) prof_land += clock64() - t_issue[s];
      if ((sender || fwd) && st.first_of_batch && credit_b != st.b) {
        if (!flag_up(st.b, true)) break;  // the (next) receiver has not drained this slot yet
        credit_b = st.b;
        if (sender && trace && lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_open[st.b % kStages]));
      }
      const uint32_t b = st.b;
      const uint64_t extent = st.extent;
      const uint64_t ts0 = prof ? clock64() : 0;
      if (reg_store)
        stream_item_store_regs(st.D, st.k, stages + static_cast<size_t>(s) * kStreamStageBytes, st_pol, lane);
      else
        stream_item_store(st.D, st.dst_contig, st.k, stages + static_cast<size_t>(s) * kStreamStageBytes, st_pol, lane,
                          fwd, st.src_contig, fwd_delta, pol_last);
      if (prof && lane == 0) prof_store += clock64() - ts0;
      const bool last = cursor_next(st, ring, sender, false, lane);
      ++g_st;
      progress = true;
      if (!last) continue;
      const uint32_t slot = b % L.slots;
      if (sender) {
        // the batch's slot writes complete, then one release publishes them
        const uint64_t tw0 = prof ? clock64() : 0;
        if (!reg_store) {
          bulk_wait_all();
          fence_proxy_async_global();
        }
        __syncwarp();
        if (prof && lane == 0) prof_pub += clock64() - tw0;
        if (lane == 0) publish_release(reinterpret_cast<uint64_t*>(L.ready_flags) + slot, epoch + b + 1, peer);
      } else {
        if (fwd) {  // relay: the batch's bytes are in the next hop's slot -> publish it there
          bulk_wait_all();
          fence_proxy_async_global();
          __syncwarp();
          if (lane == 0) publish_release(reinterpret_cast<uint64_t*>(L.fwd_ready_flags) + slot, epoch + b + 1, fpeer);
        }
        // every slot byte of batch b is in shared memory: drop the slot's
        // lines from L2 and hand the slot back (the shard stores still run)
        if ((flags & kExDiscard) && extent && ((L.slot_base_rx | L.slot_bytes) & 127) == 0) {
          const uint64_t base = L.slot_base_rx + static_cast<uint64_t>(slot) * L.slot_bytes;
          const uint64_t lines = (extent + 127) >> 7;
          for (uint64_t i = lane; i < lines; i += 32) discard_l2_line(base + (i << 7));
        }
        __syncwarp();
        if (lane == 0) publish_release(reinterpret_cast<uint64_t*>(L.credit_flags) + slot, epoch + b + 1, peer);
      }
      if (trace && lane == 0) record_batch(trace, L, batches[L.batch0 + b], b, sender ? 0 : 1, t_open[b % kStages]);
      if (sync.nlayers) {
        // strict: this lane end's batches of the layers before the next
        // batch's are done (a receiver's shard stores written) -> barriers
        if (!sender) {
          bulk_wait_all();
          fence_proxy_async_global();
        }
        __syncwarp();
        const bool done = st.b >= L.nbatches;
        if (!pass_to(!done ? ring.batch(st.b).layer_idx : (scoped ? barriers + 1 : sync.nlayers), done && scoped)) {
          bulk_wait_all();
          return;
        }
      }
    }
    if (progress) {
      idle = 0;
      continue;
    }
    int stop = 0;
    const uint64_t ti0 = prof ? clock64() : 0;
    if (lane == 0) {
      if (*reinterpret_cast<volatile unsigned int*>(error_flag)) stop = 1;
      else if (++idle > spin_limit) {
        atomicExch(error_flag, 1u);
        stop = 1;
      } else {
        __nanosleep(32);
      }
    }
    if (prof && lane == 0) prof_idle += clock64() - ti0;
    if (__shfl_sync(0xffffffffu, stop, 0)) break;
  }
  bulk_wait_all();  // shared memory stays valid until every store has read it
  if (prof && lane == 0) {  // diagnostic: cycles per phase, per lane end
    unsigned long long* p = prof + 8ull * vb;
    p[0] = clock64() - prof_t0;
    p[1] = prof_reuse;
    p[2] = prof_store;
    p[3] = prof_pub;
    p[4] = prof_idle;
    p[5] = g_st;
    p[6] = sender;
    p[7] = prof_land;
    p[1] = prof_reuse | (prof_loadloop << 32);  // (packed: reuse wait low, load loop high; both < 2^32 per slice run)
    (void)prof_items;
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

cudaError_t rs_launch_stream_exchange(const rs_lane_desc* lanes_tx, uint32_t ntx, const rs_lane_desc* lanes_rx,
                                      uint32_t nrx, const rs_batch_desc* batches, const rs_copy_desc* frames,
                                      uint64_t epoch, unsigned int* error_flag, uint64_t spin_limit, int flags,
                                      int stages, rs_trace_record* trace, unsigned long long* prof,
                                      const rs_copy_desc* local_descs, const uint64_t* local_item0, uint32_t nlocal,
                                      int local_ctas, const rs_layer_sync* sync_in, cudaStream_t stream) {
  rs_layer_sync sync{};
  if (sync_in) sync = *sync_in;
  const int grid = static_cast<int>(ntx + nrx) + (sync.nlayers ? std::max(local_ctas, 1) : 0);
  if (grid == 0) return cudaSuccess;
  const int smem = stages * static_cast<int>(kStreamStageBytes);
#define RS_STREAM_LAUNCH(S)                                                                                    \
  do {                                                                                                         \
    cudaError_t e = cudaFuncSetAttribute(rs_stream_lane_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                         smem);                                                                \
    if (e != cudaSuccess) return e;                                                                            \
    rs_stream_lane_kernel<S><<<grid, 32, smem, stream>>>(lanes_tx, ntx, lanes_rx, nrx, batches, frames, epoch, \
                                                         error_flag, spin_limit, flags, trace, prof,           \
                                                         local_descs, local_item0, nlocal, sync);              \
  } while (0)
  switch (stages) {
    case 1: RS_STREAM_LAUNCH(1); break;
    case 2: RS_STREAM_LAUNCH(2); break;
    case 3: RS_STREAM_LAUNCH(3); break;
    case 4: RS_STREAM_LAUNCH(4); break;
    case 8: RS_STREAM_LAUNCH(8); break;
    case 10: RS_STREAM_LAUNCH(10); break;
    case 13: RS_STREAM_LAUNCH(13); break;
    default: RS_STREAM_LAUNCH(6); break;
  }
#undef RS_STREAM_LAUNCH
  return cudaGetLastError();
}

int stream_max_blocks_per_sm(int stages) {
  int n = 0;
  const int smem = stages * static_cast<int>(kStreamStageBytes);
#define RS_STREAM_OCC(S)                                                                                         \
  cudaFuncSetAttribute(rs_stream_lane_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);             \
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, rs_stream_lane_kernel<S>, 32, smem)
  switch (stages) {
    case 1: RS_STREAM_OCC(1); break;
    case 2: RS_STREAM_OCC(2); break;
    case 3: RS_STREAM_OCC(3); break;
    case 4: RS_STREAM_OCC(4); break;
    case 8: RS_STREAM_OCC(8); break;
    case 10: RS_STREAM_OCC(10); break;
    case 13: RS_STREAM_OCC(13); break;
    default: RS_STREAM_OCC(6); break;
  }
#undef RS_STREAM_OCC
  return n;
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
