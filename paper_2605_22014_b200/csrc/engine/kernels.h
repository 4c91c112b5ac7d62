// Host-callable launchers of copy_kernels.cu, pattern_kernel.cu and
// exchange_kernel.cu (C linkage, no templates exposed).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "desc.h"

#ifdef __cplusplus
extern "C" {
#endif

// variant: 1 LDG x4 (default), 2 LDG x8, 3 TMA bulk ring (16 B aligned descriptors only)
cudaError_t rs_launch_copy(const rs_copy_desc* descs, const uint64_t* item0, uint32_t ndesc,
                           uint64_t item_begin, uint64_t item_end, int grid, int variant,
                           cudaStream_t stream);

cudaError_t rs_launch_pattern(const rs_pattern_desc* descs, const uint64_t* item0, uint32_t ndesc,
                              uint64_t nitems, uint64_t seed, int verify,
                              unsigned long long* mismatches, unsigned long long* first_bad,
                              int grid, cudaStream_t stream);

cudaError_t rs_launch_exchange(const rs_lane_desc* lanes_tx, uint32_t ntx,
                               const rs_lane_desc* lanes_rx, uint32_t nrx,
                               const rs_batch_desc* batches, const rs_copy_desc* frames,
                               const rs_copy_desc* local_descs, const uint64_t* local_item0,
                               uint32_t nlocal, uint64_t local_items, uint64_t epoch,
                               unsigned int* error_flag, uint64_t spin_limit, int flags,
                               int local_blocks, int threads, rs_trace_record* trace,
                               const rs_layer_sync* sync,  // NULL or nlayers == 0: fused layers
                               cudaStream_t stream);  // flags: 1 fault-inject, 2 L2 discard, 4 L2 policies

// TMA-pipelined ring lanes (one 1-warp CTA per lane end, `stages` x 16 KB of
// shared memory); the local copies run as a separate copy launch.
// sync (strict layers, nlayers > 0): `local_ctas` more CTAs copy the local
// descriptors layer by layer and every CTA meets a barrier after each layer
cudaError_t rs_launch_stream_exchange(const rs_lane_desc* lanes_tx, uint32_t ntx, const rs_lane_desc* lanes_rx,
                                      uint32_t nrx, const rs_batch_desc* batches, const rs_copy_desc* frames,
                                      uint64_t epoch, unsigned int* error_flag, uint64_t spin_limit, int flags,
                                      int stages, rs_trace_record* trace, unsigned long long* prof,
                                      const rs_copy_desc* local_descs, const uint64_t* local_item0, uint32_t nlocal,
                                      int local_ctas, const rs_layer_sync* sync, cudaStream_t stream);
int stream_max_blocks_per_sm(int stages);

// which: 0 LDG4, 3 LDG8, 5 LDG16, 6 CTA8, 4 bulk, 1 pattern, 2/7/8 exchange 256/512/1024 threads
int rs_kernel_max_blocks_per_sm(int which);
// per-file occupancy helpers behind rs_kernel_max_blocks_per_sm
int copy_max_blocks_per_sm(int which);
int pattern_max_blocks_per_sm(void);
int exchange_max_blocks_per_sm(int which);

#ifdef __cplusplus
}
#endif
