// Device work descriptors shared by the host descriptor compiler
// (compile.cpp) and the sm_100a kernels (copy_kernels.cu, exchange_kernel.cu,
// pattern_kernel.cu).  Plain C layout.
//
// A CopyDesc is one strided->strided byte copy of a sub-box between two
// row-major shard buffers, after dimension coalescing: `rows` contiguous runs
// of `row_bytes`, the run start of row r given by decomposing r over up to
// RS_MAX_OUTER outer extents (innermost first) with independent source and
// destination byte strides.  This one shape covers the reference's
// slice_local (strided -> packed), scatter_local (packed -> strided), the local
// task / carryover copy (strided -> strided) and ring pack/unpack
// (proj/src/executor.cpp:23-93).
#pragma once
#include <stdint.h>

#define RS_MAX_OUTER 4

typedef struct {
  uint64_t src;           // byte address of row 0 (local or peer-mapped)
  uint64_t dst;
  uint64_t row_bytes;     // contiguous run length
  uint64_t rows;          // product of ext[0..nouter)
  uint64_t item0;         // global index of this descriptor's first work item
  uint64_t ext[RS_MAX_OUTER];
  int64_t sstr[RS_MAX_OUTER];
  int64_t dstr[RS_MAX_OUTER];
  uint32_t rows_per_item;
  uint32_t nouter;
  uint32_t vec_log2;      // access width: 1 << vec_log2 bytes (0..4)
  uint32_t tag;           // layer (diagnostics)
  // DP broadcast (DIRECT copy kernels): every row is also stored at
  // dst + dst2_delta -- a second destination with the same layout, written
  // from the same load (0: none).  Keeps the descriptor 160 B: tables stay
  // bulk-copyable in 16 B granules.
  int64_t dst2_delta;
} rs_copy_desc;

// Synthetic-state descriptor: one shard buffer (row-major over its view),
// filled with / checked against the reference pattern
// byte b of global element g of tensor ti =
//   byte (b % 8) of splitmix64(seed ^ 0x1000003*ti ^ g)   (shard_store.cpp:51-56)
typedef struct {
  uint64_t ptr;           // buffer base
  uint64_t row_elems;     // elements per (coalesced) row
  uint64_t rows;
  uint64_t item0;
  int64_t g0;             // global element index of the view origin
  uint64_t ext[RS_MAX_OUTER];   // outer extents, innermost first
  int64_t gstr[RS_MAX_OUTER];   // global element strides of the outer dims
  uint32_t rows_per_item;
  uint32_t nouter;
  uint32_t elem_bytes;
  uint32_t tensor_index;
  uint32_t entry;         // store entry id (mismatch reporting)
  uint32_t pad;
} rs_pattern_desc;

// Ring-staged transfer (STAGED mode): a batch is the set of frames packed
// into one ring slot; frames are CopyDescs whose destination (pack) or source
// (unpack) is the slot.  One lane = one single-producer / single-consumer ring
// between a sender CTA and a receiver CTA.
typedef struct {
  uint64_t slot_base;       // lane's slot 0 address (receiver memory, as mapped for the sender)
  uint64_t slot_base_rx;    // same slots as addressed by the receiver
  uint64_t slot_bytes;
  uint64_t ready_flags;     // uint64[slots] in receiver memory (sender addressing)
  uint64_t ready_flags_rx;  // receiver addressing
  uint64_t credit_flags;    // uint64[slots] in sender memory (receiver addressing)
  uint64_t credit_flags_tx; // sender addressing
  uint32_t slots;
  uint32_t nbatches;
  uint32_t batch0;          // index of the lane's first batch in the batch table
  uint32_t flags;           // RS_LANE_PEER: sender and receiver are not one device of one process
  // Relay (receiver lanes of a relay chain's hop k < n-1, stream lanes only):
  // every drained batch is also stored into the next hop's ring at the same
  // slot offsets, published there, and credited back by the next receiver.
  uint64_t fwd_slot_base;     // next hop's slot 0 as mapped here (0: this lane does not forward)
  uint64_t fwd_ready_flags;   // next hop's ready flags (next receiver's memory, as mapped here)
  uint64_t fwd_credit_flags;  // next hop's credit flags (this slot's memory)
  uint32_t fwd_flags;         // RS_LANE_PEER: the next hop crosses slots
  // The lane's frames per role, contiguous in batch order (stream lanes
  // stage them into shared memory with bulk copies)
  uint32_t tx_frame0, tx_nframes;  // pack frames
  uint32_t rx_frame0, rx_nframes;  // unpack frames
  uint32_t fwd_pad;
} rs_lane_desc;

#define RS_LANE_PEER 1u       // flags / fences at .sys scope (else .gpu)

typedef struct {
  uint32_t pack0, npack;     // frame descriptors packing into the slot (sender side)
  uint32_t unpack0, nunpack; // frame descriptors unpacking out of the slot (receiver side)
  uint32_t pack_items;       // work items over the pack frames (frame item0 is batch-relative)
  uint32_t unpack_items;     // work items over the unpack frames
  uint64_t bytes;            // payload bytes in this batch
  uint64_t extent;           // slot bytes in use (last frame end), for the L2 discard
  uint32_t layer;            // layer of the batch's frames (trace)
  uint32_t layer_idx;        // index of that layer in the plan's layer order (strict layer barriers)
} rs_batch_desc;

// Strict layer order in STAGED mode (executor.cpp:208: all
// layer-l traffic before any layer-(l+1) traffic): every CTA of the exchange
// launch meets a barrier after each plan layer.  Two levels: the CTAs of one
// GPU count in `arrive`; the last one publishes this slot's `done_self` flag
// and, in a multi-GPU job, waits for every slot's flag (peer-mapped,
// system scope) before releasing its GPU's CTAs through `release`.
//
// Stream lanes run layer-scoped roles: a CTA takes a role by ticket (roles
// sorted by first layer, so the CTAs of the earliest layers are resident
// first), meets only the barriers of its lane's layer range, and layer l's
// barrier waits for expect[l] arrivals -- the CTAs active in l.  Lanes of
// links that never share a layer (the PP stages) then reuse the same CTA
// slots instead of idling through each other's layers.  Classic lanes:
// expect == roles == null, every CTA arrives at every barrier (cumulative).
typedef struct {
  uint32_t nlayers;                 // 0: no barriers (fused layers)
  uint32_t nslots;                  // slots whose flags `done_all` lists (1: this GPU only)
  unsigned long long* arrive;       // arrival counters (zeroed before the launch): one, or one per layer with expect
  const uint32_t* expect;           // arrivals that complete barrier l (CTAs active in layer l), or null
  const uint32_t* local_n;          // local-copy roles sharing layer l's local items, or null (all of them)
  const uint32_t* roles;            // ticket -> CTA role (the blockIdx the role stands for), or null
  const uint32_t* local_roles;      // local role q: [2q] = its share index in every layer of its run,
                                    // [2q + 1] = first layer | last layer << 16 (with local_n)
  unsigned long long* tickets;      // role ticket counter (zeroed with `arrive`)
  uint64_t* release;                // this GPU's release flag (epoch + layer + 1)
  uint64_t* done_self;              // this slot's layer-done flag (in its comm arena)
  const uint64_t* const* done_all;  // every slot's layer-done flag as mapped here (device array)
  const uint64_t* local_layer_end;  // local-copy item end of each layer (device array, nlayers)
} rs_layer_sync;

// Transport trace (the RecordingTransport of proj/include/reshard/transport.hpp:50-75
// on the device): one record per (batch, role) of the last STAGED run;
// globaltimer nanoseconds.  t_end == 0: not recorded (role ran elsewhere).
typedef struct {
  uint32_t lane;             // the lane's first batch index (a lane identifier)
  uint32_t batch;            // batch index within the lane
  uint32_t layer;
  uint32_t role;             // 0 sender (pack + publish), 1 receiver (unpack + credit)
  uint64_t bytes;
  uint64_t t_begin;          // flag acquired (slot free / data ready)
  uint64_t t_end;            // flag published
} rs_trace_record;
