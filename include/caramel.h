/*
 * caramel.h -- C ABI of the B200 data-parallel aggregation hot path.
 *
 * The reference (overlapsim, /root/reference/pkg/src/overlapsim) has no FFI:
 * its aggregation is an analytic call, `collective_time(spec, model, reduce)`
 * (collective.py:106-157), made once per fusion bucket from the pipeline's
 * bucket loop (pipeline.py:80-94).  This library is what replaces that call
 * with a real launch.  Every entry point below names the reference interface
 * it stands in for.  Conventions:
 *   - plain C types only (no torch types); device memory is passed as
 *     uint64_t device addresses or typed pointers, streams as `void*`
 *     (a cudaStream_t);
 *   - every function returns 0 on success and a negative CARAMEL_E* code on
 *     failure, with a message retrievable through caramel_last_error();
 *     no C++ exception ever crosses the ABI;
 *   - all GPU work is stream ordered; only init/import/finalize/status block.
 *
 * Element type is fp32 throughout (gradients and parameters).
 */
#ifndef CARAMEL_H
#define CARAMEL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CARAMEL_ABI_VERSION 1
#define CARAMEL_MAX_RANKS 8     /* one 8xB200 NVSwitch box */
#define CARAMEL_MAX_DEPTH 8     /* MAX_DEPTH, collective.py:32 */

/* Error codes. */
#define CARAMEL_OK 0
#define CARAMEL_EINVAL -1       /* bad argument (mirrors ValueError) */
#define CARAMEL_EWORKERS -2     /* UnsupportedWorkerCount, collective.py:77-81 */
#define CARAMEL_ECUDA -3        /* CUDA runtime failure */
#define CARAMEL_ETIMEOUT -4     /* a cross-rank flag wait hit the watchdog */
#define CARAMEL_ESTATE -5       /* call made in the wrong context state */

/* Aggregation patterns, same values/order as overlapsim Pattern
 * (collective.py:35-38: ring, hd, shuffle). */
#define CARAMEL_RING 0
#define CARAMEL_HD 1
#define CARAMEL_SHUFFLE 2

/* What the shard owner applies to the rank-ordered sum before all-gather. */
#define CARAMEL_EPI_SUM 0       /* out = sum_r g_r                              */
#define CARAMEL_EPI_SCALE 1     /* out = (sum_r g_r) * scale                    */
#define CARAMEL_EPI_SGD 2       /* out = theta - lr * ((sum_r g_r) * scale)     */
                                /* the postponed update (transfer.py:156-160)   */

/* Bucket flags. */
#define CARAMEL_F_PACK 1u        /* gather member grads into the bucket (K1)   */
#define CARAMEL_F_UNPACK 2u      /* scatter the result back to the members:
                                    into .grad for SUM/SCALE, .param for SGD   */
#define CARAMEL_F_PARAM_ARENA 4u /* SGD result is stored straight into every
                                    rank's symmetric parameter arena            */
#define CARAMEL_F_FLAT 8u        /* caller asserts: the members form ONE
                                    contiguous, 16-byte aligned gradient segment
                                    (nseg == 1) -- enables the TMA bulk-copy
                                    streaming path                              */
#define CARAMEL_F_AUTO_EPOCH 16u /* caramel_allreduce[_update] with epoch 0 only:
                                    the launch uses the device epoch counter + 1
                                    and its last CTA advances the counter -- one
                                    kernel per call, graph-replayable (instead of
                                    caramel_epoch_advance + the call); rejected
                                    by list / stream-engine calls               */

/* One member tensor of a fusion bucket.  Members are listed in bucket order
 * (BatchGroup.param_ids, batching.py:28-33) with contiguous offsets. */
typedef struct caramel_segment {
  uint64_t grad;    /* device address of the member's fp32 gradient          */
  uint64_t param;   /* device address of the member's fp32 parameter, or 0   */
  uint64_t offset;  /* element offset of the member inside the bucket        */
  uint64_t numel;   /* element count                                         */
} caramel_segment;

/* One fusion bucket's collective: BatchGroup (batching.py:27-34) +
 * CollectiveSpec (collective.py:70-83) + its placement in the arenas. */
typedef struct caramel_bucket {
  uint64_t numel;       /* bucket elements (= total_bytes / 4)                  */
  uint64_t bucket_off;  /* byte offset of the bucket in each rank's arena (16B)  */
  uint64_t param_off;   /* byte offset in each rank's param arena (PARAM_ARENA)  */
  uint64_t flag_off;    /* byte offset of the bucket's flag block in the arena   */
  uint64_t segs;        /* device address of caramel_segment[nlocal][nseg]       */
  int32_t nseg;
  int32_t depth;        /* chunks, 1..8: adaptive_depth (collective.py:160-164)  */
  int32_t pattern;      /* CARAMEL_RING / _HD / _SHUFFLE                         */
  int32_t epilogue;     /* CARAMEL_EPI_*                                         */
  uint32_t flags;       /* CARAMEL_F_*                                           */
  int32_t ctas;         /* CTAs per rank; from caramel_bucket_layout()           */
  float lr;             /* SGD learning rate                                     */
  float scale;          /* multiplier on the sum (1/p for a mean)                */
} caramel_bucket;

typedef struct caramel_ctx caramel_ctx;

/* ---- library ----------------------------------------------------------- */
int caramel_abi_version(void);
const char* caramel_last_error(void);

/* Integer chunk/shard rule.  The reference only defines float bytes per chunk
 * (stage.transfer_bytes / k, collective.py:124, with transfer_bytes = d/p,
 * collective.py:90).  Chunk c of an n-element bucket is
 * [floor(c*n/k), floor((c+1)*n/k)); shard s of an m-element chunk is
 * [floor(s*m/p), floor((s+1)*m/p)).  Writes depth*(workers+1) absolute
 * element bounds, row c = shard starts of chunk c plus the chunk end. */
int caramel_chunk_bounds(uint64_t numel, int depth, int workers, uint64_t* out);

/* Launch geometry and arena footprint of one bucket (identical on every
 * rank, so every rank launches the same grid): CTAs per rank, bytes of the
 * bucket region and bytes of its flag block.  Bucket region: shuffle = the
 * bucket itself (packed input, all-gathered in place); ring/hd = input and
 * partials + a second, output half (a fast neighbour never overwrites a
 * partial sum still to be pulled).  SHUFFLE with world > 1 adds world-1
 * staging slots of ceil(numel/world)+3 elements (256-byte aligned, after the
 * kernels' part) that peers' copy engines push into (caramel_allreduce_ce). */
int caramel_bucket_layout(uint64_t numel, int depth, int pattern, int world,
                          int32_t* ctas, uint64_t* bucket_bytes,
                          uint64_t* flag_bytes);

/* ---- context: symmetric arenas + bootstrap ----------------------------- */
/* Allocates this process's arenas on the current CUDA device.  `nlocal` is
 * 1 for one-process-per-GPU; nlocal == world hosts every rank in this process
 * on one GPU (rank emulation, used when fewer GPUs than ranks are present).
 * Arenas are zero-filled (flag words start at epoch 0). */
int caramel_init(int rank, int world, int nlocal, uint64_t arena_bytes,
                 uint64_t param_arena_bytes, caramel_ctx** out);
/* Bytes of one rank's bootstrap blob (CUDA IPC handles). */
int caramel_handle_size(void);
/* Writes this rank's bootstrap blob; exchanged by the caller (torch.distributed
 * all_gather over NCCL/gloo: bootstrap only, never on the data path). */
int caramel_export(caramel_ctx* ctx, void* blob);
/* Maps every peer's arenas from `world` blobs in rank order. */
int caramel_import(caramel_ctx* ctx, const void* blobs);
/* Device addresses of local rank `lr`'s arenas (lr < nlocal). */
int caramel_arena(caramel_ctx* ctx, int lr, uint64_t* bucket_arena,
                  uint64_t* param_arena);
/* Watchdog state: 0, or CARAMEL_ETIMEOUT if a cross-rank flag wait ever
 * exceeded the watchdog (synchronizes the device).  A timeout POISONS the
 * context: the waiting CTAs leave their kernel before any further store (no
 * epilogue writes a result computed from inputs that never arrived), every
 * later launch exits at entry, and the status stays set -- finalize the
 * context and bootstrap a new one.  The reference's analogue is its plan
 * consistency checks raising DeadlockDetected (sim.py:136-153). */
int caramel_status(caramel_ctx* ctx);
/* Same state without synchronizing: reads a host-mapped mirror of the status
 * word that the device writes when the watchdog fires (cheap enough to call
 * once per iteration). */
int caramel_poll(caramel_ctx* ctx);
int caramel_set_timeout_ms(caramel_ctx* ctx, uint64_t ms);
int caramel_finalize(caramel_ctx* ctx);

/* ---- K1 / K4: bucket pack and unpack ----------------------------------- */
/* Gather members' .grad into `bucket` in member order (batching.py:76,122).
 * 128-bit vectorised where the member is 16-byte aligned. */
int caramel_pack(const caramel_segment* segs, int32_t nseg, uint64_t numel,
                 float* bucket, void* stream);
/* Scatter `bucket` back into the members' .grad (to_param == 0) or
 * .param (to_param != 0). */
int caramel_unpack(const caramel_segment* segs, int32_t nseg, uint64_t numel,
                   const float* bucket, int32_t to_param, void* stream);

/* ---- K2/K3 (+K4): the per-bucket collective ------------------------------ */
/* Replaces collective_time(CollectiveSpec(pattern, world, 4*numel, depth))
 * (collective.py:106-157) at pipeline.py:94 with a real launch: a chunked
 * ring / halving-doubling / two-shot all-reduce that loads and stores peer
 * HBM over NVLink with per-chunk epoch flags, the reduction fused in, summing
 * each element in the pattern's fixed order.  `epoch` must be identical on
 * every rank and strictly increase per bucket (1, 2, 3, ...).  Result lands
 * in every rank's bucket (and members, with CARAMEL_F_UNPACK).
 * epoch == 0 selects the context's device epoch counter instead (see
 * caramel_epoch_advance), which makes launches replayable in a CUDA graph. */
int caramel_allreduce(caramel_ctx* ctx, const caramel_bucket* bucket,
                      uint32_t epoch, void* stream);
/* Stream-ordered increment of the context's device epoch counter: call once
 * per iteration before that iteration's epoch==0 launches (every rank the
 * same number of times). */
int caramel_epoch_advance(caramel_ctx* ctx, void* stream);
/* Same collective with the postponed SGD update fused into the all-gather
 * epilogue: the shard owner computes theta - lr*(sum*scale) once and stores
 * it to every rank (transfer.py:156-160). */
int caramel_allreduce_update(caramel_ctx* ctx, const caramel_bucket* bucket,
                             uint32_t epoch, void* stream);

/* caramel_allreduce_many modes. */
#define CARAMEL_MANY_FUSED 0  /* flat phases + cross-rank grid barriers: fastest;
                                 every rank must issue the identical list */
#define CARAMEL_MANY_FLAGS 1  /* per-(bucket, chunk, tile) flags, the same words
                                 single-bucket launches use: ranks may group the
                                 same launch order into different lists */

/* A list of buckets in launch order as ONE launch (every listed bucket's
 * gradients already produced).  `host` is the descriptor list (validated);
 * `dev_buckets` a device copy of the same caramel_bucket[count];
 * `dev_prefix` / `dev_segprefix` device uint64_t[count+1] prefix sums of the
 * buckets' element counts / member-segment counts (absolute values are fine,
 * so a sub-range of a longer list is passed by offsetting all three
 * pointers).  All buckets share pattern, epilogue and flags.  `ctas`: CTAs per
 * rank, 0 = library default (the whole GPU).  `mode`: CARAMEL_MANY_*.  In
 * FUSED mode the two-shot runs as three flat
 * phases (pack / pull-reduce-epilogue-push / unpack) separated by cross-rank
 * grid barriers, every element owned per the bucket's chunk/shard rule; with
 * world == 1 the concatenated element space is tiled over the grid.  Per
 * bucket the result equals caramel_allreduce[_update] on that bucket. */
int caramel_allreduce_many(caramel_ctx* ctx, const caramel_bucket* host, int32_t count,
                           uint64_t dev_buckets, uint64_t dev_prefix,
                           uint64_t dev_segprefix, int32_t ctas, int32_t mode,
                           uint32_t epoch, void* stream);

/* Copy-engine two-shot (the overlapped path's engine while backward kernels
 * own the SMs; same reference call it replaces, pipeline.py:94).  The NVLink
 * transfers of a two-shot run on the GPU's copy engines (each rank pushes its
 * gradients of peer q's shard into q's staging slot, then its result shard
 * into every peer's output) and the cross-rank flags are stream memory
 * operations, so no SM is held while bytes move or while a rank waits for
 * its peers; the reduction + epilogue is one short kernel.  Buckets [0, count) of `host` are launch positions index0 ..
 * index0+count-1 of this iteration's launch order; every rank must make the
 * same sequence of calls (a stream wait stalls its hardware queue, so
 * differently grouped calls could wait on each other).  `epoch`: the
 * iteration number, > 0 and increasing.  `grad_stream`: the stream that
 * produced the buckets' gradients -- the READY signal is issued there, not
 * behind this rank's earlier all-gather waits; `stream` must already be
 * ordered after the gradients (e.g. waited on grad_stream).  Per element the result equals
 * caramel_allreduce[_update] with the SHUFFLE pattern (sum in ascending rank
 * order).  Requires one rank per process, SHUFFLE buckets without
 * PACK/UNPACK (gradients live in the bucket arena) and, for SGD,
 * PARAM_ARENA.  Returns CARAMEL_ESTATE if the device lacks 64-bit stream
 * memory operations (caramel_ce_available). */
int caramel_allreduce_ce(caramel_ctx* ctx, const caramel_bucket* host, int32_t count,
                         uint32_t index0, uint32_t epoch, void* grad_stream, void* stream);
/* 1 if caramel_allreduce_ce / caramel_allreduce_gated can run on this
 * context, else 0. */
int caramel_ce_available(caramel_ctx* ctx);
/* The gated SM engine: the same two-shot as caramel_allreduce with every wait
 * moved from the SMs to the stream front end.  READY (a 64-bit stream write
 * of (epoch << 32 | index0 + count) into every peer, issued after
 * `grad_stream`'s gradients), a stream wait on every peer's READY, one
 * k_gated launch of at most CARAMEL_GATED_CTAS CTAs (default 32) that pulls
 * my shard of every bucket from every rank, sums in ascending rank order,
 * applies the epilogue and stores into every replica, then DONE and a stream
 * wait on every peer's DONE.  No CTA spins on a peer, so while it overlaps a
 * backward pass the kernel holds SMs only while bytes move.  Arguments,
 * requirements, tags and results as caramel_allreduce_ce (the two engines
 * share the READY / DONE words and may alternate in one launch order); no
 * staging slots are used.  Replaces, like caramel_allreduce, the modelled
 * collective of pipeline.py:94. */
int caramel_allreduce_gated(caramel_ctx* ctx, const caramel_bucket* host, int32_t count,
                            uint32_t index0, uint32_t epoch, void* grad_stream, void* stream);
/* Engines of caramel_ce_submit. */
#define CARAMEL_ENGINE_CE 0  /* caramel_allreduce_ce                                  */
#define CARAMEL_ENGINE_SM 1  /* caramel_allreduce[_update] per bucket, epoch 0 (device counter) */
#define CARAMEL_ENGINE_GATED 2  /* caramel_allreduce_gated                            */

/* Asynchronous launch: validates, records "gradients ready" on grad_stream in
 * the caller's stream order, and hands the call to the context's worker
 * thread, which issues it on `stream` -- the calling thread (autograd's) pays
 * a few microseconds instead of the whole issue cost.  CARAMEL_ENGINE_CE
 * issues caramel_allreduce_ce(host, count, index0, epoch), CARAMEL_ENGINE_GATED
 * caramel_allreduce_gated(host, count, index0, epoch); CARAMEL_ENGINE_SM
 * launches the SM kernel of each bucket with the device epoch counter
 * (caramel_epoch_advance on `stream` once per iteration).  Calls are issued in
 * submission order, so both engines can share `stream` in launch order.
 * `done_event` (a cudaEvent_t, or NULL) is recorded on `stream` after the
 * call.  Work submitted here is ordered on `stream` only after
 * caramel_ce_flush returns: flush before enqueueing anything else on `stream`
 * or waiting on it / on done_event.  Worker errors are reported by the next
 * submit or flush. */
int caramel_ce_submit(caramel_ctx* ctx, const caramel_bucket* host, int32_t count,
                      uint32_t index0, uint32_t epoch, int32_t engine, void* grad_stream,
                      void* stream, void* done_event);
/* Blocks until every submitted call has been issued to its streams. */
int caramel_ce_flush(caramel_ctx* ctx);

/* ---- NVLS (NVLink SHARP) multicast: the non-fixed-order mode ------------- */
/* The two-shot with the reduction done inside the NVSwitch: the owner of each
 * shard issues multimem.ld_reduce on a multicast address (the switch sums every
 * GPU's copy, in its own order) and multimem.st (the switch writes the result
 * into every GPU's copy) -- S bytes per GPU and direction instead of
 * 2(p-1)/p x S (collective.py:12-13,98-100 is the pattern; its byte count is
 * the one thing this mode changes).  Results agree with the rank-order sum to
 * 1e-6 x sum_r |g_r| per element, not bit for bit: the bit-exact contract stays
 * with caramel_allreduce.  Setup, in this order on every rank (the caller puts
 * a barrier between the steps): */
/* 1 if this context can use multicast objects (one rank per process, world > 1). */
int caramel_mc_available(caramel_ctx* ctx);
/* Allocate `bytes` (rounded up to the multicast granularity) of multicast-
 * capable memory on this GPU.  Rank 0 also creates the multicast object and
 * listens on an abstract Unix socket named after `token` (a string identical on
 * every rank and unique per job). */
int caramel_mc_create(caramel_ctx* ctx, uint64_t bytes, const char* token);
/* Concurrently on every rank: rank 0 passes the multicast handle's file
 * descriptor to every peer (SCM_RIGHTS); every rank adds its GPU. */
int caramel_mc_exchange(caramel_ctx* ctx);
/* After every rank's exchange: bind this GPU's memory to the multicast object,
 * map both views; writes this rank's unicast address of the (zeroed) arena. */
int caramel_mc_bind(caramel_ctx* ctx, uint64_t* unicast_base);
/* One bucket through the switch: `bucket_off` is relative to the multicast
 * arena (the gradients are written there through the unicast view), results
 * land in place (SUM / SCALE) or, with CARAMEL_EPI_SGD, in the parameter
 * arena (every rank updates its own copy from the identical broadcast
 * sum x scale).  `flag_off`/`ctas`/`depth` as for caramel_allreduce (the flag
 * block lives in the IPC bucket arena; size it with caramel_bucket_layout). */
int caramel_allreduce_nvls(caramel_ctx* ctx, const caramel_bucket* bucket, uint32_t epoch, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CARAMEL_H */
