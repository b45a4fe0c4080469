/*
 * fsdp_b200.h — C ABI of the B200-native FSDP hot path.
 *
 * Plain pointers, sizes and a CUDA stream handle (`void* stream` is a
 * cudaStream_t); no torch types.  Every entry point returns 0 on success or a
 * non-zero code (a cudaError_t value, or one of FSDP_E_*) and records a
 * message retrievable with fsdp_last_error().  All device work is enqueued on
 * the given stream; nothing blocks the host.
 *
 * Each entry point replaces a function of the reference `shardsim` package
 * (paths relative to /root/reference/pkg/src/shardsim/).  The reference binds
 * nothing natively (it is numpy); the binding a maintainer would add is the
 * ctypes stub shown in INTEGRATION.md, which is exactly what
 * paper_2304_11277_b200/_lib.py does.
 */
#ifndef FSDP_B200_H_
#define FSDP_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* element types */
enum { FSDP_F32 = 0, FSDP_BF16 = 1 };

/* error codes beyond cudaError_t */
enum {
  FSDP_E_INVALID = 10001,    /* bad argument (CollectiveError-class contract) */
  FSDP_E_TIMEOUT = 10002,    /* cross-GPU flag wait timed out (DeadlockError) */
  FSDP_E_IPC = 10003,        /* IPC handle export/import failed */
  FSDP_E_UNSUPPORTED = 10004
};

#define FSDP_MAX_RANKS 8
#define FSDP_MAX_CTAS 160
#define FSDP_MAX_TENSORS 96
#define FSDP_IPC_HANDLE_BYTES 64

const char* fsdp_last_error(void);
int fsdp_abi_version(void);
/* number of kernels this library has launched (process lifetime) */
uint64_t fsdp_launch_count(void);
int fsdp_num_sms(int device);

/* ------------------------------------------------------------------------
 * Layout / copy kernels                                  (flatparam.py)
 * ---------------------------------------------------------------------- */

/* Gather n tensors into a flat buffer of psi elements: tensor i lands at
 * [offsets[i], offsets[i] + numels[i]); every other element of [0, psi) is
 * written 0 (padding, flatparam.py:93, :180-181).  With accumulate != 0 the
 * result is added to the existing flat contents (engine.py:534, `ru.grad +=
 * flat`) and missing/padding regions are left unchanged.  A NULL src means
 * "no gradient": zero-filled (flatparam.py:181-185).
 * Replaces: writeback_grad (flatparam.py:167-191); the layout+concat of the
 * init materialisation paths (deferred_init.py:156-176, :244-260). */
int fsdp_flatten(const void* const* srcs, const int64_t* numels, const int64_t* offsets,
                 int n_tensors, int src_dtype, void* flat, int64_t psi, int flat_dtype,
                 int accumulate, void* stream);

/* Scatter [offsets[i], +numels[i]) of a flat buffer into n tensors.
 * Replaces: FlatParameter.views materialised (flatparam.py:159-164),
 * gather_full_params (engine.py:824-834), streamed-init copy
 * (deferred_init.py:256). */
int fsdp_unflatten(const void* flat, int flat_dtype, void* const* dsts, const int64_t* numels,
                   const int64_t* offsets, int n_tensors, int dst_dtype, void* stream);

/* shard[i] = flat[shard_index * shard_numel + i] (same dtype).
 * Replaces: FlatParameter.shard (flatparam.py:139-147). */
int fsdp_shard_copy(const void* flat, void* shard, int64_t shard_numel, int shard_index,
                    int dtype, void* stream);

/* dst[i] = cast(src[i]) (RNE for fp32 -> bf16).
 * Replaces: the full -> low cast before the gather (engine.py:661-662) and the
 * F=1 mixed-precision local cast (engine.py:651-660). */
int fsdp_cast(const void* src, int src_dtype, void* dst, int dst_dtype, int64_t n, void* stream);

/* ------------------------------------------------------------------------
 * Optimizer epilogue on the local shard         (numerics.py, engine.py)
 * ---------------------------------------------------------------------- */

/* g *= inv_scale; if any g is non-finite, *found_inf = 1.0f (else unchanged).
 * Replaces: engine.py:566-571 (`ru.accum *= inv`; isfinite check). */
int fsdp_unscale_found_inf(float* g, int64_t n, float inv_scale, float* found_inf, void* stream);

/* Adam (numerics.py:273-285), float32 operation-for-operation as numpy runs
 * it: m = b1*m + omb1*g; v = b2*v + (omb2*g)*g; mh = m/bc1; vh = v/bc2;
 * p -= (lr*mh)/(sqrt(vh)+eps).  The scalars are the float32 roundings of the
 * double-precision expressions (b1, 1-b1, b2, 1-b2, 1-b1^t, 1-b2^t, lr, eps).
 * If skip_flag != NULL and *skip_flag > 0 the step is skipped on device
 * (engine.py:578-586 verdict).  If p_lowp != NULL the updated parameter is
 * also written there as bf16 (the next gather's source).
 * Replaces: Adam.step / the optimizer loop of _rank_step (engine.py:585). */
int fsdp_adam_step(float* p, const float* g, float* m, float* v, int64_t n, float lr, float b1,
                   float omb1, float b2, float omb2, float bc1, float bc2, float eps,
                   const float* skip_flag, void* p_lowp, void* stream);

/* p -= lr * g (numerics.py:248-253), same skip/p_lowp contract. */
int fsdp_sgd_step(float* p, const float* g, int64_t n, float lr, const float* skip_flag,
                  void* p_lowp, void* stream);

/* The same two steps reading a bf16 gradient (W = 1: the write-back lands in
 * a bf16 arena and the optimizer reads it directly, 2 B/elem less on each
 * side).  bf16 -> fp32 is exact, so the result is bit-identical to running
 * fsdp_adam_step / fsdp_sgd_step on the fp32 copy of the same gradient. */
int fsdp_adam_step_bf16g(float* p, const void* g_bf16, float* m, float* v, int64_t n, float lr,
                         float b1, float omb1, float b2, float omb2, float bc1, float bc2, float eps,
                         const float* skip_flag, void* p_lowp, void* stream);
int fsdp_sgd_step_bf16g(float* p, const void* g_bf16, int64_t n, float lr, const float* skip_flag,
                        void* p_lowp, void* stream);

/* ------------------------------------------------------------------------
 * Communicator: CUDA-IPC symmetric pool + SM-driven collectives over
 * NVLink/NVSwitch peer pointers                           (collectives.py)
 *
 * Every rank allocates a pool of identical size; all collective buffers are
 * addressed by POOL OFFSET, identical on every rank.  Group = ranks
 * {start + j*stride}, j < size, with start derived from the caller's rank:
 * stride == 1 -> consecutive blocks of `size` (sharded groups,
 * collectives.py:89-92); stride > 1 -> {r % stride + j*stride} (replicated
 * groups, collectives.py:94-96).  The k-th call on a (channel, group) pairs
 * with every member's k-th call (collectives.py:238-251) via epoch counters.
 * ---------------------------------------------------------------------- */
typedef struct fsdp_comm fsdp_comm_t;

/* channels: independent flag sets, one per stream that issues collectives */
enum { FSDP_CH_AG = 0, FSDP_CH_RS = 1, FSDP_CH_AR = 2, FSDP_CH_SCALAR = 3, FSDP_NUM_CH = 4 };

/* Create a communicator for `rank` of `world`; allocates the local pool.
 * max_ctas bounds every collective's grid (<= FSDP_MAX_CTAS). */
int fsdp_comm_create(int rank, int world, int64_t pool_bytes, int max_ctas, fsdp_comm_t** out);
/* Emulated communicator: all `world` ranks' pools on the CURRENT device,
 * collectives launched as ONE cooperative kernel over every rank's data
 * (single-GPU testing of the cross-rank protocol). */
int fsdp_comm_create_emulated(int world, int64_t pool_bytes, int max_ctas, fsdp_comm_t** out);
int fsdp_comm_ipc_handle(fsdp_comm_t* c, void* handle_out /* FSDP_IPC_HANDLE_BYTES */);
/* handles: world * FSDP_IPC_HANDLE_BYTES, indexed by rank */
int fsdp_comm_open_peers(fsdp_comm_t* c, const void* handles);
/* device base address of rank r's pool as seen by this process (emulated:
 * each emulated rank's pool; real: r == own rank only) */
void* fsdp_comm_pool_ptr(fsdp_comm_t* c, int r);
int64_t fsdp_comm_pool_bytes(fsdp_comm_t* c);
/* bytes at the start of every pool reserved for flags + error word */
int64_t fsdp_comm_reserved_bytes(void);
/* device-side error word (FSDP_E_TIMEOUT after a flag-wait timeout); 0 = ok.
 * Synchronous read; call after synchronising the streams. */
int fsdp_comm_device_error(fsdp_comm_t* c);
int fsdp_comm_set_timeout_ms(fsdp_comm_t* c, int64_t ms);
/* A timed-out wait ABORTS the communicator: it sets the error word of every
 * rank whose pool this process maps (own + peers), and from then on every
 * SM/LL data kernel skips its peer loads and stores (the flag waits bail out
 * at once).  Copy-engine DMA already enqueued still runs; the optimizer must
 * therefore read the word before updating: fsdp_comm_fold_error writes
 * *flag = 1 if any local error word is set, else (keep ? *flag : 0), and
 * mirrors the word into `host_mirror` (pinned host memory, may be NULL) so the
 * host raises DeadlockError at the next step boundary without a sync.
 * Replaces: the DeadlockError raise and the verdict agreement of
 * collectives.py:461-483 / engine.py:410-411. */
int fsdp_comm_fold_error(fsdp_comm_t* c, float* flag, int keep, int* host_mirror, void* stream);
/* Diagnostics of the first local timeout (synchronous read): out[0..5] =
 * {set, polled word index in the pool, last value seen, epoch, channel,
 * group size << 8 | stride}.  A word index below the flag area's size decodes
 * as ((channel * 3 + phase) * FSDP_MAX_RANKS + src) * FSDP_MAX_CTAS + cta. */
int fsdp_comm_timeout_info(fsdp_comm_t* c, uint32_t* out);
/* Zero the local error word(s) (synchronous; tests and re-use after a handled abort). */
int fsdp_comm_clear_error(fsdp_comm_t* c);
/* Fault injection for verify-sensitivity (collectives.py:176, :296; cli.py:568-574):
 * misorder_reduce_scatter != 0 makes every reduce-scatter hand member k the
 * reduced chunk (k + 1) % size instead of chunk k (all engines).  Test use only. */
int fsdp_comm_set_fault(fsdp_comm_t* c, int misorder_reduce_scatter);
/* split != 0 (default): collectives run as [1-CTA enter barrier] [data kernel
 * that only signals] [1-CTA exit barrier], so a late peer never parks the
 * data kernel's CTAs on SMs.  timing != 0: CUDA events around every data
 * kernel, read back (and recycled) by fsdp_comm_timing_drain. */
enum { FSDP_KIND_AG = 0, FSDP_KIND_RS = 1, FSDP_KIND_AR = 2, FSDP_NUM_KINDS = 3 };
int fsdp_comm_set_mode(fsdp_comm_t* c, int split, int timing);
/* on == 0: split-mode collectives launch ONLY their data kernel (no enter /
 * exit barrier kernels).  Profiling harness only: the caller must order the
 * ranks itself (one process driving every device, synchronising all devices
 * between collectives), so that nothing ever spins under a profiler. */
int fsdp_comm_set_barriers(fsdp_comm_t* c, int on);
/* Grid cap for the data kernels of one collective kind (0 = max_ctas).  Every
 * member of a group must use the same value (per-CTA flags pair by index). */
int fsdp_comm_set_ctas(fsdp_comm_t* c, int kind, int ctas);
/* Synchronises on the recorded events of `kind`; writes up to max_n
 * durations (ms) and the total count. */
int fsdp_comm_timing_drain(fsdp_comm_t* c, int kind, float* ms_out, int max_n, int* count);
int fsdp_comm_destroy(fsdp_comm_t* c);

/* All-gather with fused cast (collectives.py:288-291 + engine.py:661-671):
 * rank at group position k pushes cast(shard[0..n)) into every member's pool
 * at byte offset dst_off + k*n*sizeof(dst) — the unsharded flat buffer is
 * written in place on every peer (no copy-out, engine.py:614/:630 removed).
 * Emulated comm: shards[e] / one entry per emulated rank e; real: shards[0]. */
int fsdp_allgather(fsdp_comm_t* c, int channel, int gsize, int gstride, const void* const* shards,
                   int src_dtype, int64_t n, int64_t dst_off, int dst_dtype, void* stream);

/* Reduce-scatter with fp32 accumulation (engine.py:789-803,
 * collectives.py:273-297): every member pushes chunk j of its flat payload
 * (gsize*n elements) to member j's staging at stage_off (slot = sender's
 * position); member k then sums its gsize slots in ascending rank order
 * starting from +0.0f, applies  (sum / postdiv)  (skipped when postdiv == 1),
 * and writes out[i] = (accumulate ? out[i] : 0.0f) + that (engine.py:817-820).
 * prediv != 1 divides every payload element before summation. */
int fsdp_reduce_scatter(fsdp_comm_t* c, int channel, int gsize, int gstride,
                        const void* const* flats, int src_dtype, int64_t n, int64_t stage_off,
                        float* const* outs, float prediv, float postdiv, int accumulate,
                        void* stream);

/* Reduce-scatter, PULL variant (same semantics as fsdp_reduce_scatter): every
 * member's flat payload lives in its own pool at src_off (gsize*n elements);
 * the member at group position k loads chunk k of every member's buffer over
 * NVLink in ascending rank order and reduces in fp32 registers; no staging.
 * The caller must not rewrite its src_off region until this call completes
 * on its stream (the kernel's exit barrier guarantees peers are done). */
int fsdp_reduce_scatter_pull(fsdp_comm_t* c, int channel, int gsize, int gstride, int64_t src_off,
                             int src_dtype, int64_t n, float* const* outs, float prediv,
                             float postdiv, int accumulate, void* stream);

/* Same contract as fsdp_reduce_scatter_pull; the NVLink reads are 1-D TMA
 * bulk copies (cp.async.bulk, mbarrier-tracked, 4-stage shared-memory ring)
 * so a few CTAs keep the link busy.  Falls back to the register-pull kernel
 * when n % 8 != 0 or buffers are not 16-byte aligned. */
int fsdp_reduce_scatter_tma(fsdp_comm_t* c, int channel, int gsize, int gstride, int64_t src_off,
                            int src_dtype, int64_t n, float* const* outs, float prediv,
                            float postdiv, int accumulate, void* stream);

/* Copy-engine variants (no SM work for the data movement; real communicator
 * only).  All-gather: same-dtype shard -> every member's pool at
 * dst_off + pos*n (DMA writes over NVLink, one side stream per peer).
 * Reduce-scatter: chunk pos of every member's payload (pool offset src_off)
 * is DMA-pulled into local staging (stage_off, gsize*n elements), then one
 * local kernel sums in ascending rank order in fp32 (/ postdiv, += out).
 * Same flag protocol (enter barrier, per-peer release, exit barrier). */
int fsdp_allgather_ce(fsdp_comm_t* c, int channel, int gsize, int gstride, const void* shard,
                      int dtype, int64_t n, int64_t dst_off, void* stream);
int fsdp_reduce_scatter_ce(fsdp_comm_t* c, int channel, int gsize, int gstride, int64_t src_off,
                           int src_dtype, int64_t n, int64_t stage_off, float* out, float prediv,
                           float postdiv, int accumulate, void* stream);
/* Same, with the result in out_dtype (FSDP_F32, or FSDP_BF16 = the fp32 sum
 * / postdiv rounded once to bf16, accumulate = 0): HYBRID_SHARD's stage-1
 * partial in the reduce dtype, which is what the reference sends to the
 * replica all-reduce (engine.py:789-790, :798-810: the reduce-scatter output
 * is the all-reduce payload). */
int fsdp_reduce_scatter_ce_out(fsdp_comm_t* c, int channel, int gsize, int gstride, int64_t src_off,
                               int src_dtype, int64_t n, int64_t stage_off, void* out, int out_dtype,
                               float prediv, float postdiv, int accumulate, void* stream);

/* All-reduce (collectives.py:298-301; hybrid stage 2, engine.py:804-816):
 * two-shot push (reduce-scatter to owners, ascending-rank fp32 sum, then
 * all-gather of the owners' results), so every member holds bit-identical
 * values.  outs[i] = (accumulate ? outs[i] : 0) + sum/postdiv.  Staging:
 * stage_off holds gsize*ceil(n/gsize) payload elements, gather_off holds
 * gsize*ceil(n/gsize) fp32. */
int fsdp_allreduce(fsdp_comm_t* c, int channel, int gsize, int gstride, const void* const* ins,
                   int src_dtype, int64_t n, int64_t stage_off, int64_t gather_off,
                   float* const* outs, float postdiv, int accumulate, void* stream);

/* Copy-engine all-reduce: same contract and bits as fsdp_allreduce, real
 * communicator only.  `in` is a local buffer of n payload elements (it need
 * not live in the pool); DMA pushes chunks to their owners' staging, the
 * owner reduces (ascending fp32, / postdiv) on SMs, DMA pushes the result to
 * every member's gather buffer, then out = (accumulate ? out : 0) + result.
 * No SM time is spent moving data, which matters when the all-reduce
 * overlaps backward GEMMs (NO_SHARD, HYBRID stage 2). */
int fsdp_allreduce_ce(fsdp_comm_t* c, int channel, int gsize, int gstride, const void* in,
                      int src_dtype, int64_t n, int64_t stage_off, int64_t gather_off, float* out,
                      float postdiv, int accumulate, void* stream);
/* Same, with the output itself a pool region: out = [out_off, +n fp32) at
 * the same offset on every member (out_off 16-byte aligned).  The owner
 * reduces its chunk straight into its own out slice and the DMA pushes that
 * slice into every member's out: no gather buffer and no epilogue pass (HBM
 * traffic per member drops by ~2n*4 bytes).  out = sum / postdiv
 * (accumulate = 0 semantics; the runtime keeps its HYBRID / NO_SHARD fp32
 * gradient arena in the pool to use this on the first micro-batch). */
int fsdp_allreduce_ce_pool(fsdp_comm_t* c, int channel, int gsize, int gstride, const void* in,
                           int src_dtype, int64_t n, int64_t stage_off, int64_t out_off, float postdiv,
                           void* stream);

/* 1-element world all-reduce of a float flag (engine.py:572-576):
 * *outs[e] = sum over ranks (ascending) of *ins[e]. */
int fsdp_allreduce_scalar(fsdp_comm_t* c, const float* const* ins, float* const* outs,
                          void* stream);

/* Low-latency (LL) one-shot variants for small messages: ONE kernel, no
 * enter/exit barrier.  Data travels as 16-byte lines {d0, epoch, d1, epoch}
 * (8 payload bytes per line, 2x wire bytes) into an LL region of the
 * receiver's pool at ll_off (16-byte aligned, fsdp_ll_bytes(gsize, n, dtype)
 * bytes, same offset on every member, one region per channel); the receiver
 * polls the flags and unpacks.  The region is double-buffered by epoch
 * parity, which is safe without barriers because a member running epoch e
 * has received every peer's epoch e-1 lines.  Lines are laid out in blocks of
 * 32 as [block][member][parity], so a line's address does not depend on the
 * message length: calls of different sizes may share the region (one region
 * per channel sized for the largest call); fsdp_ll_bytes rounds to blocks.
 * fsdp_allgather_ll: same contract and destination as fsdp_allgather
 *   (collectives.py:288-291 + engine.py:661-671); the lines carry the
 *   dst-dtype (cast) payload.
 * fsdp_reduce_scatter_ll: same semantics as fsdp_reduce_scatter (ascending
 *   fp32 sum from +0, prediv, / postdiv, accumulate; collectives.py:273-297,
 *   engine.py:789-820); payload read locally only, no staging offset. */
int64_t fsdp_ll_bytes(int gsize, int64_t n, int dtype);
int fsdp_allgather_ll(fsdp_comm_t* c, int channel, int gsize, int gstride, const void* const* shards,
                      int src_dtype, int64_t n, int64_t dst_off, int dst_dtype, int64_t ll_off,
                      void* stream);
int fsdp_reduce_scatter_ll(fsdp_comm_t* c, int channel, int gsize, int gstride,
                           const void* const* flats, int src_dtype, int64_t n, int64_t ll_off,
                           float* const* outs, float prediv, float postdiv, int accumulate,
                           void* stream);


/* ------------------------------------------------------------------------
 * VMM pool + NVLink SHARP (NVLS) multicast                (B200 + NVSwitch)
 *
 * A VMM communicator's pool is one exportable cuMemCreate allocation per
 * rank; peers map it from the exported handle (replacing cudaMalloc +
 * cudaIpc*).  Its pool can then be bound whole to the multicast object of
 * the rank's shard group (consecutive groups of gsize ranks), so a single
 * multimem.st lands at the same pool offset in every member.  Setup order
 * (every rank; the host exchanges the 64-byte handles — for
 * FSDP_HANDLE_POSIX_FD the first int is a file descriptor that the host
 * must pass to the peer process, e.g. SCM_RIGHTS):
 *   create_vmm -> export_pool -> import_pool(every peer)
 *   leader: nvls_create -> (handle) -> members: nvls_import
 *   all: nvls_add_device -> barrier -> all: nvls_bind
 * ---------------------------------------------------------------------- */
enum { FSDP_HANDLE_FABRIC = 1, FSDP_HANDLE_POSIX_FD = 2 };
#define FSDP_SHAREABLE_BYTES 64

/* 1 if `device` supports multicast objects and VMM, else 0. */
int fsdp_nvls_supported(int device);
int fsdp_comm_create_vmm(int rank, int world, int64_t pool_bytes, int max_ctas, int handle_type,
                         fsdp_comm_t** out);
int fsdp_comm_export_pool(fsdp_comm_t* c, void* handle_out /* FSDP_SHAREABLE_BYTES */);
int fsdp_comm_import_pool(fsdp_comm_t* c, int r, const void* handle);
int fsdp_nvls_create(fsdp_comm_t* c, int gsize, void* handle_out);
int fsdp_nvls_import(fsdp_comm_t* c, int gsize, const void* handle);
int fsdp_nvls_add_device(fsdp_comm_t* c);
int fsdp_nvls_bind(fsdp_comm_t* c);
/* group size of the bound multicast object, 0 if none */
int fsdp_nvls_group_size(fsdp_comm_t* c);

/* All-gather through the multicast object (same contract as fsdp_allgather,
 * real communicator, one shard): member k stores cast(shard) ONCE with
 * multimem.st at dst_off + k*n*sizeof(dst) and the switch replicates it to
 * every member.  Falls back to fsdp_allgather when the group is not the
 * bound shard group, n % 8 != 0 or the buffers are not 16-byte aligned.
 * Replaces: _issue_unshard cast + AG (engine.py:661-671, collectives.py:288-291). */
int fsdp_allgather_nvls(fsdp_comm_t* c, int channel, int gsize, int gstride, const void* shard,
                        int src_dtype, int64_t n, int64_t dst_off, int dst_dtype, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FSDP_B200_H_ */
