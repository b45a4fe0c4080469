// CUDA-IPC communicator and SM-driven collectives over NVLink/NVSwitch.
//
// Design (B200-first, not a port of the reference's in-process fabric):
//  * every rank owns a symmetric pool (same size, same sub-allocation offsets
//    on every rank); peers map it with cudaIpcOpenMemHandle, so a collective
//    addresses any member's buffer as bases[member] + offset;
//  * all data movement is PUSH (st.global to peer memory): NVLink stores need
//    no round trip, loads would need ~2 us of latency hiding per request;
//  * cross-GPU ordering uses per-(channel, phase, sender, CTA) epoch flags
//    written with st.release.sys after a system fence and polled with
//    ld.acquire.sys.  Every member launches the same grid and partitions the
//    work into the same tiles, so CTA c only waits for the CTAs c of its
//    peers (no grid-wide barrier, no co-residency requirement);
//  * waits time out (default 20 s) into a device error word instead of
//    hanging the GPU — the analogue of shardsim's DeadlockError;
//  * reductions sum in fp32 in ascending rank order from +0.0f with explicit
//    __fadd_rn, which makes them bit-identical to the reference fabric's
//    deterministic mode (collectives.py:273-278) on fp32-upcast payloads.
//
// Emulated mode runs all W ranks of one communicator on the current GPU as a
// single cooperative launch (blockIdx.y = rank) over W pools, exercising the
// exact same flag protocol and address arithmetic without multiple GPUs.
#include <cooperative_groups.h>

#include <cstring>
#include <type_traits>
#include <map>
#include <vector>

#include "common.cuh"
#include "vmm.h"

namespace fsdp {

constexpr int kPhases = 3;
constexpr int64_t kFlagBytes =
    (int64_t)FSDP_NUM_CH * kPhases * FSDP_MAX_RANKS * FSDP_MAX_CTAS * sizeof(uint32_t);
constexpr int64_t kErrOff = kFlagBytes;                 // uint32 error word
constexpr int64_t kDiagOff = kFlagBytes + 64;           // uint32[6]: first local timeout (diagnostics)
constexpr int64_t kScalarOff = kFlagBytes + 256;        // float[FSDP_MAX_RANKS]
constexpr int64_t kReserved = 65536;
static_assert(kScalarOff + 4 * FSDP_MAX_RANKS <= kReserved, "reserved region too small");

constexpr int kCommThreads = 512;
constexpr int kVec = 8;                                  // elements per vector
constexpr int kU = 4;                                    // vectors per thread per tile
constexpr int kTileElems = kCommThreads * kVec * kU;     // 16384 elements per tile

struct CollParams {
  char* bases[FSDP_MAX_RANKS];
  const void* in[FSDP_MAX_RANKS];
  float* out[FSDP_MAX_RANKS];
  int rank0;        // >= 0: real mode, this process's rank; -1: emulated
  int gsize, gstride, channel;
  uint32_t epoch;
  int64_t n;
  int64_t off_a, off_b;
  float prediv, postdiv;
  int accumulate;
  int64_t timeout_ns;
  int split;        // 1: waits live in 1-CTA enter/exit kernels, data kernels only signal
  int data_ctas;    // exit kernel: grid of the data kernel it waits for
  char* mc_base;    // NVLS multicast VA of the pool (shard group), or null
  int rot;          // reduce-scatter fault hook: member k receives chunk (k + rot) % size
};

// chunk of the payload that member position `pos` reduces (rot = 0 except
// under the misorder fault, collectives.py:296)
__device__ __forceinline__ int rs_chunk(const CollParams& p, int pos, int size) {
  return (pos + p.rot) % size;
}

// flag slot (CTA index) reserved for the whole-collective enter barrier
constexpr int kEnterSlot = FSDP_MAX_CTAS - 1;

// ------------------------------------------------------------ primitives ----
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t* flag_ptr(char* base, int ch, int phase, int src, int cta) {
  return reinterpret_cast<uint32_t*>(base) +
         (((int64_t)(ch * kPhases + phase) * FSDP_MAX_RANKS + src) * FSDP_MAX_CTAS + cta);
}

template <typename T> __device__ __forceinline__ T ldcg_elem(const T* p);
template <> __device__ __forceinline__ float ldcg_elem<float>(const float* p) { return __ldcg(p); }
template <> __device__ __forceinline__ __nv_bfloat16 ldcg_elem<__nv_bfloat16>(const __nv_bfloat16* p) {
  unsigned short v;
  asm volatile("ld.global.cg.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return __ushort_as_bfloat16(v);
}

struct Group {
  int rank, start, pos, size, stride;
  __device__ int member(int j) const { return start + j * stride; }
};

__device__ __forceinline__ Group make_group(const CollParams& p) {
  Group g;
  g.rank = p.rank0 >= 0 ? p.rank0 : (int)blockIdx.y;
  g.size = p.gsize;
  g.stride = p.gstride;
  if (p.gstride == 1) {
    g.start = (g.rank / p.gsize) * p.gsize;
    g.pos = g.rank - g.start;
  } else {
    g.start = g.rank % p.gstride;
    g.pos = g.rank / p.gstride;
  }
  return g;
}

// A flag wait that timed out aborts the communicator: the error word of
// EVERY rank whose pool this process maps is set, so a late member sees the
// failure at its next collective or optimizer step (its skip predicate reads
// the word, fsdp_comm_fold_error) instead of computing on with a slot a
// timed-out peer may have written.  collectives.py:461-483 (DeadlockError).
// `what` = the polled word (flag or LL line), `seen` = its last value: the
// first local timeout records {1, word index in the pool, seen, epoch,
// channel, group (size << 8 | stride)} at kDiagOff for the host's message.
__device__ __noinline__ void comm_abort(const CollParams& p, const Group& g, const void* what, uint32_t seen) {
  uint32_t* diag = reinterpret_cast<uint32_t*>(p.bases[g.rank] + kDiagOff);
  if (atomicCAS(diag, 0u, 1u) == 0u) {
    diag[1] = (uint32_t)(((const char*)what - p.bases[g.rank]) / 4);
    diag[2] = seen;
    diag[3] = p.epoch;
    diag[4] = (uint32_t)p.channel;
    diag[5] = (uint32_t)((g.size << 8) | g.stride);
  }
  atomicExch(reinterpret_cast<uint32_t*>(p.bases[g.rank] + kErrOff), (uint32_t)FSDP_E_TIMEOUT);
  for (int r = 0; r < FSDP_MAX_RANKS; ++r)
    if (p.bases[r] != nullptr && r != g.rank)
      st_release_sys(reinterpret_cast<uint32_t*>(p.bases[r] + kErrOff), (uint32_t)FSDP_E_TIMEOUT);
  __threadfence_system();
}

// This rank's communicator has failed (own error word set, locally or by a
// peer's abort): data kernels then skip every peer load and store.
__device__ __forceinline__ bool comm_failed(const CollParams& p, const Group& g) {
  return *reinterpret_cast<volatile const uint32_t*>(p.bases[g.rank] + kErrOff) != 0u;
}
// Same, one read per CTA so every thread of the CTA takes the same branch
// (must be called by all threads; contains __syncthreads).
__device__ __forceinline__ bool cta_failed(const CollParams& p, const Group& g) {
  __shared__ int failed;
  __syncthreads();
  if (threadIdx.x == 0) failed = comm_failed(p, g) ? 1 : 0;
  __syncthreads();
  return failed != 0;
}

// CTA-level barrier with the matching CTA of every group member.  `release`
// fences this CTA's prior peer stores (data phases).
__device__ __noinline__ void cta_barrier(const CollParams& p, const Group& g, int phase,
                                         bool release) {
  __syncthreads();
  const int j = threadIdx.x;
  if (j < g.size) {
    const int peer = g.member(j);
    if (release) __threadfence_system();
    st_release_sys(flag_ptr(p.bases[peer], p.channel, phase, g.rank, blockIdx.x), p.epoch);
    const uint32_t* mine = flag_ptr(p.bases[g.rank], p.channel, phase, peer, blockIdx.x);
    uint32_t* err = reinterpret_cast<uint32_t*>(p.bases[g.rank] + kErrOff);
    const uint64_t t0 = globaltimer();
    uint32_t spins = 0;
    while ((int32_t)(ld_acquire_sys(mine) - p.epoch) < 0) {
      if ((++spins & 1023u) == 0) {
        if (*(volatile uint32_t*)err != 0) break;           // already failed: bail out
        if (globaltimer() - t0 > (uint64_t)p.timeout_ns) {
          comm_abort(p, g, mine, ld_acquire_sys(mine));
          break;
        }
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
}

// ------------------------------------------------- vector memory helpers ----
// Non-volatile loads/stores so the compiler can keep kU independent 16-byte
// requests in flight per thread (a dependent load->use->load chain caps a
// thread at one outstanding request).
template <typename T> __device__ __forceinline__ Packed8<T> ldg8(const T* p);
template <> __device__ __forceinline__ Packed8<float> ldg8<float>(const float* p) {
  return {__ldg(reinterpret_cast<const uint4*>(p)), __ldg(reinterpret_cast<const uint4*>(p) + 1)};
}
template <> __device__ __forceinline__ Packed8<__nv_bfloat16> ldg8<__nv_bfloat16>(const __nv_bfloat16* p) {
  return {__ldg(reinterpret_cast<const uint4*>(p))};
}
// L2-coherent (peer-written during this kernel)
template <typename T> __device__ __forceinline__ Packed8<T> ldcg8(const T* p);
template <> __device__ __forceinline__ Packed8<float> ldcg8<float>(const float* p) {
  return {__ldcg(reinterpret_cast<const uint4*>(p)), __ldcg(reinterpret_cast<const uint4*>(p) + 1)};
}
template <> __device__ __forceinline__ Packed8<__nv_bfloat16> ldcg8<__nv_bfloat16>(const __nv_bfloat16* p) {
  return {__ldcg(reinterpret_cast<const uint4*>(p))};
}
template <typename T> __device__ __forceinline__ void st8(T* p, const Packed8<T>& v);
template <> __device__ __forceinline__ void st8<float>(float* p, const Packed8<float>& v) {
  reinterpret_cast<uint4*>(p)[0] = v.a;
  reinterpret_cast<uint4*>(p)[1] = v.b;
}
template <> __device__ __forceinline__ void st8<__nv_bfloat16>(__nv_bfloat16* p, const Packed8<__nv_bfloat16>& v) {
  reinterpret_cast<uint4*>(p)[0] = v.a;
}
template <typename Tin, typename Tout>
__device__ __forceinline__ Packed8<Tout> convert8(const Packed8<Tin>& r) {
  if constexpr (std::is_same<Tin, Tout>::value) return r;
  else return pack8<Tout>(unpack8<Tin>(r));
}

// index of the u-th vector of this thread inside tile t
__device__ __forceinline__ int64_t vec_index(int64_t t, int u) {
  return t * kTileElems + ((int64_t)u * kCommThreads + threadIdx.x) * kVec;
}

// Bounded spin on one flag (timeout -> device error word, never a hang).
__device__ __forceinline__ void wait_flag(const CollParams& p, const Group& g, const uint32_t* f) {
  uint32_t* err = reinterpret_cast<uint32_t*>(p.bases[g.rank] + kErrOff);
  const uint64_t t0 = globaltimer();
  uint32_t spins = 0;
  while ((int32_t)(ld_acquire_sys(f) - p.epoch) < 0) {
    if ((++spins & 1023u) == 0) {
      if (*(volatile uint32_t*)err != 0) break;
      if (globaltimer() - t0 > (uint64_t)p.timeout_ns) {
        comm_abort(p, g, f, ld_acquire_sys(f));
        break;
      }
    }
    __nanosleep(128);
  }
}

// Data kernels in split mode: signal this CTA's completion, never wait.
__device__ __forceinline__ void cta_signal(const CollParams& p, const Group& g, int phase,
                                           bool release) {
  __syncthreads();
  if ((int)threadIdx.x < g.size) {
    if (release) __threadfence_system();
    st_release_sys(flag_ptr(p.bases[g.member(threadIdx.x)], p.channel, phase, g.rank, blockIdx.x),
                   p.epoch);
  }
}

// Whole-collective enter barrier: one CTA per rank, one flag per peer.  Only
// this CTA spins while a late peer catches up; the data kernel behind it in
// stream order never occupies SMs waiting.
__global__ void __launch_bounds__(32) coll_enter_kernel(const __grid_constant__ CollParams p) {
  const Group g = make_group(p);
  if ((int)threadIdx.x < g.size) {
    const int peer = g.member(threadIdx.x);
    st_release_sys(flag_ptr(p.bases[peer], p.channel, 0, g.rank, kEnterSlot), p.epoch);
    wait_flag(p, g, flag_ptr(p.bases[g.rank], p.channel, 0, peer, kEnterSlot));
  }
}

// Exit barrier: wait for every (member, data-CTA) completion flag.
__global__ void __launch_bounds__(256) coll_exit_kernel(const __grid_constant__ CollParams p) {
  const Group g = make_group(p);
  for (int t = threadIdx.x; t < g.size * p.data_ctas; t += blockDim.x) {
    const int peer = g.member(t / p.data_ctas);
    wait_flag(p, g, flag_ptr(p.bases[g.rank], p.channel, 1, peer, t % p.data_ctas));
  }
}

// Copy-engine path: after the data has been moved by DMA (cudaMemcpyAsync,
// ordered before this kernel on the stream), publish "my part is done" to
// every member with one system-scope release per peer (phase 1, slot 0).
__global__ void __launch_bounds__(32) coll_signal_kernel(const __grid_constant__ CollParams p) {
  const Group g = make_group(p);
  if ((int)threadIdx.x < g.size) {
    __threadfence_system();
    st_release_sys(flag_ptr(p.bases[g.member(threadIdx.x)], p.channel, 1, g.rank, 0), p.epoch);
  }
}

// Copy-engine path, fused signal + exit barrier (one launch instead of two):
// publish "my DMA is done" to every member, then wait for every member's.
__global__ void __launch_bounds__(32) coll_signal_exit_kernel(const __grid_constant__ CollParams p) {
  const Group g = make_group(p);
  if ((int)threadIdx.x < g.size) {
    const int peer = g.member(threadIdx.x);
    __threadfence_system();
    st_release_sys(flag_ptr(p.bases[peer], p.channel, 1, g.rank, 0), p.epoch);
    wait_flag(p, g, flag_ptr(p.bases[g.rank], p.channel, 1, peer, 0));
  }
}

// Pipelined copy-engine push: after piece q's DMA writes into every member's
// staging (stream order on the copy side stream), publish "piece q landed"
// (phase 1, slot q) to every member; the receiving stream waits for slot q
// from every member before reducing piece q.
__global__ void __launch_bounds__(32) coll_signal_slot_kernel(const __grid_constant__ CollParams p, int slot,
                                                              int phase = 1) {
  const Group g = make_group(p);
  if ((int)threadIdx.x < g.size) {
    __threadfence_system();
    st_release_sys(flag_ptr(p.bases[g.member(threadIdx.x)], p.channel, phase, g.rank, slot), p.epoch);
  }
}
__global__ void __launch_bounds__(32) coll_wait_slot_kernel(const __grid_constant__ CollParams p, int slot,
                                                            int phase = 1) {
  const Group g = make_group(p);
  if ((int)threadIdx.x < g.size)
    wait_flag(p, g, flag_ptr(p.bases[g.rank], p.channel, phase, g.member(threadIdx.x), slot));
}

// Local reduction of a copy-engine reduce-scatter, one piece [e0, e0+len)
// of the member's chunk: member chunks j != pos sit in local staging
// (stage + j*stride), the own chunk in the own payload buffer; ascending-rank
// fp32 sum from +0, / postdiv, += out.
struct CeReduceArgs {
  const void* own;        // own payload, chunk pos (element 0 of the chunk)
  const void* stage;      // staging base (slot 0, element 0)
  int64_t stride;         // elements between staging slots (= chunk length n)
  void* out;              // output chunk (element 0): fp32, or bf16 when out_bf16
  int64_t e0, len;        // this piece
  int gsize, pos;
  float prediv, postdiv;
  int accumulate;
  int store_raw;          // 1: out = sum/postdiv as is (all-reduce owner phase), else (acc ? out : 0) + that
  int out_bf16;           // 1: the fp32 result is rounded to bf16 (hybrid stage-1 partial; no accumulate)
};

// Tout = bf16: the reduce-scatter result is the next stage's payload
// (hybrid stage 2 in the reduce dtype); the fp32 value is rounded once.
template <typename Tin, typename Tout, int MAXW>
__global__ void __launch_bounds__(256)
ce_reduce_kernel(const __grid_constant__ CeReduceArgs a) {
  constexpr int U = 2;                                 // vectors per thread per iteration
  const Tin* own = (const Tin*)a.own + a.e0;
  const Tin* stage = (const Tin*)a.stage + a.e0;
  Tout* __restrict__ out = (Tout*)a.out + a.e0;
  const int64_t n = a.len;
  const bool pre = a.prediv != 1.0f, post = a.postdiv != 1.0f;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const bool vec = (n % kVec == 0) && aligned16(own) && aligned16(stage) && aligned16(out) &&
                   ((a.stride * (int64_t)sizeof(Tin)) % 16 == 0);
  if (vec) {
    const Tin* src[MAXW];
#pragma unroll
    for (int j = 0; j < MAXW; ++j) src[j] = j == a.pos ? own : stage + (int64_t)j * a.stride;
    const int64_t nv = n / kVec;
    for (int64_t v0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v0 < nv; v0 += U * nthr) {
      Packed8<Tin> r[U][MAXW];
#pragma unroll
      for (int u = 0; u < U; ++u)                      // every load in flight before any add
#pragma unroll
        for (int j = 0; j < MAXW; ++j)
          if (j < a.gsize && v0 + u * nthr < nv) r[u][j] = ldg8<Tin>(src[j] + (v0 + u * nthr) * kVec);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t v = v0 + u * nthr;
        if (v >= nv) continue;
        V8F acc;
#pragma unroll
        for (int q = 0; q < 8; ++q) acc.v[q] = 0.0f;
#pragma unroll
        for (int j = 0; j < MAXW; ++j) {
          if (j >= a.gsize) break;
          const V8F x = unpack8<Tin>(r[u][j]);
#pragma unroll
          for (int q = 0; q < 8; ++q) acc.v[q] = __fadd_rn(acc.v[q], pre ? __fdiv_rn(x.v[q], a.prediv) : x.v[q]);
        }
        V8F base;
        if (a.accumulate) base = unpack8<Tout>(ldcg8<Tout>(out + v * kVec));
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float rr = post ? __fdiv_rn(acc.v[q], a.postdiv) : acc.v[q];
          acc.v[q] = a.store_raw ? rr : __fadd_rn(a.accumulate ? base.v[q] : 0.0f, rr);
        }
        st8<Tout>(out + v * kVec, pack8<Tout>(acc));
      }
    }
  } else {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += nthr) {
      float acc = 0.0f;
      for (int j = 0; j < a.gsize; ++j) {
        const float x = to_f<Tin>(j == a.pos ? own[i] : stage[(int64_t)j * a.stride + i]);
        acc = __fadd_rn(acc, pre ? __fdiv_rn(x, a.prediv) : x);
      }
      const float r = post ? __fdiv_rn(acc, a.postdiv) : acc;
      out[i] = from_f<Tout>(a.store_raw ? r : __fadd_rn(a.accumulate ? to_f<Tout>(out[i]) : 0.0f, r));
    }
  }
}

// All-reduce epilogue (copy-engine path): out = (accumulate ? out : 0) + gathered.
__global__ void __launch_bounds__(256)
ar_epilogue_kernel(const float* __restrict__ gath, float* __restrict__ out, int64_t n, int accumulate) {
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (aligned16(gath) && aligned16(out)) {
    const int64_t n4 = n / 4;
    for (int64_t i = t; i < n4; i += nthr) {
      const float4 x = __ldcg(reinterpret_cast<const float4*>(gath) + i);
      float4 b = accumulate ? reinterpret_cast<const float4*>(out)[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      b.x = __fadd_rn(b.x, x.x); b.y = __fadd_rn(b.y, x.y); b.z = __fadd_rn(b.z, x.z); b.w = __fadd_rn(b.w, x.w);
      reinterpret_cast<float4*>(out)[i] = b;
    }
    for (int64_t i = n4 * 4 + t; i < n; i += nthr) out[i] = __fadd_rn(accumulate ? out[i] : 0.0f, __ldcg(gath + i));
  } else {
    for (int64_t i = t; i < n; i += nthr) out[i] = __fadd_rn(accumulate ? out[i] : 0.0f, __ldcg(gath + i));
  }
}

// ------------------------------------------------------------ all-gather ----
template <typename Tin, typename Tout>
__global__ void __launch_bounds__(kCommThreads)
allgather_kernel(const __grid_constant__ CollParams p) {
  const Group g = make_group(p);
  const int e = p.rank0 >= 0 ? 0 : blockIdx.y;
  const Tin* __restrict__ src = (const Tin*)p.in[e];
  const int64_t n = p.n;
  const int64_t my_off = p.off_a + (int64_t)g.pos * n * (int64_t)sizeof(Tout);
  if (!p.split) cta_barrier(p, g, 0, false);   // every member's destination slot is free
  const bool aborted = cta_failed(p, g);       // no peer stores after a timeout

  const bool vec = (n % kVec == 0) && aligned16(src) && (my_off % 16 == 0);
  const int64_t ntiles = aborted ? 0 : (n + kTileElems - 1) / kTileElems;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if (vec) {
      Packed8<Tout> o[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t i = vec_index(t, u);
        if (i < n) o[u] = convert8<Tin, Tout>(ldg8<Tin>(src + i));
      }
      for (int jj = 0; jj < g.size; ++jj) {
        const int j = (g.pos + 1 + jj) % g.size;     // stagger destinations
        Tout* d = (Tout*)(p.bases[g.member(j)] + my_off);
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int64_t i = vec_index(t, u);
          if (i < n) st8<Tout>(d + i, o[u]);
        }
      }
    } else {
      const int64_t t0 = t * kTileElems, t1 = min(t0 + (int64_t)kTileElems, n);
      for (int64_t i = t0 + threadIdx.x; i < t1; i += kCommThreads) {
        const Tout v = from_f<Tout>(to_f<Tin>(src[i]));
        for (int jj = 0; jj < g.size; ++jj) {
          const int j = (g.pos + 1 + jj) % g.size;
          ((Tout*)(p.bases[g.member(j)] + my_off))[i] = v;
        }
      }
    }
  }
  if (p.split) cta_signal(p, g, 1, true);     // my pieces have landed everywhere
  else cta_barrier(p, g, 1, true);            // all members' pieces have landed here
}

// ------------------------------------------------- all-gather (NVLS) -----
// NVLink SHARP multicast: the pool of every member of the shard group is
// bound to one multicast object, so ONE multimem.st from the member at
// position k writes its (cast) shard into every member's unsharded buffer at
// dst_off + k*n: egress per GPU is the shard once (S/W) instead of W-1 copies,
// and each vector costs one store instruction instead of W.  Bit-exact (pure
// copy + RNE cast).  Split mode only: enter barrier (slots free everywhere),
// this signal-only kernel, exit barrier (every member's stores landed).
__device__ __forceinline__ void multimem_st16(void* p, const uint4& v) {
  asm volatile("multimem.st.global.v4.f32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
template <typename T> __device__ __forceinline__ void mc_st8(T* p, const Packed8<T>& v);
template <> __device__ __forceinline__ void mc_st8<float>(float* p, const Packed8<float>& v) {
  multimem_st16(p, v.a);
  multimem_st16(p + 4, v.b);
}
template <> __device__ __forceinline__ void mc_st8<__nv_bfloat16>(__nv_bfloat16* p,
                                                                  const Packed8<__nv_bfloat16>& v) {
  multimem_st16(p, v.a);
}

template <typename Tin, typename Tout>
__global__ void __launch_bounds__(kCommThreads)
allgather_nvls_kernel(const __grid_constant__ CollParams p) {
  const Group g = make_group(p);
  const Tin* __restrict__ src = (const Tin*)p.in[0];
  const int64_t n = p.n;
  Tout* dst = (Tout*)(p.mc_base + p.off_a + (int64_t)g.pos * n * (int64_t)sizeof(Tout));
  const int64_t ntiles = cta_failed(p, g) ? 0 : (n + kTileElems - 1) / kTileElems;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    Packed8<Tout> o[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = vec_index(t, u);
      if (i < n) o[u] = convert8<Tin, Tout>(ldg8<Tin>(src + i));
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = vec_index(t, u);
      if (i < n) mc_st8<Tout>(dst + i, o[u]);
    }
  }
  __threadfence_system();          // each thread orders its own multicast stores
  cta_signal(p, g, 1, true);       // ... before this CTA's completion flags
}

// -------------------------------------------------------- reduce-scatter ----
template <typename Tin>
__global__ void __launch_bounds__(kCommThreads)
reduce_scatter_kernel(const __grid_constant__ CollParams p) {
  const Group g = make_group(p);
  const int e = p.rank0 >= 0 ? 0 : blockIdx.y;
  const Tin* __restrict__ flat = (const Tin*)p.in[e];
  float* __restrict__ out = p.out[e];
  const int64_t n = p.n;
  const int64_t slot_bytes = n * (int64_t)sizeof(Tin);
  cta_barrier(p, g, 0, false);   // every member's staging is free

  const bool vec = (n % kVec == 0) && aligned16(flat) && (p.off_a % 16 == 0) && aligned16(out);
  const int64_t ntiles = cta_failed(p, g) ? 0 : (n + kTileElems - 1) / kTileElems;
  // phase 1: chunk j of my flat payload -> member j's staging slot [my pos]
  // (my own chunk stays in place and is read directly in phase 2)
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    for (int jj = 1; jj < g.size; ++jj) {
      const int j = (g.pos + jj) % g.size;
      Tin* dst = (Tin*)(p.bases[g.member(j)] + p.off_a + (int64_t)g.pos * slot_bytes);
      const Tin* s = flat + (int64_t)rs_chunk(p, j, g.size) * n;
      if (vec) {
        Packed8<Tin> r[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int64_t i = vec_index(t, u);
          if (i < n) r[u] = ldg8<Tin>(s + i);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int64_t i = vec_index(t, u);
          if (i < n) st8<Tin>(dst + i, r[u]);
        }
      } else {
        const int64_t t0 = t * kTileElems, t1 = min(t0 + (int64_t)kTileElems, n);
        for (int64_t i = t0 + threadIdx.x; i < t1; i += kCommThreads) dst[i] = s[i];
      }
    }
  }
  cta_barrier(p, g, 1, true);    // my tiles of every member's chunk arrived
  if (cta_failed(p, g)) return;  // staging incomplete: leave out untouched
  // phase 2: ascending-rank fp32 sum of the group's chunks, post-divide, accumulate
  const Tin* stage = (const Tin*)(p.bases[g.rank] + p.off_a);
  const Tin* mine = flat + (int64_t)rs_chunk(p, g.pos, g.size) * n;
  const bool pre = p.prediv != 1.0f, post = p.postdiv != 1.0f;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if (vec) {
      V8F acc[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u)
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[u].v[k] = 0.0f;
      for (int j = 0; j < g.size; ++j) {
        Packed8<Tin> r[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int64_t i = vec_index(t, u);
          if (i < n) r[u] = (j == g.pos) ? ldg8<Tin>(mine + i) : ldcg8<Tin>(stage + (int64_t)j * n + i);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const V8F x = unpack8<Tin>(r[u]);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            acc[u].v[k] = __fadd_rn(acc[u].v[k], pre ? __fdiv_rn(x.v[k], p.prediv) : x.v[k]);
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t i = vec_index(t, u);
        if (i >= n) continue;
        V8F base;
        if (p.accumulate) base = unpack8<float>(ldcg8<float>(out + i));
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float r = post ? __fdiv_rn(acc[u].v[k], p.postdiv) : acc[u].v[k];
          acc[u].v[k] = __fadd_rn(p.accumulate ? base.v[k] : 0.0f, r);
        }
        st8<float>(out + i, pack8<float>(acc[u]));
      }
    } else {
      const int64_t t0 = t * kTileElems, t1 = min(t0 + (int64_t)kTileElems, n);
      for (int64_t i = t0 + threadIdx.x; i < t1; i += kCommThreads) {
        float acc = 0.0f;
        for (int j = 0; j < g.size; ++j) {
          const float x = to_f<Tin>(j == g.pos ? mine[i] : ldcg_elem(stage + (int64_t)j * n + i));
          acc = __fadd_rn(acc, pre ? __fdiv_rn(x, p.prediv) : x);
        }
        const float r = post ? __fdiv_rn(acc, p.postdiv) : acc;
        out[i] = __fadd_rn(p.accumulate ? out[i] : 0.0f, r);
      }
    }
  }
}

// --------------------------------------------------- reduce-scatter (pull) --
// Member at position k reads chunk k of every member's symmetric flat buffer
// (pool offset off_a) over NVLink in ascending rank order and sums in fp32
// registers: no staging round trip, no mid-kernel phase barrier.  Loads of
// all MAXW members x U vectors are issued before the adds (MLP ~16 x 16 B per
// thread), masked to the runtime group size.  Entry barrier: every member's
// buffer is written; exit barrier: every member finished reading mine.
template <typename Tin, int MAXW>
__global__ void __launch_bounds__(kCommThreads)
reduce_scatter_pull_kernel(const __grid_constant__ CollParams p) {
  constexpr int U = (16 / MAXW) / (int)(sizeof(Tin) / 2) > 0 ? (16 / MAXW) / (int)(sizeof(Tin) / 2) : 1;
  constexpr int64_t TILE = (int64_t)kCommThreads * kVec * U;
  const Group g = make_group(p);
  const int e = p.rank0 >= 0 ? 0 : blockIdx.y;
  float* __restrict__ out = p.out[e];
  const int64_t n = p.n;
  // off_b > 0: the members' chunks are off_b elements apart (a sub-range of each chunk)
  const int64_t chunk_off = p.off_a + (int64_t)rs_chunk(p, g.pos, g.size) * (p.off_b > 0 ? p.off_b : n) * (int64_t)sizeof(Tin);
  const Tin* src[MAXW];
#pragma unroll
  for (int j = 0; j < MAXW; ++j)
    src[j] = j < g.size ? (const Tin*)(p.bases[g.member(j)] + chunk_off) : nullptr;
  if (!p.split) cta_barrier(p, g, 0, false);   // every member's payload is in place
  const bool vec = (n % kVec == 0) && (chunk_off % 16 == 0) && aligned16(out);
  const bool pre = p.prediv != 1.0f, post = p.postdiv != 1.0f;
  const int64_t ntiles = cta_failed(p, g) ? 0 : (n + TILE - 1) / TILE;   // no peer loads after a timeout
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if (vec) {
      Packed8<Tin> r[MAXW][U];
#pragma unroll
      for (int j = 0; j < MAXW; ++j)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t i = t * TILE + ((int64_t)u * kCommThreads + threadIdx.x) * kVec;
          if (j < g.size && i < n) r[j][u] = ldcg8<Tin>(src[j] + i);
        }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = t * TILE + ((int64_t)u * kCommThreads + threadIdx.x) * kVec;
        if (i >= n) continue;
        V8F acc;
#pragma unroll
        for (int k = 0; k < 8; ++k) acc.v[k] = 0.0f;
#pragma unroll
        for (int j = 0; j < MAXW; ++j) {
          if (j >= g.size) break;
          const V8F x = unpack8<Tin>(r[j][u]);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            acc.v[k] = __fadd_rn(acc.v[k], pre ? __fdiv_rn(x.v[k], p.prediv) : x.v[k]);
        }
        V8F base;
        if (p.accumulate) base = unpack8<float>(ldcg8<float>(out + i));
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float rr = post ? __fdiv_rn(acc.v[k], p.postdiv) : acc.v[k];
          acc.v[k] = __fadd_rn(p.accumulate ? base.v[k] : 0.0f, rr);
        }
        st8<float>(out + i, pack8<float>(acc));
      }
    } else {
      const int64_t t0 = t * TILE, t1 = min(t0 + TILE, n);
      for (int64_t i = t0 + threadIdx.x; i < t1; i += kCommThreads) {
        float acc = 0.0f;
        for (int j = 0; j < g.size; ++j) {
          const float x = to_f<Tin>(ldcg_elem(src[j] + i));
          acc = __fadd_rn(acc, pre ? __fdiv_rn(x, p.prediv) : x);
        }
        const float rr = post ? __fdiv_rn(acc, p.postdiv) : acc;
        out[i] = __fadd_rn(p.accumulate ? out[i] : 0.0f, rr);
      }
    }
  }
  if (p.split) cta_signal(p, g, 1, false);   // I am done reading my tiles of everyone
  else cta_barrier(p, g, 1, false);          // every member is done reading my buffer
}

// ------------------------------------------- reduce-scatter (TMA pull) -----
// Same contract as reduce_scatter_pull_kernel, but the NVLink reads are 1-D
// TMA bulk copies (cp.async.bulk -> UBLKCP) issued by one thread into a
// kStages-deep shared-memory ring, completion tracked by mbarrier
// transaction counts: the bytes in flight are no longer bounded by the SM's
// load queue, so a handful of CTAs saturates the link.  Every stage holds one
// tile of each member's chunk; all threads reduce a landed stage in
// ascending rank order (fp32, from +0) while later stages are in flight.
constexpr int kTmaThreads = 256;
constexpr int kTmaStages = 4;                // default ring: 4 stages x 32 KB
constexpr int kTmaStageBytes = 32 * 1024;   // summed over the group's members

template <typename Tin, int STAGES, int STAGE_BYTES>
__global__ void __launch_bounds__(kTmaThreads, 1)
reduce_scatter_tma_kernel(const __grid_constant__ CollParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[STAGES];
  const Group g = make_group(p);
  const int e = p.rank0 >= 0 ? 0 : blockIdx.y;
  float* __restrict__ out = p.out[e];
  const int64_t n = p.n;
  const int W = g.size;
  // elements per member tile: a multiple of 8 (16-byte bulk-copy granule)
  const int64_t T = (STAGE_BYTES / (W * (int)sizeof(Tin))) / kVec * kVec;
  // off_b > 0: the members' chunks are off_b elements apart (a sub-range of each chunk)
  const int64_t chunk_off = p.off_a + (int64_t)rs_chunk(p, g.pos, g.size) * (p.off_b > 0 ? p.off_b : n) * (int64_t)sizeof(Tin);
  const int64_t ntiles = (n + T - 1) / T;
  const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  cta_barrier(p, g, 0, false);   // every member's payload is in place (+ mbarrier init visible)
  if (cta_failed(p, g)) {        // no peer loads after a timeout
    cta_barrier(p, g, 1, false);
    return;
  }

  auto issue = [&](int64_t k) {   // tile iteration k -> stage k % STAGES
    const int s = (int)(k % STAGES);
    const int64_t t = blockIdx.x + k * gridDim.x;
    const int64_t i0 = t * T;
    const uint32_t bytes = (uint32_t)((min(T, n - i0)) * (int64_t)sizeof(Tin));
    mbar_expect_tx(&full[s], bytes * W);
    for (int j = 0; j < W; ++j) {
      const Tin* src = (const Tin*)(p.bases[g.member(j)] + chunk_off) + i0;
      tma_load_1d(smem + (size_t)s * STAGE_BYTES + (size_t)j * T * sizeof(Tin), src, bytes, &full[s]);
    }
  };
  if (threadIdx.x == 0)
    for (int64_t k = 0; k < my_tiles && k < STAGES; ++k) issue(k);

  const bool pre = p.prediv != 1.0f, post = p.postdiv != 1.0f;
  for (int64_t k = 0; k < my_tiles; ++k) {
    const int s = (int)(k % STAGES);
    mbar_wait(&full[s], (uint32_t)((k / STAGES) & 1));
    const int64_t i0 = (blockIdx.x + k * gridDim.x) * T;
    const int64_t len = min(T, n - i0);
    const Tin* st = (const Tin*)(smem + (size_t)s * STAGE_BYTES);
    for (int64_t v = threadIdx.x; v * kVec < len; v += kTmaThreads) {
      V8F acc;
#pragma unroll
      for (int q = 0; q < 8; ++q) acc.v[q] = 0.0f;
      for (int j = 0; j < W; ++j) {
        Packed8<Tin> r;
        if constexpr (sizeof(Tin) == 2) {
          r.a = *reinterpret_cast<const uint4*>(st + (size_t)j * T + v * kVec);
        } else {
          r.a = *reinterpret_cast<const uint4*>(st + (size_t)j * T + v * kVec);
          r.b = *(reinterpret_cast<const uint4*>(st + (size_t)j * T + v * kVec) + 1);
        }
        const V8F x = unpack8<Tin>(r);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          acc.v[q] = __fadd_rn(acc.v[q], pre ? __fdiv_rn(x.v[q], p.prediv) : x.v[q]);
      }
      float* o = out + i0 + v * kVec;
      V8F base;
      if (p.accumulate) base = unpack8<float>(ldcg8<float>(o));
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float rr = post ? __fdiv_rn(acc.v[q], p.postdiv) : acc.v[q];
        acc.v[q] = __fadd_rn(p.accumulate ? base.v[q] : 0.0f, rr);
      }
      st8<float>(o, pack8<float>(acc));
    }
    __syncthreads();   // stage s fully consumed
    if (threadIdx.x == 0 && k + STAGES < my_tiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(k + STAGES);
    }
  }
  cta_barrier(p, g, 1, false);   // every member is done reading my buffer
}

// ------------------------------------------------------------ all-reduce ----
// Two-shot: RS-push to chunk owners, ascending fp32 sum, AG-push of results.
// Chunk stride c is a multiple of 8; the last chunk may be short (tail
// elements take the scalar path).
template <typename Tin>
__global__ void __launch_bounds__(kCommThreads)
allreduce_kernel(const __grid_constant__ CollParams p) {
  const Group g = make_group(p);
  const int e = p.rank0 >= 0 ? 0 : blockIdx.y;
  const Tin* __restrict__ in = (const Tin*)p.in[e];
  float* __restrict__ out = p.out[e];
  const int64_t n = p.n;
  int64_t c = (n + g.size - 1) / g.size;
  c = (c + kVec - 1) / kVec * kVec;                       // chunk stride (elements)
  auto clen = [&](int j) -> int64_t {
    const int64_t s = (int64_t)j * c;
    return s >= n ? 0 : min(c, n - s);
  };
  const bool vec = aligned16(in) && aligned16(out) && (p.off_a % 16 == 0) && (p.off_b % 16 == 0);
  cta_barrier(p, g, 0, false);

  const int64_t ntiles = cta_failed(p, g) ? 0 : (c + kTileElems - 1) / kTileElems;
  // phase A: my chunk j -> member j's stage slot [my pos] (own chunk stays)
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    for (int jj = 1; jj < g.size; ++jj) {
      const int j = (g.pos + jj) % g.size;
      const int64_t len = clen(j);
      Tin* dst = (Tin*)(p.bases[g.member(j)] + p.off_a) + (int64_t)g.pos * c;
      const Tin* s = in + (int64_t)j * c;
      Packed8<Tin> r[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t i = vec_index(t, u);
        if (vec && i + kVec <= len) r[u] = ldg8<Tin>(s + i);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t i = vec_index(t, u);
        if (vec && i + kVec <= len) st8<Tin>(dst + i, r[u]);
        else for (int64_t k = i; k < min(i + kVec, len); ++k) dst[k] = s[k];
      }
    }
  }
  cta_barrier(p, g, 1, true);
  // phase B: reduce my chunk (ascending), push fp32 result to every member
  if (!cta_failed(p, g)) {
    const Tin* stage = (const Tin*)(p.bases[g.rank] + p.off_a);
    const Tin* mine = in + (int64_t)g.pos * c;
    const int64_t len = clen(g.pos);
    const bool post = p.postdiv != 1.0f;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      V8F acc[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u)
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[u].v[k] = 0.0f;
      for (int j = 0; j < g.size; ++j) {
        const Tin* s = (j == g.pos) ? mine : stage + (int64_t)j * c;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int64_t i = vec_index(t, u);
          if (vec && i + kVec <= len) {
            const V8F x = unpack8<Tin>(j == g.pos ? ldg8<Tin>(s + i) : ldcg8<Tin>(s + i));
#pragma unroll
            for (int k = 0; k < 8; ++k) acc[u].v[k] = __fadd_rn(acc[u].v[k], x.v[k]);
          } else {
            for (int k = 0; k < 8 && i + k < len; ++k)
              acc[u].v[k] = __fadd_rn(acc[u].v[k], to_f<Tin>(j == g.pos ? s[i + k] : ldcg_elem(s + i + k)));
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t i = vec_index(t, u);
        if (i >= len) continue;
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[u].v[k] = post ? __fdiv_rn(acc[u].v[k], p.postdiv) : acc[u].v[k];
        const Packed8<float> pk = pack8<float>(acc[u]);
        for (int jj = 0; jj < g.size; ++jj) {
          const int j = (g.pos + 1 + jj) % g.size;
          float* d = (float*)(p.bases[g.member(j)] + p.off_b) + (int64_t)g.pos * c;
          if (vec && i + kVec <= len) st8<float>(d + i, pk);
          else for (int k = 0; k < 8 && i + k < len; ++k) d[i + k] = acc[u].v[k];
        }
      }
    }
  }
  cta_barrier(p, g, 2, true);
  if (cta_failed(p, g)) return;
  // phase C: out = (accumulate ? out : 0) + gathered, for my tiles of every chunk
  const float* gath = (const float*)(p.bases[g.rank] + p.off_b);
  for (int j = 0; j < g.size; ++j) {
    const int64_t len = clen(j);
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t i = vec_index(t, u);
        const int64_t k0 = (int64_t)j * c + i;
        if (vec && i + kVec <= len) {
          V8F x = unpack8<float>(ldcg8<float>(gath + k0));
          V8F b;
          if (p.accumulate) b = unpack8<float>(ldcg8<float>(out + k0));
#pragma unroll
          for (int k = 0; k < 8; ++k) x.v[k] = __fadd_rn(p.accumulate ? b.v[k] : 0.0f, x.v[k]);
          st8<float>(out + k0, pack8<float>(x));
        } else {
          for (int k = 0; k < 8 && i + k < len; ++k)
            out[k0 + k] = __fadd_rn(p.accumulate ? out[k0 + k] : 0.0f, __ldcg(gath + k0 + k));
        }
      }
    }
  }
}

// 1-element world all-reduce of a float (found_inf verdict).
__global__ void __launch_bounds__(32) scalar_allreduce_kernel(const __grid_constant__ CollParams p) {
  const Group g = make_group(p);
  const int e = p.rank0 >= 0 ? 0 : blockIdx.y;
  cta_barrier(p, g, 0, false);
  if (cta_failed(p, g)) {        // verdict "skip" wherever the abort is seen
    if (threadIdx.x == 0) *p.out[e] = 1.0f;
    return;
  }
  if ((int)threadIdx.x < g.size) {
    const float v = *(const float*)p.in[e];
    ((float*)(p.bases[g.member(threadIdx.x)] + kScalarOff))[g.rank] = v;
  }
  cta_barrier(p, g, 1, true);
  if (threadIdx.x == 0) {
    const float* s = (const float*)(p.bases[g.rank] + kScalarOff);
    float acc = 0.0f;
    for (int j = 0; j < g.size; ++j) acc = __fadd_rn(acc, __ldcg(s + g.member(j)));
    *p.out[e] = acc;
  }
}

// ------------------------------------------------ low-latency (LL) path ----
// One-shot protocol for small collectives: ONE kernel, no enter/exit barrier.
// Every 16-byte line {d0, flag, d1, flag} carries 8 payload bytes; each
// 8-byte half {data, flag} is stored and loaded atomically, so a receiver
// that reads flag == epoch in both halves holds that line's data.  Lines
// land in a per-(epoch parity, sender) region of the receiver's pool at
// off_b; the receiver unpacks them itself (cast, reduction, final layout).
// Double buffering by epoch parity needs no barrier: a sender running epoch e
// has received every member's epoch e-1 lines, so every member has started
// e-1 and (stream order) finished reading its epoch e-2 region.
// Wire bytes are 2x the payload: this path is for messages where the split
// path's three launches and two flag round trips dominate.
constexpr int kLLThreads = 512;
constexpr int kLLUnroll = 4;

__device__ __forceinline__ void st_ll(void* p, uint32_t d0, uint32_t d1, uint32_t f) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "r"(d0), "r"(f), "r"(d1), "r"(f) : "memory");
}
__device__ __forceinline__ uint4 ld_ll(const void* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ bool ll_ready(const uint4& v, uint32_t f) { return v.y == f && v.w == f; }

// Spin until line `p` carries epoch f (bounded: timeout -> device error word).
__device__ __noinline__ uint4 ll_wait(const CollParams& p, const Group& g, const char* line, uint4 v) {
  const uint32_t f = p.epoch;
  uint32_t* err = reinterpret_cast<uint32_t*>(p.bases[g.rank] + kErrOff);
  const uint64_t t0 = globaltimer();
  uint32_t spins = 0;
  while (!ll_ready(v, f)) {
    if ((++spins & 255u) == 0) {
      if (*(volatile uint32_t*)err != 0) break;
      if (globaltimer() - t0 > (uint64_t)p.timeout_ns) {
        comm_abort(p, g, line, v.y);
        break;
      }
    }
    v = ld_ll(line);
  }
  return v;
}

// Line L of a chunk of n elements, converted to Tout and packed into 8 bytes
// (8/sizeof(Tout) elements; zero beyond n).  Same dtype: a raw bit copy.
template <typename Tin, typename Tout>
__device__ __forceinline__ uint2 ll_load_line(const Tin* src, int64_t L, int64_t n) {
  constexpr int EPL = 8 / (int)sizeof(Tout);
  const int64_t e0 = L * EPL;
  uint2 d = make_uint2(0u, 0u);
  if constexpr (std::is_same<Tin, Tout>::value) {
    if (e0 + EPL <= n && (reinterpret_cast<uintptr_t>(src + e0) & 7) == 0) {
      d = __ldg(reinterpret_cast<const uint2*>(src + e0));
    } else {
      Tout tmp[EPL];
      unsigned char* b = reinterpret_cast<unsigned char*>(tmp);
      for (int q = 0; q < 8; ++q) b[q] = 0;
      for (int q = 0; q < EPL && e0 + q < n; ++q) tmp[q] = src[e0 + q];
      d.x = reinterpret_cast<uint32_t*>(tmp)[0];
      d.y = reinterpret_cast<uint32_t*>(tmp)[1];
    }
  } else if constexpr (sizeof(Tout) == 2) {   // fp32 -> bf16 (RNE), 4 elements
    float x[4] = {0.f, 0.f, 0.f, 0.f};
    if (e0 + 4 <= n && aligned16(src + e0)) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(src + e0));
      x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
    } else {
      for (int q = 0; q < 4 && e0 + q < n; ++q) x[q] = to_f<Tin>(src[e0 + q]);
    }
    d.x = pack_bf16x2(x[0], x[1]);
    d.y = pack_bf16x2(x[2], x[3]);
  } else {                                    // bf16 -> fp32, 2 elements
    float x[2] = {0.f, 0.f};
    for (int q = 0; q < 2 && e0 + q < n; ++q) x[q] = to_f<Tin>(src[e0 + q]);
    d.x = __float_as_uint(x[0]);
    d.y = __float_as_uint(x[1]);
  }
  return d;
}

// Store line L (packed T elements) into a chunk of n elements (skip beyond n).
template <typename T>
__device__ __forceinline__ void ll_store_line(T* dst, int64_t L, int64_t n, uint32_t d0, uint32_t d1) {
  constexpr int EPL = 8 / (int)sizeof(T);
  const int64_t e0 = L * EPL;
  if (e0 + EPL <= n && (reinterpret_cast<uintptr_t>(dst + e0) & 7) == 0) {
    *reinterpret_cast<uint2*>(dst + e0) = make_uint2(d0, d1);
  } else {
    uint32_t w[2] = {d0, d1};
    const T* t = reinterpret_cast<const T*>(w);
    for (int q = 0; q < EPL && e0 + q < n; ++q) dst[e0 + q] = t[q];
  }
}

// Address of line L from member `pos` in the LL region of the receiver whose
// pool base is `base`.  Lines go in blocks of kLLBlock (one warp's 512
// contiguous bytes per store instruction), blocks interleaved as
// [block][member][epoch parity]: a line's address depends on (L, pos,
// parity) only, never on the message length, so consecutive calls of
// different sizes on one channel can never overlap the other parity's lines
// (a length-dependent layout let a large epoch e+1 overwrite a small epoch
// e's lines before a slow receiver read them).
constexpr int kLLBlock = 32;
__device__ __forceinline__ char* ll_line(const CollParams& p, char* base, int pos, int64_t L) {
  const int64_t blk = L / kLLBlock;
  return base + p.off_b +
         ((((blk * p.gsize + pos) * 2 + (int64_t)(p.epoch & 1u)) * kLLBlock) + (L % kLLBlock)) * 16;
}

// All-gather: member k sends cast(shard) as LL lines to every other member,
// copies its own chunk locally, then unpacks every peer's lines into its own
// unsharded buffer at off_a + j*n (the same destination as fsdp_allgather).
template <typename Tin, typename Tout>
__global__ void __launch_bounds__(kLLThreads)
allgather_ll_kernel(const __grid_constant__ CollParams p) {
  constexpr int EPL = 8 / (int)sizeof(Tout);
  const Group g = make_group(p);
  const int e = p.rank0 >= 0 ? 0 : blockIdx.y;
  const Tin* __restrict__ src = (const Tin*)p.in[e];
  const int64_t n = p.n;
  const int64_t nl = (n + EPL - 1) / EPL;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  Tout* dst = (Tout*)(p.bases[g.rank] + p.off_a);
  if (comm_failed(p, g)) return;   // no peer stores after a timeout
  for (int64_t L = tid; L < nl; L += nt) {
    const uint2 d = ll_load_line<Tin, Tout>(src, L, n);
    for (int jj = 1; jj < g.size; ++jj) {
      const int j = (g.pos + jj) % g.size;   // stagger destinations
      st_ll(ll_line(p, p.bases[g.member(j)], g.pos, L), d.x, d.y, p.epoch);
    }
    ll_store_line<Tout>(dst + (int64_t)g.pos * n, L, n, d.x, d.y);
  }
  for (int jj = 1; jj < g.size; ++jj) {
    const int j = (g.pos + jj) % g.size;
    Tout* dj = dst + (int64_t)j * n;
    for (int64_t L0 = tid; L0 < nl; L0 += nt * kLLUnroll) {
      uint4 v[kLLUnroll];
#pragma unroll
      for (int u = 0; u < kLLUnroll; ++u) {
        const int64_t L = L0 + u * nt;
        if (L < nl) v[u] = ld_ll(ll_line(p, p.bases[g.rank], j, L));
      }
#pragma unroll
      for (int u = 0; u < kLLUnroll; ++u) {
        const int64_t L = L0 + u * nt;
        if (L >= nl) continue;
        if (!ll_ready(v[u], p.epoch)) v[u] = ll_wait(p, g, ll_line(p, p.bases[g.rank], j, L), v[u]);
        ll_store_line<Tout>(dj, L, n, v[u].x, v[u].z);
      }
    }
  }
}

// Reduce-scatter: member k sends chunk j of its payload as LL lines to member
// j; then, per line of its own chunk, sums the group's lines in ascending
// rank order in fp32 from +0 (own chunk read locally), / postdiv, += out.
template <typename Tin, int MAXW>
__global__ void __launch_bounds__(kLLThreads)
reduce_scatter_ll_kernel(const __grid_constant__ CollParams p) {
  constexpr int EPL = 8 / (int)sizeof(Tin);
  const Group g = make_group(p);
  const int e = p.rank0 >= 0 ? 0 : blockIdx.y;
  const Tin* __restrict__ flat = (const Tin*)p.in[e];
  float* __restrict__ out = p.out[e];
  const int64_t n = p.n;
  const int64_t nl = (n + EPL - 1) / EPL;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (comm_failed(p, g)) return;   // no peer stores after a timeout
  for (int64_t L = tid; L < nl; L += nt) {
    for (int jj = 1; jj < g.size; ++jj) {
      const int j = (g.pos + jj) % g.size;
      const uint2 d = ll_load_line<Tin, Tin>(flat + (int64_t)rs_chunk(p, j, g.size) * n, L, n);
      st_ll(ll_line(p, p.bases[g.member(j)], g.pos, L), d.x, d.y, p.epoch);
    }
  }
  const bool pre = p.prediv != 1.0f, post = p.postdiv != 1.0f;
  const Tin* mine = flat + (int64_t)rs_chunk(p, g.pos, g.size) * n;
  for (int64_t L = tid; L < nl; L += nt) {
    uint4 v[MAXW];
#pragma unroll
    for (int j = 0; j < MAXW; ++j)      // every peer's line in flight before any wait
      if (j < g.size && j != g.pos) v[j] = ld_ll(ll_line(p, p.bases[g.rank], j, L));
    float acc[EPL];
#pragma unroll
    for (int q = 0; q < EPL; ++q) acc[q] = 0.0f;
#pragma unroll
    for (int j = 0; j < MAXW; ++j) {
      if (j >= g.size) break;
      uint2 d;
      if (j == g.pos) {
        d = ll_load_line<Tin, Tin>(mine, L, n);
      } else {
        if (!ll_ready(v[j], p.epoch)) v[j] = ll_wait(p, g, ll_line(p, p.bases[g.rank], j, L), v[j]);
        d = make_uint2(v[j].x, v[j].z);
      }
      float x[EPL];
      if constexpr (EPL == 4) {
        x[0] = bf16lo(d.x); x[1] = bf16hi(d.x); x[2] = bf16lo(d.y); x[3] = bf16hi(d.y);
      } else {
        x[0] = __uint_as_float(d.x); x[1] = __uint_as_float(d.y);
      }
#pragma unroll
      for (int q = 0; q < EPL; ++q) acc[q] = __fadd_rn(acc[q], pre ? __fdiv_rn(x[q], p.prediv) : x[q]);
    }
    const int64_t e0 = L * EPL;
    float r[EPL];
#pragma unroll
    for (int q = 0; q < EPL; ++q) r[q] = post ? __fdiv_rn(acc[q], p.postdiv) : acc[q];
    if (e0 + EPL <= n && (reinterpret_cast<uintptr_t>(out + e0) & (4 * EPL - 1)) == 0) {
      if constexpr (EPL == 4) {
        float4 b = p.accumulate ? *reinterpret_cast<const float4*>(out + e0) : make_float4(0.f, 0.f, 0.f, 0.f);
        *reinterpret_cast<float4*>(out + e0) =
            make_float4(__fadd_rn(b.x, r[0]), __fadd_rn(b.y, r[1]), __fadd_rn(b.z, r[2]), __fadd_rn(b.w, r[3]));
      } else {
        float2 b = p.accumulate ? *reinterpret_cast<const float2*>(out + e0) : make_float2(0.f, 0.f);
        *reinterpret_cast<float2*>(out + e0) = make_float2(__fadd_rn(b.x, r[0]), __fadd_rn(b.y, r[1]));
      }
    } else {
#pragma unroll
      for (int q = 0; q < EPL; ++q) {
        if (e0 + q >= n) break;
        out[e0 + q] = __fadd_rn(p.accumulate ? out[e0 + q] : 0.0f, r[q]);
      }
    }
  }
}

}  // namespace fsdp

using namespace fsdp;

struct fsdp_comm {
  int rank = 0, world = 1;
  bool emulated = false;
  int64_t pool_bytes = 0;
  int max_ctas = 32;
  int device = 0;
  char* pool = nullptr;                       // own pool (emulated: all pools)
  char* bases[FSDP_MAX_RANKS] = {};
  bool opened[FSDP_MAX_RANKS] = {};
  uint32_t epoch[FSDP_NUM_CH] = {};
  int64_t timeout_ns = 20LL * 1000 * 1000 * 1000;
  int kind_ctas[FSDP_NUM_KINDS] = {};         // per-kind grid caps (0: max_ctas)
  bool split = true;                          // 1-CTA enter/exit kernels around data kernels
  bool barriers = true;                       // false: data kernels only (profiling harness)
  bool timing = false;                        // record events around every data kernel
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timed[FSDP_NUM_KINDS];
  std::vector<cudaEvent_t> spare;
  // copy-engine path: one side stream per (collective kind, peer, piece) —
  // all-gather and reduce-scatter copies never queue behind each other —
  // and an event pool
  cudaStream_t ce_stream[3][FSDP_MAX_RANKS * 4] = {};   // [AG, RS, AR][...]
  int ce_split = 1;                           // pieces per peer copy (FSDP_CE_SPLIT, <= 4)
  bool ce_shared_streams = false;             // FSDP_CE_SHARED_STREAMS=1: AG and RS share side streams
  // one destination at a time, staggered (FSDP_CE_SERIAL=0: one side stream
  // per peer, all concurrent).  Measured at W=4, 2 GB: AG 704 vs 498 GB/s,
  // RS 546 vs 308 GB/s bus bandwidth.
  bool ce_serial = true;
  // reduce-scatter data direction: 0 = pull (DMA reads of the peers' chunks),
  // 1 = push (DMA writes into the peers' staging), -1 (default) = push when
  // the chunk is pipelined in pieces, else pull.  Measured at W=4, 2 GiB:
  // pipelined push 647-654 GB/s vs pipelined pull 590-624 (FSDP_CE_RS_PUSH)
  int ce_rs_push = -1;
  int ce_rs_pieces = 8;                       // FSDP_CE_RS_PIECES: max pipeline pieces of a CE reduce-scatter
  int64_t ce_rs_pipe_min = 64LL << 20;        // FSDP_CE_RS_PIPE_MIN: pipeline chunks of at least this many elements
  int64_t ce_rs_min_piece = 4LL << 20;        // FSDP_CE_RS_MIN_PIECE: smallest geometric piece (about)
  int ce_reduce_ctas = 0;                     // FSDP_CE_REDUCE_CTAS: grid of non-final piece reductions (0: full)
  bool ce_rs_geom = true;                     // FSDP_CE_RS_GEOM: halving pieces (else uniform)
  int ce_reduce_cap = 0;                      // FSDP_CE_REDUCE_CAP: grid cap of every CE reduction (0: 4 CTAs/SM)
  bool ce_rs_noreduce = false;
  int misorder_rs = 0;                        // fault hook (fsdp_comm_set_fault)
  int64_t ce_ag_piece = -1;                   // FSDP_CE_AG_PIECE: piece-major all-gather DMA (-1 auto, 0 off, N bytes)
  int rs_tma_ring = -1;
  float ce_rs_sm_frac = 0.f;                  // FSDP_CE_RS_SM_FRAC: tail fraction of a pipelined chunk pulled by SM TMA                       // FSDP_RS_TMA_RING: TMA-pull ring geometry (-1: not read yet)                // FSDP_CE_RS_NOREDUCE=1: DIAGNOSTIC ONLY, skip the reductions (wrong results)
  std::vector<cudaEvent_t> ce_events;
  size_t ce_next = 0;
  // VMM pool (fsdp_comm_create_vmm): own allocation + peer mappings
  bool vmm = false;
  int handle_type = 0;
  vmm::Mapping own_map;
  vmm::Mapping peer_map[FSDP_MAX_RANKS];
  // NVLS: multicast object of this rank's shard group (consecutive mc_gsize ranks)
  CUmemGenericAllocationHandle mc_handle = 0;
  vmm::Mapping mc_map;
  int mc_gsize = 0;
  bool mc_added = false;
};

namespace {

int validate_group(fsdp_comm_t* c, int channel, int gsize, int gstride) {
  if (!c) return fail(FSDP_E_INVALID, "null communicator");
  if (channel < 0 || channel >= FSDP_NUM_CH) return fail(FSDP_E_INVALID, "bad channel");
  if (gsize < 1 || gstride < 1 || gsize * gstride > c->world ||
      (gstride == 1 ? c->world % gsize : c->world % (gsize * gstride)))
    return fail(FSDP_E_INVALID, "group does not partition the world");
  if (!c->emulated)
    for (int j = 0; j < gsize; ++j) {
      const int start = gstride == 1 ? (c->rank / gsize) * gsize : c->rank % gstride;
      const int m = start + j * gstride;
      if (!c->bases[m]) return fail(FSDP_E_INVALID, "peer pool not opened (fsdp_comm_open_peers)");
    }
  return 0;
}

void fill_common(fsdp_comm_t* c, CollParams& p, int channel, int gsize, int gstride, int64_t n) {
  std::memset(&p, 0, sizeof(p));
  for (int r = 0; r < FSDP_MAX_RANKS; ++r) p.bases[r] = c->bases[r];
  p.rank0 = c->emulated ? -1 : c->rank;
  p.gsize = gsize;
  p.gstride = gstride;
  p.channel = channel;
  p.epoch = ++c->epoch[channel];
  p.n = n;
  p.prediv = 1.0f;
  p.postdiv = 1.0f;
  p.timeout_ns = c->timeout_ns;
  p.mc_base = (char*)c->mc_map.va;
}

int grid_for(fsdp_comm_t* c, int64_t elems, int kind = -1) {
  int64_t tiles = (elems + kTileElems - 1) / kTileElems;
  const int cap = (kind >= 0 && c->kind_ctas[kind] > 0) ? c->kind_ctas[kind] : c->max_ctas;
  int g = (int)std::min<int64_t>(std::max<int64_t>(tiles, 1), cap);
  if (c->emulated) g = std::min(g, std::max(1, 128 / c->world));
  return g;
}

template <typename K>
int launch(fsdp_comm_t* c, K kernel, const CollParams& p, int grid, int threads, cudaStream_t s) {
  if (c->emulated) {
    dim3 gd(grid, c->world), bd(threads);
    void* args[] = {(void*)&p};
    FSDP_CUDA(cudaLaunchCooperativeKernel((void*)kernel, gd, bd, args, 0, s));
  } else {
    kernel<<<grid, threads, 0, s>>>(p);
  }
  FSDP_LAUNCHED();
  return 0;
}

int nranks_args(fsdp_comm_t* c) { return c->emulated ? c->world : 1; }

cudaEvent_t take_event(fsdp_comm_t* c) {
  if (!c->spare.empty()) {
    cudaEvent_t e = c->spare.back();
    c->spare.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// enter barrier -> data kernel (signal-only) -> exit barrier, one epoch.
// Only the 1-CTA barrier kernels ever spin.
template <typename K>
int launch_split(fsdp_comm_t* c, int kind, K kernel, CollParams& p, int grid, int threads,
                 size_t smem, cudaStream_t s) {
  p.split = 1;
  p.data_ctas = grid;
  if (c->barriers)
    if (int rc = launch(c, coll_enter_kernel, p, 1, 32, s)) return rc;
  cudaEvent_t a = nullptr, b = nullptr;
  if (c->timing) {
    a = take_event(c);
    b = take_event(c);
    FSDP_CUDA(cudaEventRecord(a, s));
  }
  void* args[] = {(void*)&p};
  if (c->emulated) {
    FSDP_CUDA(cudaLaunchCooperativeKernel((void*)kernel, dim3(grid, c->world), dim3(threads), args, smem, s));
  } else {
    FSDP_CUDA(cudaLaunchKernel((void*)kernel, dim3(grid), dim3(threads), args, smem, s));
  }
  FSDP_LAUNCHED();
  if (c->timing) {
    FSDP_CUDA(cudaEventRecord(b, s));
    c->timed[kind].emplace_back(a, b);
  }
  if (!c->barriers) return 0;
  return launch(c, coll_exit_kernel, p, 1, 256, s);
}

}  // namespace

extern "C" int fsdp_comm_set_ctas(fsdp_comm_t* c, int kind, int ctas) {
  if (!c || kind < 0 || kind >= FSDP_NUM_KINDS || ctas < 0 || ctas > FSDP_MAX_CTAS - 1)
    return fail(FSDP_E_INVALID, "fsdp_comm_set_ctas: bad args");
  c->kind_ctas[kind] = ctas;
  return 0;
}

extern "C" int fsdp_comm_set_barriers(fsdp_comm_t* c, int on) {
  if (!c) return fail(FSDP_E_INVALID, "null communicator");
  c->barriers = on != 0;
  return 0;
}

extern "C" int fsdp_comm_set_mode(fsdp_comm_t* c, int split, int timing) {
  if (!c) return fail(FSDP_E_INVALID, "null communicator");
  c->split = split != 0;
  c->timing = timing != 0;
  return 0;
}

extern "C" int fsdp_comm_timing_drain(fsdp_comm_t* c, int kind, float* ms_out, int max_n,
                                      int* count) {
  if (!c || kind < 0 || kind >= FSDP_NUM_KINDS || !count) return fail(FSDP_E_INVALID, "bad args");
  auto& v = c->timed[kind];
  int k = 0;
  for (auto& pr : v) {
    float ms = 0.f;
    FSDP_CUDA(cudaEventSynchronize(pr.second));
    FSDP_CUDA(cudaEventElapsedTime(&ms, pr.first, pr.second));
    if (ms_out && k < max_n) ms_out[k] = ms;
    ++k;
    c->spare.push_back(pr.first);
    c->spare.push_back(pr.second);
  }
  v.clear();
  *count = k;
  return 0;
}

extern "C" int64_t fsdp_comm_reserved_bytes(void) { return kReserved; }

extern "C" int fsdp_comm_create(int rank, int world, int64_t pool_bytes, int max_ctas,
                                fsdp_comm_t** out) {
  if (!out) return fail(FSDP_E_INVALID, "null out");
  if (world < 1 || world > FSDP_MAX_RANKS || rank < 0 || rank >= world)
    return fail(FSDP_E_INVALID, "rank/world out of range (world <= 8)");
  if (max_ctas < 1 || max_ctas > FSDP_MAX_CTAS - 1) return fail(FSDP_E_INVALID, "max_ctas out of range (1..159)");
  if (pool_bytes < kReserved) pool_bytes = kReserved;
  pool_bytes = (pool_bytes + 4095) / 4096 * 4096;
  fsdp_comm_t* c = new fsdp_comm_t();
  c->rank = rank; c->world = world; c->pool_bytes = pool_bytes; c->max_ctas = max_ctas;
  cudaGetDevice(&c->device);
  cudaError_t e = cudaMalloc(&c->pool, pool_bytes);
  if (e != cudaSuccess) { delete c; return check_cuda(e, "cudaMalloc(pool)"); }
  e = cudaMemset(c->pool, 0, kReserved);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { cudaFree(c->pool); delete c; return check_cuda(e, "cudaMemset(pool)"); }
  c->bases[rank] = c->pool;
  c->opened[rank] = true;
  *out = c;
  return 0;
}

extern "C" int fsdp_comm_create_emulated(int world, int64_t pool_bytes, int max_ctas,
                                         fsdp_comm_t** out) {
  if (!out) return fail(FSDP_E_INVALID, "null out");
  if (world < 1 || world > FSDP_MAX_RANKS) return fail(FSDP_E_INVALID, "world out of range");
  if (max_ctas < 1 || max_ctas > FSDP_MAX_CTAS - 1) return fail(FSDP_E_INVALID, "max_ctas out of range (1..159)");
  if (pool_bytes < kReserved) pool_bytes = kReserved;
  pool_bytes = (pool_bytes + 4095) / 4096 * 4096;
  fsdp_comm_t* c = new fsdp_comm_t();
  c->rank = 0; c->world = world; c->emulated = true; c->pool_bytes = pool_bytes;
  c->max_ctas = max_ctas;
  cudaGetDevice(&c->device);
  cudaError_t e = cudaMalloc(&c->pool, pool_bytes * world);
  if (e != cudaSuccess) { delete c; return check_cuda(e, "cudaMalloc(emulated pools)"); }
  for (int r = 0; r < world; ++r) {
    c->bases[r] = c->pool + r * pool_bytes;
    c->opened[r] = true;
    e = cudaMemset(c->bases[r], 0, kReserved);
    if (e != cudaSuccess) break;
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { cudaFree(c->pool); delete c; return check_cuda(e, "cudaMemset(pools)"); }
  *out = c;
  return 0;
}

extern "C" int fsdp_comm_ipc_handle(fsdp_comm_t* c, void* handle_out) {
  if (!c || !handle_out) return fail(FSDP_E_INVALID, "null argument");
  if (c->emulated) return fail(FSDP_E_UNSUPPORTED, "emulated communicator has no IPC handle");
  static_assert(sizeof(cudaIpcMemHandle_t) == FSDP_IPC_HANDLE_BYTES, "ipc handle size");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, c->pool);
  if (e != cudaSuccess) return fail(FSDP_E_IPC, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
  std::memcpy(handle_out, &h, sizeof(h));
  return 0;
}

extern "C" int fsdp_comm_open_peers(fsdp_comm_t* c, const void* handles) {
  if (!c || !handles) return fail(FSDP_E_INVALID, "null argument");
  if (c->emulated) return 0;
  const char* hs = (const char*)handles;
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank || c->opened[r]) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, hs + (size_t)r * FSDP_IPC_HANDLE_BYTES, sizeof(h));
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
      return fail(FSDP_E_IPC, "cudaIpcOpenMemHandle(rank " + std::to_string(r) + "): " +
                                  cudaGetErrorString(e));
    c->bases[r] = (char*)ptr;
    c->opened[r] = true;
  }
  return 0;
}

extern "C" void* fsdp_comm_pool_ptr(fsdp_comm_t* c, int r) {
  if (!c || r < 0 || r >= c->world) return nullptr;
  if (!c->emulated && r != c->rank) return nullptr;
  return c->bases[r];
}

extern "C" int64_t fsdp_comm_pool_bytes(fsdp_comm_t* c) { return c ? c->pool_bytes : -1; }

extern "C" int fsdp_comm_set_timeout_ms(fsdp_comm_t* c, int64_t ms) {
  if (!c || ms <= 0) return fail(FSDP_E_INVALID, "bad timeout");
  c->timeout_ns = ms * 1000000LL;
  return 0;
}

extern "C" int fsdp_comm_device_error(fsdp_comm_t* c) {
  if (!c) return fail(FSDP_E_INVALID, "null communicator");
  int worst = 0;
  const int n = c->emulated ? c->world : 1;
  for (int i = 0; i < n; ++i) {
    uint32_t v = 0;
    char* base = c->emulated ? c->bases[i] : c->pool;
    cudaError_t e = cudaMemcpy(&v, base + kErrOff, sizeof(v), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return check_cuda(e, "read device error word");
    if (v) worst = (int)v;
  }
  return worst;
}

// Device-side fold of the error word(s) into a skip predicate: *flag = 1 if
// any local pool's error word is set, else (keep ? *flag : 0); also mirrors
// the word into host-visible memory (pinned, UVA) so the host can raise
// DeadlockError at a step boundary without a synchronisation.
namespace {
struct ErrWords { const uint32_t* w[FSDP_MAX_RANKS]; int n; };
__global__ void __launch_bounds__(32) fold_error_kernel(ErrWords e, float* flag, int keep, int* mirror) {
  if (threadIdx.x != 0) return;
  uint32_t worst = 0;
  for (int i = 0; i < e.n; ++i) {
    const uint32_t v = *reinterpret_cast<volatile const uint32_t*>(e.w[i]);
    if (v) worst = v;
  }
  if (flag) *flag = worst ? 1.0f : (keep ? *flag : 0.0f);
  if (mirror) *reinterpret_cast<volatile int*>(mirror) = (int)worst;
}
}  // namespace

extern "C" int fsdp_comm_fold_error(fsdp_comm_t* c, float* flag, int keep, int* host_mirror,
                                    void* stream) {
  if (!c) return fail(FSDP_E_INVALID, "null communicator");
  ErrWords e;
  e.n = c->emulated ? c->world : 1;
  for (int i = 0; i < e.n; ++i)
    e.w[i] = reinterpret_cast<const uint32_t*>((c->emulated ? c->bases[i] : c->pool) + kErrOff);
  fold_error_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(e, flag, keep ? 1 : 0, host_mirror);
  FSDP_LAUNCHED();
  return 0;
}

// First local timeout: out[0..5] = {set, word index, seen, epoch, channel,
// size << 8 | stride}; word index < flag words decodes as
// ((channel * 3 + phase) * MAX_RANKS + src) * MAX_CTAS + cta.
extern "C" int fsdp_comm_timeout_info(fsdp_comm_t* c, uint32_t* out) {
  if (!c || !out) return fail(FSDP_E_INVALID, "null argument");
  const int n = c->emulated ? c->world : 1;
  for (int i = 0; i < 6; ++i) out[i] = 0;
  for (int i = 0; i < n && !out[0]; ++i)
    FSDP_CUDA(cudaMemcpy(out, (c->emulated ? c->bases[i] : c->pool) + kDiagOff, 6 * sizeof(uint32_t),
                         cudaMemcpyDeviceToHost));
  return 0;
}

extern "C" int fsdp_comm_set_fault(fsdp_comm_t* c, int misorder_reduce_scatter) {
  if (!c) return fail(FSDP_E_INVALID, "null communicator");
  c->misorder_rs = misorder_reduce_scatter ? 1 : 0;
  return 0;
}

extern "C" int fsdp_comm_clear_error(fsdp_comm_t* c) {
  if (!c) return fail(FSDP_E_INVALID, "null communicator");
  const int n = c->emulated ? c->world : 1;
  for (int i = 0; i < n; ++i)
    FSDP_CUDA(cudaMemset((c->emulated ? c->bases[i] : c->pool) + kErrOff, 0, kScalarOff - kErrOff));
  FSDP_CUDA(cudaDeviceSynchronize());
  return 0;
}

extern "C" int fsdp_comm_destroy(fsdp_comm_t* c) {
  if (!c) return 0;
  if (c->vmm) {
    cudaDeviceSynchronize();
    if (c->mc_map.va) vmm::mc_unbind(c->mc_handle, c->device, &c->mc_map);
    if (c->mc_handle) vmm::release_handle(c->mc_handle);
    for (int r = 0; r < c->world; ++r)
      if (r != c->rank) vmm::unmap(&c->peer_map[r]);
  } else if (!c->emulated) {
    for (int r = 0; r < c->world; ++r)
      if (r != c->rank && c->bases[r]) cudaIpcCloseMemHandle(c->bases[r]);
  }
  for (auto& v : c->timed)
    for (auto& pr : v) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
  for (auto e : c->spare) cudaEventDestroy(e);
  for (auto e : c->ce_events) cudaEventDestroy(e);
  for (auto& row : c->ce_stream)
    for (auto s : row)
      if (s) cudaStreamDestroy(s);
  if (c->vmm) vmm::unmap(&c->own_map);
  else cudaFree(c->pool);
  delete c;
  return 0;
}

static int check_range(fsdp_comm_t* c, int64_t off, int64_t bytes, const char* who) {
  if (off < kReserved || bytes < 0 || off + bytes > c->pool_bytes)
    return fail(FSDP_E_INVALID, std::string(who) + ": pool region out of range (offset " +
                                    std::to_string(off) + ", " + std::to_string(bytes) +
                                    " bytes, pool " + std::to_string(c->pool_bytes) + ")");
  return 0;
}

extern "C" int fsdp_allgather(fsdp_comm_t* c, int channel, int gsize, int gstride,
                              const void* const* shards, int src_dtype, int64_t n, int64_t dst_off,
                              int dst_dtype, void* stream) {
  if (int rc = validate_group(c, channel, gsize, gstride)) return rc;
  if (n < 0 || !shards) return fail(FSDP_E_INVALID, "fsdp_allgather: bad args");
  const int os = elem_size(dst_dtype);
  if (!os || !elem_size(src_dtype)) return fail(FSDP_E_INVALID, "fsdp_allgather: bad dtype");
  if (int rc = check_range(c, dst_off, n * gsize * os, "fsdp_allgather")) return rc;
  CollParams p;
  fill_common(c, p, channel, gsize, gstride, n);
  for (int e = 0; e < nranks_args(c); ++e) p.in[e] = shards[e];
  p.off_a = dst_off;
  const int grid = grid_for(c, n, FSDP_KIND_AG);
  cudaStream_t s = (cudaStream_t)stream;
  if (c->split) {
    void* k = src_dtype == FSDP_F32
                  ? (dst_dtype == FSDP_BF16 ? (void*)allgather_kernel<float, __nv_bfloat16>
                                            : (void*)allgather_kernel<float, float>)
                  : (dst_dtype == FSDP_BF16 ? (void*)allgather_kernel<__nv_bfloat16, __nv_bfloat16>
                                            : (void*)allgather_kernel<__nv_bfloat16, float>);
    return launch_split(c, FSDP_KIND_AG, k, p, grid, kCommThreads, 0, s);
  }
  if (src_dtype == FSDP_F32 && dst_dtype == FSDP_BF16)
    return launch(c, allgather_kernel<float, __nv_bfloat16>, p, grid, kCommThreads, s);
  if (src_dtype == FSDP_F32 && dst_dtype == FSDP_F32)
    return launch(c, allgather_kernel<float, float>, p, grid, kCommThreads, s);
  if (src_dtype == FSDP_BF16 && dst_dtype == FSDP_BF16)
    return launch(c, allgather_kernel<__nv_bfloat16, __nv_bfloat16>, p, grid, kCommThreads, s);
  return launch(c, allgather_kernel<__nv_bfloat16, float>, p, grid, kCommThreads, s);
}

extern "C" int fsdp_reduce_scatter(fsdp_comm_t* c, int channel, int gsize, int gstride,
                                   const void* const* flats, int src_dtype, int64_t n,
                                   int64_t stage_off, float* const* outs, float prediv,
                                   float postdiv, int accumulate, void* stream) {
  if (int rc = validate_group(c, channel, gsize, gstride)) return rc;
  if (n < 0 || !flats || !outs) return fail(FSDP_E_INVALID, "fsdp_reduce_scatter: bad args");
  const int is = elem_size(src_dtype);
  if (!is) return fail(FSDP_E_INVALID, "fsdp_reduce_scatter: bad dtype");
  if (!(prediv > 0.f) || !(postdiv > 0.f)) return fail(FSDP_E_INVALID, "divisors must be > 0");
  if (int rc = check_range(c, stage_off, n * gsize * is, "fsdp_reduce_scatter")) return rc;
  CollParams p;
  fill_common(c, p, channel, gsize, gstride, n);
  p.rot = c->misorder_rs && gsize > 1 ? 1 : 0;
  for (int e = 0; e < nranks_args(c); ++e) { p.in[e] = flats[e]; p.out[e] = outs[e]; }
  p.off_a = stage_off;
  p.prediv = prediv; p.postdiv = postdiv; p.accumulate = accumulate ? 1 : 0;
  const int grid = grid_for(c, n);
  cudaStream_t s = (cudaStream_t)stream;
  if (src_dtype == FSDP_BF16)
    return launch(c, reduce_scatter_kernel<__nv_bfloat16>, p, grid, kCommThreads, s);
  return launch(c, reduce_scatter_kernel<float>, p, grid, kCommThreads, s);
}

extern "C" int fsdp_reduce_scatter_pull(fsdp_comm_t* c, int channel, int gsize, int gstride,
                                        int64_t src_off, int src_dtype, int64_t n,
                                        float* const* outs, float prediv, float postdiv,
                                        int accumulate, void* stream) {
  if (int rc = validate_group(c, channel, gsize, gstride)) return rc;
  if (n < 0 || !outs) return fail(FSDP_E_INVALID, "fsdp_reduce_scatter_pull: bad args");
  const int is = elem_size(src_dtype);
  if (!is) return fail(FSDP_E_INVALID, "fsdp_reduce_scatter_pull: bad dtype");
  if (!(prediv > 0.f) || !(postdiv > 0.f)) return fail(FSDP_E_INVALID, "divisors must be > 0");
  if (int rc = check_range(c, src_off, n * gsize * is, "fsdp_reduce_scatter_pull")) return rc;
  CollParams p;
  fill_common(c, p, channel, gsize, gstride, n);
  p.rot = c->misorder_rs && gsize > 1 ? 1 : 0;
  for (int e = 0; e < nranks_args(c); ++e) p.out[e] = outs[e];
  p.off_a = src_off;
  p.prediv = prediv; p.postdiv = postdiv; p.accumulate = accumulate ? 1 : 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int mw = gsize <= 2 ? 2 : (gsize <= 4 ? 4 : 8);
  const int u = std::max(1, (16 / mw) / (is / 2));
  const int grid = std::max(1, grid_for(c, n * 4 / u, FSDP_KIND_RS));
#define RSP(T, W)                                                                        \
  (c->split ? launch_split(c, FSDP_KIND_RS, (void*)reduce_scatter_pull_kernel<T, W>, p, grid, \
                           kCommThreads, 0, s)                                           \
            : launch(c, reduce_scatter_pull_kernel<T, W>, p, grid, kCommThreads, s))
  if (src_dtype == FSDP_BF16) {
    if (mw == 2) return RSP(__nv_bfloat16, 2);
    if (mw == 4) return RSP(__nv_bfloat16, 4);
    return RSP(__nv_bfloat16, 8);
  }
  if (mw == 2) return RSP(float, 2);
  if (mw == 4) return RSP(float, 4);
  return RSP(float, 8);
#undef RSP
}

extern "C" int fsdp_reduce_scatter_tma(fsdp_comm_t* c, int channel, int gsize, int gstride,
                                       int64_t src_off, int src_dtype, int64_t n,
                                       float* const* outs, float prediv, float postdiv,
                                       int accumulate, void* stream) {
  if (int rc = validate_group(c, channel, gsize, gstride)) return rc;
  if (n < 0 || !outs) return fail(FSDP_E_INVALID, "fsdp_reduce_scatter_tma: bad args");
  const int is = elem_size(src_dtype);
  if (!is) return fail(FSDP_E_INVALID, "fsdp_reduce_scatter_tma: bad dtype");
  if (!(prediv > 0.f) || !(postdiv > 0.f)) return fail(FSDP_E_INVALID, "divisors must be > 0");
  if (int rc = check_range(c, src_off, n * gsize * is, "fsdp_reduce_scatter_tma")) return rc;
  bool aligned = (n % kVec == 0) && (src_off % 16 == 0);
  for (int e = 0; e < nranks_args(c); ++e)
    aligned = aligned && outs[e] && ((uintptr_t)outs[e] % 16 == 0);
  if (!aligned)   // bulk copies need 16-byte granules: take the register-pull path
    return fsdp_reduce_scatter_pull(c, channel, gsize, gstride, src_off, src_dtype, n, outs, prediv,
                                    postdiv, accumulate, stream);
  CollParams p;
  fill_common(c, p, channel, gsize, gstride, n);
  p.rot = c->misorder_rs && gsize > 1 ? 1 : 0;
  for (int e = 0; e < nranks_args(c); ++e) p.out[e] = outs[e];
  p.off_a = src_off;
  p.prediv = prediv; p.postdiv = postdiv; p.accumulate = accumulate ? 1 : 0;
  // ring geometry (FSDP_RS_TMA_RING: 0 = 4 x 32 KB, 1 = 3 x 64 KB, 2 = 6 x 32 KB, 3 = 2 x 96 KB)
  if (c->rs_tma_ring < 0) {       // read once per communicator
    const char* e = getenv("FSDP_RS_TMA_RING");
    c->rs_tma_ring = e ? std::max(0, std::min(3, atoi(e))) : 0;
  }
  const int ring = c->rs_tma_ring;
  static const struct { void* bf; void* f; int stages, bytes; } kRings[] = {
      {(void*)reduce_scatter_tma_kernel<__nv_bfloat16, 4, 32768>, (void*)reduce_scatter_tma_kernel<float, 4, 32768>, 4, 32768},
      {(void*)reduce_scatter_tma_kernel<__nv_bfloat16, 3, 65536>, (void*)reduce_scatter_tma_kernel<float, 3, 65536>, 3, 65536},
      {(void*)reduce_scatter_tma_kernel<__nv_bfloat16, 6, 32768>, (void*)reduce_scatter_tma_kernel<float, 6, 32768>, 6, 32768},
      {(void*)reduce_scatter_tma_kernel<__nv_bfloat16, 2, 98304>, (void*)reduce_scatter_tma_kernel<float, 2, 98304>, 2, 98304},
  };
  const auto& rg = kRings[ring];
  const int64_t T = (rg.bytes / (gsize * is)) / kVec * kVec;
  const int64_t ntiles = (n + T - 1) / T;
  int grid = (int)std::min<int64_t>(std::max<int64_t>(ntiles, 1), c->max_ctas);
  if (c->emulated) grid = std::min(grid, std::max(1, 128 / c->world));
  const size_t smem = (size_t)rg.stages * rg.bytes;
  cudaStream_t s = (cudaStream_t)stream;
  void* fn = src_dtype == FSDP_BF16 ? rg.bf : rg.f;
  FSDP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  void* args[] = {(void*)&p};
  if (c->emulated) {
    FSDP_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid, c->world), dim3(kTmaThreads), args, smem, s));
  } else {
    FSDP_CUDA(cudaLaunchKernel(fn, dim3(grid), dim3(kTmaThreads), args, smem, s));
  }
  FSDP_LAUNCHED();
  return 0;
}

// ---------------------------------------------------- copy-engine variants --
// Local ascending reduction of [e0, e0+len) (grid_cap 0: full occupancy grid).
static int launch_ce_reduce(CeReduceArgs ra, int64_t e0, int64_t len, int src_dtype, int grid_cap,
                            cudaStream_t s) {
  if (len <= 0) return 0;
  ra.e0 = e0; ra.len = len;
  const int64_t nv = std::max<int64_t>(1, (len + kVec - 1) / kVec);
  int grid = (int)std::min<int64_t>((nv + 255) / 256, (int64_t)kNumSMs * 4);
  if (grid_cap > 0) grid = std::min(grid, grid_cap);
  const int mw = ra.gsize <= 2 ? 2 : (ra.gsize <= 4 ? 4 : 8);
  using bf = __nv_bfloat16;
  if (ra.out_bf16) {
    if (src_dtype == FSDP_BF16) {
      if (mw == 2) ce_reduce_kernel<bf, bf, 2><<<grid, 256, 0, s>>>(ra);
      else if (mw == 4) ce_reduce_kernel<bf, bf, 4><<<grid, 256, 0, s>>>(ra);
      else ce_reduce_kernel<bf, bf, 8><<<grid, 256, 0, s>>>(ra);
    } else {
      if (mw == 2) ce_reduce_kernel<float, bf, 2><<<grid, 256, 0, s>>>(ra);
      else if (mw == 4) ce_reduce_kernel<float, bf, 4><<<grid, 256, 0, s>>>(ra);
      else ce_reduce_kernel<float, bf, 8><<<grid, 256, 0, s>>>(ra);
    }
  } else if (src_dtype == FSDP_BF16) {
    if (mw == 2) ce_reduce_kernel<bf, float, 2><<<grid, 256, 0, s>>>(ra);
    else if (mw == 4) ce_reduce_kernel<bf, float, 4><<<grid, 256, 0, s>>>(ra);
    else ce_reduce_kernel<bf, float, 8><<<grid, 256, 0, s>>>(ra);
  } else {
    if (mw == 2) ce_reduce_kernel<float, float, 2><<<grid, 256, 0, s>>>(ra);
    else if (mw == 4) ce_reduce_kernel<float, float, 4><<<grid, 256, 0, s>>>(ra);
    else ce_reduce_kernel<float, float, 8><<<grid, 256, 0, s>>>(ra);
  }
  FSDP_LAUNCHED();
  return 0;
}

static int ce_prepare(fsdp_comm_t* c) {
  if (c->ce_events.empty()) {
    if (const char* e = getenv("FSDP_CE_SPLIT")) c->ce_split = std::max(1, std::min(4, atoi(e)));
    if (const char* e = getenv("FSDP_CE_SHARED_STREAMS")) c->ce_shared_streams = atoi(e) != 0;
    if (const char* e = getenv("FSDP_CE_SERIAL")) c->ce_serial = atoi(e) != 0;
    if (const char* e = getenv("FSDP_CE_RS_PUSH")) c->ce_rs_push = atoi(e) != 0 ? 1 : 0;
    if (const char* e = getenv("FSDP_CE_RS_PIECES")) c->ce_rs_pieces = std::max(1, std::min(16, atoi(e)));
    if (const char* e = getenv("FSDP_CE_RS_MIN_PIECE")) c->ce_rs_min_piece = std::max<int64_t>(1 << 16, atoll(e));
    if (const char* e = getenv("FSDP_CE_RS_PIPE_MIN")) c->ce_rs_pipe_min = std::max<int64_t>(1 << 16, atoll(e));
    if (const char* e = getenv("FSDP_CE_REDUCE_CTAS")) c->ce_reduce_ctas = std::max(0, atoi(e));
    if (const char* e = getenv("FSDP_CE_RS_GEOM")) c->ce_rs_geom = atoi(e) != 0;
    if (const char* e = getenv("FSDP_CE_RS_NOREDUCE")) c->ce_rs_noreduce = atoi(e) != 0;
    if (const char* e = getenv("FSDP_CE_REDUCE_CAP")) c->ce_reduce_cap = std::max(0, atoi(e));
    if (const char* e = getenv("FSDP_CE_RS_SM_FRAC")) c->ce_rs_sm_frac = std::max(0.f, std::min(0.9f, (float)atof(e)));
    if (const char* e = getenv("FSDP_CE_AG_PIECE")) c->ce_ag_piece = std::max<int64_t>(-1, atoll(e));
    for (int k = 0; k < 3; ++k)
      for (int r = 0; r < FSDP_MAX_RANKS * c->ce_split; ++r)
        FSDP_CUDA(cudaStreamCreateWithFlags(&c->ce_stream[k][r], cudaStreamNonBlocking));
    c->ce_events.resize(256);
    for (auto& e : c->ce_events) FSDP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  return 0;
}
static cudaEvent_t ce_event(fsdp_comm_t* c) {
  cudaEvent_t e = c->ce_events[c->ce_next % c->ce_events.size()];
  ++c->ce_next;
  return e;
}

// copies[j] = (dst, src, bytes) for member j (skipped when bytes == 0); each on
// its own side stream so distinct peers' transfers use distinct copy engines
static int ce_fork_join(fsdp_comm_t* c, int kind, cudaStream_t s, int gsize, int pos,
                        void* const* dst, const void* const* src, size_t bytes) {
  cudaEvent_t fork = ce_event(c);
  FSDP_CUDA(cudaEventRecord(fork, s));
  if (c->ce_serial) {
    // one side stream, one destination at a time, staggered (member pos+1
    // first): every copy gets the whole NVSwitch port, and no two members
    // start on the same destination
    // (the member's own chunk is a local copy: it runs beside them on a
    // second side stream, it needs no NVLink)
    cudaStream_t* row = c->ce_stream[c->ce_shared_streams ? 0 : kind];
    cudaStream_t cs = row[0];
    FSDP_CUDA(cudaStreamWaitEvent(cs, fork, 0));
    // piece-major all-gather: every destination gets piece q while q is
    // still in L2, so the shard is read from DRAM once instead of once per
    // peer (measured: a 134 MB shard was read 3.95x at W = 4), at one copy
    // start per piece and peer.  Auto (ce_ag_piece < 0): 32 MB pieces for
    // shards of 48-256 MB -- below that L2 already absorbs the re-reads,
    // above it the extra copy starts cost more than the DRAM reads saved
    // (T5-11B 134 MB shards: +2 %; GPT-30B 308 MB shards: -2 %, N = 4).
    size_t ag_piece = 0;
    if (kind == 0) {
      if (c->ce_ag_piece > 0) ag_piece = (size_t)c->ce_ag_piece;
      else if (c->ce_ag_piece < 0 && gsize >= 3 && bytes > (48u << 20) && bytes <= (256u << 20))
        ag_piece = 32u << 20;   // (with one peer there is no re-read to save)
    }
    const size_t piece = (ag_piece > 0 && bytes > ag_piece) ? (ag_piece + 255) / 256 * 256 : bytes;
    for (size_t off = 0; off < bytes; off += piece) {
      const size_t len = std::min(piece, bytes - off);
      for (int jj = 0; jj + 1 < gsize; ++jj) {
        const int j = (pos + 1 + jj) % gsize;
        if (!dst[j] || !bytes) continue;
        FSDP_CUDA(cudaMemcpyAsync((char*)dst[j] + off, (const char*)src[j] + off, len,
                                  cudaMemcpyDeviceToDevice, cs));
      }
    }
    cudaEvent_t done = ce_event(c);
    FSDP_CUDA(cudaEventRecord(done, cs));
    FSDP_CUDA(cudaStreamWaitEvent(s, done, 0));
    if (dst[pos] && bytes) {
      FSDP_CUDA(cudaStreamWaitEvent(row[1], fork, 0));
      FSDP_CUDA(cudaMemcpyAsync(dst[pos], src[pos], bytes, cudaMemcpyDeviceToDevice, row[1]));
      cudaEvent_t own = ce_event(c);
      FSDP_CUDA(cudaEventRecord(own, row[1]));
      FSDP_CUDA(cudaStreamWaitEvent(s, own, 0));
    }
    return 0;
  }
  const int k = c->ce_split;
  const size_t piece = ((bytes + k - 1) / k + 255) / 256 * 256;
  for (int j = 0; j < gsize; ++j) {
    if (!dst[j] || !bytes) continue;
    for (int q = 0; q < k; ++q) {
      const size_t off = (size_t)q * piece;
      if (off >= bytes) break;
      const size_t len = std::min(piece, bytes - off);
      cudaStream_t cs = c->ce_stream[c->ce_shared_streams ? 0 : kind][j * k + q];
      FSDP_CUDA(cudaStreamWaitEvent(cs, fork, 0));
      FSDP_CUDA(cudaMemcpyAsync((char*)dst[j] + off, (const char*)src[j] + off, len,
                                cudaMemcpyDeviceToDevice, cs));
      cudaEvent_t done = ce_event(c);
      FSDP_CUDA(cudaEventRecord(done, cs));
      FSDP_CUDA(cudaStreamWaitEvent(s, done, 0));
    }
  }
  return 0;
}

extern "C" int fsdp_allgather_ce(fsdp_comm_t* c, int channel, int gsize, int gstride,
                                 const void* shard, int dtype, int64_t n, int64_t dst_off,
                                 void* stream) {
  if (int rc = validate_group(c, channel, gsize, gstride)) return rc;
  if (c->emulated) return fail(FSDP_E_UNSUPPORTED, "copy-engine collectives need a real communicator");
  const int es = elem_size(dtype);
  if (n < 0 || !shard || !es) return fail(FSDP_E_INVALID, "fsdp_allgather_ce: bad args");
  if (int rc = check_range(c, dst_off, n * gsize * es, "fsdp_allgather_ce")) return rc;
  if (int rc = ce_prepare(c)) return rc;
  CollParams p;
  fill_common(c, p, channel, gsize, gstride, n);
  p.data_ctas = 1;
  cudaStream_t s = (cudaStream_t)stream;
  if (int rc = launch(c, coll_enter_kernel, p, 1, 32, s)) return rc;
  const int start = gstride == 1 ? (c->rank / gsize) * gsize : c->rank % gstride;
  const int pos = gstride == 1 ? c->rank - start : c->rank / gstride;
  void* dst[FSDP_MAX_RANKS] = {};
  const void* src[FSDP_MAX_RANKS] = {};
  for (int j = 0; j < gsize; ++j) {
    dst[j] = c->bases[start + j * gstride] + dst_off + (int64_t)pos * n * es;
    src[j] = shard;
  }
  cudaEvent_t a = nullptr, b = nullptr;
  if (c->timing) { a = take_event(c); b = take_event(c); FSDP_CUDA(cudaEventRecord(a, s)); }
  if (int rc = ce_fork_join(c, 0, s, gsize, pos, dst, src, (size_t)n * es)) return rc;
  if (c->timing) { FSDP_CUDA(cudaEventRecord(b, s)); c->timed[FSDP_KIND_AG].emplace_back(a, b); }
  return launch(c, coll_signal_exit_kernel, p, 1, 32, s);   // my copies landed; so did everyone's
}

extern "C" int fsdp_reduce_scatter_ce_out(fsdp_comm_t* c, int channel, int gsize, int gstride,
                                          int64_t src_off, int src_dtype, int64_t n,
                                          int64_t stage_off, void* out, int out_dtype, float prediv,
                                          float postdiv, int accumulate, void* stream) {
  if (int rc = validate_group(c, channel, gsize, gstride)) return rc;
  if (c->emulated) return fail(FSDP_E_UNSUPPORTED, "copy-engine collectives need a real communicator");
  const int es = elem_size(src_dtype);
  if (n < 0 || !out || !es) return fail(FSDP_E_INVALID, "fsdp_reduce_scatter_ce: bad args");
  if (out_dtype != FSDP_F32 && out_dtype != FSDP_BF16)
    return fail(FSDP_E_INVALID, "fsdp_reduce_scatter_ce: out dtype must be fp32 or bf16");
  const bool out_bf16 = out_dtype == FSDP_BF16;
  if (out_bf16 && accumulate)
    return fail(FSDP_E_INVALID, "fsdp_reduce_scatter_ce: a bf16 result cannot accumulate");
  if (!(prediv > 0.f) || !(postdiv > 0.f)) return fail(FSDP_E_INVALID, "divisors must be > 0");
  if (int rc = check_range(c, src_off, n * gsize * es, "fsdp_reduce_scatter_ce(src)")) return rc;
  if (int rc = check_range(c, stage_off, n * gsize * es, "fsdp_reduce_scatter_ce(stage)")) return rc;
  if (int rc = ce_prepare(c)) return rc;
  CollParams p;
  fill_common(c, p, channel, gsize, gstride, n);
  p.rot = c->misorder_rs && gsize > 1 ? 1 : 0;
  p.data_ctas = 1;
  cudaStream_t s = (cudaStream_t)stream;
  if (int rc = launch(c, coll_enter_kernel, p, 1, 32, s)) return rc;
  const int start = gstride == 1 ? (c->rank / gsize) * gsize : c->rank % gstride;
  const int pos = gstride == 1 ? c->rank - start : c->rank / gstride;
  const int rot = p.rot;                           // misorder fault: chunk (k + rot) % gsize
  auto chunk = [&](int k) { return (k + rot) % gsize; };
  const int cpos = chunk(pos);
  char* mine = c->bases[c->rank];
  CeReduceArgs ra;
  ra.own = mine + src_off + (int64_t)cpos * n * es;
  ra.stage = mine + stage_off;
  ra.stride = n;
  ra.out = out;
  ra.gsize = gsize; ra.pos = pos;
  ra.prediv = prediv; ra.postdiv = postdiv; ra.accumulate = accumulate ? 1 : 0;
  ra.store_raw = 0;
  ra.out_bf16 = out_bf16 ? 1 : 0;
  cudaEvent_t a = nullptr, b = nullptr;
  if (c->timing) { a = take_event(c); b = take_event(c); FSDP_CUDA(cudaEventRecord(a, s)); }

  // Pieces: the side stream pulls piece q+1 from every peer (serial,
  // staggered, NVLink reads into local staging) while the stream reduces
  // piece q, so the HBM-bound reduction hides behind the transfers.
  // (smaller DMA copies lose efficiency: pieces of at least ce_rs_min_piece elements)
  // Chunks of at least ce_rs_pipe_min elements are pipelined.  Geometric
  // (default): halving pieces n/2, n/4, ... down to ~2*min_piece, so the one
  // exposed reduction (the last piece's) is small while the large early
  // pieces keep the DMA copies long.  Uniform (FSDP_CE_RS_GEOM=0): up to
  // ce_rs_pieces equal pieces of at least ce_rs_pipe_min/2.
  std::vector<std::pair<int64_t, int64_t>> pcs;      // (first element, length)
  auto round8 = [](int64_t x) { return (x + kVec - 1) / kVec * kVec; };
  // Hybrid (FSDP_CE_RS_SM_FRAC > 0, pipelined push only): the copy engines
  // move [0, nA) of every chunk while an SM TMA-pull kernel reduces [nA, n)
  // straight from the peers' payloads on a third side stream, so the tail of
  // the chunk needs no staging round trip.
  const bool hyb = c->ce_rs_sm_frac > 0.f && !out_bf16 && c->ce_serial && n >= c->ce_rs_pipe_min &&
                   c->ce_rs_push != 0 && (n % kVec == 0) && (src_off % 16 == 0) && aligned16(out);
  const int64_t nA = hyb ? std::min(n, round8((int64_t)((double)n * (1.0 - c->ce_rs_sm_frac)))) : n;
  if (!c->ce_serial || n < c->ce_rs_pipe_min) {
    pcs.emplace_back(0, n);
  } else if (c->ce_rs_geom) {
    int64_t e0 = 0, rem = nA;
    while (rem > 2 * c->ce_rs_min_piece && (int)pcs.size() + 1 < c->ce_rs_pieces) {
      const int64_t len = round8(rem / 2);
      pcs.emplace_back(e0, len);
      e0 += len; rem -= len;
    }
    pcs.emplace_back(e0, rem);
  } else {
    const int np = (int)std::min<int64_t>(c->ce_rs_pieces, std::max<int64_t>(1, 2 * nA / c->ce_rs_pipe_min));
    const int64_t plen = round8((nA + np - 1) / np);
    for (int64_t e0 = 0; e0 < nA || pcs.empty(); e0 += plen) pcs.emplace_back(e0, std::min(plen, nA - e0));
  }
  const int pieces = (int)pcs.size();
  const bool push = c->ce_rs_push < 0 ? pieces > 1 : c->ce_rs_push == 1;
  auto reduce_piece = [&](int64_t e0, int64_t len) -> int {
    if (c->ce_rs_noreduce) return 0;
    // a piece reduced behind the next piece's transfer needs only enough
    // HBM bandwidth to keep pace; the final piece is exposed: full grid
    return launch_ce_reduce(ra, e0, len, src_dtype,
                            (c->ce_reduce_ctas > 0 && e0 + len < n) ? c->ce_reduce_ctas : c->ce_reduce_cap, s);
  };

  if (pieces > 1 && push) {
    // pipelined push: piece q of my chunk j -> member j's staging slot pos
    // (NVLink writes, serial staggered), then a per-piece flag; my stream
    // reduces piece q once every member's piece q has landed here.  My
    // payload is read only by my own copies and peers read nothing of mine,
    // so no exit barrier: the next call's enter barrier guards the staging.
    // The per-piece signals run on a second side stream behind an event, so
    // the copy stream issues every piece's DMA back to back (a signal kernel
    // between pieces on the copy stream would leave a bubble per piece:
    // transfers alone measured 666 vs 759 GB/s at W=4, 2 GiB).
    cudaEvent_t fork = ce_event(c);
    FSDP_CUDA(cudaEventRecord(fork, s));
    cudaStream_t cs = c->ce_stream[c->ce_shared_streams ? 0 : 1][0];
    cudaStream_t ss = c->ce_stream[c->ce_shared_streams ? 0 : 1][1];
    FSDP_CUDA(cudaStreamWaitEvent(cs, fork, 0));
    // hybrid: piece flags move to phase 2 (the TMA kernel's in-kernel
    // barriers use phases 0 and 1, slot = CTA index, same epoch)
    const int fph = hyb && nA < n ? 2 : 1;
    cudaEvent_t pulled = nullptr;
    if (hyb && nA < n) {
      cudaStream_t ps = c->ce_stream[c->ce_shared_streams ? 0 : 1][2];
      FSDP_CUDA(cudaStreamWaitEvent(ps, fork, 0));
      CollParams p2 = p;
      p2.n = n - nA;
      p2.off_a = src_off + nA * es;
      p2.off_b = n;                                  // members' chunks stay n elements apart
      p2.out[0] = (float*)out + nA;
      p2.prediv = prediv; p2.postdiv = postdiv; p2.accumulate = accumulate ? 1 : 0;
      p2.split = 0;
      const int64_t T = (kTmaStageBytes / (gsize * es)) / kVec * kVec;
      const int grid = (int)std::min<int64_t>(std::max<int64_t>((p2.n + T - 1) / T, 1), c->max_ctas);
      void* fn = src_dtype == FSDP_BF16 ? (void*)reduce_scatter_tma_kernel<__nv_bfloat16, kTmaStages, kTmaStageBytes>
                                        : (void*)reduce_scatter_tma_kernel<float, kTmaStages, kTmaStageBytes>;
      const size_t smem = (size_t)kTmaStages * kTmaStageBytes;
      FSDP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      void* args[] = {(void*)&p2};
      FSDP_CUDA(cudaLaunchKernel(fn, dim3(grid), dim3(kTmaThreads), args, smem, ps));
      FSDP_LAUNCHED();
      pulled = ce_event(c);
      FSDP_CUDA(cudaEventRecord(pulled, ps));
    }
    for (int q = 0; q < pieces; ++q) {
      const int64_t e0 = pcs[q].first, len = pcs[q].second;
      for (int jj = 0; jj + 1 < gsize; ++jj) {
        const int j = (pos + 1 + jj) % gsize;
        FSDP_CUDA(cudaMemcpyAsync(c->bases[start + j * gstride] + stage_off + ((int64_t)pos * n + e0) * es,
                                  mine + src_off + ((int64_t)chunk(j) * n + e0) * es,
                                  (size_t)len * es, cudaMemcpyDeviceToDevice, cs));
      }
      cudaEvent_t landed = ce_event(c);
      FSDP_CUDA(cudaEventRecord(landed, cs));
      FSDP_CUDA(cudaStreamWaitEvent(ss, landed, 0));
      coll_signal_slot_kernel<<<1, 32, 0, ss>>>(p, q, fph);
      FSDP_LAUNCHED();
    }
    cudaEvent_t sent = ce_event(c);
    FSDP_CUDA(cudaEventRecord(sent, ss));        // after the last signal, hence after every copy
    for (int q = 0; q < pieces; ++q) {
      const int64_t e0 = pcs[q].first, len = pcs[q].second;
      coll_wait_slot_kernel<<<1, 32, 0, s>>>(p, q, fph);
      FSDP_LAUNCHED();
      if (q + 1 == pieces)
        if (c->timing) { FSDP_CUDA(cudaEventRecord(b, s)); c->timed[FSDP_KIND_RS].emplace_back(a, b); }
      if (int rc = reduce_piece(e0, len)) return rc;
    }
    FSDP_CUDA(cudaStreamWaitEvent(s, sent, 0));   // my payload is free once my copies are done
    if (pulled) FSDP_CUDA(cudaStreamWaitEvent(s, pulled, 0));   // ... and peers finished pulling its tail
    return 0;
  }
  if (pieces > 1) {
    cudaEvent_t fork = ce_event(c);
    FSDP_CUDA(cudaEventRecord(fork, s));
    cudaStream_t cs = c->ce_stream[c->ce_shared_streams ? 0 : 1][0];
    FSDP_CUDA(cudaStreamWaitEvent(cs, fork, 0));
    for (int q = 0; q < pieces; ++q) {
      const int64_t e0 = pcs[q].first, len = pcs[q].second;
      for (int jj = 0; jj + 1 < gsize; ++jj) {
        const int j = (pos + 1 + jj) % gsize;
        FSDP_CUDA(cudaMemcpyAsync(mine + stage_off + ((int64_t)j * n + e0) * es,
                                  c->bases[start + j * gstride] + src_off + ((int64_t)cpos * n + e0) * es,
                                  (size_t)len * es, cudaMemcpyDeviceToDevice, cs));
      }
      cudaEvent_t landed = ce_event(c);
      FSDP_CUDA(cudaEventRecord(landed, cs));
      FSDP_CUDA(cudaStreamWaitEvent(s, landed, 0));
      if (q + 1 == pieces) {
        if (c->timing) { FSDP_CUDA(cudaEventRecord(b, s)); c->timed[FSDP_KIND_RS].emplace_back(a, b); }
        if (int rc = launch(c, coll_signal_kernel, p, 1, 32, s)) return rc;   // done reading peers
      }
      if (int rc = reduce_piece(e0, len)) return rc;
    }
    return launch(c, coll_exit_kernel, p, 1, 256, s);     // peers done reading mine
  }

  void* dst[FSDP_MAX_RANKS] = {};
  const void* src[FSDP_MAX_RANKS] = {};
  for (int j = 0; j < gsize; ++j) {
    if (j == pos) continue;   // own chunk is reduced in place
    if (push) {               // my chunk j -> member j's staging, slot pos (NVLink writes)
      dst[j] = c->bases[start + j * gstride] + stage_off + (int64_t)pos * n * es;
      src[j] = mine + src_off + (int64_t)chunk(j) * n * es;
    } else {                  // member j's chunk pos -> my staging, slot j (NVLink reads)
      dst[j] = mine + stage_off + (int64_t)j * n * es;
      src[j] = c->bases[start + j * gstride] + src_off + (int64_t)cpos * n * es;
    }
  }
  if (int rc = ce_fork_join(c, 1, s, gsize, pos, dst, src, (size_t)n * es)) return rc;
  if (c->timing) { FSDP_CUDA(cudaEventRecord(b, s)); c->timed[FSDP_KIND_RS].emplace_back(a, b); }
  if (push) {
    // my copies are done and every member's pushes into my staging have
    // landed; my payload was only read by my own copies, so nothing waits
    // after the reduction
    if (int rc = launch(c, coll_signal_exit_kernel, p, 1, 32, s)) return rc;
    return reduce_piece(0, n);
  }
  if (int rc = launch(c, coll_signal_kernel, p, 1, 32, s)) return rc;   // done reading my peers
  if (int rc = reduce_piece(0, n)) return rc;
  return launch(c, coll_exit_kernel, p, 1, 256, s);     // peers done reading mine
}

// Copy-engine all-reduce (same contract and bits as fsdp_allreduce; real
// communicator): enter barrier; DMA-push chunk j of my input to member j's
// staging (slot pos) + per-member flag; ascending fp32 reduction of my chunk
// (/ postdiv) into my slot of the gather buffer; DMA-push that result into
// every member's gather buffer + flag; out = (accumulate ? out : 0) +
// gathered.  Peers read nothing of mine and the next call's enter barrier
// guards the staging/gather buffers, so there is no exit barrier.
// out_off >= 0: `out` is the pool region [out_off, +n fp32) on every member
// (same offset everywhere): the owner reduces its chunk straight into its own
// out slice and the DMA pushes that slice into every member's out, so there
// is no gather buffer and no epilogue (accumulate must be 0).
static int allreduce_ce_impl(fsdp_comm_t* c, int channel, int gsize, int gstride, const void* in,
                             int src_dtype, int64_t n, int64_t stage_off, int64_t gather_off, float* out,
                             int64_t out_off, float postdiv, int accumulate, cudaStream_t s) {
  const int is = elem_size(src_dtype);
  if (int rc = ce_prepare(c)) return rc;
  int64_t ch = (n + gsize - 1) / gsize;
  ch = (ch + kVec - 1) / kVec * kVec;
  const bool direct = out_off >= 0;
  const int64_t res_off = direct ? out_off : gather_off;   // where results land on every member
  CollParams p;
  fill_common(c, p, channel, gsize, gstride, n);
  if (int rc = launch(c, coll_enter_kernel, p, 1, 32, s)) return rc;
  const int start = gstride == 1 ? (c->rank / gsize) * gsize : c->rank % gstride;
  const int pos = gstride == 1 ? c->rank - start : c->rank / gstride;
  auto clen = [&](int j) -> int64_t { const int64_t b = (int64_t)j * ch; return b >= n ? 0 : std::min(ch, n - b); };
  char* mine = c->bases[c->rank];
  // own side stream: a HYBRID stage-2 all-reduce of unit u overlaps the
  // reduce-scatter of unit u+1 (caller streams differ), DMA included
  cudaStream_t cs = c->ce_stream[c->ce_shared_streams ? 0 : 2][0];
  cudaEvent_t a = nullptr, b = nullptr;
  if (c->timing) { a = take_event(c); b = take_event(c); FSDP_CUDA(cudaEventRecord(a, s)); }
  // 1. reduce-scatter push: chunk j -> member j's staging slot pos
  cudaEvent_t fork = ce_event(c);
  FSDP_CUDA(cudaEventRecord(fork, s));
  FSDP_CUDA(cudaStreamWaitEvent(cs, fork, 0));
  for (int jj = 0; jj + 1 < gsize; ++jj) {
    const int j = (pos + 1 + jj) % gsize;
    if (clen(j) > 0)
      FSDP_CUDA(cudaMemcpyAsync(c->bases[start + j * gstride] + stage_off + (int64_t)pos * ch * is,
                                (const char*)in + (int64_t)j * ch * is, (size_t)(clen(j) * is),
                                cudaMemcpyDeviceToDevice, cs));
  }
  coll_signal_slot_kernel<<<1, 32, 0, cs>>>(p, 0);
  FSDP_LAUNCHED();
  coll_wait_slot_kernel<<<1, 32, 0, s>>>(p, 0);
  FSDP_LAUNCHED();
  // 2. owner reduction of my chunk -> my slot of the result buffer
  CeReduceArgs ra;
  ra.own = (const char*)in + (int64_t)pos * ch * is;
  ra.stage = mine + stage_off;
  ra.stride = ch;
  ra.out = (float*)(mine + res_off) + (int64_t)pos * ch;
  ra.gsize = gsize; ra.pos = pos;
  ra.prediv = 1.0f; ra.postdiv = postdiv; ra.accumulate = 0; ra.store_raw = 1; ra.out_bf16 = 0;
  if (int rc = launch_ce_reduce(ra, 0, clen(pos), src_dtype, c->ce_reduce_cap, s)) return rc;
  // 3. all-gather push of my reduced chunk
  cudaEvent_t reduced = ce_event(c);
  FSDP_CUDA(cudaEventRecord(reduced, s));
  FSDP_CUDA(cudaStreamWaitEvent(cs, reduced, 0));
  for (int jj = 0; jj + 1 < gsize; ++jj) {
    const int j = (pos + 1 + jj) % gsize;
    if (clen(pos) > 0)
      FSDP_CUDA(cudaMemcpyAsync(c->bases[start + j * gstride] + res_off + (int64_t)pos * ch * 4,
                                mine + res_off + (int64_t)pos * ch * 4, (size_t)(clen(pos) * 4),
                                cudaMemcpyDeviceToDevice, cs));
  }
  coll_signal_slot_kernel<<<1, 32, 0, cs>>>(p, 1);
  FSDP_LAUNCHED();
  cudaEvent_t sent = ce_event(c);
  FSDP_CUDA(cudaEventRecord(sent, cs));
  coll_wait_slot_kernel<<<1, 32, 0, s>>>(p, 1);
  FSDP_LAUNCHED();
  if (c->timing) { FSDP_CUDA(cudaEventRecord(b, s)); c->timed[FSDP_KIND_AR].emplace_back(a, b); }
  if (!direct) {
    // 4. out = (accumulate ? out : 0) + gathered
    const int grid = (int)std::min<int64_t>(std::max<int64_t>((n / 4 + 255) / 256, 1), (int64_t)kNumSMs * 4);
    ar_epilogue_kernel<<<grid, 256, 0, s>>>((const float*)(mine + gather_off), out, n, accumulate ? 1 : 0);
    FSDP_LAUNCHED();
  }
  FSDP_CUDA(cudaStreamWaitEvent(s, sent, 0));   // my input and result slot are free once my copies are done
  return 0;
}

extern "C" int fsdp_reduce_scatter_ce(fsdp_comm_t* c, int channel, int gsize, int gstride,
                                      int64_t src_off, int src_dtype, int64_t n,
                                      int64_t stage_off, float* out, float prediv, float postdiv,
                                      int accumulate, void* stream) {
  return fsdp_reduce_scatter_ce_out(c, channel, gsize, gstride, src_off, src_dtype, n, stage_off, out,
                                    FSDP_F32, prediv, postdiv, accumulate, stream);
}
extern "C" int fsdp_allreduce_ce(fsdp_comm_t* c, int channel, int gsize, int gstride, const void* in,
                                 int src_dtype, int64_t n, int64_t stage_off, int64_t gather_off,
                                 float* out, float postdiv, int accumulate, void* stream) {
  if (int rc = validate_group(c, channel, gsize, gstride)) return rc;
  if (c->emulated) return fail(FSDP_E_UNSUPPORTED, "copy-engine collectives need a real communicator");
  const int is = elem_size(src_dtype);
  if (n < 0 || !in || !out || !is) return fail(FSDP_E_INVALID, "fsdp_allreduce_ce: bad args");
  if (!(postdiv > 0.f)) return fail(FSDP_E_INVALID, "postdiv must be > 0");
  int64_t ch = (n + gsize - 1) / gsize;
  ch = (ch + kVec - 1) / kVec * kVec;
  if (int rc = check_range(c, stage_off, ch * gsize * is, "fsdp_allreduce_ce(stage)")) return rc;
  if (int rc = check_range(c, gather_off, ch * gsize * 4, "fsdp_allreduce_ce(gather)")) return rc;
  return allreduce_ce_impl(c, channel, gsize, gstride, in, src_dtype, n, stage_off, gather_off, out, -1,
                           postdiv, accumulate, (cudaStream_t)stream);
}

extern "C" int fsdp_allreduce_ce_pool(fsdp_comm_t* c, int channel, int gsize, int gstride, const void* in,
                                      int src_dtype, int64_t n, int64_t stage_off, int64_t out_off,
                                      float postdiv, void* stream) {
  if (int rc = validate_group(c, channel, gsize, gstride)) return rc;
  if (c->emulated) return fail(FSDP_E_UNSUPPORTED, "copy-engine collectives need a real communicator");
  const int is = elem_size(src_dtype);
  if (n < 0 || !in || !is) return fail(FSDP_E_INVALID, "fsdp_allreduce_ce_pool: bad args");
  if (!(postdiv > 0.f)) return fail(FSDP_E_INVALID, "postdiv must be > 0");
  if (out_off % 16) return fail(FSDP_E_INVALID, "fsdp_allreduce_ce_pool: out region must be 16-byte aligned");
  int64_t ch = (n + gsize - 1) / gsize;
  ch = (ch + kVec - 1) / kVec * kVec;
  if (int rc = check_range(c, stage_off, ch * gsize * is, "fsdp_allreduce_ce_pool(stage)")) return rc;
  if (int rc = check_range(c, out_off, n * 4, "fsdp_allreduce_ce_pool(out)")) return rc;
  return allreduce_ce_impl(c, channel, gsize, gstride, in, src_dtype, n, stage_off, -1,
                           (float*)(c->bases[c->rank] + out_off), out_off, postdiv, 0, (cudaStream_t)stream);
}

extern "C" int fsdp_allreduce(fsdp_comm_t* c, int channel, int gsize, int gstride,
                              const void* const* ins, int src_dtype, int64_t n, int64_t stage_off,
                              int64_t gather_off, float* const* outs, float postdiv, int accumulate,
                              void* stream) {
  if (int rc = validate_group(c, channel, gsize, gstride)) return rc;
  if (n < 0 || !ins || !outs) return fail(FSDP_E_INVALID, "fsdp_allreduce: bad args");
  const int is = elem_size(src_dtype);
  if (!is) return fail(FSDP_E_INVALID, "fsdp_allreduce: bad dtype");
  if (!(postdiv > 0.f)) return fail(FSDP_E_INVALID, "postdiv must be > 0");
  int64_t ch = (n + gsize - 1) / gsize;
  ch = (ch + kVec - 1) / kVec * kVec;
  if (int rc = check_range(c, stage_off, ch * gsize * is, "fsdp_allreduce(stage)")) return rc;
  if (int rc = check_range(c, gather_off, ch * gsize * 4, "fsdp_allreduce(gather)")) return rc;
  CollParams p;
  fill_common(c, p, channel, gsize, gstride, n);
  for (int e = 0; e < nranks_args(c); ++e) { p.in[e] = ins[e]; p.out[e] = outs[e]; }
  p.off_a = stage_off; p.off_b = gather_off;
  p.postdiv = postdiv; p.accumulate = accumulate ? 1 : 0;
  const int grid = grid_for(c, ch);
  cudaStream_t s = (cudaStream_t)stream;
  if (src_dtype == FSDP_BF16)
    return launch(c, allreduce_kernel<__nv_bfloat16>, p, grid, kCommThreads, s);
  return launch(c, allreduce_kernel<float>, p, grid, kCommThreads, s);
}

extern "C" int fsdp_allreduce_scalar(fsdp_comm_t* c, const float* const* ins, float* const* outs,
                                     void* stream) {
  if (int rc = validate_group(c, FSDP_CH_SCALAR, c ? c->world : 1, 1)) return rc;
  if (!ins || !outs) return fail(FSDP_E_INVALID, "fsdp_allreduce_scalar: bad args");
  CollParams p;
  fill_common(c, p, FSDP_CH_SCALAR, c->world, 1, 1);
  for (int e = 0; e < nranks_args(c); ++e) { p.in[e] = ins[e]; p.out[e] = outs[e]; }
  return launch(c, scalar_allreduce_kernel, p, 1, 32, (cudaStream_t)stream);
}

// ------------------------------------------------------ low-latency path ---
extern "C" int64_t fsdp_ll_bytes(int gsize, int64_t n, int dtype) {
  const int es = elem_size(dtype);
  if (gsize < 1 || n < 0 || !es) return -1;
  const int64_t nl = (n * es + 7) / 8;
  const int64_t blocks = (nl + kLLBlock - 1) / kLLBlock;      // whole line blocks (ll_line layout)
  return 2 * (int64_t)gsize * blocks * kLLBlock * 16;
}

static int ll_grid(fsdp_comm_t* c, int64_t nl, int kind) {
  const int cap = c->kind_ctas[kind] > 0 ? c->kind_ctas[kind] : c->max_ctas;
  int g = (int)std::min<int64_t>(std::max<int64_t>((nl + 2 * kLLThreads - 1) / (2 * kLLThreads), 1), cap);
  if (c->emulated) g = std::min(g, std::max(1, 128 / c->world));
  return g;
}

extern "C" int fsdp_allgather_ll(fsdp_comm_t* c, int channel, int gsize, int gstride,
                                 const void* const* shards, int src_dtype, int64_t n,
                                 int64_t dst_off, int dst_dtype, int64_t ll_off, void* stream) {
  if (int rc = validate_group(c, channel, gsize, gstride)) return rc;
  if (n < 0 || !shards) return fail(FSDP_E_INVALID, "fsdp_allgather_ll: bad args");
  const int os = elem_size(dst_dtype);
  if (!os || !elem_size(src_dtype)) return fail(FSDP_E_INVALID, "fsdp_allgather_ll: bad dtype");
  if (int rc = check_range(c, dst_off, n * gsize * os, "fsdp_allgather_ll(dst)")) return rc;
  if (ll_off % 16) return fail(FSDP_E_INVALID, "fsdp_allgather_ll: LL region must be 16-byte aligned");
  if (int rc = check_range(c, ll_off, fsdp_ll_bytes(gsize, n, dst_dtype), "fsdp_allgather_ll(ll)")) return rc;
  CollParams p;
  fill_common(c, p, channel, gsize, gstride, n);
  for (int e = 0; e < nranks_args(c); ++e) p.in[e] = shards[e];
  p.off_a = dst_off;
  p.off_b = ll_off;
  const int grid = ll_grid(c, (n * os + 7) / 8, FSDP_KIND_AG);
  cudaStream_t s = (cudaStream_t)stream;
  if (src_dtype == FSDP_F32 && dst_dtype == FSDP_BF16)
    return launch(c, allgather_ll_kernel<float, __nv_bfloat16>, p, grid, kLLThreads, s);
  if (src_dtype == FSDP_F32 && dst_dtype == FSDP_F32)
    return launch(c, allgather_ll_kernel<float, float>, p, grid, kLLThreads, s);
  if (src_dtype == FSDP_BF16 && dst_dtype == FSDP_BF16)
    return launch(c, allgather_ll_kernel<__nv_bfloat16, __nv_bfloat16>, p, grid, kLLThreads, s);
  return launch(c, allgather_ll_kernel<__nv_bfloat16, float>, p, grid, kLLThreads, s);
}

extern "C" int fsdp_reduce_scatter_ll(fsdp_comm_t* c, int channel, int gsize, int gstride,
                                      const void* const* flats, int src_dtype, int64_t n,
                                      int64_t ll_off, float* const* outs, float prediv,
                                      float postdiv, int accumulate, void* stream) {
  if (int rc = validate_group(c, channel, gsize, gstride)) return rc;
  if (n < 0 || !flats || !outs) return fail(FSDP_E_INVALID, "fsdp_reduce_scatter_ll: bad args");
  const int is = elem_size(src_dtype);
  if (!is) return fail(FSDP_E_INVALID, "fsdp_reduce_scatter_ll: bad dtype");
  if (!(prediv > 0.f) || !(postdiv > 0.f)) return fail(FSDP_E_INVALID, "divisors must be > 0");
  if (ll_off % 16) return fail(FSDP_E_INVALID, "fsdp_reduce_scatter_ll: LL region must be 16-byte aligned");
  if (int rc = check_range(c, ll_off, fsdp_ll_bytes(gsize, n, src_dtype), "fsdp_reduce_scatter_ll")) return rc;
  CollParams p;
  fill_common(c, p, channel, gsize, gstride, n);
  p.rot = c->misorder_rs && gsize > 1 ? 1 : 0;
  for (int e = 0; e < nranks_args(c); ++e) { p.in[e] = flats[e]; p.out[e] = outs[e]; }
  p.off_b = ll_off;
  p.prediv = prediv; p.postdiv = postdiv; p.accumulate = accumulate ? 1 : 0;
  const int grid = ll_grid(c, (n * is + 7) / 8, FSDP_KIND_RS);
  cudaStream_t s = (cudaStream_t)stream;
  const int mw = gsize <= 2 ? 2 : (gsize <= 4 ? 4 : 8);
#define RSLL(T, W) launch(c, reduce_scatter_ll_kernel<T, W>, p, grid, kLLThreads, s)
  if (src_dtype == FSDP_BF16)
    return mw == 2 ? RSLL(__nv_bfloat16, 2) : (mw == 4 ? RSLL(__nv_bfloat16, 4) : RSLL(__nv_bfloat16, 8));
  return mw == 2 ? RSLL(float, 2) : (mw == 4 ? RSLL(float, 4) : RSLL(float, 8));
#undef RSLL
}

// ------------------------------------------------------ VMM pool + NVLS ----
extern "C" int fsdp_nvls_supported(int device) { return vmm::multicast_supported(device); }

extern "C" int fsdp_comm_create_vmm(int rank, int world, int64_t pool_bytes, int max_ctas,
                                    int handle_type, fsdp_comm_t** out) {
  if (!out) return fail(FSDP_E_INVALID, "null out");
  if (world < 1 || world > FSDP_MAX_RANKS || rank < 0 || rank >= world)
    return fail(FSDP_E_INVALID, "rank/world out of range (world <= 8)");
  if (max_ctas < 1 || max_ctas > FSDP_MAX_CTAS - 1) return fail(FSDP_E_INVALID, "max_ctas out of range (1..159)");
  if (handle_type != vmm::kFabric && handle_type != vmm::kPosixFd)
    return fail(FSDP_E_INVALID, "handle_type must be FSDP_HANDLE_FABRIC or FSDP_HANDLE_POSIX_FD");
  int device = 0;
  FSDP_CUDA(cudaGetDevice(&device));
  size_t gran = 0;
  if (int rc = vmm::granularity(device, handle_type, world, &gran)) return rc;
  if (pool_bytes < kReserved) pool_bytes = kReserved;
  pool_bytes = (int64_t)(((size_t)pool_bytes + gran - 1) / gran * gran);
  fsdp_comm_t* c = new fsdp_comm_t();
  c->rank = rank; c->world = world; c->pool_bytes = pool_bytes; c->max_ctas = max_ctas;
  c->device = device;
  c->vmm = true;
  c->handle_type = handle_type;
  if (int rc = vmm::create(device, (size_t)pool_bytes, handle_type, &c->own_map)) { delete c; return rc; }
  c->pool = (char*)c->own_map.va;
  cudaError_t e = cudaMemset(c->pool, 0, kReserved);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { vmm::unmap(&c->own_map); delete c; return check_cuda(e, "cudaMemset(pool)"); }
  c->bases[rank] = c->pool;
  c->opened[rank] = true;
  *out = c;
  return 0;
}

extern "C" int fsdp_comm_export_pool(fsdp_comm_t* c, void* handle_out) {
  if (!c || !handle_out) return fail(FSDP_E_INVALID, "null argument");
  if (!c->vmm) return fail(FSDP_E_UNSUPPORTED, "not a VMM communicator");
  return vmm::export_handle(c->own_map.handle, c->handle_type, handle_out);
}

extern "C" int fsdp_comm_import_pool(fsdp_comm_t* c, int r, const void* handle) {
  if (!c || !handle) return fail(FSDP_E_INVALID, "null argument");
  if (!c->vmm) return fail(FSDP_E_UNSUPPORTED, "not a VMM communicator");
  if (r < 0 || r >= c->world || r == c->rank) return fail(FSDP_E_INVALID, "bad peer rank");
  if (c->opened[r]) return 0;
  if (int rc = vmm::import_map(c->device, handle, c->handle_type, (size_t)c->pool_bytes, &c->peer_map[r]))
    return rc;
  c->bases[r] = (char*)c->peer_map[r].va;
  c->opened[r] = true;
  return 0;
}

static int nvls_check(fsdp_comm_t* c, int gsize) {
  if (!c) return fail(FSDP_E_INVALID, "null communicator");
  if (!c->vmm) return fail(FSDP_E_UNSUPPORTED, "NVLS needs a VMM communicator (fsdp_comm_create_vmm)");
  if (gsize < 2 || c->world % gsize) return fail(FSDP_E_INVALID, "NVLS group size must divide the world");
  if (c->mc_gsize && c->mc_gsize != gsize) return fail(FSDP_E_INVALID, "NVLS group already set up");
  return 0;
}

extern "C" int fsdp_nvls_create(fsdp_comm_t* c, int gsize, void* handle_out) {
  if (int rc = nvls_check(c, gsize)) return rc;
  if (c->rank % gsize != 0) return fail(FSDP_E_INVALID, "fsdp_nvls_create: only the group leader creates");
  if (!handle_out) return fail(FSDP_E_INVALID, "null handle_out");
  if (!c->mc_handle) {
    if (int rc = vmm::mc_create(gsize, (size_t)c->pool_bytes, c->handle_type, &c->mc_handle)) return rc;
  }
  c->mc_gsize = gsize;
  return vmm::export_handle(c->mc_handle, c->handle_type, handle_out);
}

extern "C" int fsdp_nvls_import(fsdp_comm_t* c, int gsize, const void* handle) {
  if (int rc = nvls_check(c, gsize)) return rc;
  if (c->rank % gsize == 0) return fail(FSDP_E_INVALID, "fsdp_nvls_import: the leader creates");
  if (!handle) return fail(FSDP_E_INVALID, "null handle");
  if (!c->mc_handle)
    if (int rc = vmm::mc_import(handle, c->handle_type, &c->mc_handle)) return rc;
  c->mc_gsize = gsize;
  return 0;
}

extern "C" int fsdp_nvls_add_device(fsdp_comm_t* c) {
  if (!c || !c->mc_handle) return fail(FSDP_E_INVALID, "fsdp_nvls_add_device: no multicast object");
  if (c->mc_added) return 0;
  if (int rc = vmm::mc_add_device(c->mc_handle, c->device)) return rc;
  c->mc_added = true;
  return 0;
}

extern "C" int fsdp_nvls_bind(fsdp_comm_t* c) {
  if (!c || !c->mc_added) return fail(FSDP_E_INVALID, "fsdp_nvls_bind: add the device first");
  if (c->mc_map.va) return 0;
  return vmm::mc_bind_map(c->mc_handle, c->device, c->own_map, &c->mc_map);
}

extern "C" int fsdp_nvls_group_size(fsdp_comm_t* c) {
  return (c && c->mc_map.va) ? c->mc_gsize : 0;
}

extern "C" int fsdp_allgather_nvls(fsdp_comm_t* c, int channel, int gsize, int gstride,
                                   const void* shard, int src_dtype, int64_t n, int64_t dst_off,
                                   int dst_dtype, void* stream) {
  if (int rc = validate_group(c, channel, gsize, gstride)) return rc;
  const int os = elem_size(dst_dtype);
  if (n < 0 || !shard || !os || !elem_size(src_dtype))
    return fail(FSDP_E_INVALID, "fsdp_allgather_nvls: bad args");
  if (int rc = check_range(c, dst_off, n * gsize * os, "fsdp_allgather_nvls")) return rc;
  const int64_t my_off = dst_off + (int64_t)(c->rank % gsize) * n * os;
  const bool usable = c->mc_map.va && gstride == 1 && gsize == c->mc_gsize && n % kVec == 0 &&
                      aligned16(shard) && my_off % 16 == 0;
  if (!usable) {   // same contract through the unicast SM kernel
    const void* shards[1] = {shard};
    return fsdp_allgather(c, channel, gsize, gstride, shards, src_dtype, n, dst_off, dst_dtype, stream);
  }
  CollParams p;
  fill_common(c, p, channel, gsize, gstride, n);
  p.in[0] = shard;
  p.off_a = dst_off;
  const int grid = grid_for(c, n, FSDP_KIND_AG);
  void* k = src_dtype == FSDP_F32
                ? (dst_dtype == FSDP_BF16 ? (void*)allgather_nvls_kernel<float, __nv_bfloat16>
                                          : (void*)allgather_nvls_kernel<float, float>)
                : (dst_dtype == FSDP_BF16 ? (void*)allgather_nvls_kernel<__nv_bfloat16, __nv_bfloat16>
                                          : (void*)allgather_nvls_kernel<__nv_bfloat16, float>);
  return launch_split(c, FSDP_KIND_AG, k, p, grid, kCommThreads, 0, (cudaStream_t)stream);
}
