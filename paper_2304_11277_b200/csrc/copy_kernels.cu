// Flat-parameter layout kernels: flatten (multi-tensor gather + pad + cast,
// optional accumulate), unflatten (multi-tensor scatter + cast), shard copy
// and elementwise cast.  HBM-bound: 8-element (16/32-byte) vectors,
// streaming loads, grid = a multiple of the 148 SMs.
//
// Reference semantics: flatparam.py:88-93 (offsets, padding), :139-147
// (shard), :159-164 (views), :167-191 (gradient write-back);
// deferred_init.py:156-176 (materialise by unit), engine.py:661-662 (cast).
#include "common.cuh"

namespace fsdp {

struct TensorTable {
  const void* ptr[FSDP_MAX_TENSORS];   // src (flatten) or dst (unflatten)
  int64_t off[FSDP_MAX_TENSORS + 1];   // flat offsets; off[n] = end of last
  int64_t numel[FSDP_MAX_TENSORS];
  int n;
};

constexpr int kCopyThreads = 256;
constexpr int kCopyUnroll = 4;

// Largest i with off[i] <= p (tensors sorted by offset, non-overlapping).
__device__ __forceinline__ int find_tensor(const TensorTable& t, int64_t p, int hint) {
  int i = hint;
  while (i + 1 < t.n && t.off[i + 1] <= p) ++i;   // monotone per thread
  if (i < t.n && t.off[i] <= p) return i;
  int lo = 0, hi = t.n - 1;                       // fallback binary search
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (t.off[mid] <= p) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// flat[p] for p in [0, psi): value of the tensor covering p, else 0.
template <typename Tin, typename Tout>
__global__ void __launch_bounds__(kCopyThreads)
flatten_kernel(const __grid_constant__ TensorTable tab, Tout* __restrict__ flat, int64_t psi,
               int accumulate) {
  const int64_t nvec = (psi + 7) >> 3;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int hint = 0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += stride) {
    const int64_t p0 = v << 3;
    int ti = find_tensor(tab, p0, hint);
    hint = ti;
    const Tin* src = (const Tin*)tab.ptr[ti];
    const int64_t t0 = tab.off[ti], t1 = t0 + tab.numel[ti];
    const bool full_vec = p0 + 8 <= psi;
    V8F x;
    if (full_vec && p0 >= t0 && p0 + 8 <= t1 && src != nullptr && aligned16(src + (p0 - t0))) {
      x = load8<Tin>(src + (p0 - t0), LD_NC);
    } else {
      // mixed vector: elements may span tensors / padding / unaligned sources
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int64_t p = p0 + k;
        float val = 0.f;
        if (p < psi) {
          int tk = find_tensor(tab, p, ti);
          const int64_t a = tab.off[tk];
          if (p >= a && p < a + tab.numel[tk] && tab.ptr[tk] != nullptr)
            val = to_f<Tin>(((const Tin*)tab.ptr[tk])[p - a]);
        }
        x.v[k] = val;
      }
    }
    Tout* dst = flat + p0;
    if (full_vec && aligned16(dst)) {
      if (accumulate) {
        V8F y = load8<Tout>(dst, LD_PLAIN);
#pragma unroll
        for (int k = 0; k < 8; ++k) x.v[k] = __fadd_rn(y.v[k], x.v[k]);
      }
      store8<Tout>(dst, pack8<Tout>(x));
    } else {
      for (int k = 0; k < 8 && p0 + k < psi; ++k) {
        float val = x.v[k];
        if (accumulate) val = __fadd_rn(to_f<Tout>(dst[k]), val);
        dst[k] = from_f<Tout>(val);
      }
    }
  }
}

// dst_i[j] = flat[off_i + j]
template <typename Tin, typename Tout>
__global__ void __launch_bounds__(kCopyThreads)
unflatten_kernel(const Tin* __restrict__ flat, const __grid_constant__ TensorTable tab) {
  const int64_t end = tab.off[tab.n];
  const int64_t v0 = tab.off[0] >> 3;
  const int64_t nvec = ((end + 7) >> 3) - v0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int hint = 0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += stride) {
    const int64_t p0 = (v0 + v) << 3;
    int ti = find_tensor(tab, p0 < tab.off[0] ? tab.off[0] : p0, hint);
    hint = ti;
    const int64_t t0 = tab.off[ti], t1 = t0 + tab.numel[ti];
    Tout* dst = (Tout*)tab.ptr[ti];
    if (p0 >= t0 && p0 + 8 <= t1 && aligned16(flat + p0) && aligned16(dst + (p0 - t0))) {
      store8<Tout>(dst + (p0 - t0), pack8<Tout>(load8<Tin>(flat + p0, LD_NC)));
    } else {
      for (int k = 0; k < 8; ++k) {
        const int64_t p = p0 + k;
        if (p < tab.off[0] || p >= end) continue;
        int tk = find_tensor(tab, p, ti);
        const int64_t a = tab.off[tk];
        if (p >= a && p < a + tab.numel[tk])
          ((Tout*)tab.ptr[tk])[p - a] = from_f<Tout>(to_f<Tin>(flat[p]));
      }
    }
  }
}

// dst[i] = cast(src[i]); vector path when both ends are 16B-aligned.
template <typename Tin, typename Tout>
__global__ void __launch_bounds__(kCopyThreads)
cast_kernel(const Tin* __restrict__ src, Tout* __restrict__ dst, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (aligned16(src) && aligned16(dst)) {
    const int64_t nvec = n >> 3;
    int64_t v = tid;
    for (; v + (kCopyUnroll - 1) * stride < nvec; v += kCopyUnroll * stride) {
      V8F x[kCopyUnroll];
#pragma unroll
      for (int u = 0; u < kCopyUnroll; ++u) x[u] = load8<Tin>(src + ((v + u * stride) << 3), LD_NC);
#pragma unroll
      for (int u = 0; u < kCopyUnroll; ++u) store8<Tout>(dst + ((v + u * stride) << 3), pack8<Tout>(x[u]));
    }
    for (; v < nvec; v += stride) store8<Tout>(dst + (v << 3), pack8<Tout>(load8<Tin>(src + (v << 3), LD_NC)));
    for (int64_t i = (nvec << 3) + tid; i < n; i += stride) dst[i] = from_f<Tout>(to_f<Tin>(src[i]));
  } else {
    for (int64_t i = tid; i < n; i += stride) dst[i] = from_f<Tout>(to_f<Tin>(src[i]));
  }
}

static int copy_grid(int64_t nvec) {
  int64_t blocks = (nvec + kCopyThreads - 1) / kCopyThreads;
  const int64_t cap = (int64_t)kNumSMs * 8;   // 8 x 256-thread CTAs per SM
  if (blocks > cap) blocks = cap;
  return blocks < 1 ? 1 : (int)blocks;
}

template <typename Tin, typename Tout>
static void launch_flatten(const TensorTable& t, void* flat, int64_t psi, int acc, cudaStream_t s) {
  flatten_kernel<Tin, Tout><<<copy_grid((psi + 7) >> 3), kCopyThreads, 0, s>>>(t, (Tout*)flat, psi, acc);
}
template <typename Tin, typename Tout>
static void launch_unflatten(const void* flat, const TensorTable& t, cudaStream_t s) {
  int64_t span = ((t.off[t.n] + 7) >> 3) - (t.off[0] >> 3);
  unflatten_kernel<Tin, Tout><<<copy_grid(span), kCopyThreads, 0, s>>>((const Tin*)flat, t);
}
template <typename Tin, typename Tout>
static void launch_cast(const void* src, void* dst, int64_t n, cudaStream_t s) {
  cast_kernel<Tin, Tout><<<copy_grid((n + 7) >> 3), kCopyThreads, 0, s>>>((const Tin*)src, (Tout*)dst, n);
}

#define DISPATCH2(sd, dd, FN, ...)                                                         \
  do {                                                                                     \
    if ((sd) == FSDP_F32 && (dd) == FSDP_F32) FN<float, float>(__VA_ARGS__);               \
    else if ((sd) == FSDP_F32 && (dd) == FSDP_BF16) FN<float, __nv_bfloat16>(__VA_ARGS__);  \
    else if ((sd) == FSDP_BF16 && (dd) == FSDP_F32) FN<__nv_bfloat16, float>(__VA_ARGS__);  \
    else if ((sd) == FSDP_BF16 && (dd) == FSDP_BF16)                                       \
      FN<__nv_bfloat16, __nv_bfloat16>(__VA_ARGS__);                                       \
    else return fail(FSDP_E_INVALID, "unsupported dtype pair");                            \
  } while (0)

// Validate and sort-check a tensor table (offsets ascending, non-overlapping).
static int build_table(TensorTable& t, const void* const* ptrs, const int64_t* numels,
                       const int64_t* offsets, int n, int64_t limit, const char* who) {
  if (n < 1 || n > FSDP_MAX_TENSORS)
    return fail(FSDP_E_INVALID, std::string(who) + ": tensor count out of range");
  t.n = n;
  for (int i = 0; i < n; ++i) {
    t.ptr[i] = ptrs ? ptrs[i] : nullptr;
    t.off[i] = offsets[i];
    t.numel[i] = numels[i];
    if (numels[i] < 0 || offsets[i] < 0)
      return fail(FSDP_E_INVALID, std::string(who) + ": negative offset/numel");
    if (i > 0 && offsets[i] < offsets[i - 1] + numels[i - 1])
      return fail(FSDP_E_INVALID, std::string(who) + ": offsets must be ascending and disjoint");
  }
  t.off[n] = offsets[n - 1] + numels[n - 1];
  if (limit >= 0 && t.off[n] > limit)
    return fail(FSDP_E_INVALID, std::string(who) + ": tensors exceed the flat buffer");
  return 0;
}

}  // namespace fsdp

using namespace fsdp;

extern "C" int fsdp_flatten(const void* const* srcs, const int64_t* numels, const int64_t* offsets,
                            int n_tensors, int src_dtype, void* flat, int64_t psi, int flat_dtype,
                            int accumulate, void* stream) {
  if (psi < 0 || (psi > 0 && flat == nullptr)) return fail(FSDP_E_INVALID, "fsdp_flatten: bad flat");
  if (psi == 0) return 0;
  TensorTable t;
  if (n_tensors == 0) {   // pure zero-fill of the padding-only buffer
    t.n = 1; t.ptr[0] = nullptr; t.off[0] = 0; t.numel[0] = 0; t.off[1] = 0;
  } else if (int rc = build_table(t, srcs, numels, offsets, n_tensors, psi, "fsdp_flatten")) {
    return rc;
  }
  cudaStream_t s = (cudaStream_t)stream;
  DISPATCH2(src_dtype, flat_dtype, launch_flatten, t, flat, psi, accumulate, s);
  FSDP_LAUNCHED();
  return 0;
}

extern "C" int fsdp_unflatten(const void* flat, int flat_dtype, void* const* dsts,
                              const int64_t* numels, const int64_t* offsets, int n_tensors,
                              int dst_dtype, void* stream) {
  if (n_tensors == 0) return 0;
  TensorTable t;
  if (int rc = build_table(t, (const void* const*)dsts, numels, offsets, n_tensors, -1,
                           "fsdp_unflatten"))
    return rc;
  for (int i = 0; i < n_tensors; ++i)
    if (!dsts[i] && numels[i] > 0) return fail(FSDP_E_INVALID, "fsdp_unflatten: null dst");
  if (t.off[t.n] == t.off[0]) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  DISPATCH2(flat_dtype, dst_dtype, launch_unflatten, flat, t, s);
  FSDP_LAUNCHED();
  return 0;
}

extern "C" int fsdp_cast(const void* src, int src_dtype, void* dst, int dst_dtype, int64_t n,
                         void* stream) {
  if (n < 0) return fail(FSDP_E_INVALID, "fsdp_cast: negative n");
  if (n == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  DISPATCH2(src_dtype, dst_dtype, launch_cast, src, dst, n, s);
  FSDP_LAUNCHED();
  return 0;
}

extern "C" int fsdp_shard_copy(const void* flat, void* shard, int64_t shard_numel, int shard_index,
                               int dtype, void* stream) {
  if (shard_index < 0 || shard_numel < 0) return fail(FSDP_E_INVALID, "fsdp_shard_copy: bad args");
  const int es = elem_size(dtype);
  if (!es) return fail(FSDP_E_INVALID, "fsdp_shard_copy: bad dtype");
  const char* src = (const char*)flat + (int64_t)shard_index * shard_numel * es;
  return fsdp_cast(src, dtype, shard, dtype, shard_numel, stream);
}
