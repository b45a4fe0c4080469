// Flat-parameter layout kernels: flatten (multi-tensor gather + pad + cast,
// optional accumulate), unflatten (multi-tensor scatter + cast), shard copy
// and elementwise cast.  HBM-bound: warp-interleaved 8-element vectors
// (every warp instruction moves one contiguous 256/512-byte span), streaming
// loads, grid = one resident wave over the 148 SMs.
//
// Reference semantics: flatparam.py:88-93 (offsets, padding), :139-147
// (shard), :159-164 (views), :167-191 (gradient write-back);
// deferred_init.py:156-176 (materialise by unit), engine.py:661-662 (cast).
#include "common.cuh"

#include <cstdlib>
#include <mutex>
#include <type_traits>

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

// ---- warp-interleaved 8-element vectors --------------------------------
// Vector v of a kernel covers two 4-element quads: elements [a, a+4) and
// [a+128, a+132) with a = (v/32)*256 + (v%32)*4.  A warp's 32 vectors tile
// 256 consecutive elements, and every load or store INSTRUCTION of the warp
// touches one contiguous span (32 x 16 B for fp32, 32 x 8 B for bf16): full
// 32-byte sectors, no half-sector writes for the 4-byte side of a cast.
__device__ __forceinline__ int64_t quad0(int64_t v) { return ((v >> 5) << 8) + ((v & 31) << 2); }
constexpr int64_t kQuadGap = 128;
constexpr int64_t kVecSpan = kQuadGap + 4;        // a .. a+132

template <typename T> struct Quad;
template <> struct Quad<float> { uint4 q; };
template <> struct Quad<__nv_bfloat16> { uint2 q; };

template <typename T> __device__ __forceinline__ Quad<T> ldq(const T* p, bool nc);
template <> __device__ __forceinline__ Quad<float> ldq<float>(const float* p, bool nc) {
  Quad<float> r;
  if (nc) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(r.q.x), "=r"(r.q.y), "=r"(r.q.z), "=r"(r.q.w) : "l"(p));
  else asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                    : "=r"(r.q.x), "=r"(r.q.y), "=r"(r.q.z), "=r"(r.q.w) : "l"(p));
  return r;
}
template <> __device__ __forceinline__ Quad<__nv_bfloat16> ldq<__nv_bfloat16>(const __nv_bfloat16* p, bool nc) {
  Quad<__nv_bfloat16> r;
  if (nc) asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.q.x), "=r"(r.q.y) : "l"(p));
  else asm volatile("ld.global.v2.u32 {%0,%1}, [%2];" : "=r"(r.q.x), "=r"(r.q.y) : "l"(p));
  return r;
}
template <typename T> __device__ __forceinline__ void stq(T* p, const Quad<T>& v);
template <> __device__ __forceinline__ void stq<float>(float* p, const Quad<float>& v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "r"(v.q.x), "r"(v.q.y), "r"(v.q.z), "r"(v.q.w) : "memory");
}
template <> __device__ __forceinline__ void stq<__nv_bfloat16>(__nv_bfloat16* p, const Quad<__nv_bfloat16>& v) {
  asm volatile("st.global.v2.u32 [%0], {%1,%2};" :: "l"(p), "r"(v.q.x), "r"(v.q.y) : "memory");
}
template <typename T> __device__ __forceinline__ float4 q2f(const Quad<T>& x);
template <> __device__ __forceinline__ float4 q2f<float>(const Quad<float>& x) {
  return make_float4(__uint_as_float(x.q.x), __uint_as_float(x.q.y), __uint_as_float(x.q.z),
                     __uint_as_float(x.q.w));
}
template <> __device__ __forceinline__ float4 q2f<__nv_bfloat16>(const Quad<__nv_bfloat16>& x) {
  return make_float4(bf16lo(x.q.x), bf16hi(x.q.x), bf16lo(x.q.y), bf16hi(x.q.y));
}
template <typename T> __device__ __forceinline__ Quad<T> f2q(const float4& x);
template <> __device__ __forceinline__ Quad<float> f2q<float>(const float4& x) {
  Quad<float> r;
  r.q = make_uint4(__float_as_uint(x.x), __float_as_uint(x.y), __float_as_uint(x.z), __float_as_uint(x.w));
  return r;
}
template <> __device__ __forceinline__ Quad<__nv_bfloat16> f2q<__nv_bfloat16>(const float4& x) {
  Quad<__nv_bfloat16> r;
  r.q = make_uint2(pack_bf16x2(x.x, x.y), pack_bf16x2(x.z, x.w));
  return r;
}
template <typename Tin, typename Tout>
__device__ __forceinline__ Quad<Tout> convq(const Quad<Tin>& x) {
  if constexpr (std::is_same<Tin, Tout>::value) return x;
  else return f2q<Tout>(q2f<Tin>(x));
}
template <typename T> __device__ __forceinline__ bool qaligned(const T* p) {
  return (reinterpret_cast<uintptr_t>(p) & (4 * sizeof(T) - 1)) == 0;
}
__device__ __forceinline__ int64_t vec_elem(int64_t a, int k) { return a + (k < 4 ? k : kQuadGap + k - 4); }
__device__ __forceinline__ float f4get(const float4& f, int k) {
  return k == 0 ? f.x : (k == 1 ? f.y : (k == 2 ? f.z : f.w));
}
__device__ __forceinline__ void f4set(float4& f, int k, float v) {
  if (k == 0) f.x = v; else if (k == 1) f.y = v; else if (k == 2) f.z = v; else f.w = v;
}

// Element-wise slow path of flatten for one vector at quad start a: its
// elements may span tensors / padding / unaligned sources.
template <typename Tin>
__device__ __noinline__ void gather_slow(const TensorTable& tab, int64_t a, int64_t psi, int ti,
                                         float4& lo, float4& hi) {
  lo = hi = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int k = 0; k < 8; ++k) {
    const int64_t p = vec_elem(a, k);
    float val = 0.f;
    if (p < psi) {
      int tk = find_tensor(tab, p, ti);
      const int64_t o = tab.off[tk];
      if (p >= o && p < o + tab.numel[tk] && tab.ptr[tk] != nullptr)
        val = to_f<Tin>(((const Tin*)tab.ptr[tk])[p - o]);
    }
    if (k < 4) f4set(lo, k, val); else f4set(hi, k - 4, val);
  }
}

// flat[p] for p in [0, psi): value of the tensor covering p, else 0 (with
// kAcc: flat[p] += value, padding untouched).  Each thread handles U
// grid-strided vectors per iteration and issues all their loads (kept
// packed) before any store.
template <typename Tin, typename Tout, bool kAcc, int U>
__global__ void __launch_bounds__(kCopyThreads)
flatten_kernel(const __grid_constant__ TensorTable tab, Tout* __restrict__ flat, int64_t psi) {
  const int64_t nvec = ((psi + 255) >> 8) << 5;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool flat_al = qaligned(flat);
  int hint = 0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += U * stride) {
    Quad<Tin> x[U][2];
    Quad<Tout> y[U][2];
    bool fast[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t vu = v + u * stride;
      fast[u] = false;
      if (vu >= nvec) break;
      const int64_t a = quad0(vu);
      if (a >= psi) continue;
      const int ti = find_tensor(tab, a, hint);
      hint = ti;
      const Tin* src = (const Tin*)tab.ptr[ti];
      const int64_t t0 = tab.off[ti], t1 = t0 + tab.numel[ti];
      fast[u] = a + kVecSpan <= psi && a >= t0 && a + kVecSpan <= t1 && src != nullptr &&
                qaligned(src + (a - t0)) && flat_al;
      if (fast[u]) {
        x[u][0] = ldq<Tin>(src + (a - t0), true);
        x[u][1] = ldq<Tin>(src + (a - t0) + kQuadGap, true);
        if (kAcc) {
          y[u][0] = ldq<Tout>(flat + a, false);
          y[u][1] = ldq<Tout>(flat + a + kQuadGap, false);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t vu = v + u * stride;
      if (vu >= nvec) break;
      const int64_t a = quad0(vu);
      if (a >= psi) continue;
      if (fast[u]) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (kAcc) {
            float4 f = q2f<Tin>(x[u][h]);
            const float4 b = q2f<Tout>(y[u][h]);
            f.x = __fadd_rn(b.x, f.x); f.y = __fadd_rn(b.y, f.y);
            f.z = __fadd_rn(b.z, f.z); f.w = __fadd_rn(b.w, f.w);
            stq<Tout>(flat + a + h * kQuadGap, f2q<Tout>(f));
          } else {
            stq<Tout>(flat + a + h * kQuadGap, convq<Tin, Tout>(x[u][h]));
          }
        }
      } else {
        float4 lo, hi;
        gather_slow<Tin>(tab, a, psi, find_tensor(tab, a, hint), lo, hi);
        for (int k = 0; k < 8; ++k) {
          const int64_t p = vec_elem(a, k);
          if (p >= psi) continue;
          float val = k < 4 ? f4get(lo, k) : f4get(hi, k - 4);
          if (kAcc) val = __fadd_rn(to_f<Tout>(flat[p]), val);
          flat[p] = from_f<Tout>(val);
        }
      }
    }
  }
}

// dst_i[j] = flat[off_i + j]; U vectors per thread per iteration, loads
// issued before stores.  Vectors cover [off[0], off[n]) from the
// 256-element block containing off[0].
template <typename Tin, typename Tout, int U>
__global__ void __launch_bounds__(kCopyThreads)
unflatten_kernel(const Tin* __restrict__ flat, const __grid_constant__ TensorTable tab) {
  const int64_t begin = tab.off[0], end = tab.off[tab.n];
  const int64_t b0 = begin >> 8;
  const int64_t nvec = (((end + 255) >> 8) - b0) << 5;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int hint = 0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += U * stride) {
    Quad<Tin> x[U][2];
    bool fast[U];
    int tis[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t vu = v + u * stride;
      fast[u] = false;
      tis[u] = 0;
      if (vu >= nvec) break;
      const int64_t a = (b0 << 8) + quad0(vu);
      const int ti = find_tensor(tab, a < begin ? begin : a, hint);
      hint = ti;
      tis[u] = ti;
      const int64_t t0 = tab.off[ti], t1 = t0 + tab.numel[ti];
      const Tout* dst = (const Tout*)tab.ptr[ti];
      fast[u] = a >= t0 && a + kVecSpan <= t1 && qaligned(flat + a) && qaligned(dst + (a - t0));
      if (fast[u]) {
        x[u][0] = ldq<Tin>(flat + a, true);
        x[u][1] = ldq<Tin>(flat + a + kQuadGap, true);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t vu = v + u * stride;
      if (vu >= nvec) break;
      const int64_t a = (b0 << 8) + quad0(vu);
      const int ti = tis[u];
      if (fast[u]) {
        Tout* dst = (Tout*)tab.ptr[ti] + (a - tab.off[ti]);
        stq<Tout>(dst, convq<Tin, Tout>(x[u][0]));
        stq<Tout>(dst + kQuadGap, convq<Tin, Tout>(x[u][1]));
      } else {
        for (int k = 0; k < 8; ++k) {
          const int64_t p = vec_elem(a, k);
          if (p < begin || p >= end) continue;
          int tk = find_tensor(tab, p, ti);
          const int64_t o = tab.off[tk];
          if (p >= o && p < o + tab.numel[tk])
            ((Tout*)tab.ptr[tk])[p - o] = from_f<Tout>(to_f<Tin>(flat[p]));
        }
      }
    }
  }
}

// dst[i] = cast(src[i]) over the same warp-interleaved vectors.
template <typename Tin, typename Tout, int U>
__global__ void __launch_bounds__(kCopyThreads)
cast_kernel(const Tin* __restrict__ src, Tout* __restrict__ dst, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nvec = ((n + 255) >> 8) << 5;
  const bool al = qaligned(src) && qaligned(dst);
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += U * stride) {
    Quad<Tin> x[U][2];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t a = quad0(v + u * stride);
      if (al && a + kVecSpan <= n) {
        x[u][0] = ldq<Tin>(src + a, true);
        x[u][1] = ldq<Tin>(src + a + kQuadGap, true);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t vu = v + u * stride;
      if (vu >= nvec) break;
      const int64_t a = quad0(vu);
      if (al && a + kVecSpan <= n) {
        stq<Tout>(dst + a, convq<Tin, Tout>(x[u][0]));
        stq<Tout>(dst + a + kQuadGap, convq<Tin, Tout>(x[u][1]));
      } else {
        for (int k = 0; k < 8; ++k) {
          const int64_t p = vec_elem(a, k);
          if (p < n) dst[p] = from_f<Tout>(to_f<Tin>(src[p]));
        }
      }
    }
  }
}

static int resident_per_sm(const void* kernel) {
  static const void* keys[96];
  static int vals[96];
  static int used = 0;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  for (int i = 0; i < used; ++i)
    if (keys[i] == kernel) return vals[i];
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, kCopyThreads, 0) != cudaSuccess || n < 1)
    n = 2;
  if (used < 96) { keys[used] = kernel; vals[used] = n; ++used; }
  return n;
}

// Grid = one full wave: resident CTAs per SM (from the kernel's register
// footprint) x 148 SMs, fewer for small inputs.  Grid-stride loops cover
// the rest, so there is no partial second wave.
template <typename K>
static int copy_grid(K kernel, int64_t nvec, int unroll) {
  const int per_sm = resident_per_sm((const void*)kernel);
  int64_t blocks = (nvec + (int64_t)kCopyThreads * unroll - 1) / ((int64_t)kCopyThreads * unroll);
  const int64_t cap = (int64_t)kNumSMs * per_sm;
  if (blocks > cap) blocks = cap;
  return blocks < 1 ? 1 : (int)blocks;
}

template <typename Tin, typename Tout>
static void launch_flatten(const TensorTable& t, void* flat, int64_t psi, int acc, cudaStream_t s) {
  const int64_t nvec = ((psi + 255) >> 8) << 5;
  if (acc) {
    auto k = flatten_kernel<Tin, Tout, true, kCopyUnroll>;
    k<<<copy_grid(k, nvec, kCopyUnroll), kCopyThreads, 0, s>>>(t, (Tout*)flat, psi);
  } else {
    auto k = flatten_kernel<Tin, Tout, false, kCopyUnroll>;
    k<<<copy_grid(k, nvec, kCopyUnroll), kCopyThreads, 0, s>>>(t, (Tout*)flat, psi);
  }
}
template <typename Tin, typename Tout>
static void launch_unflatten(const void* flat, const TensorTable& t, cudaStream_t s) {
  const int64_t nvec = (((t.off[t.n] + 255) >> 8) - (t.off[0] >> 8)) << 5;
  auto k = unflatten_kernel<Tin, Tout, kCopyUnroll>;
  k<<<copy_grid(k, nvec, kCopyUnroll), kCopyThreads, 0, s>>>((const Tin*)flat, t);
}
template <typename Tin, typename Tout>
static void launch_cast(const void* src, void* dst, int64_t n, cudaStream_t s) {
  const int64_t nvec = ((n + 255) >> 8) << 5;
  auto k = cast_kernel<Tin, Tout, kCopyUnroll>;
  k<<<copy_grid(k, nvec, kCopyUnroll), kCopyThreads, 0, s>>>((const Tin*)src, (Tout*)dst, n);
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
