// Shared device/host helpers for the FSDP B200 runtime (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string>

#include "../../include/fsdp_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "fsdp_b200 is written for sm_100a (B200) only"
#endif

namespace fsdp {

// ---------------------------------------------------------------- errors ----
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int check_cuda(cudaError_t e, const char* what);
void count_launch(uint64_t n = 1);

#define FSDP_CUDA(expr)                                              \
  do {                                                               \
    cudaError_t _e = (expr);                                         \
    if (_e != cudaSuccess) return ::fsdp::check_cuda(_e, #expr);     \
  } while (0)

#define FSDP_LAUNCHED()                                              \
  do {                                                               \
    cudaError_t _e = cudaGetLastError();                             \
    if (_e != cudaSuccess) return ::fsdp::check_cuda(_e, "launch"); \
    ::fsdp::count_launch();                                          \
  } while (0)

constexpr int kNumSMs = 148;

inline int elem_size(int dtype) {
  switch (dtype) {
    case FSDP_F32: return 4;
    case FSDP_BF16: return 2;
    default: return 0;
  }
}

// ------------------------------------------------------- device helpers ----
// 8-element vector: the unit of work of every copy/cast kernel.  8 bf16 are
// one 16-byte access, 8 fp32 are two.
struct alignas(16) V8F { float v[8]; };

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  // cvt.rn.bf16x2.f32 d, a, b: d.hi = cvt(a), d.lo = cvt(b); RNE.
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float bf16lo(uint32_t x) { return __uint_as_float(x << 16); }
__device__ __forceinline__ float bf16hi(uint32_t x) { return __uint_as_float(x & 0xFFFF0000u); }

__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
// L2-coherent load (bypasses L1): for data peers wrote during this kernel.
__device__ __forceinline__ uint4 ld_cg(const void* p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
enum LdMode { LD_NC = 0, LD_PLAIN = 1, LD_CG = 2 };
__device__ __forceinline__ uint4 ld_mode(const void* p, int mode) {
  return mode == LD_NC ? ld_stream(p) : (mode == LD_CG ? ld_cg(p) : ld_v4(p));
}
__device__ __forceinline__ void st_v4(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

template <typename T> struct DT;
template <> struct DT<float> { static constexpr int id = FSDP_F32; };
template <> struct DT<__nv_bfloat16> { static constexpr int id = FSDP_BF16; };

// Load 8 consecutive elements (16B-aligned start) as floats.
template <typename T> __device__ __forceinline__ V8F load8(const T* p, int mode);
template <> __device__ __forceinline__ V8F load8<float>(const float* p, int mode) {
  uint4 a = ld_mode(p, mode);
  uint4 b = ld_mode(p + 4, mode);
  V8F r;
  r.v[0] = __uint_as_float(a.x); r.v[1] = __uint_as_float(a.y);
  r.v[2] = __uint_as_float(a.z); r.v[3] = __uint_as_float(a.w);
  r.v[4] = __uint_as_float(b.x); r.v[5] = __uint_as_float(b.y);
  r.v[6] = __uint_as_float(b.z); r.v[7] = __uint_as_float(b.w);
  return r;
}
template <> __device__ __forceinline__ V8F load8<__nv_bfloat16>(const __nv_bfloat16* p, int mode) {
  uint4 a = ld_mode(p, mode);
  V8F r;
  r.v[0] = bf16lo(a.x); r.v[1] = bf16hi(a.x); r.v[2] = bf16lo(a.y); r.v[3] = bf16hi(a.y);
  r.v[4] = bf16lo(a.z); r.v[5] = bf16hi(a.z); r.v[6] = bf16lo(a.w); r.v[7] = bf16hi(a.w);
  return r;
}

// Pack 8 floats into the raw bytes of T (1 or 2 uint4).
template <typename T> struct Packed8;
template <> struct Packed8<float> { uint4 a, b; };
template <> struct Packed8<__nv_bfloat16> { uint4 a; };

template <typename T> __device__ __forceinline__ Packed8<T> pack8(const V8F& x);
template <> __device__ __forceinline__ Packed8<float> pack8<float>(const V8F& x) {
  Packed8<float> r;
  r.a = make_uint4(__float_as_uint(x.v[0]), __float_as_uint(x.v[1]), __float_as_uint(x.v[2]),
                   __float_as_uint(x.v[3]));
  r.b = make_uint4(__float_as_uint(x.v[4]), __float_as_uint(x.v[5]), __float_as_uint(x.v[6]),
                   __float_as_uint(x.v[7]));
  return r;
}
template <> __device__ __forceinline__ Packed8<__nv_bfloat16> pack8<__nv_bfloat16>(const V8F& x) {
  Packed8<__nv_bfloat16> r;
  r.a = make_uint4(pack_bf16x2(x.v[0], x.v[1]), pack_bf16x2(x.v[2], x.v[3]),
                   pack_bf16x2(x.v[4], x.v[5]), pack_bf16x2(x.v[6], x.v[7]));
  return r;
}
template <typename T> __device__ __forceinline__ void store8(T* p, const Packed8<T>& v);
template <> __device__ __forceinline__ void store8<float>(float* p, const Packed8<float>& v) {
  st_v4(p, v.a); st_v4(p + 4, v.b);
}
template <> __device__ __forceinline__ void store8<__nv_bfloat16>(__nv_bfloat16* p,
                                                                  const Packed8<__nv_bfloat16>& v) {
  st_v4(p, v.a);
}

// Raw (still-packed) 8-element loads: half the registers of V8F for bf16,
// so more vectors stay in flight per thread.
template <typename T> __device__ __forceinline__ Packed8<T> ld_raw8(const T* p, int mode);
template <> __device__ __forceinline__ Packed8<float> ld_raw8<float>(const float* p, int mode) {
  Packed8<float> r; r.a = ld_mode(p, mode); r.b = ld_mode(p + 4, mode); return r;
}
template <> __device__ __forceinline__ Packed8<__nv_bfloat16> ld_raw8<__nv_bfloat16>(
    const __nv_bfloat16* p, int mode) {
  Packed8<__nv_bfloat16> r; r.a = ld_mode(p, mode); return r;
}
template <typename T> __device__ __forceinline__ V8F unpack8(const Packed8<T>& x);
template <> __device__ __forceinline__ V8F unpack8<float>(const Packed8<float>& x) {
  V8F r;
  r.v[0] = __uint_as_float(x.a.x); r.v[1] = __uint_as_float(x.a.y);
  r.v[2] = __uint_as_float(x.a.z); r.v[3] = __uint_as_float(x.a.w);
  r.v[4] = __uint_as_float(x.b.x); r.v[5] = __uint_as_float(x.b.y);
  r.v[6] = __uint_as_float(x.b.z); r.v[7] = __uint_as_float(x.b.w);
  return r;
}
template <> __device__ __forceinline__ V8F unpack8<__nv_bfloat16>(const Packed8<__nv_bfloat16>& x) {
  V8F r;
  r.v[0] = bf16lo(x.a.x); r.v[1] = bf16hi(x.a.x); r.v[2] = bf16lo(x.a.y); r.v[3] = bf16hi(x.a.y);
  r.v[4] = bf16lo(x.a.z); r.v[5] = bf16hi(x.a.z); r.v[6] = bf16lo(x.a.w); r.v[7] = bf16hi(x.a.w);
  return r;
}

template <typename T> __device__ __forceinline__ float to_f(T x);
template <> __device__ __forceinline__ float to_f<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) {
  return __bfloat162float(x);
}
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

__host__ __device__ __forceinline__ bool aligned16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15) == 0;
}

// ---------------------------------------------- TMA bulk copy + mbarrier ----
// 1-D bulk copies (cp.async.bulk -> UBLKCP) completing on an mbarrier's
// transaction count.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}"
      :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gsrc, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      :: "r"(smem_u32(smem_dst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

}  // namespace fsdp
