// Sharded optimizer epilogue on the rank-local fp32 shard arena.
//
// Adam follows numerics.py:273-285 operation for operation in float32 with
// explicit round-to-nearest intrinsics (no FMA contraction), so the result is
// bit-identical to numpy running the reference's Adam.step on float32 arrays
// (python-float scalars are weak under NEP 50 -> rounded to float32 first).
// HBM-bound: p, g, m, v read (16 B) + p, m, v written (12 B) [+ 2 B bf16 copy].
#include "common.cuh"

#include <algorithm>
#include <cstdlib>

namespace fsdp {

constexpr int kOptThreads = 256;

struct AdamScalars {
  float lr, b1, omb1, b2, omb2, bc1, bc2, eps;
};

__device__ __forceinline__ void adam1(float& p, float g, float& m, float& v, const AdamScalars& s) {
  // state["m"] = b1 * m + (1.0 - b1) * grad
  m = __fadd_rn(__fmul_rn(s.b1, m), __fmul_rn(s.omb1, g));
  // state["v"] = b2 * v + (1.0 - b2) * grad * grad      ((c*g)*g, left to right)
  v = __fadd_rn(__fmul_rn(s.b2, v), __fmul_rn(__fmul_rn(s.omb2, g), g));
  const float mh = __fdiv_rn(m, s.bc1);
  const float vh = __fdiv_rn(v, s.bc2);
  // param -= lr * m_hat / (sqrt(v_hat) + eps)
  const float den = __fadd_rn(__fsqrt_rn(vh), s.eps);
  p = __fsub_rn(p, __fdiv_rn(__fmul_rn(s.lr, mh), den));
}

// 4 gradient elements as floats (bf16 -> fp32 is exact: same bits as an
// fp32 gradient arena holding the bf16 write-back)
__device__ __forceinline__ float4 ld_grad4(const float* g, int64_t i4) {
  return __ldcs(reinterpret_cast<const float4*>(g) + i4);
}
__device__ __forceinline__ float4 ld_grad4(const __nv_bfloat16* g, int64_t i4) {
  const uint2 r = __ldcs(reinterpret_cast<const uint2*>(g) + i4);
  return make_float4(bf16lo(r.x), bf16hi(r.x), bf16lo(r.y), bf16hi(r.y));
}

template <typename G>
__global__ void __launch_bounds__(kOptThreads)
adam_kernel(float* __restrict__ p, const G* __restrict__ g, float* __restrict__ m,
            float* __restrict__ v, int64_t n, AdamScalars s, const float* __restrict__ skip,
            __nv_bfloat16* __restrict__ plow) {
  if (skip != nullptr && *skip > 0.f) return;      // world verdict: skip step
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool vec = aligned16(p) && ((uintptr_t)g % (4 * sizeof(G)) == 0) && aligned16(m) && aligned16(v) &&
                   (plow == nullptr || aligned16(plow));
  int64_t done = 0;
  if (vec) {
    const int64_t n4 = n >> 2;
    float4* p4 = (float4*)p;
    float4* m4 = (float4*)m; float4* v4 = (float4*)v;
    for (int64_t i = tid; i < n4; i += stride) {
      float4 pp = p4[i], gg = ld_grad4(g, i), mm = m4[i], vv = v4[i];
      adam1(pp.x, gg.x, mm.x, vv.x, s); adam1(pp.y, gg.y, mm.y, vv.y, s);
      adam1(pp.z, gg.z, mm.z, vv.z, s); adam1(pp.w, gg.w, mm.w, vv.w, s);
      p4[i] = pp; __stcs(m4 + i, mm); __stcs(v4 + i, vv);
      if (plow) {
        uint2 b = make_uint2(pack_bf16x2(pp.x, pp.y), pack_bf16x2(pp.z, pp.w));
        *(uint2*)(plow + 4 * i) = b;
      }
    }
    done = n4 << 2;
  }
  for (int64_t i = done + tid; i < n; i += stride) {
    float pp = p[i], mm = m[i], vv = v[i];
    adam1(pp, to_f<G>(g[i]), mm, vv, s);
    p[i] = pp; m[i] = mm; v[i] = vv;
    if (plow) plow[i] = __float2bfloat16_rn(pp);
  }
}

// TMA-pipelined Adam: p, g, m, v tiles are streamed into a shared-memory
// ring by 1-D bulk copies (one elected thread, mbarrier transaction counts),
// so the bytes in flight per SM are set by the ring depth rather than by the
// registers each thread can hold.  All threads then run the same adam1 math
// on their float4s of the landed stage and store p, m, v (+ bf16 copy)
// straight from registers.  Persistent grid (ctas_per_sm CTAs per SM).  Same
// bits as adam_kernel.
template <int TILE, int STAGES, bool CONTIG, int THREADS, typename G = float>
__global__ void __launch_bounds__(THREADS)
adam_tma_kernel(float* __restrict__ p, const G* __restrict__ g, float* __restrict__ m,
                float* __restrict__ v, int64_t n, AdamScalars s, const float* __restrict__ skip,
                __nv_bfloat16* __restrict__ plow) {
  // stage = [p fp32 | m fp32 | v fp32 | g G] tiles
  constexpr int kStageBytes = TILE * (12 + (int)sizeof(G));
  constexpr int kPer = TILE / THREADS;                // elements per thread per stage (multiple of 4)
  static_assert(kPer % 4 == 0, "tile must give every thread whole float4s");
  if (skip != nullptr && *skip > 0.f) return;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes);
  const int64_t ntiles = n / TILE;                    // full tiles; the tail is scalar
  // CONTIG: CTA b streams the contiguous tile range [b*T/G, (b+1)*T/G);
  // else tiles are dealt round-robin (tile b + k*G)
  const int64_t tbeg = CONTIG ? ntiles * blockIdx.x / gridDim.x : 0;
  const int64_t mine = CONTIG ? ntiles * (blockIdx.x + 1) / gridDim.x - tbeg
                              : (ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0);
  auto tile_of = [&](int64_t k) -> int64_t { return CONTIG ? tbeg + k : blockIdx.x + k * gridDim.x; };
  if (threadIdx.x == 0) {
    for (int st = 0; st < STAGES; ++st) mbar_init(&full[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t k) {
    const int st = (int)(k % STAGES);
    const int64_t e0 = tile_of(k) * (int64_t)TILE;
    float* base = reinterpret_cast<float*>(smem + (size_t)st * kStageBytes);
    mbar_expect_tx(&full[st], kStageBytes);
    tma_load_1d(base, p + e0, TILE * 4, &full[st]);
    tma_load_1d(base + TILE, m + e0, TILE * 4, &full[st]);
    tma_load_1d(base + 2 * TILE, v + e0, TILE * 4, &full[st]);
    tma_load_1d(base + 3 * TILE, g + e0, TILE * (int)sizeof(G), &full[st]);
  };
  if (threadIdx.x == 0)
    for (int64_t k = 0; k < mine && k < STAGES; ++k) issue(k);
  for (int64_t k = 0; k < mine; ++k) {
    const int st = (int)(k % STAGES);
    mbar_wait(&full[st], (uint32_t)((k / STAGES) & 1));
    const float* base = reinterpret_cast<const float*>(smem + (size_t)st * kStageBytes);
    const G* gbase = reinterpret_cast<const G*>(base + 3 * TILE);
    const int64_t e0 = tile_of(k) * (int64_t)TILE;
    float4 pp[kPer / 4], gg[kPer / 4], mm[kPer / 4], vv[kPer / 4];
#pragma unroll
    for (int q = 0; q < kPer / 4; ++q) {               // warp-contiguous float4s
      const int i = (q * THREADS + threadIdx.x) * 4;
      pp[q] = *reinterpret_cast<const float4*>(base + i);
      mm[q] = *reinterpret_cast<const float4*>(base + TILE + i);
      vv[q] = *reinterpret_cast<const float4*>(base + 2 * TILE + i);
      if constexpr (sizeof(G) == 4) {
        gg[q] = *reinterpret_cast<const float4*>(gbase + i);
      } else {
        const uint2 r = *reinterpret_cast<const uint2*>(gbase + i);
        gg[q] = make_float4(bf16lo(r.x), bf16hi(r.x), bf16lo(r.y), bf16hi(r.y));
      }
    }
    __syncthreads();                                  // stage st fully read: refill it
    if (threadIdx.x == 0 && k + STAGES < mine) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic reads -> async writes
      issue(k + STAGES);
    }
#pragma unroll
    for (int q = 0; q < kPer / 4; ++q) {
      adam1(pp[q].x, gg[q].x, mm[q].x, vv[q].x, s); adam1(pp[q].y, gg[q].y, mm[q].y, vv[q].y, s);
      adam1(pp[q].z, gg[q].z, mm[q].z, vv[q].z, s); adam1(pp[q].w, gg[q].w, mm[q].w, vv[q].w, s);
      const int64_t e = e0 + (q * THREADS + threadIdx.x) * 4;
      reinterpret_cast<float4*>(p + e)[0] = pp[q];
      __stcs(reinterpret_cast<float4*>(m + e), mm[q]);
      __stcs(reinterpret_cast<float4*>(v + e), vv[q]);
      if (plow) {
        uint2 b = make_uint2(pack_bf16x2(pp[q].x, pp[q].y), pack_bf16x2(pp[q].z, pp[q].w));
        *reinterpret_cast<uint2*>(plow + e) = b;
      }
    }
  }
  // scalar tail (n % TILE elements), spread over the grid
  const int64_t t0 = ntiles * TILE;
  for (int64_t i = t0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float pp = p[i], mm = m[i], vv = v[i];
    adam1(pp, to_f<G>(g[i]), mm, vv, s);
    p[i] = pp; m[i] = mm; v[i] = vv;
    if (plow) plow[i] = __float2bfloat16_rn(pp);
  }
}

// (tile elements, stages, CTAs per SM) variants, FSDP_ADAM_VARIANT=<index>
struct AdamVariant {
  void* fn;
  int tile, stages, ctas_per_sm, threads;
  void* fn_bf16g;                 // bf16 gradient (W = 1 write-back arena), with its own
  int stages_bf16g, tile_bf16g;   // ring (14 B/elem stages fit deeper rings) and CTA size
  int threads_bf16g;
};
// Measured in the step at N=1 on the GPT-1.3B arena (1.32 G elements;
// bench.py FSDP_ADAM_VARIANT=k, profiles/r2/adam_ring/; round 1:
// profiles/r1/adam/).  The SM clock is power-capped (~1.6 GHz) there, so the
// exact-rounding math (3 IEEE divides + a sqrt per element) must overlap the
// DRAM stream: what matters is how many bytes are still in flight while a
// CTA computes on a landed stage.  Two 6144-element stages leave one stage
// (86 KB) in flight; four 3072-element stages leave three (129 KB): bf16-g
// Adam 5.67 vs 6.36 ms (0.99 vs 0.89 of the measured copy peak).  For fp32
// gradients (16 B/elem) six 2048-element stages of 512 threads give 6.40 vs
// 6.73 ms.  256-thread CTAs starve the math of warps (round 1: 0.78).
static const AdamVariant kAdamVariants[] = {
    {(void*)adam_tma_kernel<2048, 6, true, 512>, 2048, 6, 1, 512,
     (void*)adam_tma_kernel<3072, 4, true, 768, __nv_bfloat16>, 4, 3072, 768},     // 0 (default)
    {(void*)adam_tma_kernel<6144, 2, true, 768>, 6144, 2, 1, 768,
     (void*)adam_tma_kernel<6144, 2, true, 768, __nv_bfloat16>, 2, 6144, 768},     // 1: round-1 default
    {(void*)adam_tma_kernel<6144, 2, true, 256>, 6144, 2, 1, 256,
     (void*)adam_tma_kernel<6144, 2, true, 256, __nv_bfloat16>, 2, 6144, 256},     // 2: best standalone (r1)
    {(void*)adam_tma_kernel<1024, 4, false, 256>, 1024, 4, 3, 256,
     (void*)adam_tma_kernel<1024, 4, false, 256, __nv_bfloat16>, 4, 1024, 256},    // 3: the first version
    {(void*)adam_tma_kernel<4096, 3, true, 1024>, 4096, 3, 1, 1024,
     (void*)adam_tma_kernel<4096, 4, true, 1024, __nv_bfloat16>, 4, 4096, 1024},    // 4
    {(void*)adam_tma_kernel<3072, 4, true, 768>, 3072, 4, 1, 768,
     (void*)adam_tma_kernel<2048, 7, true, 512, __nv_bfloat16>, 7, 2048, 512},     // 5
};

template <typename G>
__global__ void __launch_bounds__(kOptThreads)
sgd_kernel(float* __restrict__ p, const G* __restrict__ g, int64_t n, float lr,
           const float* __restrict__ skip, __nv_bfloat16* __restrict__ plow) {
  if (skip != nullptr && *skip > 0.f) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float pp = __fsub_rn(p[i], __fmul_rn(lr, to_f<G>(g[i])));   // param -= lr * grad
    p[i] = pp;
    if (plow) plow[i] = __float2bfloat16_rn(pp);
  }
}

__global__ void __launch_bounds__(kOptThreads)
unscale_kernel(float* __restrict__ g, int64_t n, float inv, float* __restrict__ found) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float x = __fmul_rn(g[i], inv);       // ru.accum *= inv
    g[i] = x;
    bad |= !isfinite(x);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) *found = 1.0f;
}

static int opt_grid(int64_t n) {
  int64_t blocks = (n / 4 + kOptThreads - 1) / kOptThreads;
  static int per_sm = 0;   // CTAs per SM in the grid cap (FSDP_OPT_CTAS_PER_SM, default 8)
  if (per_sm == 0) {
    const char* e = getenv("FSDP_OPT_CTAS_PER_SM");
    per_sm = e ? std::max(1, std::min(32, atoi(e))) : 8;
  }
  const int64_t cap = (int64_t)kNumSMs * per_sm;
  if (blocks > cap) blocks = cap;
  return blocks < 1 ? 1 : (int)blocks;
}

}  // namespace fsdp

using namespace fsdp;

static int adam_launch(float* p, const void* g, int g_bf16, float* m, float* v, int64_t n,
                       const AdamScalars& s, const float* skip_flag, void* p_lowp, cudaStream_t stream) {
  static int use_tma = -1;      // FSDP_ADAM_TMA=0 selects the register-streaming kernel
  static int var = 0;
  if (use_tma < 0) {
    const char* e = getenv("FSDP_ADAM_TMA");
    use_tma = e ? (atoi(e) != 0) : 1;
    if (const char* ev = getenv("FSDP_ADAM_VARIANT"))
      var = std::max(0, std::min((int)(sizeof(kAdamVariants) / sizeof(kAdamVariants[0])) - 1, atoi(ev)));
    const AdamVariant& av = kAdamVariants[var];
    if (use_tma && (cudaFuncSetAttribute(av.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         av.stages * 16 * av.tile + 64) != cudaSuccess ||
                    cudaFuncSetAttribute(av.fn_bf16g, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         av.stages_bf16g * 14 * av.tile_bf16g + 64) != cudaSuccess))
      use_tma = 0;
  }
  const AdamVariant& av = kAdamVariants[var];
  const size_t gs = g_bf16 ? 2 : 4;
  const bool al = aligned16(p) && aligned16(g) && aligned16(m) && aligned16(v) &&
                  (p_lowp == nullptr || ((uintptr_t)p_lowp & 7) == 0);
  const int tile = g_bf16 ? av.tile_bf16g : av.tile;
  const int stages = g_bf16 ? av.stages_bf16g : av.stages;
  if (use_tma && al && n >= (int64_t)tile * kNumSMs) {
    const int64_t tiles = n / tile;
    const int grid = (int)std::min<int64_t>(tiles, (int64_t)kNumSMs * av.ctas_per_sm);
    __nv_bfloat16* pl = (__nv_bfloat16*)p_lowp;
    AdamScalars sc = s;
    void* args[] = {&p, (void*)&g, &m, &v, &n, &sc, (void*)&skip_flag, &pl};
    FSDP_CUDA(cudaLaunchKernel(g_bf16 ? av.fn_bf16g : av.fn, dim3(grid), dim3(g_bf16 ? av.threads_bf16g : av.threads), args,
                               (size_t)stages * (12 + gs) * tile + 64, stream));
  } else if (g_bf16) {
    adam_kernel<__nv_bfloat16><<<opt_grid(n), kOptThreads, 0, stream>>>(
        p, (const __nv_bfloat16*)g, m, v, n, s, skip_flag, (__nv_bfloat16*)p_lowp);
  } else {
    adam_kernel<float><<<opt_grid(n), kOptThreads, 0, stream>>>(
        p, (const float*)g, m, v, n, s, skip_flag, (__nv_bfloat16*)p_lowp);
  }
  FSDP_LAUNCHED();
  return 0;
}

extern "C" int fsdp_adam_step(float* p, const float* g, float* m, float* v, int64_t n, float lr,
                              float b1, float omb1, float b2, float omb2, float bc1, float bc2,
                              float eps, const float* skip_flag, void* p_lowp, void* stream) {
  if (n < 0) return fail(FSDP_E_INVALID, "fsdp_adam_step: negative n");
  if (n == 0) return 0;
  if (!p || !g || !m || !v) return fail(FSDP_E_INVALID, "fsdp_adam_step: null buffer");
  AdamScalars s{lr, b1, omb1, b2, omb2, bc1, bc2, eps};
  return adam_launch(p, g, 0, m, v, n, s, skip_flag, p_lowp, (cudaStream_t)stream);
}

extern "C" int fsdp_adam_step_bf16g(float* p, const void* g_bf16, float* m, float* v, int64_t n, float lr,
                                    float b1, float omb1, float b2, float omb2, float bc1, float bc2,
                                    float eps, const float* skip_flag, void* p_lowp, void* stream) {
  if (n < 0) return fail(FSDP_E_INVALID, "fsdp_adam_step_bf16g: negative n");
  if (n == 0) return 0;
  if (!p || !g_bf16 || !m || !v) return fail(FSDP_E_INVALID, "fsdp_adam_step_bf16g: null buffer");
  AdamScalars s{lr, b1, omb1, b2, omb2, bc1, bc2, eps};
  return adam_launch(p, g_bf16, 1, m, v, n, s, skip_flag, p_lowp, (cudaStream_t)stream);
}

extern "C" int fsdp_sgd_step(float* p, const float* g, int64_t n, float lr, const float* skip_flag,
                             void* p_lowp, void* stream) {
  if (n < 0) return fail(FSDP_E_INVALID, "fsdp_sgd_step: negative n");
  if (n == 0) return 0;
  sgd_kernel<float><<<opt_grid(n), kOptThreads, 0, (cudaStream_t)stream>>>(p, g, n, lr, skip_flag,
                                                                           (__nv_bfloat16*)p_lowp);
  FSDP_LAUNCHED();
  return 0;
}

extern "C" int fsdp_sgd_step_bf16g(float* p, const void* g_bf16, int64_t n, float lr, const float* skip_flag,
                                   void* p_lowp, void* stream) {
  if (n < 0) return fail(FSDP_E_INVALID, "fsdp_sgd_step_bf16g: negative n");
  if (n == 0) return 0;
  sgd_kernel<__nv_bfloat16><<<opt_grid(n), kOptThreads, 0, (cudaStream_t)stream>>>(
      p, (const __nv_bfloat16*)g_bf16, n, lr, skip_flag, (__nv_bfloat16*)p_lowp);
  FSDP_LAUNCHED();
  return 0;
}

extern "C" int fsdp_unscale_found_inf(float* g, int64_t n, float inv_scale, float* found_inf,
                                      void* stream) {
  if (n < 0 || !found_inf) return fail(FSDP_E_INVALID, "fsdp_unscale_found_inf: bad args");
  if (n == 0) return 0;
  unscale_kernel<<<opt_grid(n), kOptThreads, 0, (cudaStream_t)stream>>>(g, n, inv_scale, found_inf);
  FSDP_LAUNCHED();
  return 0;
}
