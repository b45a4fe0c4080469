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

__global__ void __launch_bounds__(kOptThreads)
adam_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
            float* __restrict__ v, int64_t n, AdamScalars s, const float* __restrict__ skip,
            __nv_bfloat16* __restrict__ plow) {
  if (skip != nullptr && *skip > 0.f) return;      // world verdict: skip step
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool vec = aligned16(p) && aligned16(g) && aligned16(m) && aligned16(v) &&
                   (plow == nullptr || aligned16(plow));
  int64_t done = 0;
  if (vec) {
    const int64_t n4 = n >> 2;
    float4* p4 = (float4*)p; const float4* g4 = (const float4*)g;
    float4* m4 = (float4*)m; float4* v4 = (float4*)v;
    for (int64_t i = tid; i < n4; i += stride) {
      float4 pp = p4[i], gg = __ldcs(g4 + i), mm = m4[i], vv = v4[i];
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
    adam1(pp, g[i], mm, vv, s);
    p[i] = pp; m[i] = mm; v[i] = vv;
    if (plow) plow[i] = __float2bfloat16_rn(pp);
  }
}

// TMA-pipelined Adam: p, g, m, v tiles are streamed into a shared-memory
// ring by 1-D bulk copies (one elected thread, mbarrier transaction counts),
// so the bytes in flight per SM are set by the ring depth rather than by the
// registers each thread can hold.  All threads then run the same adam1 math
// on their float4 of the landed stage and store p, m, v (+ bf16 copy)
// straight from registers.  Persistent grid: kAdamCtasPerSm CTAs per SM,
// tiles assigned round-robin.  Same bits as adam_kernel.
constexpr int kAdamTile = 1024;                       // elements per array per stage
constexpr int kAdamStages = 4;
constexpr int kAdamStageBytes = 4 * kAdamTile * 4;    // p, g, m, v
constexpr int kAdamSmem = kAdamStages * kAdamStageBytes + 64;
constexpr int kAdamCtasPerSm = 3;

__global__ void __launch_bounds__(kOptThreads)
adam_tma_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                float* __restrict__ v, int64_t n, AdamScalars s, const float* __restrict__ skip,
                __nv_bfloat16* __restrict__ plow) {
  if (skip != nullptr && *skip > 0.f) return;
  extern __shared__ __align__(128) unsigned char smem[];
  float* ring = reinterpret_cast<float*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kAdamStages * kAdamStageBytes);
  const int64_t ntiles = n / kAdamTile;               // full tiles; the tail is scalar
  const int64_t mine = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kAdamStages; ++st) mbar_init(&full[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t k) {
    const int st = (int)(k % kAdamStages);
    const int64_t e0 = (blockIdx.x + k * gridDim.x) * (int64_t)kAdamTile;
    float* base = ring + st * (4 * kAdamTile);
    mbar_expect_tx(&full[st], kAdamStageBytes);
    tma_load_1d(base, p + e0, kAdamTile * 4, &full[st]);
    tma_load_1d(base + kAdamTile, g + e0, kAdamTile * 4, &full[st]);
    tma_load_1d(base + 2 * kAdamTile, m + e0, kAdamTile * 4, &full[st]);
    tma_load_1d(base + 3 * kAdamTile, v + e0, kAdamTile * 4, &full[st]);
  };
  if (threadIdx.x == 0)
    for (int64_t k = 0; k < mine && k < kAdamStages; ++k) issue(k);
  for (int64_t k = 0; k < mine; ++k) {
    const int st = (int)(k % kAdamStages);
    mbar_wait(&full[st], (uint32_t)((k / kAdamStages) & 1));
    const float* base = ring + st * (4 * kAdamTile);
    const int64_t e0 = (blockIdx.x + k * gridDim.x) * (int64_t)kAdamTile;
    const int i = threadIdx.x * 4;                    // kOptThreads * 4 == kAdamTile
    float4 pp = *reinterpret_cast<const float4*>(base + i);
    const float4 gg = *reinterpret_cast<const float4*>(base + kAdamTile + i);
    float4 mm = *reinterpret_cast<const float4*>(base + 2 * kAdamTile + i);
    float4 vv = *reinterpret_cast<const float4*>(base + 3 * kAdamTile + i);
    __syncthreads();                                  // stage st fully read: refill it
    if (threadIdx.x == 0 && k + kAdamStages < mine) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic reads -> async writes
      issue(k + kAdamStages);
    }
    adam1(pp.x, gg.x, mm.x, vv.x, s); adam1(pp.y, gg.y, mm.y, vv.y, s);
    adam1(pp.z, gg.z, mm.z, vv.z, s); adam1(pp.w, gg.w, mm.w, vv.w, s);
    const int64_t e = e0 + i;
    reinterpret_cast<float4*>(p + e)[0] = pp;
    __stcs(reinterpret_cast<float4*>(m + e), mm);
    __stcs(reinterpret_cast<float4*>(v + e), vv);
    if (plow) {
      uint2 b = make_uint2(pack_bf16x2(pp.x, pp.y), pack_bf16x2(pp.z, pp.w));
      *reinterpret_cast<uint2*>(plow + e) = b;
    }
  }
  // scalar tail (n % kAdamTile elements), spread over the grid
  const int64_t t0 = ntiles * kAdamTile;
  for (int64_t i = t0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float pp = p[i], mm = m[i], vv = v[i];
    adam1(pp, g[i], mm, vv, s);
    p[i] = pp; m[i] = mm; v[i] = vv;
    if (plow) plow[i] = __float2bfloat16_rn(pp);
  }
}

__global__ void __launch_bounds__(kOptThreads)
sgd_kernel(float* __restrict__ p, const float* __restrict__ g, int64_t n, float lr,
           const float* __restrict__ skip, __nv_bfloat16* __restrict__ plow) {
  if (skip != nullptr && *skip > 0.f) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float pp = __fsub_rn(p[i], __fmul_rn(lr, g[i]));   // param -= lr * grad
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

extern "C" int fsdp_adam_step(float* p, const float* g, float* m, float* v, int64_t n, float lr,
                              float b1, float omb1, float b2, float omb2, float bc1, float bc2,
                              float eps, const float* skip_flag, void* p_lowp, void* stream) {
  if (n < 0) return fail(FSDP_E_INVALID, "fsdp_adam_step: negative n");
  if (n == 0) return 0;
  if (!p || !g || !m || !v) return fail(FSDP_E_INVALID, "fsdp_adam_step: null buffer");
  AdamScalars s{lr, b1, omb1, b2, omb2, bc1, bc2, eps};
  static int use_tma = -1;      // FSDP_ADAM_TMA=0 selects the register-streaming kernel
  if (use_tma < 0) {
    const char* e = getenv("FSDP_ADAM_TMA");
    use_tma = e ? (atoi(e) != 0) : 1;
    if (use_tma && cudaFuncSetAttribute(adam_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        kAdamSmem) != cudaSuccess)
      use_tma = 0;
  }
  const bool al = aligned16(p) && aligned16(g) && aligned16(m) && aligned16(v) &&
                  (p_lowp == nullptr || ((uintptr_t)p_lowp & 7) == 0);
  if (use_tma && al && n >= (int64_t)kAdamTile * kNumSMs) {
    const int64_t tiles = n / kAdamTile;
    const int grid = (int)std::min<int64_t>(tiles, (int64_t)kNumSMs * kAdamCtasPerSm);
    adam_tma_kernel<<<grid, kOptThreads, kAdamSmem, (cudaStream_t)stream>>>(
        p, g, m, v, n, s, skip_flag, (__nv_bfloat16*)p_lowp);
  } else {
    adam_kernel<<<opt_grid(n), kOptThreads, 0, (cudaStream_t)stream>>>(
        p, g, m, v, n, s, skip_flag, (__nv_bfloat16*)p_lowp);
  }
  FSDP_LAUNCHED();
  return 0;
}

extern "C" int fsdp_sgd_step(float* p, const float* g, int64_t n, float lr, const float* skip_flag,
                             void* p_lowp, void* stream) {
  if (n < 0) return fail(FSDP_E_INVALID, "fsdp_sgd_step: negative n");
  if (n == 0) return 0;
  sgd_kernel<<<opt_grid(n), kOptThreads, 0, (cudaStream_t)stream>>>(p, g, n, lr, skip_flag,
                                                                    (__nv_bfloat16*)p_lowp);
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
