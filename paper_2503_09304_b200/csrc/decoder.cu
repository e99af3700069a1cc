// Fused decoder-side helpers around the MoE path (not the north-star hot path itself): RMSNorm
// with an optional fused residual add, and in-place RoPE on q/k.  They replace ~30 small torch
// elementwise launches per layer of the Mixtral/Qwen serving plugin, which made decode
// iterations host-launch-bound.
#include "common.cuh"

namespace qmoe {
namespace {

constexpr int kNormThreads = 256;

// out = rmsnorm(x [+ add]) * w; if add != nullptr, sum_out = x + add (bf16) is written too.
__global__ void __launch_bounds__(kNormThreads)
rmsnorm_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ add,
               const __nv_bfloat16* __restrict__ w, float eps, int d, __nv_bfloat16* __restrict__ out,
               __nv_bfloat16* __restrict__ sum_out) {
  pdl_wait();  // launched with programmatic dependent launch (launch_pdl): x comes from the predecessor
  pdl_trigger();
  const int row = blockIdx.x;
  const __nv_bfloat16* xr = x + (size_t)row * d;
  const __nv_bfloat16* ar = add ? add + (size_t)row * d : nullptr;
  __shared__ float s_red[kNormThreads / 32];
  float ss = 0.f;
  // d <= 8192: each thread keeps up to 4 vectors of 8 in registers
  float v[4][8];
  const int nv = d / 8;
  int c = 0;
  for (int i = threadIdx.x; i < nv; i += kNormThreads, ++c) {
    uint4 u = reinterpret_cast<const uint4*>(xr)[i];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
    float a[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float2 f = __bfloat1622float2(h[q]);
      a[2 * q] = f.x;
      a[2 * q + 1] = f.y;
    }
    if (ar) {
      uint4 ua = reinterpret_cast<const uint4*>(ar)[i];
      const __nv_bfloat162* ha = reinterpret_cast<const __nv_bfloat162*>(&ua);
      uint4 o;
      __nv_bfloat162* ho = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float2 f = __bfloat1622float2(ha[q]);
        ho[q] = __floats2bfloat162_rn(a[2 * q] + f.x, a[2 * q + 1] + f.y);
        float2 r = __bfloat1622float2(ho[q]);  // the residual stream is bf16: norm what is stored
        a[2 * q] = r.x;
        a[2 * q + 1] = r.y;
      }
      reinterpret_cast<uint4*>(sum_out + (size_t)row * d)[i] = o;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      v[c][q] = a[q];
      ss += a[q] * a[q];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int i = 0; i < kNormThreads / 32; ++i) tot += s_red[i];
  const float inv = rsqrtf(tot / d + eps);
  c = 0;
  for (int i = threadIdx.x; i < nv; i += kNormThreads, ++c) {
    uint4 uw = reinterpret_cast<const uint4*>(w)[i];
    const __nv_bfloat162* hw = reinterpret_cast<const __nv_bfloat162*>(&uw);
    uint4 o;
    __nv_bfloat162* ho = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float2 f = __bfloat1622float2(hw[q]);
      // match HF: normalise in fp32, round to the activation dtype, then scale by the weight
      const float n0 = __bfloat162float(__float2bfloat16_rn(v[c][2 * q] * inv));
      const float n1 = __bfloat162float(__float2bfloat16_rn(v[c][2 * q + 1] * inv));
      ho[q] = __floats2bfloat162_rn(n0 * f.x, n1 * f.y);
    }
    reinterpret_cast<uint4*>(out + (size_t)row * d)[i] = o;
  }
}

// In-place rotate-half RoPE on q [T, H, hd] and k [T, KV, hd] (HF Llama/Mixtral convention).
// One warp per (token, head); lanes cover the first half of head_dim.
__global__ void rope_kernel(__nv_bfloat16* __restrict__ q, __nv_bfloat16* __restrict__ k, const int64_t* __restrict__ pos,
                            const float* __restrict__ cos_t, const float* __restrict__ sin_t, int T, int H, int KV,
                            int hd, int q_stride, int k_stride) {
  pdl_wait();
  pdl_trigger();
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int heads = H + KV;
  if (gw >= T * heads) return;
  const int t = gw / heads, h = gw - t * heads;
  __nv_bfloat16* v = h < H ? q + (size_t)t * q_stride + (size_t)h * hd : k + (size_t)t * k_stride + (size_t)(h - H) * hd;
  const int half = hd / 2;
  const float* cr = cos_t + pos[t] * hd;
  const float* sr = sin_t + pos[t] * hd;
  for (int i = threadIdx.x & 31; i < half; i += 32) {
    const float a = __bfloat162float(v[i]), b = __bfloat162float(v[i + half]);
    v[i] = __float2bfloat16_rn(a * cr[i] - b * sr[i]);
    v[i + half] = __float2bfloat16_rn(b * cr[i + half] + a * sr[i + half]);
  }
}

}  // namespace
}  // namespace qmoe

extern "C" int qmoe_rmsnorm(const void* x, const void* residual_add, const void* weight, float eps, int T, int d,
                            void* out, void* sum_out, void* stream) {
  using namespace qmoe;
  QMOE_REQUIRE(T >= 0 && d > 0 && d % 8 == 0 && d <= 8 * 4 * kNormThreads, "qmoe_rmsnorm: bad sizes T=%d d=%d", T, d);
  QMOE_REQUIRE((residual_add == nullptr) == (sum_out == nullptr), "qmoe_rmsnorm: residual_add and sum_out go together");
  if (T == 0) return QMOE_OK;
  return launch_pdl("qmoe_rmsnorm", rmsnorm_kernel, dim3(T), dim3(kNormThreads), 0, as_stream(stream),
                    (const __nv_bfloat16*)x, (const __nv_bfloat16*)residual_add, (const __nv_bfloat16*)weight, eps, d,
                    (__nv_bfloat16*)out, (__nv_bfloat16*)sum_out);
}

extern "C" int qmoe_rope(void* q, void* k, const int64_t* positions, const float* cos_table, const float* sin_table,
                         int T, int n_heads, int n_kv_heads, int head_dim, int q_stride, int k_stride, void* stream) {
  using namespace qmoe;
  QMOE_REQUIRE(T >= 0 && head_dim % 2 == 0, "qmoe_rope: bad sizes");
  if (T == 0) return QMOE_OK;
  const int warps = T * (n_heads + n_kv_heads);
  return launch_pdl("qmoe_rope", rope_kernel, dim3((warps + 7) / 8), dim3(256), 0, as_stream(stream), (__nv_bfloat16*)q,
                    (__nv_bfloat16*)k, positions, cos_table, sin_table, T, n_heads, n_kv_heads, head_dim, q_stride,
                    k_stride);
}
