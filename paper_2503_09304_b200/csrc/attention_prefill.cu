// Causal varlen GQA prefill attention (the prefill half; the reference's
// attention stage is engine.py:252-301 with _prefill_attention / attend at model.py:58-68, a toy
// single-head attention -- the decoders' GQA attention with RoPE follows HF MixtralAttention /
// Qwen2MoeAttention).  Replaces flash-attn's varlen kernel on the decoders' prefill passes.
//
// Sequences are packed: sequence b owns rows [cu[b], cu[b+1]) of q / k / v, each row a token of a
// packed qkv projection (row strides q_stride / kv_stride elements, heads dense).  Every query
// attends the keys of its own sequence at positions <= its own (the prompt's K/V; a prefill pass
// starts from an empty cache, so these are exactly the entries the pass appends to the page pool).
//
// Flash-attention forward on mma.sync m16n8k16 (bf16 in, fp32 accumulate): CTA = (16 W-query
// block, head, sequence), W = 4 or 8 warps x 16 query rows.  Q is staged once and held as A fragments; 64-key
// blocks of K and V stream through a 2-stage cp.async ring (padded rows, ldmatrix / ldmatrix.trans);
// S = Q K^T stays in registers, online softmax in the exp2 domain with quad shuffles, P is re-packed
// from the S accumulators straight into A fragments for O += P V.  Keys beyond the query (causal)
// or beyond the sequence are masked; the last key block is the diagonal one.
#include <stdlib.h>

#include "common.cuh"

namespace qmoe {
namespace {

constexpr int kKB = 64;  // keys per block

__device__ __forceinline__ void ldsm_x4(const void* p, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
}
__device__ __forceinline__ void ldsm_x4_t(const void* p, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
}
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void cp16(void* dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(ok ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

template <int HD, int W>  // W warps x 16 query rows per CTA
__global__ void __launch_bounds__(W * 32)
prefill_attn_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
                    const __nv_bfloat16* __restrict__ v, int q_stride, int kv_stride, const int32_t* __restrict__ cu,
                    int H, int KV, float scale_log2, __nv_bfloat16* __restrict__ out, int out_stride) {
  pdl_wait();
  pdl_trigger();
  constexpr int kQB = 16 * W;  // query rows per CTA
  constexpr int kThreads = W * 32;
  constexpr int LD = HD + 8;  // padded smem row (bf16): ldmatrix rows 16 B apart mod 128 B
  constexpr int NT = HD / 8;  // n8 tiles of the output
  constexpr int KS = HD / 16; // k16 steps of Q K^T
  extern __shared__ __align__(16) __nv_bfloat16 smem[];
  __nv_bfloat16* sQ = smem;                    // [kQB][LD]
  __nv_bfloat16* sK = sQ + kQB * LD;           // [2][kKB][LD]
  __nv_bfloat16* sV = sK + 2 * kKB * LD;       // [2][kKB][LD]
  // longest CTAs (the most key blocks under the causal mask) first: query blocks in reverse order
  const int b = blockIdx.z, h = blockIdx.y, qb = gridDim.x - 1 - blockIdx.x;
  const int start = cu[b], len = cu[b + 1] - start;
  const int q0 = qb * kQB;
  if (q0 >= len) return;
  const int g = h / (H / KV);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int kPieces = HD / 8;  // 16-byte pieces per row
  // Q tile
  for (int i = tid; i < kQB * kPieces; i += kThreads) {
    const int r = i / kPieces, c = (i % kPieces) * 8;
    const int t = q0 + r;
    cp16(sQ + r * LD + c, q + (size_t)(start + min(t, len - 1)) * q_stride + h * HD + c, t < len);
  }
  auto load_kv = [&](int kb, int st) {
    const int k0 = kb * kKB;
    __nv_bfloat16* dk = sK + st * kKB * LD;
    __nv_bfloat16* dv = sV + st * kKB * LD;
    for (int i = tid; i < kKB * kPieces; i += kThreads) {
      const int r = i / kPieces, c = (i % kPieces) * 8;
      const int t = k0 + r;
      const size_t row = (size_t)(start + min(t, len - 1)) * kv_stride + g * HD + c;
      cp16(dk + r * LD + c, k + row, t < len);
      cp16(dv + r * LD + c, v + row, t < len);
    }
  };
  const int nkb = min((len + kKB - 1) / kKB, (q0 + kQB - 1) / kKB + 1);  // causal: blocks up to the diagonal
  load_kv(0, 0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  // this warp's 16 query rows and the thread's two rows in the accumulator layout
  const int qr0 = warp * 16;
  const int row_a = q0 + qr0 + (lane >> 2), row_b = row_a + 8;  // query positions (within the sequence)
  uint32_t qa[KS][4];
  float o[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float m_a = -INFINITY, m_b = -INFINITY, l_a = 0.f, l_b = 0.f;
  for (int kb = 0; kb < nkb; ++kb) {
    const int st = kb & 1;
    if (kb + 1 < nkb) load_kv(kb + 1, st ^ 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // block kb (and Q) landed
    __syncthreads();
    if (kb == 0) {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks)
        ldsm_x4(sQ + (qr0 + (lane & 15)) * LD + ks * 16 + (lane >> 4) * 8, qa[ks][0], qa[ks][1], qa[ks][2],
                qa[ks][3]);
    }
    const __nv_bfloat16* bk = sK + st * kKB * LD;
    const __nv_bfloat16* bv = sV + st * kKB * LD;
    // S = Q K^T: 16 rows x 64 keys per warp
    float s[kKB / 8][4];
#pragma unroll
    for (int n = 0; n < kKB / 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int np = 0; np < kKB / 16; ++np) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(bk + (16 * np + (lane >> 4) * 8 + (lane & 7)) * LD + ks * 16 + ((lane >> 3) & 1) * 8, b0, b1, b2, b3);
        mma16816(s[2 * np], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b0, b1);
        mma16816(s[2 * np + 1], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b2, b3);
      }
    // scale (log2 domain), causal / length mask, online softmax
    const int k0 = kb * kKB;
    float mx_a = m_a, mx_b = m_b;
#pragma unroll
    for (int n = 0; n < kKB / 8; ++n) {
      const int key = k0 + 8 * n + 2 * (lane & 3);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int kk = key + c;
        s[n][c] = (kk <= row_a && kk < len) ? s[n][c] * scale_log2 : -INFINITY;
        s[n][2 + c] = (kk <= row_b && kk < len) ? s[n][2 + c] * scale_log2 : -INFINITY;
        mx_a = fmaxf(mx_a, s[n][c]);
        mx_b = fmaxf(mx_b, s[n][2 + c]);
      }
    }
#pragma unroll
    for (int off = 1; off < 4; off <<= 1) {
      mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, off));
      mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, off));
    }
    // rows past the sequence end see only masked keys: keep their state finite
    const float base_a = mx_a == -INFINITY ? 0.f : mx_a, base_b = mx_b == -INFINITY ? 0.f : mx_b;
    const float corr_a = exp2f(m_a - base_a), corr_b = exp2f(m_b - base_b);
    m_a = mx_a;
    m_b = mx_b;
    float sum_a = 0.f, sum_b = 0.f;
#pragma unroll
    for (int n = 0; n < kKB / 8; ++n) {
      s[n][0] = exp2f(s[n][0] - base_a);
      s[n][1] = exp2f(s[n][1] - base_a);
      s[n][2] = exp2f(s[n][2] - base_b);
      s[n][3] = exp2f(s[n][3] - base_b);
      sum_a += s[n][0] + s[n][1];
      sum_b += s[n][2] + s[n][3];
    }
    l_a = l_a * corr_a + sum_a;  // per-thread partial row sums; reduced over the quad at the end
    l_b = l_b * corr_b + sum_b;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      o[n][0] *= corr_a;
      o[n][1] *= corr_a;
      o[n][2] *= corr_b;
      o[n][3] *= corr_b;
    }
    // O += P V: P's accumulator tiles re-packed as A fragments (k = keys)
#pragma unroll
    for (int kk = 0; kk < kKB / 16; ++kk) {
      const uint32_t a0 = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
      const uint32_t a1 = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
      const uint32_t a2 = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      const uint32_t a3 = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int np = 0; np < NT / 2; ++np) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(bv + (16 * kk + (lane & 15)) * LD + 16 * np + (lane >> 4) * 8, b0, b1, b2, b3);
        mma16816(o[2 * np], a0, a1, a2, a3, b0, b1);
        mma16816(o[2 * np + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    __syncthreads();  // stage st is refilled by the next iteration's prefetch
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
  for (int off = 1; off < 4; off <<= 1) {
    l_a += __shfl_xor_sync(0xffffffffu, l_a, off);
    l_b += __shfl_xor_sync(0xffffffffu, l_b, off);
  }
  const float inv_a = l_a > 0.f ? 1.f / l_a : 0.f, inv_b = l_b > 0.f ? 1.f / l_b : 0.f;
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    const int c = h * HD + 8 * n + 2 * (lane & 3);
    if (row_a < len)
      *reinterpret_cast<__nv_bfloat162*>(out + (size_t)(start + row_a) * out_stride + c) =
          __floats2bfloat162_rn(o[n][0] * inv_a, o[n][1] * inv_a);
    if (row_b < len)
      *reinterpret_cast<__nv_bfloat162*>(out + (size_t)(start + row_b) * out_stride + c) =
          __floats2bfloat162_rn(o[n][2] * inv_b, o[n][3] * inv_b);
  }
}

// The same computation with two 16-row m tiles per warp (4 warps x 32 query rows = 128-query CTAs):
// every K / V fragment loaded from shared memory feeds both m tiles, halving the ldmatrix traffic
// per MMA; Q is re-read from shared memory per k step instead of held in registers.  Per query row
// the arithmetic (MMA order, masking, softmax updates, P.V order) is exactly prefill_attn_kernel's,
// so the two kernels return the same bits.
template <int HD>
__global__ void __launch_bounds__(128, 1)
prefill_attn_wide_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
                         const __nv_bfloat16* __restrict__ v, int q_stride, int kv_stride,
                         const int32_t* __restrict__ cu, int H, int KV, float scale_log2,
                         __nv_bfloat16* __restrict__ out, int out_stride) {
  pdl_wait();
  pdl_trigger();
  constexpr int kQB = 128, kThreads = 128, MT = 2;
  constexpr int LD = HD + 8;
  constexpr int NT = HD / 8;
  constexpr int KS = HD / 16;
  extern __shared__ __align__(16) __nv_bfloat16 smem[];
  __nv_bfloat16* sQ = smem;
  __nv_bfloat16* sK = sQ + kQB * LD;
  __nv_bfloat16* sV = sK + 2 * kKB * LD;
  const int b = blockIdx.z, h = blockIdx.y, qb = gridDim.x - 1 - blockIdx.x;
  const int start = cu[b], len = cu[b + 1] - start;
  const int q0 = qb * kQB;
  if (q0 >= len) return;
  const int g = h / (H / KV);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int kPieces = HD / 8;
  for (int i = tid; i < kQB * kPieces; i += kThreads) {
    const int r = i / kPieces, c = (i % kPieces) * 8;
    const int t = q0 + r;
    cp16(sQ + r * LD + c, q + (size_t)(start + min(t, len - 1)) * q_stride + h * HD + c, t < len);
  }
  auto load_kv = [&](int kb, int st) {
    const int k0 = kb * kKB;
    __nv_bfloat16* dk = sK + st * kKB * LD;
    __nv_bfloat16* dv = sV + st * kKB * LD;
    for (int i = tid; i < kKB * kPieces; i += kThreads) {
      const int r = i / kPieces, c = (i % kPieces) * 8;
      const int t = k0 + r;
      const size_t row = (size_t)(start + min(t, len - 1)) * kv_stride + g * HD + c;
      cp16(dk + r * LD + c, k + row, t < len);
      cp16(dv + r * LD + c, v + row, t < len);
    }
  };
  const int nkb = min((len + kKB - 1) / kKB, (q0 + kQB - 1) / kKB + 1);
  load_kv(0, 0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  const int qr0 = warp * 32;  // m tile mt: rows qr0 + 16 mt .. + 15
  int row_a[MT], row_b[MT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    row_a[mt] = q0 + qr0 + 16 * mt + (lane >> 2);
    row_b[mt] = row_a[mt] + 8;
  }
  float o[MT][NT][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int n = 0; n < NT; ++n) o[mt][n][0] = o[mt][n][1] = o[mt][n][2] = o[mt][n][3] = 0.f;
  float m_a[MT], m_b[MT], l_a[MT], l_b[MT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    m_a[mt] = m_b[mt] = -INFINITY;
    l_a[mt] = l_b[mt] = 0.f;
  }
  for (int kb = 0; kb < nkb; ++kb) {
    const int st = kb & 1;
    if (kb + 1 < nkb) load_kv(kb + 1, st ^ 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    const __nv_bfloat16* bk = sK + st * kKB * LD;
    const __nv_bfloat16* bv = sV + st * kKB * LD;
    float s[MT][kKB / 8][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int n = 0; n < kKB / 8; ++n) s[mt][n][0] = s[mt][n][1] = s[mt][n][2] = s[mt][n][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      uint32_t qa[MT][4];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
        ldsm_x4(sQ + (qr0 + 16 * mt + (lane & 15)) * LD + ks * 16 + (lane >> 4) * 8, qa[mt][0], qa[mt][1], qa[mt][2],
                qa[mt][3]);
#pragma unroll
      for (int np = 0; np < kKB / 16; ++np) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(bk + (16 * np + (lane >> 4) * 8 + (lane & 7)) * LD + ks * 16 + ((lane >> 3) & 1) * 8, b0, b1, b2, b3);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          mma16816(s[mt][2 * np], qa[mt][0], qa[mt][1], qa[mt][2], qa[mt][3], b0, b1);
          mma16816(s[mt][2 * np + 1], qa[mt][0], qa[mt][1], qa[mt][2], qa[mt][3], b2, b3);
        }
      }
    }
    const int k0 = kb * kKB;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      float mx_a = m_a[mt], mx_b = m_b[mt];
#pragma unroll
      for (int n = 0; n < kKB / 8; ++n) {
        const int key = k0 + 8 * n + 2 * (lane & 3);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int kk = key + c;
          s[mt][n][c] = (kk <= row_a[mt] && kk < len) ? s[mt][n][c] * scale_log2 : -INFINITY;
          s[mt][n][2 + c] = (kk <= row_b[mt] && kk < len) ? s[mt][n][2 + c] * scale_log2 : -INFINITY;
          mx_a = fmaxf(mx_a, s[mt][n][c]);
          mx_b = fmaxf(mx_b, s[mt][n][2 + c]);
        }
      }
#pragma unroll
      for (int off = 1; off < 4; off <<= 1) {
        mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, off));
        mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, off));
      }
      const float base_a = mx_a == -INFINITY ? 0.f : mx_a, base_b = mx_b == -INFINITY ? 0.f : mx_b;
      const float corr_a = exp2f(m_a[mt] - base_a), corr_b = exp2f(m_b[mt] - base_b);
      m_a[mt] = mx_a;
      m_b[mt] = mx_b;
      float sum_a = 0.f, sum_b = 0.f;
#pragma unroll
      for (int n = 0; n < kKB / 8; ++n) {
        s[mt][n][0] = exp2f(s[mt][n][0] - base_a);
        s[mt][n][1] = exp2f(s[mt][n][1] - base_a);
        s[mt][n][2] = exp2f(s[mt][n][2] - base_b);
        s[mt][n][3] = exp2f(s[mt][n][3] - base_b);
        sum_a += s[mt][n][0] + s[mt][n][1];
        sum_b += s[mt][n][2] + s[mt][n][3];
      }
      l_a[mt] = l_a[mt] * corr_a + sum_a;
      l_b[mt] = l_b[mt] * corr_b + sum_b;
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        o[mt][n][0] *= corr_a;
        o[mt][n][1] *= corr_a;
        o[mt][n][2] *= corr_b;
        o[mt][n][3] *= corr_b;
      }
    }
#pragma unroll
    for (int kk = 0; kk < kKB / 16; ++kk) {
      uint32_t pa[MT][4];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        pa[mt][0] = pack_bf16(s[mt][2 * kk][0], s[mt][2 * kk][1]);
        pa[mt][1] = pack_bf16(s[mt][2 * kk][2], s[mt][2 * kk][3]);
        pa[mt][2] = pack_bf16(s[mt][2 * kk + 1][0], s[mt][2 * kk + 1][1]);
        pa[mt][3] = pack_bf16(s[mt][2 * kk + 1][2], s[mt][2 * kk + 1][3]);
      }
#pragma unroll
      for (int np = 0; np < NT / 2; ++np) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(bv + (16 * kk + (lane & 15)) * LD + 16 * np + (lane >> 4) * 8, b0, b1, b2, b3);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          mma16816(o[mt][2 * np], pa[mt][0], pa[mt][1], pa[mt][2], pa[mt][3], b0, b1);
          mma16816(o[mt][2 * np + 1], pa[mt][0], pa[mt][1], pa[mt][2], pa[mt][3], b2, b3);
        }
      }
    }
    __syncthreads();
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    float la = l_a[mt], lb = l_b[mt];
#pragma unroll
    for (int off = 1; off < 4; off <<= 1) {
      la += __shfl_xor_sync(0xffffffffu, la, off);
      lb += __shfl_xor_sync(0xffffffffu, lb, off);
    }
    const float inv_a = la > 0.f ? 1.f / la : 0.f, inv_b = lb > 0.f ? 1.f / lb : 0.f;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int c = h * HD + 8 * n + 2 * (lane & 3);
      if (row_a[mt] < len)
        *reinterpret_cast<__nv_bfloat162*>(out + (size_t)(start + row_a[mt]) * out_stride + c) =
            __floats2bfloat162_rn(o[mt][n][0] * inv_a, o[mt][n][1] * inv_a);
      if (row_b[mt] < len)
        *reinterpret_cast<__nv_bfloat162*>(out + (size_t)(start + row_b[mt]) * out_stride + c) =
            __floats2bfloat162_rn(o[mt][n][2] * inv_b, o[mt][n][3] * inv_b);
    }
  }
}

template <int HD>
int launch_prefill_wide(const void* q, const void* k, const void* v, int q_stride, int kv_stride, const int32_t* cu,
                        int B, int max_len, int H, int KV, float scale, void* out, int out_stride, cudaStream_t s) {
  constexpr int smem = (128 + 4 * kKB) * (HD + 8) * 2;
  static uint64_t attr_set = 0;  // devices already configured
  if (!(attr_set & current_device_bit())) {
    QMOE_CUDA_TRY(
        cudaFuncSetAttribute(prefill_attn_wide_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set |= current_device_bit();
  }
  const dim3 grid((max_len + 127) / 128, H, B);
  return launch_pdl("qmoe_prefill_attention(wide)", prefill_attn_wide_kernel<HD>, grid, dim3(128), smem, s,
                    (const __nv_bfloat16*)q, (const __nv_bfloat16*)k, (const __nv_bfloat16*)v, q_stride, kv_stride, cu,
                    H, KV, scale * 1.4426950408889634f, (__nv_bfloat16*)out, out_stride);
}

template <int HD, int W>
int launch_prefill(const void* q, const void* k, const void* v, int q_stride, int kv_stride, const int32_t* cu, int B,
                   int max_len, int H, int KV, float scale, void* out, int out_stride, cudaStream_t s) {
  constexpr int smem = (16 * W + 4 * kKB) * (HD + 8) * 2;
  static uint64_t attr_set = 0;  // devices already configured
  if (!(attr_set & current_device_bit())) {
    QMOE_CUDA_TRY(cudaFuncSetAttribute(prefill_attn_kernel<HD, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set |= current_device_bit();
  }
  const dim3 grid((max_len + 16 * W - 1) / (16 * W), H, B);
  return launch_pdl("qmoe_prefill_attention", prefill_attn_kernel<HD, W>, grid, dim3(W * 32), smem, s,
                    (const __nv_bfloat16*)q, (const __nv_bfloat16*)k, (const __nv_bfloat16*)v, q_stride, kv_stride, cu,
                    H, KV, scale * 1.4426950408889634f, (__nv_bfloat16*)out, out_stride);
}

// 128-query CTAs halve the K/V tile loads per query row (and the 32-row warps halve the ldmatrix
// traffic per MMA); 64-query CTAs keep short prompts spread over more CTAs.  QMOE_PREFILL_W forces one: 4 / 8 = prefill_attn_kernel with 4 / 8 warps of 16
// rows, 2 = prefill_attn_wide_kernel (4 warps of 32 rows).
template <int HD>
int dispatch_prefill(const void* q, const void* k, const void* v, int q_stride, int kv_stride, const int32_t* cu,
                     int B, int max_len, int H, int KV, float scale, void* out, int out_stride, cudaStream_t s) {
  static const int w_env = [] {
    const char* e = getenv("QMOE_PREFILL_W");
    return e == nullptr ? 0 : atoi(e);
  }();
  // measured (tools/prefill_attn_ab.py): the 32-row kernel wins from 256-token prompts (Mixtral heads
  // 8 x 256: 0.051 vs 0.058 ms; 1 x 4096: 0.553 vs 0.680), the 64-query one for 16 x 64 (0.030 vs 0.033)
  if (w_env == 2 || (w_env == 0 && max_len >= 256))  // 4 warps x 32 rows
    return launch_prefill_wide<HD>(q, k, v, q_stride, kv_stride, cu, B, max_len, H, KV, scale, out, out_stride, s);
  return w_env == 8 ? launch_prefill<HD, 8>(q, k, v, q_stride, kv_stride, cu, B, max_len, H, KV, scale, out, out_stride, s)
                    : launch_prefill<HD, 4>(q, k, v, q_stride, kv_stride, cu, B, max_len, H, KV, scale, out, out_stride, s);
}

}  // namespace
}  // namespace qmoe

extern "C" int qmoe_prefill_attention(const void* q, const void* k, const void* v, int q_stride, int kv_stride,
                                      const int32_t* cu_seqlens, int B, int max_len, int H, int KV, int head_dim,
                                      float scale, void* out, int out_stride, void* stream) {
  using namespace qmoe;
  QMOE_REQUIRE(B >= 0 && max_len >= 0, "qmoe_prefill_attention: bad sizes B=%d max_len=%d", B, max_len);
  QMOE_REQUIRE(H >= 1 && KV >= 1 && H % KV == 0, "qmoe_prefill_attention: H=%d must be a multiple of KV=%d", H, KV);
  QMOE_REQUIRE(head_dim == 64 || head_dim == 128, "qmoe_prefill_attention: head_dim %d (64 or 128)", head_dim);
  QMOE_REQUIRE(q_stride >= H * head_dim && kv_stride >= KV * head_dim && out_stride >= H * head_dim &&
                   q_stride % 8 == 0 && kv_stride % 8 == 0 && out_stride % 2 == 0,
               "qmoe_prefill_attention: row strides q=%d kv=%d out=%d", q_stride, kv_stride, out_stride);
  if (B == 0 || max_len == 0) return QMOE_OK;
  QMOE_REQUIRE(q && k && v && cu_seqlens && out, "qmoe_prefill_attention: null pointer");
  QMOE_REQUIRE(((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) & 15) ==
                   0,
               "qmoe_prefill_attention: q / k / v must be 16-byte aligned");
  QMOE_REQUIRE(B <= 65535 && H <= 65535, "qmoe_prefill_attention: B=%d H=%d exceed the grid", B, H);
  cudaStream_t s = as_stream(stream);
  return head_dim == 128 ? dispatch_prefill<128>(q, k, v, q_stride, kv_stride, cu_seqlens, B, max_len, H, KV, scale, out,
                                               out_stride, s)
                         : dispatch_prefill<64>(q, k, v, q_stride, kv_stride, cu_seqlens, B, max_len, H, KV, scale, out,
                                              out_stride, s);
}
