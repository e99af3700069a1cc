// Paged decode attention over the engine's KV page pool (the reference's
// attention stage is engine.py:252-301 / model.py:58-68, a toy single-head softmax attention --
// the decoders' GQA attention with RoPE has no reference counterpart and follows HF
// MixtralAttention / Qwen2MoeAttention).
//
// One query token per sequence (decode).  pool layout (kvcache.py): [n_pages, page, 2, KV, hd]
// bf16, K at [.., 0, ..], V at [.., 1, ..]; block_table[b] lists sequence b's pages; seq_lens[b]
// counts its cached tokens including the new one (the query sits at position seq_lens[b] - 1 and
// attends every cached token).
//
// Flash-decoding split over pages: CTA (b, g, s) owns KV head g of sequence b and page s of its
// block table, for the G = H / KV query heads of that group.  Memory-bound: a page is page*hd*2*2
// bytes of K+V per KV head.  Warp w takes 32-token blocks of the page:
//   scores  lane i owns token i of the block and reads its whole K row (16 x 16-byte loads) -> G
//           dot products with the query heads held in registers (fp32);
//   softmax online per head with warp max / sum reductions;
//   values  lanes switch to owning 4 feature columns: for each token of the block the warp reads
//           its V row (coalesced 256 B), p broadcast by shuffle, o[h][4 cols] += p * v.
// The CTA merges its warps' (m, l, o) in shared memory and stores one partial per page; the last
// CTA of (b, g) (atomic arrival count, re-zeroed) merges the pages in page order (deterministic)
// and writes o in bf16.
#include "common.cuh"

namespace qmoe {
namespace {

constexpr int kHd = 128;
constexpr int kAttnWarps = 4;
constexpr int kMaxG = 8;
// Arrival counters sit at a FIXED offset (the head of the workspace) with a fixed capacity, so a
// workspace reused across calls of different shapes keeps them zero: the page partials, which
// every call fully rewrites before reading, never overlap them.
constexpr int kMaxCounters = 8192;  // B * KV per call

struct AttnPartial {
  float m[kMaxG], l[kMaxG];
  float o[kMaxG][kHd];
};

template <int G, int HD>
__global__ void __launch_bounds__(kAttnWarps * 32)
paged_decode_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ pool,
                    const int32_t* __restrict__ block_table, const int32_t* __restrict__ seq_lens, int H, int KV,
                    int page, int max_pages, float scale, __nv_bfloat16* __restrict__ out,
                    AttnPartial* __restrict__ parts, int* __restrict__ arrivals, int q_stride) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.x, g = blockIdx.y, sp = blockIdx.z;
  const int len = seq_lens[b];
  const int npages = (len + page - 1) / page;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ float s_m[kAttnWarps][G], s_l[kAttnWarps][G];
  constexpr int CPL = HD / 32;  // feature columns per lane in the value pass
  __shared__ float s_o[kAttnWarps][G][HD];
  __shared__ int s_last;
  float m[G], l[G], o[G][CPL];
#pragma unroll
  for (int h = 0; h < G; ++h) {
    m[h] = -INFINITY;
    l[h] = 0.f;
#pragma unroll
    for (int c = 0; c < CPL; ++c) o[h][c] = 0.f;
  }
  // query heads g*G .. g*G+G-1 (scaled, fp32) in shared memory: every lane reads them as
  // broadcasts while it walks its own token's K row
  __shared__ __align__(16) float s_q[G][HD];
  for (int i = threadIdx.x; i < G * HD; i += blockDim.x)
    s_q[i / HD][i % HD] = __bfloat162float(q[(size_t)b * q_stride + (size_t)g * G * HD + i]) * scale;
  __syncthreads();
  if (sp < npages) {
    const int pg = block_table[(size_t)b * max_pages + sp];
    const int t0 = sp * page;
    const int tn = min(page, len - t0);  // tokens of this page
    const size_t tok_stride = (size_t)2 * KV * HD;  // elements between consecutive tokens
    const __nv_bfloat16* kbase = pool + (size_t)pg * page * tok_stride + (size_t)g * HD;
    const __nv_bfloat16* vbase = kbase + (size_t)KV * HD;
    for (int blk = warp * 32; blk < tn; blk += kAttnWarps * 32) {
      const int t = blk + lane;
      const bool valid = t < tn;
      float s[G];
#pragma unroll
      for (int h = 0; h < G; ++h) s[h] = 0.f;
      if (valid) {
        const uint4* kr = reinterpret_cast<const uint4*>(kbase + (size_t)t * tok_stride);
#pragma unroll 4
        for (int i = 0; i < HD / 8; ++i) {
          const uint4 u = __ldg(kr + i);
          const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&u);
          float kf[8];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 f = __bfloat1622float2(p2[j]);
            kf[2 * j] = f.x;
            kf[2 * j + 1] = f.y;
          }
#pragma unroll
          for (int h = 0; h < G; ++h) {
            const float4 qa = *reinterpret_cast<const float4*>(&s_q[h][8 * i]);
            const float4 qb = *reinterpret_cast<const float4*>(&s_q[h][8 * i + 4]);
            s[h] += qa.x * kf[0] + qa.y * kf[1] + qa.z * kf[2] + qa.w * kf[3] + qb.x * kf[4] + qb.y * kf[5] +
                    qb.z * kf[6] + qb.w * kf[7];
          }
        }
      }
      float p[G];
#pragma unroll
      for (int h = 0; h < G; ++h) {
        float bm = valid ? s[h] : -INFINITY;
#pragma unroll
        for (int o2 = 16; o2 > 0; o2 >>= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, o2));
        const float mn = fmaxf(m[h], bm);
        const float corr = __expf(m[h] - mn);  // m = -inf initially: corr = 0
        p[h] = valid ? __expf(s[h] - mn) : 0.f;
        float ps = p[h];
#pragma unroll
        for (int o2 = 16; o2 > 0; o2 >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o2);
        l[h] = l[h] * corr + ps;
        m[h] = mn;
#pragma unroll
        for (int c = 0; c < CPL; ++c) o[h][c] *= corr;
      }
      // values: lane owns columns CPL*lane .. CPL*lane+CPL-1; token j's V row is read by the whole warp
      const int nb = min(32, tn - blk);
      for (int j = 0; j < nb; ++j) {
        float vf[CPL];
        const __nv_bfloat16* vr = vbase + (size_t)(blk + j) * tok_stride;
        if constexpr (CPL == 4) {
          const uint2 u = __ldg(reinterpret_cast<const uint2*>(vr) + lane);
          const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&u);
          const float2 a = __bfloat1622float2(p2[0]), c2 = __bfloat1622float2(p2[1]);
          vf[0] = a.x; vf[1] = a.y; vf[2] = c2.x; vf[3] = c2.y;
        } else {
          const unsigned u = __ldg(reinterpret_cast<const unsigned*>(vr) + lane);
          const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u));
          vf[0] = a.x; vf[1] = a.y;
        }
#pragma unroll
        for (int h = 0; h < G; ++h) {
          const float pj = __shfl_sync(0xffffffffu, p[h], j);
#pragma unroll
          for (int c = 0; c < CPL; ++c) o[h][c] += pj * vf[c];
        }
      }
    }
  }
  // merge the CTA's warps, then store this page's partial
#pragma unroll
  for (int h = 0; h < G; ++h) {
    if (lane == 0) {
      s_m[warp][h] = m[h];
      s_l[warp][h] = l[h];
    }
#pragma unroll
    for (int c = 0; c < CPL; ++c) s_o[warp][h][CPL * lane + c] = o[h][c];
  }
  __syncthreads();
  AttnPartial* part = parts + ((size_t)b * KV + g) * max_pages + sp;
  for (int i = threadIdx.x; i < G * HD; i += blockDim.x) {
    const int h = i / HD, c = i - h * HD;
    float mm = -INFINITY;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) mm = fmaxf(mm, s_m[w][h]);
    float acc = 0.f, ll = 0.f;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) {
      const float f = s_m[w][h] == -INFINITY ? 0.f : __expf(s_m[w][h] - mm);
      acc += f * s_o[w][h][c];
      ll += f * s_l[w][h];
    }
    part->o[h][c] = acc;
    if (c == 0) {
      part->m[h] = mm;
      part->l[h] = ll;
    }
  }
  // last CTA of (b, g) merges the pages in order
  __threadfence();
  __syncthreads();
  const int nsp = gridDim.z;
  if (threadIdx.x == 0) s_last = atomicAdd(&arrivals[b * KV + g], 1) == nsp - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const AttnPartial* ps = parts + ((size_t)b * KV + g) * max_pages;
  const int used = min(npages, nsp);
  for (int i = threadIdx.x; i < G * HD; i += blockDim.x) {
    const int h = i / HD, c = i - h * HD;
    float mm = -INFINITY;
    for (int s2 = 0; s2 < used; ++s2) mm = fmaxf(mm, ps[s2].m[h]);
    float acc = 0.f, ll = 0.f;
    for (int s2 = 0; s2 < used; ++s2) {
      const float pm = ps[s2].m[h];
      const float f = pm == -INFINITY ? 0.f : __expf(pm - mm);
      acc += f * ps[s2].o[h][c];
      ll += f * ps[s2].l[h];
    }
    out[((size_t)b * H + g * G + h) * HD + c] = __float2bfloat16_rn(ll > 0.f ? acc / ll : 0.f);
  }
  if (threadIdx.x == 0) arrivals[b * KV + g] = 0;
}

template <int G, int HD>
int launch_decode(const void* q, int q_stride, const void* pool, const int32_t* bt, const int32_t* lens, int B, int H,
                  int KV, int page, int max_pages, int splits, float scale, void* out, void* ws, cudaStream_t s) {
  int* arrivals = reinterpret_cast<int*>(ws);
  AttnPartial* parts = reinterpret_cast<AttnPartial*>(arrivals + kMaxCounters);
  return launch_pdl("qmoe_paged_decode_attention", paged_decode_kernel<G, HD>, dim3(B, KV, splits),
                    dim3(kAttnWarps * 32), 0, s, (const __nv_bfloat16*)q, (const __nv_bfloat16*)pool, bt, lens, H, KV,
                    page, max_pages, scale, (__nv_bfloat16*)out, parts, arrivals, q_stride);
}

}  // namespace
}  // namespace qmoe

extern "C" size_t qmoe_paged_decode_attention_workspace_bytes(int B, int KV, int max_pages) {
  return sizeof(int) * (size_t)qmoe::kMaxCounters + sizeof(qmoe::AttnPartial) * (size_t)B * KV * max_pages;
}

extern "C" int qmoe_paged_decode_attention(const void* q, int q_stride, const void* pool, const int32_t* block_table,
                                           const int32_t* seq_lens, int B, int H, int KV, int head_dim,
                                           int page_size, int max_pages, int max_len, float scale, void* out,
                                           void* workspace, size_t workspace_bytes, void* stream) {
  using namespace qmoe;
  QMOE_REQUIRE(head_dim == 128 || head_dim == 64, "qmoe_paged_decode_attention: head_dim must be 64 or 128 (got %d)",
               head_dim);
  QMOE_REQUIRE(B >= 0 && KV >= 1 && H % KV == 0 && H / KV <= kMaxG, "qmoe_paged_decode_attention: bad heads H=%d KV=%d",
               H, KV);
  QMOE_REQUIRE((size_t)B * KV <= (size_t)kMaxCounters, "qmoe_paged_decode_attention: B * KV %d > %d", B * KV,
               kMaxCounters);
  QMOE_REQUIRE(q_stride >= H * head_dim, "qmoe_paged_decode_attention: q_stride %d < H * head_dim", q_stride);
  QMOE_REQUIRE(page_size >= 1 && max_pages >= 1 && max_len >= 1 && max_len <= page_size * max_pages,
               "qmoe_paged_decode_attention: bad paging (page %d, pages %d, max_len %d)", page_size, max_pages,
               max_len);
  QMOE_REQUIRE(workspace != nullptr &&
                   workspace_bytes >= qmoe_paged_decode_attention_workspace_bytes(B, KV, max_pages),
               "qmoe_paged_decode_attention: workspace too small");
  if (B == 0) return QMOE_OK;
  QMOE_REQUIRE(q && pool && block_table && seq_lens && out, "qmoe_paged_decode_attention: null pointer");
  QMOE_REQUIRE(((uintptr_t)q | (uintptr_t)pool) % 16 == 0, "qmoe_paged_decode_attention: 16-byte alignment");
  const int splits = (max_len + page_size - 1) / page_size;  // one CTA per page of the longest sequence
  cudaStream_t s = as_stream(stream);
#define QMOE_ATTN_G(G_)                                                                                          \
  case G_:                                                                                                       \
    return head_dim == 128 ? launch_decode<G_, 128>(q, q_stride, pool, block_table, seq_lens, B, H, KV, page_size,   \
                                                    max_pages, splits, scale, out, workspace, s)                  \
                           : launch_decode<G_, 64>(q, q_stride, pool, block_table, seq_lens, B, H, KV, page_size,    \
                                                   max_pages, splits, scale, out, workspace, s);
  switch (H / KV) {
    QMOE_ATTN_G(1)
    QMOE_ATTN_G(2)
    QMOE_ATTN_G(4)
    default:
      set_error("qmoe_paged_decode_attention: group size %d unsupported (1, 2, 4)", H / KV);
      return QMOE_ERR_UNSUPPORTED;
  }
#undef QMOE_ATTN_G
}
