// Router kernel: gate GEMV/skinny GEMM + top-k (lower id wins ties) + softmax over the picks.
//
// Replaces MoEModel.route / route_many (reference model.py:115-134) and select_top_k /
// softmax_over (model.py:71-80).  HBM-bound on X: each token row is read once; W_router (E x d)
// stays L1/L2-resident and is reused across the TPC tokens a CTA owns (register blocking).
#include "common.cuh"

namespace qmoe {
namespace {

constexpr int kWarps = 4;      // warps per CTA
constexpr int kExpChunk = 8;   // experts accumulated per pass over d
constexpr int kMaxE = 64;

template <typename T> struct Vec;
template <> struct Vec<__nv_bfloat16> { static constexpr int N = 8; using U = uint4; };
template <> struct Vec<float> { static constexpr int N = 4; using U = float4; };
template <> struct Vec<double> { static constexpr int N = 2; using U = double2; };

template <typename T, typename A>
__device__ __forceinline__ void unpack(const typename Vec<T>::U& u, A* out);
template <> __device__ __forceinline__ void unpack<__nv_bfloat16, float>(const uint4& u, float* o) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    o[2 * i] = f.x;
    o[2 * i + 1] = f.y;
  }
}
template <> __device__ __forceinline__ void unpack<float, float>(const float4& u, float* o) {
  o[0] = u.x; o[1] = u.y; o[2] = u.z; o[3] = u.w;
}
template <> __device__ __forceinline__ void unpack<double, double>(const double2& u, double* o) {
  o[0] = u.x; o[1] = u.y;
}

template <typename A> __device__ __forceinline__ A warp_sum(A v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float exp_acc(float v) { return expf(v); }
__device__ __forceinline__ double exp_acc(double v) { return exp(v); }

// One CTA owns TPC tokens; its kWarps warps split the hidden dimension (so a decode batch still
// spreads over many CTAs), every lane keeps TPC x kExpChunk partial dot products in registers,
// and all loads of one step (TPC token vectors + kExpChunk weight vectors) are issued before any
// FMA so they are in flight together.  Partials are reduced across lanes (shuffles) and warps
// (shared memory); then one thread per token does the top-k selection.
// VEC: true -> 16-byte vector loads (requires d % Vec<T>::N == 0 and aligned rows).
template <typename T, int TPC, bool VEC>
__global__ void __launch_bounds__(kWarps * 32)
router_kernel(const T* __restrict__ x, const T* __restrict__ wr, int ntok, int d, int E, int k,
              int mode, int32_t* __restrict__ ids_out, typename AccOf<T>::type* __restrict__ w_out,
              typename AccOf<T>::type* __restrict__ logits_out) {
  using A = typename AccOf<T>::type;
  __shared__ A s_part[kWarps][TPC][kExpChunk];
  __shared__ A s_logit[TPC][kMaxE];
  const int warp = warp_id(), lane = lane_id();
  const int tok0 = blockIdx.x * TPC;
  constexpr int N = VEC ? Vec<T>::N : 1;
  // d range of this warp, in units of N elements
  const int nvec = d / N;
  const int per_warp = (nvec + kWarps - 1) / kWarps;
  const int v0 = warp * per_warp, v1 = min(nvec, v0 + per_warp);

  // Few experts (E <= 16): the warps split d and every warp covers all experts.  Many experts
  // (Qwen: 60): the warps take 8-expert chunks in parallel over the full d (no serial chunk loop).
  const bool split_d = E <= 2 * kExpChunk;
  const int c_begin = split_d ? 0 : warp * kExpChunk;
  const int c_step = split_d ? kExpChunk : kWarps * kExpChunk;
  const int w_v0 = split_d ? v0 : 0, w_v1 = split_d ? v1 : nvec;
  for (int ec = c_begin; ec < E; ec += c_step) {
    A acc[TPC][kExpChunk];
#pragma unroll
    for (int t = 0; t < TPC; ++t)
#pragma unroll
      for (int j = 0; j < kExpChunk; ++j) acc[t][j] = A(0);
    const T* wrow[kExpChunk];
#pragma unroll
    for (int j = 0; j < kExpChunk; ++j) wrow[j] = wr + (size_t)min(ec + j, E - 1) * d;  // clamp: no branch
    const T* xrow[TPC];
#pragma unroll
    for (int t = 0; t < TPC; ++t) xrow[t] = x + (size_t)min(tok0 + t, ntok - 1) * d;

    for (int v = w_v0 + lane; v < w_v1; v += 32) {
      A xv[TPC][N], wv[kExpChunk][N];
      if constexpr (VEC) {
        using U = typename Vec<T>::U;
        U xu[TPC], wu[kExpChunk];
#pragma unroll
        for (int t = 0; t < TPC; ++t) xu[t] = *reinterpret_cast<const U*>(xrow[t] + (size_t)v * N);
#pragma unroll
        for (int j = 0; j < kExpChunk; ++j) wu[j] = __ldg(reinterpret_cast<const U*>(wrow[j] + (size_t)v * N));
#pragma unroll
        for (int t = 0; t < TPC; ++t) unpack<T, A>(xu[t], xv[t]);
#pragma unroll
        for (int j = 0; j < kExpChunk; ++j) unpack<T, A>(wu[j], wv[j]);
      } else {
#pragma unroll
        for (int t = 0; t < TPC; ++t) xv[t][0] = load_as<T, A>(xrow[t] + v);
#pragma unroll
        for (int j = 0; j < kExpChunk; ++j) wv[j][0] = load_as<T, A>(wrow[j] + v);
      }
#pragma unroll
      for (int t = 0; t < TPC; ++t)
#pragma unroll
        for (int j = 0; j < kExpChunk; ++j)
#pragma unroll
          for (int q = 0; q < N; ++q) acc[t][j] += xv[t][q] * wv[j][q];
    }
    if (split_d) {
#pragma unroll
      for (int t = 0; t < TPC; ++t)
#pragma unroll
        for (int j = 0; j < kExpChunk; ++j) {
          const A sum = warp_sum(acc[t][j]);
          if (lane == 0) s_part[warp][t][j] = sum;
        }
      __syncthreads();
      if (threadIdx.x < TPC * kExpChunk) {
        const int t = threadIdx.x / kExpChunk, j = threadIdx.x % kExpChunk;
        A sum = A(0);
#pragma unroll
        for (int w = 0; w < kWarps; ++w) sum += s_part[w][t][j];
        if (ec + j < E) s_logit[t][ec + j] = sum;
      }
      __syncthreads();
    } else {
#pragma unroll
      for (int t = 0; t < TPC; ++t)
#pragma unroll
        for (int j = 0; j < kExpChunk; ++j) {
          const A sum = warp_sum(acc[t][j]);
          if (lane == 0 && ec + j < E) s_logit[t][ec + j] = sum;
        }
    }
  }
  if (!split_d) __syncthreads();

  // Selection: thread t owns token tok0 + t.
  if (threadIdx.x < TPC) {
    const int tok = tok0 + threadIdx.x;
    if (tok < ntok) {
      const A* lg = s_logit[threadIdx.x];
      if (logits_out != nullptr)
        for (int e = 0; e < E; ++e) logits_out[(size_t)tok * E + e] = lg[e];
      A score[kMaxE];  // value the top-k ranks on
      if (mode == QMOE_ROUTE_SOFTMAX_TOPK) {
        A m_all = lg[0];
        for (int e = 1; e < E; ++e) m_all = lg[e] > m_all ? lg[e] : m_all;
        A tot = A(0);
        for (int e = 0; e < E; ++e) {
          score[e] = exp_acc(lg[e] - m_all);
          tot += score[e];
        }
        for (int e = 0; e < E; ++e) score[e] = score[e] / tot;
      } else {
        for (int e = 0; e < E; ++e) score[e] = lg[e];
      }
      // top-k by (score desc, id asc): scanning ascending ids with a strict '>' keeps the lower
      // id on ties (model.py:74 sorts by (-value, id)).
      uint64_t chosen = 0;
      for (int r = 0; r < k; ++r) {
        int best = -1;
        A bv = A(0);
        for (int e = 0; e < E; ++e) {
          if ((chosen >> e) & 1ull) continue;
          if (best < 0 || score[e] > bv) { best = e; bv = score[e]; }
        }
        chosen |= 1ull << best;
      }
      // ids ascending (model.py:75 / :129), weights in the same order.
      int pick[8];
      int n = 0;
      for (int e = 0; e < E; ++e)
        if ((chosen >> e) & 1ull) pick[n++] = e;
      A wv[8];
      if (mode == QMOE_ROUTE_SOFTMAX_TOPK) {
        for (int j = 0; j < k; ++j) wv[j] = score[pick[j]];
      } else {
        A m = lg[pick[0]];
        for (int j = 1; j < k; ++j) m = lg[pick[j]] > m ? lg[pick[j]] : m;
        A tot = A(0);
        for (int j = 0; j < k; ++j) {
          wv[j] = exp_acc(lg[pick[j]] - m);
          tot += wv[j];
        }
        for (int j = 0; j < k; ++j) wv[j] = wv[j] / tot;
      }
      for (int j = 0; j < k; ++j) {
        ids_out[(size_t)tok * k + j] = pick[j];
        w_out[(size_t)tok * k + j] = wv[j];
      }
    }
  }
}

template <typename T, int TPC>
int launch_router(const void* x, const void* wr, int T_, int d, int E, int k, int mode, int32_t* ids,
                  void* w, void* logits, cudaStream_t s) {
  using A = typename AccOf<T>::type;
  dim3 grid((T_ + TPC - 1) / TPC);
  const bool vec = (d % Vec<T>::N == 0) && (reinterpret_cast<uintptr_t>(x) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(wr) % 16 == 0);
  if (vec)
    router_kernel<T, TPC, true><<<grid, kWarps * 32, 0, s>>>(
        (const T*)x, (const T*)wr, T_, d, E, k, mode, ids, (A*)w, (A*)logits);
  else
    router_kernel<T, TPC, false><<<grid, kWarps * 32, 0, s>>>(
        (const T*)x, (const T*)wr, T_, d, E, k, mode, ids, (A*)w, (A*)logits);
  return check_launch("qmoe_router");
}

}  // namespace
}  // namespace qmoe

extern "C" int qmoe_router(const void* x, const void* w_router, int T, int d, int E, int k, int dtype,
                           int route_mode, int32_t* ids_out, void* w_out, void* logits_out,
                           void* stream) {
  using namespace qmoe;
  QMOE_REQUIRE(T >= 0 && d >= 1, "qmoe_router: bad sizes T=%d d=%d", T, d);
  QMOE_REQUIRE(E >= 1 && E <= kMaxE, "qmoe_router: E=%d outside [1, %d]", E, kMaxE);
  QMOE_REQUIRE(k >= 1 && k <= E && k <= 8, "qmoe_router: k=%d must satisfy 1 <= k <= min(E, 8)", k);
  QMOE_REQUIRE(route_mode == QMOE_ROUTE_TOPK_SOFTMAX || route_mode == QMOE_ROUTE_SOFTMAX_TOPK,
               "qmoe_router: unknown route_mode %d", route_mode);
  if (T == 0) return QMOE_OK;
  QMOE_REQUIRE(x && w_router && ids_out && w_out, "qmoe_router: null pointer");
  cudaStream_t s = as_stream(stream);
  // Few tokens (decode): one token per CTA maximises the CTA count; many tokens: 4 per CTA so
  // every W_router load feeds 4 dot products.
  const bool small = T < 148 * 8;
  switch (dtype) {
    case QMOE_BF16:
      return small ? launch_router<__nv_bfloat16, 1>(x, w_router, T, d, E, k, route_mode, ids_out, w_out, logits_out, s)
                   : launch_router<__nv_bfloat16, 4>(x, w_router, T, d, E, k, route_mode, ids_out, w_out, logits_out, s);
    case QMOE_F32:
      return small ? launch_router<float, 1>(x, w_router, T, d, E, k, route_mode, ids_out, w_out, logits_out, s)
                   : launch_router<float, 4>(x, w_router, T, d, E, k, route_mode, ids_out, w_out, logits_out, s);
    case QMOE_F64:
      return launch_router<double, 1>(x, w_router, T, d, E, k, route_mode, ids_out, w_out, logits_out, s);
    default:
      set_error("qmoe_router: unknown dtype %d", dtype);
      return QMOE_ERR_INVALID;
  }
}
