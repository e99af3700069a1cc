// Router kernel: gate GEMV/skinny GEMM + top-k (lower id wins ties) + softmax over the picks.
//
// Replaces MoEModel.route / route_many (reference model.py:115-134) and select_top_k /
// softmax_over (model.py:71-80).  HBM-bound on X: each token row is read once; W_router (E x d)
// stays L1/L2-resident and is reused across the TPC tokens a CTA owns (register blocking).
#include <stdlib.h>

#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace qmoe {
int tc_init_driver();  // expert_tc.cu: cuTensorMapEncodeTiled entry point (sm_100 check)
int tc_make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows);
namespace {

constexpr int kExpChunk = 8;   // experts accumulated per pass over d
constexpr int kNoSelect = 1 << 16;  // router_tc_kernel mode bit: skip the selection (timing runs)
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

// E logit rows.  ns > 0 (Qwen2-MoE shared expert run as ns sub-experts of the routed width): the
// last logit row is the shared expert's gate; top-k runs over the first E - 1 experts and the
// token's slots k .. k+ns-1 get ids E-1 .. E-2+ns with weight sigmoid(gate logit)
// (HF Qwen2MoeSparseMoeBlock: sigmoid(shared_expert_gate(h)) * shared_expert(h)).
// The kernels carry ns in bits 8.. of `mode` (set by qmoe_router_shared).
template <typename A>
__device__ __noinline__ void select_token(const A* lg, A* s_score, int tok, int E, int k, int mode, int lane,
                                             int32_t* __restrict__ ids_out, A* __restrict__ w_out,
                                             A* __restrict__ logits_out) {
  const int ns = mode >> 8;
  mode &= 0xFF;
  if (logits_out != nullptr) {
    if (lane < E) logits_out[(size_t)tok * E + lane] = lg[lane];
    if (lane + 32 < E) logits_out[(size_t)tok * E + lane + 32] = lg[lane + 32];
  }
  const int Er = ns > 0 ? E - 1 : E;  // experts eligible for the top-k
  const int ko = k + ns;              // slots per token
  const bool ok0 = lane < Er, ok1 = lane + 32 < Er;
  const A l0 = ok0 ? lg[lane] : A(0), l1 = ok1 ? lg[lane + 32] : A(0);
  A s0 = l0, s1 = l1;  // value the top-k ranks on
  if (mode == QMOE_ROUTE_SOFTMAX_TOPK) {
    A m = ok0 ? l0 : l1;
    if (ok1 && l1 > m) m = l1;
    for (int o = 16; o > 0; o >>= 1) {
      const A v = __shfl_xor_sync(0xffffffffu, m, o);
      m = v > m ? v : m;
    }
    // lanes >= E contribute nothing; E >= 1 so lane 0 always holds a real expert
    const A z0 = ok0 ? exp_acc(l0 - m) : A(0), z1 = ok1 ? exp_acc(l1 - m) : A(0);
    const A tot = warp_sum(z0 + z1);
    s0 = z0 / tot;
    s1 = z1 / tot;
    if (ok0) s_score[lane] = s0;
    if (ok1) s_score[lane + 32] = s1;
  }
  // top-k by (score desc, id asc): k warp-wide argmax rounds (model.py:74 sorts by (-value, id)).
  bool c0 = !ok0, c1 = !ok1;  // "taken" (or not an expert)
#pragma unroll 1
  for (int r = 0; r < k; ++r) {
    int bid = -1;
    A bv = A(0);
    if (!c0) { bid = lane; bv = s0; }
    if (!c1 && (bid < 0 || s1 > bv)) { bid = lane + 32; bv = s1; }
    for (int o = 16; o > 0; o >>= 1) {
      const A ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oid = __shfl_xor_sync(0xffffffffu, bid, o);
      if (oid >= 0 && (bid < 0 || ov > bv || (ov == bv && oid < bid))) { bv = ov; bid = oid; }
    }
    if (bid == lane) c0 = true;
    if (bid == lane + 32) c1 = true;
  }
  const unsigned lo = __ballot_sync(0xffffffffu, ok0 && c0), hi = __ballot_sync(0xffffffffu, ok1 && c1);
  if (lane != 0) return;
  uint64_t chosen = (uint64_t)lo | ((uint64_t)hi << 32);
  // ids ascending (model.py:75 / :129), weights in the same order.
  int pick[8];
  for (int j = 0; j < k; ++j) {
    pick[j] = __ffsll((long long)chosen) - 1;
    chosen &= chosen - 1;
  }
  A wv[8];
  if (mode == QMOE_ROUTE_SOFTMAX_TOPK) {
    for (int j = 0; j < k; ++j) wv[j] = s_score[pick[j]];
  } else {
    // softmax over the picked logits, summed in ascending id order (model.py:78-80)
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
    ids_out[(size_t)tok * ko + j] = pick[j];
    w_out[(size_t)tok * ko + j] = wv[j];
  }
  if (ns > 0) {
    const A g = A(1) / (A(1) + exp_acc(-lg[Er]));
    for (int s = 0; s < ns; ++s) {
      ids_out[(size_t)tok * ko + k + s] = Er + s;
      w_out[(size_t)tok * ko + k + s] = g;
    }
  }
}

// select_token for a group of G consecutive lanes (G | 32) instead of a warp, bit for bit: lane j of
// the group holds the logits of select_token's "lanes" L = j + G i (i < 32 / G), i.e. logit rows L
// and L + 32.  The maxima and the top-k winner are order-free (exact max; value desc, id asc); the
// softmax denominator replays warp_sum's butterfly (bit 4 of L first): the bits of L above log2 G
// are the bits of i, combined locally, then xor shuffles G/2 .. 1.  So one token costs
// log2 G shuffle levels instead of 5, and 256 / G tokens are selected at once by a CTA.
template <int G>
__device__ __forceinline__ void select_group(const float (&l0)[32 / G], const float (&l1)[32 / G], bool live, int tok,
                                             int E, int k, int mode, int j, int32_t* __restrict__ ids_out,
                                             float* __restrict__ w_out, float* __restrict__ logits_out) {
  constexpr int C = 32 / G;
  const int ns = mode >> 8;
  mode &= 0xFF;
  const int Er = ns > 0 ? E - 1 : E;
  const int ko = k + ns;
  if (live && logits_out != nullptr) {
#pragma unroll
    for (int i = 0; i < C; ++i) {
      const int L = j + G * i;
      if (L < E) logits_out[(size_t)tok * E + L] = l0[i];
      if (L + 32 < E) logits_out[(size_t)tok * E + L + 32] = l1[i];
    }
  }
  float s0[C], s1[C];
#pragma unroll
  for (int i = 0; i < C; ++i) {
    const int L = j + G * i;
    s0[i] = L < Er ? l0[i] : 0.f;
    s1[i] = L + 32 < Er ? l1[i] : 0.f;
  }
  if (mode == QMOE_ROUTE_SOFTMAX_TOPK) {
    float m = 0.f;
#pragma unroll
    for (int i = 0; i < C; ++i) {  // select_token's per-lane start value, then the max
      const int L = j + G * i;
      float v = L < Er ? s0[i] : s1[i];
      if (L + 32 < Er && s1[i] > v) v = s1[i];
      m = (i == 0 || v > m) ? v : m;
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      const float v = __shfl_xor_sync(0xffffffffu, m, o);
      m = v > m ? v : m;
    }
    float z0[C], z1[C], t[C];
#pragma unroll
    for (int i = 0; i < C; ++i) {
      const int L = j + G * i;
      z0[i] = L < Er ? exp_acc(s0[i] - m) : 0.f;
      z1[i] = L + 32 < Er ? exp_acc(s1[i] - m) : 0.f;
      t[i] = z0[i] + z1[i];
    }
#pragma unroll
    for (int h = C / 2; h > 0; h >>= 1)
#pragma unroll
      for (int i = 0; i < h; ++i) t[i] = t[i] + t[i + h];
    float tot = t[0];
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
#pragma unroll
    for (int i = 0; i < C; ++i) {
      s0[i] = z0[i] / tot;
      s1[i] = z1[i] / tot;
    }
  }
  // top-k by (score desc, id asc)
  uint32_t taken0 = 0, taken1 = 0;  // bit i: leaf i's row L (resp. L + 32) taken or not an expert
#pragma unroll
  for (int i = 0; i < C; ++i) {
    const int L = j + G * i;
    if (!(L < Er)) taken0 |= 1u << i;
    if (!(L + 32 < Er)) taken1 |= 1u << i;
  }
  int pick[8];
  float pv[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    pick[q] = 0x7fffffff;
    pv[q] = 0.f;
    if (q < k) {
      int bid = -1;
      float bv = 0.f;
#pragma unroll
      for (int i = 0; i < C; ++i) {
        const int L = j + G * i;
        if (!(taken0 >> i & 1) && (bid < 0 || s0[i] > bv || (s0[i] == bv && L < bid))) { bid = L; bv = s0[i]; }
        if (!(taken1 >> i & 1) && (bid < 0 || s1[i] > bv || (s1[i] == bv && L + 32 < bid))) { bid = L + 32; bv = s1[i]; }
      }
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oid = __shfl_xor_sync(0xffffffffu, bid, o);
        if (oid >= 0 && (bid < 0 || ov > bv || (ov == bv && oid < bid))) { bv = ov; bid = oid; }
      }
      pick[q] = bid;
      pv[q] = bv;
      if (bid >= 0 && (bid & 31) % G == j) {
        if (bid < 32) taken0 |= 1u << ((bid & 31) / G);
        else taken1 |= 1u << ((bid & 31) / G);
      }
    }
  }
  // ids ascending (model.py:75 / :129): an 8-element sorting network on (id, value)
#define QMOE_CX(a, b)                                                         \
  if (pick[b] < pick[a]) {                                                    \
    const int ti = pick[a]; pick[a] = pick[b]; pick[b] = ti;                  \
    const float tv = pv[a]; pv[a] = pv[b]; pv[b] = tv;                        \
  }
  QMOE_CX(0, 1) QMOE_CX(2, 3) QMOE_CX(4, 5) QMOE_CX(6, 7)
  QMOE_CX(0, 2) QMOE_CX(1, 3) QMOE_CX(4, 6) QMOE_CX(5, 7)
  QMOE_CX(1, 2) QMOE_CX(5, 6) QMOE_CX(0, 4) QMOE_CX(3, 7)
  QMOE_CX(1, 5) QMOE_CX(2, 6)
  QMOE_CX(1, 4) QMOE_CX(3, 6)
  QMOE_CX(2, 4) QMOE_CX(3, 5)
  QMOE_CX(3, 4)
#undef QMOE_CX
  float gl = 0.f;  // the shared expert's gate logit (row Er), from the lane that holds it
  if (ns > 0) {
    const int gi = (Er & 31) / G, gj = (Er & 31) % G;
#pragma unroll
    for (int i = 0; i < C; ++i)
      if (i == gi) gl = Er >= 32 ? l1[i] : l0[i];
    gl = __shfl_sync(0xffffffffu, gl, (threadIdx.x & 31 & ~(G - 1)) + gj);
  }
  if (!live || j != 0) return;
  float wv[8];
  if (mode == QMOE_ROUTE_SOFTMAX_TOPK) {
#pragma unroll
    for (int q = 0; q < 8; ++q) wv[q] = pv[q];
  } else {
    // softmax over the picked logits, summed in ascending id order (model.py:78-80)
    float m = pv[0];
#pragma unroll
    for (int q = 1; q < 8; ++q)
      if (q < k) m = pv[q] > m ? pv[q] : m;
    float tot = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < k) {
        wv[q] = exp_acc(pv[q] - m);
        tot += wv[q];
      }
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < k) wv[q] = wv[q] / tot;
  }
#pragma unroll
  for (int q = 0; q < 8; ++q)
    if (q < k) {
      ids_out[(size_t)tok * ko + q] = pick[q];
      w_out[(size_t)tok * ko + q] = wv[q];
    }
  if (ns > 0) {
    const float g = 1.f / (1.f + exp_acc(-gl));
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < ns) {
        ids_out[(size_t)tok * ko + k + q] = Er + q;
        w_out[(size_t)tok * ko + k + q] = g;
      }
  }
}

// Selection of a 16-token tile whose logits sit in shared memory (row stride kMaxE): the block's
// NT threads form 16 groups of G = NT / 16 lanes, one token each (select_group, bit-identical to
// select_token), instead of kWarps warps walking the 16 tokens in turn.
template <int NT>
__device__ __forceinline__ void select_tile16(const float* s_logit, int tok0, int ntok, int E, int k, int mode,
                                              int32_t* __restrict__ ids_out, float* __restrict__ w_out,
                                              float* __restrict__ logits_out) {
  constexpr int G = NT / 16, C = 32 / G;
  static_assert(G >= 1 && G <= 32 && 32 % G == 0, "16 groups of a power-of-two size");
  const int r = threadIdx.x / G, j = threadIdx.x % G;
  float l0[C], l1[C];
#pragma unroll
  for (int i = 0; i < C; ++i) {
    const int L = j + G * i;
    l0[i] = L < E ? s_logit[r * kMaxE + L] : 0.f;
    l1[i] = L + 32 < E ? s_logit[r * kMaxE + L + 32] : 0.f;
  }
  select_group<G>(l0, l1, tok0 + r < ntok, tok0 + r, E, k, mode, j, ids_out, w_out, logits_out);
}

// One CTA owns TPC tokens, split into TPC/TPW groups of TPW tokens; each group gets kWarps/groups
// warps laid out as (d slice) x (8-expert chunk).  Decode (TPC = 1): with few experts (Mixtral's 8)
// all 8 warps split d, with many (Qwen's 60) each warp owns one chunk over the whole of d, so a
// small batch still spreads over many warps.  Large batches: a warp owns TPW tokens over all of d
// (few shuffles per byte of X, HBM-bound on X).  Every lane keeps TPW x kExpChunk partial dot
// products in registers and issues all loads of a step (TPW token vectors + kExpChunk weight
// vectors) before any FMA.  Partials are reduced across lanes (shuffles) and d slices (shared
// memory, fixed slice order); then one warp per token does the selection with warp-wide argmax
// rounds.  Requires ceil(E/8) <= warps per group (checked by the host dispatch).
// VEC: true -> 16-byte vector loads (requires d % Vec<T>::N == 0 and aligned rows).
template <typename T, int TPC, int TPW, bool VEC, int kWarps = 8>
__global__ void __launch_bounds__(kWarps * 32)
router_kernel(const T* __restrict__ x, const T* __restrict__ wr, int ntok, int d, int E, int k,
              int mode, int32_t* __restrict__ ids_out, typename AccOf<T>::type* __restrict__ w_out,
              typename AccOf<T>::type* __restrict__ logits_out, int rounds) {
  pdl_wait();
  pdl_trigger();
  using A = typename AccOf<T>::type;
  constexpr int kGroups = TPC / TPW;
  constexpr int kWpg = kWarps / kGroups;  // warps per token group
  static_assert(kGroups * TPW == TPC && kWpg * kGroups == kWarps, "bad router tiling");
  __shared__ A s_part[kWpg][TPC][kMaxE];
  __shared__ A s_logit[TPC][kMaxE];
  __shared__ A s_score[TPC][kMaxE];
  const int warp = warp_id(), lane = lane_id();
  constexpr int N = VEC ? Vec<T>::N : 1;
  const int nvec = d / N;
  const int nchunk = (E + kExpChunk - 1) / kExpChunk;  // <= kWpg
  const int dsplit = kWpg / nchunk;                     // >= 1
  const int group = warp / kWpg, wig = warp % kWpg;
  const int chunk = wig % nchunk, slice = wig / nchunk;
  // `rounds` batches of TPC tokens per CTA: with many experts W_router (Qwen: 245 KB) is then
  // re-read from L1 instead of from L2 for every 4 tokens.
  for (int rnd = 0; rnd < rounds; ++rnd) {
  const int tok0 = (blockIdx.x * rounds + rnd) * TPC;
  if (tok0 >= ntok) break;
  if (slice < dsplit) {
    const int per = (nvec + dsplit - 1) / dsplit;
    const int v0 = slice * per, v1 = min(nvec, v0 + per);
    const int ec = chunk * kExpChunk;
    const int gt0 = group * TPW;  // first token of this group within the CTA
    A acc[TPW][kExpChunk];
#pragma unroll
    for (int t = 0; t < TPW; ++t)
#pragma unroll
      for (int j = 0; j < kExpChunk; ++j) acc[t][j] = A(0);
    const T* wrow[kExpChunk];
#pragma unroll
    for (int j = 0; j < kExpChunk; ++j) wrow[j] = wr + (size_t)min(ec + j, E - 1) * d;  // clamp: no branch
    const T* xrow[TPW];
#pragma unroll
    for (int t = 0; t < TPW; ++t) xrow[t] = x + (size_t)min(tok0 + gt0 + t, ntok - 1) * d;

#pragma unroll 2
    for (int v = v0 + lane; v < v1; v += 32) {
      A xv[TPW][N], wv[kExpChunk][N];
      if constexpr (VEC) {
        using U = typename Vec<T>::U;
        U xu[TPW], wu[kExpChunk];
#pragma unroll
        for (int t = 0; t < TPW; ++t) xu[t] = *reinterpret_cast<const U*>(xrow[t] + (size_t)v * N);
#pragma unroll
        for (int j = 0; j < kExpChunk; ++j) wu[j] = __ldg(reinterpret_cast<const U*>(wrow[j] + (size_t)v * N));
#pragma unroll
        for (int t = 0; t < TPW; ++t) unpack<T, A>(xu[t], xv[t]);
#pragma unroll
        for (int j = 0; j < kExpChunk; ++j) unpack<T, A>(wu[j], wv[j]);
      } else {
#pragma unroll
        for (int t = 0; t < TPW; ++t) xv[t][0] = load_as<T, A>(xrow[t] + v);
#pragma unroll
        for (int j = 0; j < kExpChunk; ++j) wv[j][0] = load_as<T, A>(wrow[j] + v);
      }
#pragma unroll
      for (int t = 0; t < TPW; ++t)
#pragma unroll
        for (int j = 0; j < kExpChunk; ++j)
#pragma unroll
          for (int q = 0; q < N; ++q) acc[t][j] += xv[t][q] * wv[j][q];
    }
#pragma unroll
    for (int t = 0; t < TPW; ++t)
#pragma unroll
      for (int j = 0; j < kExpChunk; ++j) {
        const A sum = warp_sum(acc[t][j]);
        if (lane == 0 && ec + j < E) s_part[slice][gt0 + t][ec + j] = sum;
      }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < TPC * E; i += kWarps * 32) {
    const int t = i / E, e = i - t * E;
    A sum = s_part[0][t][e];
    for (int sl = 1; sl < dsplit; ++sl) sum += s_part[sl][t][e];
    s_logit[t][e] = sum;
  }
  __syncthreads();

  // Selection: warp w owns tokens tok0 + w, tok0 + w + kWarps, ...; lane l holds experts l, l + 32.
#pragma unroll 1
  for (int ti = warp; ti < TPC; ti += kWarps) {
    const int tok = tok0 + ti;
    if (tok >= ntok) break;
    select_token<A>(s_logit[ti], s_score[ti], tok, E, k, mode, lane, ids_out, w_out, logits_out);
  }
  __syncthreads();  // s_part / s_logit / s_score are reused by the next round
  }
}


template <typename T, int TPC, int TPW, int NW = 8>
int launch_router(const void* x, const void* wr, int T_, int d, int E, int k, int mode, int32_t* ids,
                  void* w, void* logits, cudaStream_t s) {
  using A = typename AccOf<T>::type;
  const int nchunk = (E + kExpChunk - 1) / kExpChunk;
  const int rounds = nchunk > 2 && TPC > 1 ? 8 : 1;
  dim3 grid((T_ + TPC * rounds - 1) / (TPC * rounds));
  const bool vec = (d % Vec<T>::N == 0) && (reinterpret_cast<uintptr_t>(x) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(wr) % 16 == 0);
  if (vec)
    return launch_pdl("qmoe_router", router_kernel<T, TPC, TPW, true, NW>, grid, dim3(NW * 32), 0, s, (const T*)x,
                      (const T*)wr, T_, d, E, k, mode, ids, (A*)w, (A*)logits, rounds);
  return launch_pdl("qmoe_router", router_kernel<T, TPC, TPW, false, NW>, grid, dim3(NW * 32), 0, s, (const T*)x,
                    (const T*)wr, T_, d, E, k, mode, ids, (A*)w, (A*)logits, rounds);
}

// ---- bf16, many tokens: the logits as a skinny GEMM on the tensor cores ------------------------
// [T, d] x [d, E] with E <= 64 is HBM-bound on X (Qwen, T = 8k: 33 MB), but as fp32 FMAs it is
// ~1 GFMA of CUDA-core work and the SIMT kernel re-reads W_router (245 KB) from L2 for every few
// tokens.  Here a CTA owns 16 tokens x all experts; its 8 warps split K (warp w takes k16-step w of
// every 128-wide chunk), chunks of X and W_router are staged by cp.async (4 stages, padded rows
// for conflict-free ldmatrix) and multiplied with mma.sync m16n8k16 (bf16 in, fp32 accumulate;
// the same products as the FMA path).  The 8 partial logit tiles are summed in warp order (fixed,
// deterministic), then the logits go through the same selection as the SIMT kernel.  Small CTAs
// keep every SM busy down to ~2k tokens.
constexpr int kMmaTok = 16;
constexpr int kMmaK = 128;
constexpr int kLd = kMmaK + 8;  // bf16 per padded smem row
constexpr int kMmaStages = 4;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const int sz = pred ? 16 : 0;  // 0 -> zero-fill (rows past T or E)
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(sz) : "memory");
}
__device__ __forceinline__ void ldsm_x4(const void* smem, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(sa));
}
__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// NP n-tile pairs (experts padded to 16 * NP); MT 16-token tiles per CTA; KC K-chunk width (128 or
// 256: a 256-wide chunk halves the chunk iterations -- each with two barriers -- and warp w then
// takes k16 steps w and w + 8 of it, the same per-warp step sequence as two 128-wide chunks, so
// the logits are bit-identical)
template <int NP, int MT, int KC = kMmaK>
__global__ void __launch_bounds__(256)
router_mma_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wr, int ntok, int d, int E,
                  int k, int mode, int32_t* __restrict__ ids_out, float* __restrict__ w_out,
                  float* __restrict__ logits_out) {
  pdl_wait();
  pdl_trigger();
  constexpr int kTok = 16 * MT;
  extern __shared__ __align__(16) __nv_bfloat16 sbuf[];  // kMmaStages x (X chunk, W chunk); reused below
  const int warp = warp_id(), lane = lane_id();
  const int tok0 = blockIdx.x * kTok;
  constexpr int kLdC = KC + 8;     // bf16 per padded smem row
  constexpr int kPieces = KC / 8;  // 16-byte pieces per row
  const int nk = d / KC;
  constexpr int wrows = 16 * NP;  // W rows staged
  constexpr int stage_elems = (kTok + wrows) * kLdC;
  auto load = [&](int kc) {
    if (kc < nk) {
      __nv_bfloat16* sx = sbuf + (kc % kMmaStages) * stage_elems;
      __nv_bfloat16* sw = sx + kTok * kLdC;
      const int k0 = kc * KC;
      // (kTok + wrows) rows x kPieces pieces of 16 B over 256 threads
      for (int piece = threadIdx.x; piece < (kTok + wrows) * kPieces; piece += 256) {
        const int r = piece / kPieces, c = (piece % kPieces) * 8;
        if (r < kTok) {
          const int t = tok0 + r;
          cp_async16(sx + r * kLdC + c, x + (size_t)min(t, ntok - 1) * d + k0 + c, t < ntok);
        } else {
          const int e = r - kTok;
          cp_async16(sw + e * kLdC + c, wr + (size_t)min(e, E - 1) * d + k0 + c, e < E);
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");  // (possibly empty) group per chunk
  };
  float acc[MT][2 * NP][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int j = 0; j < 2 * NP; ++j) acc[mt][j][0] = acc[mt][j][1] = acc[mt][j][2] = acc[mt][j][3] = 0.f;
#pragma unroll
  for (int i = 0; i < kMmaStages - 1; ++i) load(i);
  for (int kc = 0; kc < nk; ++kc) {
    load(kc + kMmaStages - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(kMmaStages - 1) : "memory");  // chunk kc landed
    __syncthreads();
    const __nv_bfloat16* sx = sbuf + (kc % kMmaStages) * stage_elems;
    const __nv_bfloat16* sw = sx + kTok * kLdC;
#pragma unroll
    for (int sub = 0; sub < KC / 128; ++sub) {
      const int ks = warp + 8 * sub;  // this warp's k16 step(s) of the chunk
      uint32_t a[MT][4];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
        ldsm_x4(sx + (16 * mt + (lane & 15)) * kLdC + ks * 16 + (lane >> 4) * 8, a[mt][0], a[mt][1], a[mt][2],
                a[mt][3]);
#pragma unroll
      for (int np = 0; np < NP; ++np) {
        uint32_t b0, b1, b2, b3;  // one B fragment load feeds every token tile
        ldsm_x4(sw + (16 * np + (lane >> 4) * 8 + (lane & 7)) * kLdC + ks * 16 + ((lane >> 3) & 1) * 8, b0, b1, b2,
                b3);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          mma_bf16_16816(acc[mt][2 * np], a[mt][0], a[mt][1], a[mt][2], a[mt][3], b0, b1);
          mma_bf16_16816(acc[mt][2 * np + 1], a[mt][0], a[mt][1], a[mt][2], a[mt][3], b2, b3);
        }
      }
    }
    __syncthreads();  // stage kc % kMmaStages is refilled by the next iteration's load
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  // partial tiles [warp][kTok tokens][64 experts], summed in warp order
  float* s_part = reinterpret_cast<float*>(sbuf);
  float* s_logit = s_part + 8 * kTok * kMaxE;
  float* s_score = s_logit + kTok * kMaxE;
  {
    float* my = s_part + warp * kTok * kMaxE;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int r0 = 16 * mt + (lane >> 2);
#pragma unroll
      for (int j = 0; j < 2 * NP; ++j) {
        const int e = 8 * j + 2 * (lane & 3);
        my[r0 * kMaxE + e] = acc[mt][j][0];
        my[r0 * kMaxE + e + 1] = acc[mt][j][1];
        my[(r0 + 8) * kMaxE + e] = acc[mt][j][2];
        my[(r0 + 8) * kMaxE + e + 1] = acc[mt][j][3];
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kTok * kMaxE; i += 256) {
    float v = s_part[i];
#pragma unroll
    for (int w = 1; w < 8; ++w) v += s_part[w * kTok * kMaxE + i];
    s_logit[i] = v;
  }
  __syncthreads();
#pragma unroll 1
  for (int ti = warp; ti < kTok; ti += 8) {
    const int tok = tok0 + ti;
    if (tok >= ntok) break;
    select_token<float>(s_logit + ti * kMaxE, s_score + ti * kMaxE, tok, E, k, mode, lane, ids_out, w_out,
                        logits_out);
  }
}

template <int NP, int MT, int KC = kMmaK>
int launch_router_mma_np(const void* x, const void* wr, int T_, int d, int E, int k, int mode, int32_t* ids, void* w,
                         void* logits, cudaStream_t s) {
  constexpr int kTok = 16 * MT;
  static uint64_t attr_set = 0;  // devices already configured
  const int smem = std::max(kMmaStages * (kTok + 16 * NP) * (KC + 8) * 2, (8 + 2) * kTok * kMaxE * 4);
  if (!(attr_set & current_device_bit())) {
    QMOE_CUDA_TRY(cudaFuncSetAttribute(router_mma_kernel<NP, MT, KC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem));
    attr_set |= current_device_bit();
  }
  return launch_pdl("qmoe_router(mma)", router_mma_kernel<NP, MT, KC>, dim3((T_ + kTok - 1) / kTok), dim3(256), smem, s,
                    (const __nv_bfloat16*)x, (const __nv_bfloat16*)wr, T_, d, E, k, mode, ids, (float*)w,
                    (float*)logits);
}

int launch_router_mma(const void* x, const void* wr, int T_, int d, int E, int k, int mode, int32_t* ids, void* w,
                      void* logits, cudaStream_t s) {
  // 32 tokens per CTA from ~6k tokens (halves the W_router re-reads and doubles the MMA work per
  // staged chunk: Qwen 8k tokens 49 -> 39 us); 16 below that, to keep every SM busy (4k tokens:
  // 22.5 vs 26.6 us Mixtral, 28.7 vs 30.7 Qwen).  Same per-token k16 order either way.
  // QMOE_ROUTER_MT=1/2 forces the tile
  static const int mt_env = [] {
    const char* v = getenv("QMOE_ROUTER_MT");
    return v == nullptr ? 0 : atoi(v);
  }();
  if (mt_env == 4 && E > 32) return launch_router_mma_np<4, 4>(x, wr, T_, d, E, k, mode, ids, w, logits, s);
  const bool two = mt_env ? mt_env == 2 : T_ >= 6144;
  if (E <= 16)
    return d % 256 == 0 ? (two ? launch_router_mma_np<1, 2, 256>(x, wr, T_, d, E, k, mode, ids, w, logits, s)
                               : launch_router_mma_np<1, 1, 256>(x, wr, T_, d, E, k, mode, ids, w, logits, s))
                        : (two ? launch_router_mma_np<1, 2>(x, wr, T_, d, E, k, mode, ids, w, logits, s)
                               : launch_router_mma_np<1, 1>(x, wr, T_, d, E, k, mode, ids, w, logits, s));
  if (E <= 32)
    return two ? launch_router_mma_np<2, 2>(x, wr, T_, d, E, k, mode, ids, w, logits, s)
               : launch_router_mma_np<2, 1>(x, wr, T_, d, E, k, mode, ids, w, logits, s);
  return two ? launch_router_mma_np<4, 2>(x, wr, T_, d, E, k, mode, ids, w, logits, s)
             : launch_router_mma_np<4, 1>(x, wr, T_, d, E, k, mode, ids, w, logits, s);
}

// ---- bf16, many tokens: register-streamed logits ------------------------------------------------
// The router reads X once (T x d bf16) and does E MACs per element: HBM-bound.  Here nothing is
// staged through shared memory and there is no barrier in the main loop: every lane streams its
// rows of X from HBM with 16-byte loads straight into mma.sync A fragments.  That works because a
// dot product may permute k freely as long as A and B use the same permutation: lane (g, t) loads
// X[row g][8t .. 8t+7] and X[row g+8][8t .. 8t+7] of a 32-wide k step and W[expert g][8t .. 8t+7]
// from L1/L2, and hands words 0-1 to one m16n8k16 and words 2-3 to a second -- logical k (2t,
// 2t+1, 2t+8, 2t+9) of each MMA is physical k (8t .. 8t+3) resp. (8t+4 .. 8t+7) for A and B
// alike.  A CTA owns 16 tokens; its DS x NQ warps split d into DS slices and the experts into NQ
// groups of NTW n8 tiles (NQ warps re-read the same X rows from L1).  U k-steps of loads are in
// flight per warp before any MMA.  The DS partial logits are summed in slice order (fixed,
// deterministic), then the selection is the SIMT kernel's.  16-token CTAs of 4-8 warps put
// ~2-4k warps in flight at 8k tokens.
// 16-byte read-only load as a volatile asm statement: the compiler keeps all U steps' loads ahead
// of the (also volatile) MMAs instead of interleaving them into a short software pipeline.
// NOALLOC: X rows no other warp reads again (NQ == 1) bypass L1 so W_router stays resident.
template <bool NOALLOC>
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  if constexpr (NOALLOC)
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

template <int DS, int NQ, int NTW, int U, int MINB = 1>
__global__ void __launch_bounds__(DS * NQ * 32, MINB)
router_stream_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wr, int ntok, int d,
                     int E, int k, int mode, int32_t* __restrict__ ids_out, float* __restrict__ w_out,
                     float* __restrict__ logits_out) {
  pdl_wait();
  pdl_trigger();
  constexpr int kWarps = DS * NQ;
  constexpr int kCols = 8 * NTW * NQ;  // experts covered (padded)
  __shared__ float s_part[DS][16][kCols];
  __shared__ float s_logit[16][kMaxE];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int slice = warp / NQ, grp = warp % NQ;
  const int tok0 = blockIdx.x * 16;
  const int dq = d / DS, k0 = slice * dq;
  const uint4* xr0 = reinterpret_cast<const uint4*>(x + (size_t)min(tok0 + g, ntok - 1) * d + k0) + t4;
  const uint4* xr1 = reinterpret_cast<const uint4*>(x + (size_t)min(tok0 + g + 8, ntok - 1) * d + k0) + t4;
  const uint4* wp[NTW];
#pragma unroll
  for (int j = 0; j < NTW; ++j)
    wp[j] = reinterpret_cast<const uint4*>(wr + (size_t)min(8 * (grp * NTW + j) + g, E - 1) * d + k0) + t4;
  float acc[NTW][4];
#pragma unroll
  for (int j = 0; j < NTW; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
  const int nsteps = dq / 32;  // 32-wide k steps (4 x uint4 per row); a multiple of U
  // two register buffers of U k-steps: the loads of batch n+1 are issued before the MMAs of batch
  // n, so 2U steps of X are in flight per warp
  uint4 a0[2][U], a1[2][U], b[2][U][NTW];
  auto load = [&](int buf, int s0) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a0[buf][u] = ld_stream<NQ == 1>(xr0 + 4 * (s0 + u));
      a1[buf][u] = ld_stream<NQ == 1>(xr1 + 4 * (s0 + u));
#pragma unroll
      for (int j = 0; j < NTW; ++j) b[buf][u][j] = ld_stream<false>(wp[j] + 4 * (s0 + u));
    }
  };
  auto mma = [&](int buf) {
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < NTW; ++j) {
        mma_bf16_16816(acc[j], a0[buf][u].x, a1[buf][u].x, a0[buf][u].y, a1[buf][u].y, b[buf][u][j].x,
                       b[buf][u][j].y);
        mma_bf16_16816(acc[j], a0[buf][u].z, a1[buf][u].z, a0[buf][u].w, a1[buf][u].w, b[buf][u][j].z,
                       b[buf][u][j].w);
      }
  };
  load(0, 0);
  for (int s0 = 0; s0 < nsteps; s0 += 2 * U) {
    if (s0 + U < nsteps) load(1, s0 + U);
    mma(0);
    if (s0 + U < nsteps) {
      if (s0 + 2 * U < nsteps) load(0, s0 + 2 * U);
      mma(1);
    }
  }
#pragma unroll
  for (int j = 0; j < NTW; ++j) {
    const int c = 8 * (grp * NTW + j) + 2 * t4;
    s_part[slice][g][c] = acc[j][0];
    s_part[slice][g][c + 1] = acc[j][1];
    s_part[slice][g + 8][c] = acc[j][2];
    s_part[slice][g + 8][c + 1] = acc[j][3];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 16 * kCols; i += kWarps * 32) {
    const int t = i / kCols, e = i - t * kCols;
    float v = s_part[0][t][e];
#pragma unroll
    for (int sl = 1; sl < DS; ++sl) v += s_part[sl][t][e];
    s_logit[t][e] = v;
  }
  __syncthreads();
  select_tile16<kWarps * 32>(&s_logit[0][0], tok0, ntok, E, k, mode, ids_out, w_out, logits_out);
}

template <int DS, int NQ, int NTW, int U, int MINB = 1>
int launch_router_stream(const void* x, const void* wr, int T_, int d, int E, int k, int mode, int32_t* ids, void* w,
                         void* logits, cudaStream_t s) {
  return launch_pdl("qmoe_router(stream)", router_stream_kernel<DS, NQ, NTW, U, MINB>, dim3((T_ + 15) / 16),
                    dim3(DS * NQ * 32), 0, s, (const __nv_bfloat16*)x, (const __nv_bfloat16*)wr, T_, d, E, k, mode,
                    ids, (float*)w, (float*)logits);
}

// ---- bf16, many tokens, <= 8 experts: persistent CTAs with W_router held in registers ------------
// The streamed kernel above re-reads W_router (8 x d) from L2 for every 16-token tile: a read probe
// of the same access pattern (tools/scratch/stream_probe.cu) streams X alone in 12.9 us at 8k
// tokens but 16.4 us with the W reads.  Here each warp loads its d slice of W_router ONCE into
// registers (KS k32 steps x 16 B per lane, in the same k permutation as the X fragments), and the
// CTAs (2 per SM) walk 16-token tiles in a grid stride, so only X streams from HBM.  Same per-warp
// k order and slice reduction as router_stream_kernel<8, 1, 1, U>: bit-identical logits.
template <int KS, int U>
__global__ void __launch_bounds__(256, 2)
router_wreg_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wr, int ntok, int d,
                   int E, int k, int mode, int32_t* __restrict__ ids_out, float* __restrict__ w_out,
                   float* __restrict__ logits_out) {
  pdl_wait();
  pdl_trigger();
  constexpr int DS = 8;
  __shared__ float s_part[DS][16][8];
  __shared__ float s_logit[16][kMaxE];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int k0 = warp * KS * 32;  // this warp's d slice: KS k32 steps
  uint4 wf[KS];                   // W_router[g][k0 + 32 s + 8 t4 .. +8] for every step s
  {
    const uint4* wp = reinterpret_cast<const uint4*>(wr + (size_t)min(g, E - 1) * d + k0) + t4;
#pragma unroll
    for (int st = 0; st < KS; ++st) wf[st] = __ldg(wp + 4 * st);
  }
  const int ntiles = (ntok + 15) / 16;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int tok0 = tile * 16;
    const uint4* xr0 = reinterpret_cast<const uint4*>(x + (size_t)min(tok0 + g, ntok - 1) * d + k0) + t4;
    const uint4* xr1 = reinterpret_cast<const uint4*>(x + (size_t)min(tok0 + g + 8, ntok - 1) * d + k0) + t4;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    uint4 a0[2][U], a1[2][U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a0[0][u] = ld_stream<true>(xr0 + 4 * u);
      a1[0][u] = ld_stream<true>(xr1 + 4 * u);
    }
#pragma unroll
    for (int s0 = 0; s0 < KS; s0 += U) {
      const int buf = (s0 / U) & 1;
      if (s0 + U < KS) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          a0[buf ^ 1][u] = ld_stream<true>(xr0 + 4 * (s0 + U + u));
          a1[buf ^ 1][u] = ld_stream<true>(xr1 + 4 * (s0 + U + u));
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint4 b = wf[s0 + u];
        mma_bf16_16816(acc, a0[buf][u].x, a1[buf][u].x, a0[buf][u].y, a1[buf][u].y, b.x, b.y);
        mma_bf16_16816(acc, a0[buf][u].z, a1[buf][u].z, a0[buf][u].w, a1[buf][u].w, b.z, b.w);
      }
    }
    const int c = 2 * t4;
    s_part[warp][g][c] = acc[0];
    s_part[warp][g][c + 1] = acc[1];
    s_part[warp][g + 8][c] = acc[2];
    s_part[warp][g + 8][c + 1] = acc[3];
    __syncthreads();
    if (threadIdx.x < 16 * 8) {
      const int t = threadIdx.x >> 3, e = threadIdx.x & 7;
      float v = s_part[0][t][e];
#pragma unroll
      for (int sl = 1; sl < DS; ++sl) v += s_part[sl][t][e];
      s_logit[t][e] = v;
    }
    __syncthreads();
    select_tile16<256>(&s_logit[0][0], tok0, ntok, E, k, mode, ids_out, w_out, logits_out);
    __syncthreads();  // s_part / s_logit are rewritten by the next tile
  }
}

int device_sm_count() {
  static int counts[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (counts[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    counts[dev] = n > 0 ? n : 148;
  }
  return counts[dev];
}

// 0 = not applicable (shape), else launched.  QMOE_ROUTER_STREAM=0 keeps the cp.async kernel.
int try_router_stream(const void* x, const void* wr, int T_, int d, int E, int k, int mode, int32_t* ids, void* w,
                      void* logits, cudaStream_t s, int* st) {
  static const int env = [] {
    const char* v = getenv("QMOE_ROUTER_STREAM");
    return v == nullptr ? 1 : atoi(v);
  }();
  static const int cfg = [] {  // QMOE_ROUTER_CFG: tiling variant (measurement sweeps)
    const char* v = getenv("QMOE_ROUTER_CFG");
    return v == nullptr ? 0 : atoi(v);
  }();
  if (!env) return 0;
#define QMOE_TRY_STREAM(DS, NQ, NTW, U)                                                       \
  if (d % ((DS) * 32 * (U)) == 0) {                                                          \
    *st = launch_router_stream<DS, NQ, NTW, U>(x, wr, T_, d, E, k, mode, ids, w, logits, s); \
    return 1;                                                                                \
  }
  // Measured on B200 (tools/router_ab.py, L2 flushed): Mixtral 1-2k tokens 12 us (16 d-slices:
  // 8 k-steps per warp, one round trip) vs 18 on the cp.async kernel, 8k/16k tokens 27/46 us vs
  // 35/59 (8 slices).  Qwen's 61 logit rows: 4 expert groups re-read X from L1 and W from L2 per
  // 16 tokens -- faster up to 2k tokens (17 vs 23 us), slower from 8k (51 vs 39 us), where the
  // cp.async kernel's 32-token tiles halve the W re-reads.
  // ncu at 8k tokens: <8,1,1,4> reads 67 MB in 24 us (2.8 TB/s) at 128 registers = 2 CTAs/SM, so
  // 512 CTAs take 1.7 waves; U = 2 halves the register buffers (4 CTAs/SM: one wave).
#define QMOE_TRY_STREAM_MINB(DS, NQ, NTW, U, MINB)                                                  \
  if (d % ((DS) * 32 * (U)) == 0) {                                                                  \
    *st = launch_router_stream<DS, NQ, NTW, U, MINB>(x, wr, T_, d, E, k, mode, ids, w, logits, s); \
    return 1;                                                                                        \
  }
  if (E <= 8) {
    // W_router in registers, persistent CTAs (d = 4096: 16 k32 steps per warp); QMOE_ROUTER_CFG=5
    // forces it at any size, -1 keeps the streamed tilings
    if (d == 4096 && (cfg == 5 || (cfg == 0 && T_ >= 4096))) {  // (8 d slices: the streamed kernels' order)
      const int ntiles = (T_ + 15) / 16;
      const int grid = std::min(ntiles, 2 * device_sm_count());
      *st = launch_pdl("qmoe_router(wreg)", router_wreg_kernel<16, 2>, dim3(grid), dim3(256), 0, s,
                       (const __nv_bfloat16*)x, (const __nv_bfloat16*)wr, T_, d, E, k, mode, ids, (float*)w,
                       (float*)logits);
      return 1;
    }
    if (cfg == 1) { QMOE_TRY_STREAM(8, 1, 1, 4) }
    // from ~6k tokens: 64 registers so 4 CTAs fit an SM and 512+ CTAs run in one wave (the
    // 3-per-SM build leaves a 15% second wave: 29.5 -> 26.5 us at 8k tokens, 52 -> 44 us at 16k)
    if (cfg == 3 || (cfg == 0 && T_ >= 6144)) { QMOE_TRY_STREAM_MINB(8, 1, 1, 2, 4) }
    if (cfg == 4) { QMOE_TRY_STREAM_MINB(4, 1, 1, 2, 8) }
    if (cfg == 2 || (cfg == 0 && T_ < 4096)) { QMOE_TRY_STREAM(16, 1, 1, 2) }
    QMOE_TRY_STREAM(8, 1, 1, 2)
  } else if (E <= 16) {
    QMOE_TRY_STREAM(8, 1, 2, 4)
  } else if (E <= 32) {
    QMOE_TRY_STREAM(4, 2, 2, 4)
  } else {
    if (cfg == 1) { QMOE_TRY_STREAM(2, 4, 2, 4) }
    if (cfg == 2) { QMOE_TRY_STREAM(2, 8, 1, 4) }
    if (T_ < 4096) { QMOE_TRY_STREAM(4, 4, 2, 2) }
  }
#undef QMOE_TRY_STREAM
#undef QMOE_TRY_STREAM_MINB
  return 0;
}

// ---- bf16 decode (<= 32 tokens): one cluster of 8 CTAs for the whole batch ---------------------
// The per-token SIMT kernel re-reads all of W_router (Qwen: 61 x 2048 bf16 = 250 KB) in every
// token's CTA and walks d in dependent rounds (14 us for 32 Qwen tokens).  Here CTA r of an
// 8-CTA cluster owns expert chunk r / DS (8 logit rows) over d slice r % DS (NCH x DS = 8), for
// all tokens: its 8 warps split the slice in k, every warp runs mma.sync m16n8k16 on up to 4
// token tiles with X and W fragments loaded straight into registers (the streamed kernel's k
// permutation), the 8 warp partials are summed in warp order in shared memory, and after a
// cluster barrier CTA r selects the tokens t = r (mod 8): it sums the DS slice partials of every
// chunk in slice order through distributed shared memory and runs select_token.  One launch,
// W_router read once per batch, deterministic.
__device__ __forceinline__ float ld_cluster_f32(const float* p, uint32_t rank) {
  float v;
  asm volatile(
      "{\n\t"
      ".reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %1, %2;\n\t"
      "ld.shared::cluster.f32 %0, [ra];\n\t"
      "}"
      : "=f"(v)
      : "r"(ptx::smem_u32(p)), "r"(rank)
      : "memory");
  return v;
}

template <int NCH, int DS, int MT, int U>
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(256)
router_decode_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wr, int ntok, int d,
                     int E, int k, int mode, int32_t* __restrict__ ids_out, float* __restrict__ w_out,
                     float* __restrict__ logits_out) {
  static_assert(NCH * DS == 8, "8 CTAs per cluster");
  pdl_trigger();  // at entry: the permute and the expert launch behind it may be scheduled now
  pdl_wait();
  __shared__ float s_part[8][16 * MT][8];   // per warp partials
  __shared__ float s_log[16 * MT][8];       // this CTA's (chunk, slice) logits
  __shared__ float s_full[8][kMaxE];        // per warp: one token's logits (selection)
  __shared__ float s_score[8][kMaxE];
  const uint32_t rank = ptx::cluster_ctarank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int chunk = (int)rank / DS, slice = (int)rank % DS;
  const int dq = d / DS, dw = dq / 8;          // this CTA's slice, each warp's share
  const int k0 = slice * dq + warp * dw;
  const uint4* wp = reinterpret_cast<const uint4*>(wr + (size_t)min(8 * chunk + g, E - 1) * d + k0) + t4;
  const uint4* xr[MT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    xr[mt][0] = reinterpret_cast<const uint4*>(x + (size_t)min(16 * mt + g, ntok - 1) * d + k0) + t4;
    xr[mt][1] = reinterpret_cast<const uint4*>(x + (size_t)min(16 * mt + g + 8, ntok - 1) * d + k0) + t4;
  }
  float acc[MT][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
  // U k32 steps of loads in flight before their MMAs (a handful of steps per warp: latency-bound;
  // volatile loads keep the compiler from interleaving them with the MMAs); dw / 32 % U == 0
  for (int st0 = 0; st0 < dw / 32; st0 += U) {
    uint4 b[U], a0[U][MT], a1[U][MT];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int st = st0 + u;
      b[u] = ld_stream<false>(wp + 4 * st);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        a0[u][mt] = ld_stream<false>(xr[mt][0] + 4 * st);
        a1[u][mt] = ld_stream<false>(xr[mt][1] + 4 * st);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        mma_bf16_16816(acc[mt], a0[u][mt].x, a1[u][mt].x, a0[u][mt].y, a1[u][mt].y, b[u].x, b[u].y);
        mma_bf16_16816(acc[mt], a0[u][mt].z, a1[u][mt].z, a0[u][mt].w, a1[u][mt].w, b[u].z, b[u].w);
      }
  }
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int r0 = 16 * mt + g, c = 2 * t4;
    s_part[warp][r0][c] = acc[mt][0];
    s_part[warp][r0][c + 1] = acc[mt][1];
    s_part[warp][r0 + 8][c] = acc[mt][2];
    s_part[warp][r0 + 8][c + 1] = acc[mt][3];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 16 * MT * 8; i += 256) {
    const int t = i >> 3, e = i & 7;
    float v = s_part[0][t][e];
#pragma unroll
    for (int w = 1; w < 8; ++w) v += s_part[w][t][e];
    s_log[t][e] = v;
  }
  ptx::cluster_sync();  // every CTA's s_log is complete and visible cluster-wide
  // CTA r selects tokens r, r + 8, ...: warp j of it takes token r + 8 j
  const int tok = (int)rank + 8 * warp;
  if (tok < ntok) {
    for (int i = lane; i < NCH * 8; i += 32) {
      const int cc = i >> 3, e = i & 7;
      float v = 0.f;
#pragma unroll
      for (int ss = 0; ss < DS; ++ss) v += ld_cluster_f32(&s_log[tok][e], (uint32_t)(cc * DS + ss));
      s_full[warp][i] = v;
    }
    __syncwarp();
    select_token<float>(s_full[warp], s_score[warp], tok, E, k, mode, lane, ids_out, w_out, logits_out);
  }
  ptx::cluster_sync();  // no CTA leaves while a peer may still read its s_log
}

template <int NCH, int DS, int U>
int launch_router_decode(const void* x, const void* wr, int T_, int d, int E, int k, int mode, int32_t* ids, void* w,
                         void* logits, cudaStream_t s) {
  if (T_ <= 16)
    return launch_pdl("qmoe_router(decode cluster)", router_decode_kernel<NCH, DS, 1, U>, dim3(8), dim3(256), 0, s,
                      (const __nv_bfloat16*)x, (const __nv_bfloat16*)wr, T_, d, E, k, mode, ids, (float*)w,
                      (float*)logits);
  return launch_pdl("qmoe_router(decode cluster)", router_decode_kernel<NCH, DS, 2, U>, dim3(8), dim3(256), 0, s,
                    (const __nv_bfloat16*)x, (const __nv_bfloat16*)wr, T_, d, E, k, mode, ids, (float*)w,
                    (float*)logits);
}

// 0 = not applicable; QMOE_ROUTER_DECODE=0 keeps the per-token SIMT kernel.
int try_router_decode(const void* x, const void* wr, int T_, int d, int E, int k, int mode, int32_t* ids, void* w,
                      void* logits, cudaStream_t s, int* st) {
  static const int env = [] {
    const char* v = getenv("QMOE_ROUTER_DECODE");
    return v == nullptr ? 1 : atoi(v);
  }();
  // up to 32 tokens (64: the 8 CTAs' X reads outweigh the per-token kernel's, measured 23 vs 17 us Qwen)
  if (!env || T_ > 32 || T_ < 1 || reinterpret_cast<uintptr_t>(x) % 16 || reinterpret_cast<uintptr_t>(wr) % 16)
    return 0;
  if (E <= 8 && d % (8 * 8 * 32 * 2) == 0) { *st = launch_router_decode<1, 8, 2>(x, wr, T_, d, E, k, mode, ids, w, logits, s); return 1; }
  if (E <= 16 && d % (4 * 8 * 32 * 4) == 0) { *st = launch_router_decode<2, 4, 4>(x, wr, T_, d, E, k, mode, ids, w, logits, s); return 1; }
  if (E <= 32 && d % (2 * 8 * 32 * 4) == 0) { *st = launch_router_decode<4, 2, 4>(x, wr, T_, d, E, k, mode, ids, w, logits, s); return 1; }
  if (E <= 64 && d % (8 * 32 * 4) == 0) { *st = launch_router_decode<8, 1, 4>(x, wr, T_, d, E, k, mode, ids, w, logits, s); return 1; }
  return 0;
}

// ---- bf16, large batches: tcgen05 logits, d split over a cluster --------------------------------
// The mma.sync kernels above pay for W_router in every 16/32-token tile (re-read from L2: Qwen's
// 61 x 2048 logit rows are 250 KB, 4x the X bytes of a 32-token tile) and move every operand
// through registers.  Here the logits are a skinny GEMM on the 5th-gen tensor core: a tile is
// 128 tokens x NB logit rows (experts padded to 16), K = d split into S slices, one CTA per
// (tile, slice), the S CTAs of a tile forming a cluster.  Warp 0 streams X (128 x 64, evict-first)
// and W_router (NB x 64, evict-last) into a STAGES-deep 128B-swizzled ring with TMA; one thread of
// warp 1 issues tcgen05.mma (M=128, N=NB, K=16) into an NB-column fp32 TMEM accumulator.  Warps
// 4-7 read the accumulator (thread = token row) into shared memory; after a cluster barrier CTA r
// sums the S slice partials of tokens [r 128/S, (r+1) 128/S) in slice order through distributed
// shared memory (deterministic) and its 8 warps run select_token.  X rows beyond T are zero-filled
// by TMA and never selected.  W_router is read from L2 once per 128 tokens.
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t"
      "}"
      : "=r"(ok)
      : "r"(ptx::smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

template <int NB, int S, int STAGES, int MINB>
__global__ void __cluster_dims__(S, 1, 1) __launch_bounds__(256, MINB)
router_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW, int ntok, int d,
                 int E, int k, int mode, int32_t* __restrict__ ids_out, float* __restrict__ w_out,
                 float* __restrict__ logits_out) {
  constexpr int kXBytes = 128 * 64 * 2, kWBytes = NB * 64 * 2, kStage = kXBytes + kWBytes;
  constexpr uint32_t kCols = NB <= 32 ? 32 : (NB <= 64 ? 64 : 128);
  constexpr int kRows = 128 / S;   // tokens this CTA selects
  constexpr int kLdP = NB + 4;     // padded partial row (float4 stores conflict-free)
  constexpr uint32_t kIdesc = ptx::idesc_bf16_f32(128, NB);
  static_assert(kStage % 1024 == 0, "stages keep the 1024-byte swizzle-atom alignment");
  static_assert(128 * kLdP * 4 <= STAGES * kStage, "the partial tile aliases the ring");
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES], done_bar;
  __shared__ uint32_t tmem_base_smem;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = S > 1 ? ptx::cluster_ctarank() : 0;
  const int tile = blockIdx.x / S;
  const int nkb = d / (64 * S), kb0 = (int)rank * nkb;  // this CTA's 64-wide K blocks
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    ptx::mbar_init(&done_bar, 1);
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tmX);
    ptx::tma_prefetch_desc(&tmW);
  }
  if (warp == 1) ptx::tmem_alloc<kCols>(&tmem_base_smem);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_smem;
  pdl_wait();  // X is the predecessor's output
  pdl_trigger();
  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sx = smem + stage * kStage;
        ptx::mbar_arrive_expect_tx(&full_bar[stage], kStage);
        ptx::tma_load_2d(&tmX, &full_bar[stage], sx, (kb0 + kb) * 64, tile * 128, ptx::kEvictFirst);
        ptx::tma_load_2d(&tmW, &full_bar[stage], sx + kXBytes, (kb0 + kb) * 64, 0, ptx::kEvictLast);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        ptx::mbar_wait(&full_bar[stage], phase);
        ptx::tc_fence_after();
        const uint32_t a = ptx::smem_u32(smem + stage * kStage), b = a + kXBytes;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          ptx::tc_mma_bf16(tmem, ptx::sw128_kmajor_desc(a + kk * 32), ptx::sw128_kmajor_desc(b + kk * 32), kIdesc,
                           (kb > 0 || kk > 0) ? 1u : 0u);
        ptx::tc_commit(&empty_bar[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      ptx::tc_commit(&done_bar);  // accumulator complete
    }
    __syncwarp();
  }
  float* s_p = reinterpret_cast<float*>(smem);  // [128][kLdP] this CTA's slice partials (ring reused)
  if (warp >= 4) {
    // every MMA retired (the ring is free).  One polling lane per warp, backing off: 128 threads
    // spinning on try_wait compete with the ring's barriers and the TMA completions.
    if (lane == 0) {
      while (!mbar_try_wait(&done_bar, 0)) __nanosleep(256);
    }
    __syncwarp();
    ptx::tc_fence_after();
    const int row = (warp - 4) * 32 + lane;
    const uint32_t t_row = tmem + ((uint32_t)((warp - 4) * 32) << 16);
#pragma unroll
    for (int c0 = 0; c0 < NB; c0 += 32) {
      uint32_t v[32];
      ptx::tmem_ld32(t_row + c0, v);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int c = 0; c < 32 && c0 + c < NB; c += 4)
        *reinterpret_cast<float4*>(s_p + row * kLdP + c0 + c) =
            make_float4(__uint_as_float(v[c]), __uint_as_float(v[c + 1]), __uint_as_float(v[c + 2]),
                        __uint_as_float(v[c + 3]));
    }
  }
  ptx::tc_fence_before();
  if constexpr (S > 1) ptx::cluster_sync(); else __syncthreads();
  // token r of this CTA's kRows is selected by the G = 256 / kRows consecutive threads r G .. r G +
  // G - 1; thread j of the group sums the slice partials (slice order) of logit rows L, L + 32 for
  // L = j + G i straight into registers
  constexpr int G = 256 / kRows, C = 32 / G;
  const int r = threadIdx.x / G, j = threadIdx.x % G;
  const int tok = tile * 128 + (int)rank * kRows + r;
  float l0[C], l1[C];
  {
    const float* p = s_p + ((int)rank * kRows + r) * kLdP;
#pragma unroll
    for (int i = 0; i < C; ++i) {
      const int L = j + G * i;
      float a = 0.f, b = 0.f;
      if (L < E) {
        a = S > 1 ? ld_cluster_f32(p + L, 0) : p[L];
#pragma unroll
        for (int sl = 1; sl < S; ++sl) a += ld_cluster_f32(p + L, (uint32_t)sl);
      }
      if (L + 32 < E && L + 32 < NB) {
        b = S > 1 ? ld_cluster_f32(p + L + 32, 0) : p[L + 32];
#pragma unroll
        for (int sl = 1; sl < S; ++sl) b += ld_cluster_f32(p + L + 32, (uint32_t)sl);
      }
      l0[i] = a;
      l1[i] = b;
    }
  }
  if constexpr (S > 1) ptx::cluster_sync(); else __syncthreads();  // peers done reading s_p
  if (!(mode & kNoSelect))
    select_group<G>(l0, l1, tok < ntok, tok, E, k, mode, j, ids_out, w_out, logits_out);
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<kCols>(tmem);
  }
}

template <int NB, int S, int STAGES, int MINB>
int launch_router_tc(const CUtensorMap& mx, const CUtensorMap& mw, int T_, int d, int E, int k, int mode,
                     int32_t* ids, void* w, void* logits, cudaStream_t s) {
  constexpr int smem = STAGES * (128 * 64 * 2 + NB * 64 * 2) + 1024;
  static uint64_t attr_set = 0;  // devices already configured
  if (!(attr_set & current_device_bit())) {
    QMOE_CUDA_TRY(cudaFuncSetAttribute(router_tc_kernel<NB, S, STAGES, MINB>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set |= current_device_bit();
  }
  const int ntiles = (T_ + 127) / 128;
  return launch_pdl("qmoe_router(tcgen05)", router_tc_kernel<NB, S, STAGES, MINB>, dim3(ntiles * S), dim3(256), smem,
                    s, mx, mw, T_, d, E, k, mode, ids, (float*)w, (float*)logits);
}

// 0 = not applicable.  QMOE_ROUTER_TC=0 disables it, QMOE_ROUTER_TC_MIN sets the token threshold,
// QMOE_ROUTER_TC_S forces the d split (1, 2, 4; default: enough CTAs for one wave, see below).
int try_router_tc(const void* x, const void* wr, int T_, int d, int E, int k, int mode, int32_t* ids, void* w,
                  void* logits, cudaStream_t s, int* st) {
  static const int env = [] {
    const char* v = getenv("QMOE_ROUTER_TC");
    return v == nullptr ? 1 : atoi(v);
  }();
  static const int tmin_env = [] {
    const char* v = getenv("QMOE_ROUTER_TC_MIN");
    return v == nullptr ? 0 : atoi(v);
  }();
  // measured crossover against the mma.sync kernels (tools/router_ab.py, L2 flushed, CUDA events):
  // Mixtral 2048 / 3072 / 4096 tokens 16.4 / 16.8 / 18.4 us vs 14.3 / 21.2 / 17.3; Qwen (61 logit
  // rows) 16.4 / 18.4 / 18.4 vs 16.4 / 26.6 / 28.7
  const int tmin = tmin_env ? tmin_env : 3072;
  static const int s_env = [] {
    const char* v = getenv("QMOE_ROUTER_TC_S");
    return v == nullptr ? 0 : atoi(v);
  }();
  static const int nosel = [] {  // timing only: logits streamed, no selection (ids/w not written)
    const char* v = getenv("QMOE_ROUTER_TC_NOSEL");
    return v != nullptr && atoi(v) != 0;
  }();
  static const int deep = [] {  // QMOE_ROUTER_TC_DEEP=1: deeper ring, 1 CTA per SM
    const char* v = getenv("QMOE_ROUTER_TC_DEEP");
    return v != nullptr && atoi(v) != 0;
  }();
  if (nosel) mode |= kNoSelect;
  if (!env || T_ < tmin || E > 64 || d % 64 != 0) return 0;
  if (tc_init_driver() != QMOE_OK) return 0;
  // d split: the smallest S that puts >= 128 CTAs on the GPU, slices of >= 256 columns (Qwen
  // 4k / 8k / 16k tokens: S = 4 / 2 / 1 -> 18.8 / 22.5 / 28.7 us; Mixtral 8k / 16k: S = 2 / 1)
  const int ntiles = (T_ + 127) / 128;
  int S = 1;
  while (S < 4 && ntiles * S < 128 && d / (2 * S) >= 256 && d % (128 * S) == 0) S *= 2;
  if (s_env == 1 || s_env == 2 || s_env == 4) S = s_env;
  if (d % (64 * S) != 0) return 0;
  const int NB = E <= 16 ? 16 : (E <= 32 ? 32 : 64);
  CUtensorMap mx, mw;
  if (tc_make_map(&mx, x, (uint64_t)T_, (uint64_t)d, 128) != QMOE_OK) return 0;
  if (tc_make_map(&mw, wr, (uint64_t)E, (uint64_t)d, (uint32_t)NB) != QMOE_OK) return 0;
#define QMOE_RTC(NB_, S_, ST_, MB_)                                                                   \
  if (NB == NB_ && S == S_) {                                                                         \
    *st = launch_router_tc<NB_, S_, ST_, MB_>(mx, mw, T_, d, E, k, mode, ids, w, logits, s);          \
    return 1;                                                                                         \
  }
  if (deep) {
    QMOE_RTC(16, 1, 12, 1) QMOE_RTC(16, 2, 12, 1) QMOE_RTC(16, 4, 12, 1)
    QMOE_RTC(64, 1, 8, 1) QMOE_RTC(64, 2, 8, 1) QMOE_RTC(64, 4, 8, 1)
  }
  QMOE_RTC(16, 1, 6, 2) QMOE_RTC(16, 2, 6, 2) QMOE_RTC(16, 4, 6, 2)
  QMOE_RTC(32, 1, 5, 2) QMOE_RTC(32, 2, 5, 2) QMOE_RTC(32, 4, 5, 2)
  QMOE_RTC(64, 1, 5, 1) QMOE_RTC(64, 2, 4, 2) QMOE_RTC(64, 4, 4, 2)
#undef QMOE_RTC
  return 0;
}

// Few tokens (decode): one token per CTA, all 8 warps on it.  Many tokens: warps own tokens (2
// each) when the experts fit one or two 8-expert chunks, else 4 tokens share the 8 warps.
template <typename T>
int dispatch_router(const void* x, const void* wr, int T_, int d, int E, int k, int mode, int32_t* ids, void* w,
                    void* logits, cudaStream_t s) {
  const int nchunk = (E + kExpChunk - 1) / kExpChunk;
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    if (T_ >= 256 && d % kMmaK == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0 &&
        reinterpret_cast<uintptr_t>(wr) % 16 == 0) {
      int st = QMOE_OK;
      if (try_router_tc(x, wr, T_, d, E, k, mode, ids, w, logits, s, &st)) return st;
      if (try_router_stream(x, wr, T_, d, E, k, mode, ids, w, logits, s, &st)) return st;
      return launch_router_mma(x, wr, T_, d, E, k, mode, ids, w, logits, s);
    }
  }
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    int st = QMOE_OK;
    if (try_router_decode(x, wr, T_, d, E, k, mode, ids, w, logits, s, &st)) return st;
  }
  // decode: 16 warps on one token halve the dependent load rounds over d (Qwen: 8 chunks x 2 slices)
  if (T_ < 148 * 8) return launch_router<T, 1, 1, 16>(x, wr, T_, d, E, k, mode, ids, w, logits, s);
  if (nchunk == 1) return launch_router<T, 16, 2>(x, wr, T_, d, E, k, mode, ids, w, logits, s);
  if (nchunk == 2) return launch_router<T, 8, 2>(x, wr, T_, d, E, k, mode, ids, w, logits, s);
  if (nchunk <= 4) return launch_router<T, 4, 2>(x, wr, T_, d, E, k, mode, ids, w, logits, s);
  return launch_router<T, 4, 4>(x, wr, T_, d, E, k, mode, ids, w, logits, s);
}

}  // namespace
}  // namespace qmoe

extern "C" int qmoe_router_shared(const void* x, const void* w_router, int T, int d, int E, int k, int n_shared,
                                  int dtype, int route_mode, int32_t* ids_out, void* w_out, void* logits_out,
                                  void* stream) {
  using namespace qmoe;
  QMOE_REQUIRE(T >= 0 && d >= 1, "qmoe_router: bad sizes T=%d d=%d", T, d);
  QMOE_REQUIRE(n_shared >= 0 && n_shared <= 8 && k + n_shared <= 8,
               "qmoe_router_shared: need 0 <= n_shared and k + n_shared <= 8 (k=%d, n_shared=%d)", k, n_shared);
  const int rows = E + (n_shared > 0 ? 1 : 0);  // logit rows: routed experts (+ the shared gate)
  QMOE_REQUIRE(E >= 1 && rows <= kMaxE, "qmoe_router: E=%d (+ shared gate) outside [1, %d]", E, kMaxE);
  QMOE_REQUIRE(k >= 1 && k <= E && k <= 8, "qmoe_router: k=%d must satisfy 1 <= k <= min(E, 8)", k);
  QMOE_REQUIRE(route_mode == QMOE_ROUTE_TOPK_SOFTMAX || route_mode == QMOE_ROUTE_SOFTMAX_TOPK,
               "qmoe_router: unknown route_mode %d", route_mode);
  if (T == 0) return QMOE_OK;
  QMOE_REQUIRE(x && w_router && ids_out && w_out, "qmoe_router: null pointer");
  cudaStream_t s = as_stream(stream);
  E = rows;
  route_mode |= n_shared << 8;  // mode word: the kernels hand n_shared to select_token in bits 8..
  switch (dtype) {
    case QMOE_BF16:
      return dispatch_router<__nv_bfloat16>(x, w_router, T, d, E, k, route_mode, ids_out, w_out, logits_out, s);
    case QMOE_F32:
      return dispatch_router<float>(x, w_router, T, d, E, k, route_mode, ids_out, w_out, logits_out, s);
    case QMOE_F64:
      return launch_router<double, 1, 1>(x, w_router, T, d, E, k, route_mode, ids_out, w_out, logits_out, s);
    default:
      set_error("qmoe_router: unknown dtype %d", dtype);
      return QMOE_ERR_INVALID;
  }
}

extern "C" int qmoe_router(const void* x, const void* w_router, int T, int d, int E, int k, int dtype,
                           int route_mode, int32_t* ids_out, void* w_out, void* logits_out,
                           void* stream) {
  return qmoe_router_shared(x, w_router, T, d, E, k, 0, dtype, route_mode, ids_out, w_out, logits_out, stream);
}
