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
namespace {

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
  __shared__ float s_score[16][kMaxE];
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
#pragma unroll 1
  for (int ti = warp; ti < 16; ti += kWarps) {
    const int tok = tok0 + ti;
    if (tok >= ntok) break;
    select_token<float>(s_logit[ti], s_score[ti], tok, E, k, mode, lane, ids_out, w_out, logits_out);
  }
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
  __shared__ float s_score[16][kMaxE];
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
#pragma unroll 1
    for (int ti = warp; ti < 16; ti += 8) {
      const int tok = tok0 + ti;
      if (tok >= ntok) break;
      select_token<float>(s_logit[ti], s_score[ti], tok, E, k, mode, lane, ids_out, w_out, logits_out);
    }
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
  pdl_wait();
  pdl_trigger();
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
