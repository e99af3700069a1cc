// Permute: stable counting sort of pending routed slots by expert (+ fused row gather).
//
// Replaces the per-(expert, layer) FIFO construction of the reference:
//   _enqueue_expert_work (engine.py:312-328) walks members -> tokens -> sorted(pending) experts
//   and appends to the (expert, layer) deque (model.py:195-200); drain (model.py:206-214) pops
//   each expert's FIFO in ascending expert id (model.py:202-204); the gather is engine.py:207-209.
// The FIFO order of expert e is therefore the flat slot order s = t*k + j restricted to
// ids[s] == e, which is what a stable counting sort by expert produces.  Stability comes from
// warp match + per-warp prefix counts, never from atomics, so the output is deterministic.
//
// Two launches: (1) per-chunk expert histograms, (2) per-chunk exclusive bases, in-chunk stable
// ranks, scatter of perm, and a cooperative (coalesced, 16 B vector) copy of the gathered rows.
#include "common.cuh"

namespace qmoe {
namespace {

constexpr int kChunk = 2048;      // slots per CTA
constexpr int kPass = 512;        // slots ranked per pass (one per thread)
constexpr int kThreads = kPass;
constexpr int kWarpsPer = kThreads / 32;
constexpr int kMaxE = 64;

__device__ __forceinline__ int slot_expert(const int32_t* ids, const int32_t* cursor, int s, int k,
                                           int E) {
  const int e = ids[s];
  if (e < 0 || e >= E) return -1;
  if (cursor != nullptr && e < cursor[s / k]) return -1;  // already drained before preemption
  return e;
}

__global__ void __launch_bounds__(256) perm_count_kernel(const int32_t* __restrict__ ids,
                                                         const int32_t* __restrict__ cursor, int S,
                                                         int k, int E, int32_t* __restrict__ hist) {
  pdl_wait();
  pdl_trigger();
  __shared__ int h[kMaxE];
  for (int e = threadIdx.x; e < E; e += blockDim.x) h[e] = 0;
  __syncthreads();
  const int s0 = blockIdx.x * kChunk;
  const int s1 = min(S, s0 + kChunk);
  for (int s = s0 + threadIdx.x; s < s1; s += blockDim.x) {
    const int e = slot_expert(ids, cursor, s, k, E);
    if (e >= 0) atomicAdd(&h[e], 1);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) hist[blockIdx.x * E + e] = h[e];
}

__device__ __forceinline__ void copy_row(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                         size_t row_bytes, int lane) {
  if ((row_bytes & 15) == 0 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    const int n = (int)(row_bytes >> 4);
    int i = lane;
    for (; i + 96 < n; i += 128) {  // 4 loads in flight per lane
      uint4 a = __ldg(s4 + i), b = __ldg(s4 + i + 32), c = __ldg(s4 + i + 64), d = __ldg(s4 + i + 96);
      d4[i] = a; d4[i + 32] = b; d4[i + 64] = c; d4[i + 96] = d;
    }
    for (; i < n; i += 32) d4[i] = __ldg(s4 + i);
  } else {
    for (size_t i = lane; i < row_bytes; i += 32) dst[i] = src[i];
  }
}

// Wide row gather for multi-chunk launches: Xp[r] = X[perm[r] / k], one warp per row.
// gather_e: rows of experts >= gather_e are not gathered (their A operand is read straight from X,
// qmoe_expert_ffn_xs: the shared sub-experts' queues are X's rows in order).
__global__ void __launch_bounds__(256) perm_gather_kernel(const int32_t* __restrict__ perm,
                                                          const int32_t* __restrict__ offsets, int gather_e, int k,
                                                          int max_rows, const uint8_t* __restrict__ x,
                                                          uint8_t* __restrict__ xp, size_t row_bytes) {
  // Decode-sized launches trigger their dependents at entry, so the expert launch is resident
  // before the permute finishes (Qwen decode layer ~190 -> ~186 us, CUPTI); large ones after the
  // wait (at 8192 Qwen tokens the entry trigger cost the grouped GEMM ~25 us).
  const bool early = max_rows <= kChunk;
  if (early) pdl_trigger();
  pdl_wait();
  if (!early) pdl_trigger();
  const int R = offsets[gather_e];
  const int lane = lane_id();
  for (int r = blockIdx.x * 8 + warp_id(); r < R && r < max_rows; r += gridDim.x * 8)
    copy_row(x + (size_t)(perm[r] / k) * row_bytes, xp + (size_t)r * row_bytes, row_bytes, lane);
}

__global__ void __launch_bounds__(kThreads)
perm_scatter_kernel(const int32_t* __restrict__ ids, const int32_t* __restrict__ cursor, int S, int k,
                    int E, int nblk, int32_t* __restrict__ hist, int32_t* __restrict__ perm,
                    int32_t* __restrict__ offsets, const uint8_t* __restrict__ x, uint8_t* __restrict__ xp,
                    size_t row_bytes) {
  if (nblk == 1) pdl_trigger();  // decode-sized: at entry (see perm_gather_kernel)
  pdl_wait();
  if (nblk > 1) pdl_trigger();
  __shared__ int base[kMaxE];
  __shared__ int warp_cnt[kWarpsPer][kMaxE];
  __shared__ int pass_tot[kMaxE];
  __shared__ int s_pos[kPass];
  __shared__ int s_src[kPass];
  const int tid = threadIdx.x, warp = warp_id(), lane = lane_id();

  // Single-chunk launches (decode-sized batches) count in-kernel: one launch does everything.
  if (nblk == 1) {
    __shared__ int h1[kMaxE];
    for (int e = tid; e < E; e += kThreads) h1[e] = 0;
    __syncthreads();
    for (int s = tid; s < S; s += kThreads) {
      const int e = slot_expert(ids, cursor, s, k, E);
      if (e >= 0) atomicAdd(&h1[e], 1);
    }
    __syncthreads();
    for (int e = tid; e < E; e += kThreads) hist[e] = h1[e];
    __syncthreads();
  }
  // Exclusive base of this chunk for every expert: expert start + counts of earlier chunks.
  if (warp == 0) {
    int tot_e[2] = {0, 0}, pre_e[2] = {0, 0};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int e = lane + 32 * q;
      if (e < E) {
        for (int b = 0; b < nblk; ++b) {
          const int c = hist[b * E + e];
          tot_e[q] += c;
          if (b < (int)blockIdx.x) pre_e[q] += c;
        }
      }
    }
    // exclusive scan of totals over experts (64 lanes worth, two halves)
    int incl0 = tot_e[0];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl0, o);
      if (lane >= o) incl0 += v;
    }
    const int sum0 = __shfl_sync(0xffffffffu, incl0, 31);
    int incl1 = tot_e[1];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl1, o);
      if (lane >= o) incl1 += v;
    }
    const int start0 = incl0 - tot_e[0];
    const int start1 = sum0 + incl1 - tot_e[1];
    if (lane < E) base[lane] = start0 + pre_e[0];
    if (lane + 32 < E) base[lane + 32] = start1 + pre_e[1];
    if (blockIdx.x == 0) {
      if (lane < E) offsets[lane] = start0;
      if (lane + 32 < E) offsets[lane + 32] = start1;
      const int total = sum0 + __shfl_sync(0xffffffffu, incl1, 31);
      if (lane == 0) offsets[E] = total;
    }
  }
  __syncthreads();

  const int s0 = blockIdx.x * kChunk;
  const int s1 = min(S, s0 + kChunk);
  for (int p0 = s0; p0 < s1; p0 += kPass) {
    for (int i = tid; i < kWarpsPer * kMaxE; i += kThreads) (&warp_cnt[0][0])[i] = 0;
    __syncthreads();
    const int s = p0 + tid;
    const int e = s < s1 ? slot_expert(ids, cursor, s, k, E) : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, e);
    const int rank = __popc(grp & ((1u << lane) - 1u));
    if (e >= 0 && rank == 0) warp_cnt[warp][e] = __popc(grp);
    __syncthreads();
    if (tid < E) {  // exclusive prefix over warps for expert tid
      int acc = 0;
#pragma unroll
      for (int w = 0; w < kWarpsPer; ++w) {
        const int c = warp_cnt[w][tid];
        warp_cnt[w][tid] = acc;
        acc += c;
      }
      pass_tot[tid] = acc;
    }
    __syncthreads();
    if (e >= 0) {
      const int pos = base[e] + warp_cnt[warp][e] + rank;
      perm[pos] = s;
      s_pos[tid] = pos;
      s_src[tid] = s / k;
    } else {
      s_pos[tid] = -1;
    }
    __syncthreads();
    if (tid < E) base[tid] += pass_tot[tid];
    if (xp != nullptr) {
      const int n = min(kPass, s1 - p0);
      for (int i = warp; i < n; i += kWarpsPer) {
        const int pos = s_pos[i];
        if (pos >= 0) copy_row(x + (size_t)s_src[i] * row_bytes, xp + (size_t)pos * row_bytes, row_bytes, lane);
      }
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace qmoe

extern "C" size_t qmoe_permute_workspace_bytes(int T, int k, int E) {
  const long S = (long)T * k;
  const long nblk = (S + qmoe::kChunk - 1) / qmoe::kChunk;
  return (size_t)((nblk < 1 ? 1 : nblk) * (E < 1 ? 1 : E)) * sizeof(int32_t);
}

extern "C" int qmoe_permute_ex(const int32_t* ids, const int32_t* cursor, int T, int k, int E, int gather_e_end,
                               int32_t* perm_out, int32_t* offsets_out, void* workspace, size_t workspace_bytes,
                               const void* x, void* xp, size_t row_bytes, void* stream);

extern "C" int qmoe_permute(const int32_t* ids, const int32_t* cursor, int T, int k, int E,
                            int32_t* perm_out, int32_t* offsets_out, void* workspace,
                            size_t workspace_bytes, const void* x, void* xp, size_t row_bytes,
                            void* stream) {
  return qmoe_permute_ex(ids, cursor, T, k, E, E, perm_out, offsets_out, workspace, workspace_bytes, x, xp, row_bytes,
                         stream);
}

extern "C" int qmoe_permute_ex(const int32_t* ids, const int32_t* cursor, int T, int k, int E, int gather_e_end,
                               int32_t* perm_out, int32_t* offsets_out, void* workspace, size_t workspace_bytes,
                               const void* x, void* xp, size_t row_bytes, void* stream) {
  using namespace qmoe;
  QMOE_REQUIRE(gather_e_end >= 0 && gather_e_end <= E, "qmoe_permute_ex: gather_e_end %d outside [0, %d]", gather_e_end,
               E);
  QMOE_REQUIRE(T >= 0 && k >= 1 && E >= 1 && E <= kMaxE, "qmoe_permute: bad sizes T=%d k=%d E=%d", T, k, E);
  QMOE_REQUIRE(offsets_out != nullptr, "qmoe_permute: offsets_out is null");
  QMOE_REQUIRE((x == nullptr) == (xp == nullptr), "qmoe_permute: x and xp must both be set or both null");
  QMOE_REQUIRE(workspace_bytes >= qmoe_permute_workspace_bytes(T, k, E),
               "qmoe_permute: workspace too small (%zu < %zu)", workspace_bytes,
               qmoe_permute_workspace_bytes(T, k, E));
  cudaStream_t s = as_stream(stream);
  const long S = (long)T * k;
  QMOE_REQUIRE(S < (1L << 30), "qmoe_permute: too many slots");
  if (S == 0) {
    QMOE_CUDA_TRY(cudaMemsetAsync(offsets_out, 0, sizeof(int32_t) * (E + 1), s));
    return QMOE_OK;
  }
  QMOE_REQUIRE(ids && perm_out && workspace, "qmoe_permute: null pointer");
  const int nblk = (int)((S + kChunk - 1) / kChunk);
  int32_t* hist = reinterpret_cast<int32_t*>(workspace);
  int st;
  if (nblk > 1) {  // multi-chunk: per-chunk histograms first
    if ((st = launch_pdl("qmoe_permute(count)", perm_count_kernel, dim3(nblk), dim3(256), 0, s, ids, cursor, (int)S, k,
                         E, hist)))
      return st;
  }
  // one CTA: count + rank + scatter + gather fused; many CTAs: gather runs wide afterwards
  const bool inline_gather = S <= 32;  // decode-sized: one launch; otherwise gather wide
  if ((st = launch_pdl("qmoe_permute(scatter)", perm_scatter_kernel, dim3(nblk), dim3(kThreads), 0, s, ids, cursor,
                       (int)S, k, E, nblk, hist, perm_out, offsets_out, (const uint8_t*)x,
                       inline_gather ? (uint8_t*)xp : nullptr, row_bytes)))
    return st;
  if (xp != nullptr && !inline_gather) {
    const int rows = (int)S;
    const int grid = rows / 8 < 148 * 16 ? (rows + 7) / 8 : 148 * 16;
    if ((st = launch_pdl("qmoe_permute(gather)", perm_gather_kernel, dim3(grid), dim3(256), 0, s, perm_out,
                         offsets_out, gather_e_end, k, rows, (const uint8_t*)x, (uint8_t*)xp, row_bytes)))
      return st;
  }
  return QMOE_OK;
}
