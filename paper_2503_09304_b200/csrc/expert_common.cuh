// Tile scheduling shared by the SIMT and tcgen05 grouped expert kernels.
//
// Tiles are numbered expert-major (ascending expert id, the reference's drain order,
// model.py:202-204), then by N block, then by M block (M fastest, so consecutive claims reuse the
// same weight block from L2).  They are claimed from one global counter, so at any instant the
// claimed set is a prefix of that order.  The device preempt flag holds 0 (run on) or s > 0:
// "stop at the first expert boundary >= s" — the scheduler answered PREEMPT at the report of
// expert s-1, so experts < s always complete (progress is guaranteed, as in the reference where
// a preemption lands after the reported expert's drain).  Seen at a claim of expert e it votes
// for max(s, e) if the tile is e's first (stop before e), else max(s, e+1).  The stop expert
// is kept as max(INT_MAX - stop) so a zeroed workspace means "no stop".  Invariant: every tile
// of every expert < final stop is executed.
#pragma once

#include <limits.h>

#include <cuda.h>

#include "common.cuh"

namespace qmoe {

struct alignas(128) FfnWorkspace {
  int next;      // next tile index to claim
  int stop_inv;  // INT_MAX - stop expert (0 == no stop yet)
  int stop;      // finalized stop (written by ffn_finalize_kernel, read by chained launches)
  int exits;     // CTAs that left a single-launch kernel (the last one finalizes, ffn_exit)
  int pad[28];
};

constexpr int kFfnWorkspaceSlots = 2;
// Workspace header: kFfnWorkspaceSlots claim slots, then one gate_up completion counter per expert
// (the single-launch kernels' gate_up -> down dependency), one down completion counter per expert
// (expert-boundary progress signals, signal_expert_done), then the split-K partials.
constexpr int kFfnMaxExperts = 64;
constexpr size_t kFfnHeaderBytes = sizeof(FfnWorkspace) * kFfnWorkspaceSlots + 2 * kFfnMaxExperts * sizeof(int);
__host__ __device__ inline int* ffn_done(FfnWorkspace* ws) { return reinterpret_cast<int*>(ws + kFfnWorkspaceSlots); }

// Workspace invariant: between launches every claim counter, vote and completion counter of the
// header is zero (the caller zeroes the header once at allocation; each launch leaves it so), so
// no launch needs a memset in front of it.  `stop` survives until the next launch's finalize.
//
// Single-launch kernels finalize in-kernel: one thread per CTA calls this after the CTA's last
// claim and store; the LAST CTA out publishes the stop expert (what ffn_finalize_kernel does for
// the multi-launch paths), writes cursor_out, and re-zeroes the header for the next launch.
// A launch that stopped before e_end because of its preempt flag leaves the flag at -1 ("void"):
// every later launch polling the same flag -- the rest of the preempted iteration, already
// enqueued by a host that runs ahead -- claims nothing, and guarded KV appends
// (qmoe_kv_append_guarded) skip, so the abandoned layers leave no state behind.
__device__ __forceinline__ void ffn_exit(FfnWorkspace* ws, int* done, int e_end, int32_t* cursor_out,
                                         const volatile int32_t* flag = nullptr) {
  __threadfence();
  const unsigned n = gridDim.x * gridDim.y * gridDim.z;
  if (atomicAdd(&ws->exits, 1) != (int)n - 1) return;
  __threadfence();
  int c = INT_MAX - atomicOr(&ws->stop_inv, 0);
  if (c > e_end) c = e_end;
  ws->stop = c;
  if (cursor_out != nullptr) *cursor_out = c;
  if (flag != nullptr && c < e_end) *const_cast<volatile int32_t*>(flag) = -1;
  ws->next = 0;
  ws->stop_inv = 0;
  ws->exits = 0;
  for (int e = 0; e < 2 * kFfnMaxExperts; ++e) done[e] = 0;
}

// Expert-boundary progress (qmoe_expert_ffn_ex, wall-clock reporting): every epilogue warp that
// finished storing a down unit of expert e counts itself (lane 0, after __syncwarp); the warp that
// completes e's count (`need` = down units of e x epilogue warps per unit) publishes `seq` into
// progress[e] -- pinned host memory the serving host polls, so it answers expert e's report when
// the GPU has actually drained expert e (reference engine.py:204-219: the report follows the drain).
__device__ __forceinline__ void signal_expert_done(int* done, int e, int need, int32_t* progress, int seq) {
  __threadfence();
  if (atomicAdd(done + kFfnMaxExperts + e, 1) == need - 1)
    asm volatile("st.release.sys.b32 [%0], %1;" ::"l"(progress + e), "r"(seq) : "memory");
}

struct TileMap {
  int e_first;              // absolute id of experts[0]
  int n_exp;                // experts covered
  int total;                // total tiles
  int tile_begin[65];       // prefix over covered experts
  int row_begin[64];        // offsets[e]
  int m_tiles[64];

  // Index of the covered expert owning `tile` (binary search over the tile prefix).
  __device__ __forceinline__ int slot_of(int tile) const {
    int lo = 0, hi = n_exp - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (tile_begin[mid] <= tile) lo = mid; else hi = mid - 1;
    }
    return lo;
  }
  // Tile -> (expert, first row, first column, split).  Within an expert tiles run N-block
  // major, M fastest; the `nsplit` K-splits of one (M, N) tile are adjacent N-block entries.
  __device__ __forceinline__ void locate(int tile, int bm, int n_tiles_n, int bn, int& e, int& m0, int& n0,
                                         int nsplit = 1, int* split = nullptr) const {
    const int i = slot_of(tile);
    const int local = tile - tile_begin[i];
    const int nt = local / m_tiles[i];
    const int mt = local - nt * m_tiles[i];
    e = e_first + i;
    m0 = row_begin[i] + mt * bm;
    n0 = (nt / nsplit) * bn;
    if (split != nullptr) *split = nt % nsplit;
  }
  __device__ __forceinline__ int expert_of(int tile, int& local) const {
    const int i = slot_of(tile);
    local = tile - tile_begin[i];
    return e_first + i;
  }
};

// Called by all 32 lanes of ONE warp: per-expert row ranges loaded in parallel, tile counts
// prefix-summed with warp shuffles (E <= 64).  e_limit (optional, device) caps the covered
// experts (chained launches).  n_tiles_n already includes any K-split factor.
// merge > 0: an expert's last M tile absorbs a remainder of <= merge rows into the tile before it
// (tile of bm + remainder rows; kernels that handle such wide tiles only).
__device__ __forceinline__ void build_tile_map(TileMap& m, const int32_t* offsets, int e_begin, int e_end,
                                               const int32_t* e_limit, int bm, int n_tiles_n, int merge = 0) {
  const int lane = threadIdx.x & 31;
  int hi = e_end;
  if (e_limit != nullptr) hi = min(hi, *e_limit);
  if (hi < e_begin) hi = e_begin;
  const int n = hi - e_begin;
  int carry = 0;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int i = lane + 32 * half;
    int tiles = 0;
    if (i < n) {
      const int r0 = offsets[e_begin + i], r1 = offsets[e_begin + i + 1];
      int mt = (r1 - r0 + bm - 1) / bm;
      if (merge > 0 && mt >= 2 && (r1 - r0) - (mt - 1) * bm <= merge) --mt;
      m.row_begin[i] = r0;
      m.m_tiles[i] = mt;
      tiles = mt * n_tiles_n;
    }
    int incl = tiles;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (i < n) m.tile_begin[i + 1] = carry + incl;
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) {
    m.tile_begin[0] = 0;
    m.e_first = e_begin;
    m.n_exp = n;
    m.total = carry;
  }
  __syncwarp();
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Claim the next tile or return -1 (no work left, or the preempt boundary was reached).
// `last_e` is the caller's previously claimed expert: the (possibly host-mapped, PCIe-latency)
// flag is only read when the claimer moves to a new expert — the only place a stop can take
// effect — while the device-side stop vote is consulted on every claim.
__device__ __forceinline__ int ffn_claim(const TileMap& m, FfnWorkspace* ws, const volatile int32_t* flag,
                                         int& last_e) {
  const int t = atomicAdd(&ws->next, 1);
  if (t >= m.total) return -1;
  int local;
  const int e = m.expert_of(t, local);
  if (flag != nullptr && e != last_e) {
    const int s = *flag;
    if (s != 0) {  // s < 0: the iteration was preempted by an earlier launch -- stop here
      int cand = (s < 0 || local == 0) ? e : e + 1;
      if (cand < s) cand = s;
      atomicMax(&ws->stop_inv, INT_MAX - cand);
    }
  }
  last_e = e;
  const int stop = INT_MAX - ld_acquire(&ws->stop_inv);
  return e < stop ? t : -1;
}

// Destination row of a down-projection output: row v of the local slot buffer, or — expert
// parallel over NVLink peer memory (qmoe_expert_ffn_peer) — row (v & 0xFFFFFF) of the slot
// buffer of rank (v >> 24), whose base address is peers[v >> 24].
template <typename T>
__device__ __forceinline__ T* out_row(T* base, void* const* peers, int32_t v, size_t ld) {
  if (peers != nullptr) return reinterpret_cast<T*>(peers[(uint32_t)v >> 24]) + (size_t)(v & 0xFFFFFF) * ld;
  return base + (size_t)v * ld;
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Single-launch gate_up + down kernels (expert_swap.cu, expert_fused.cu).  Resolve a unit index
// t taken from the claim counter: gate_up units [0, N1) under the expert-boundary stop protocol of
// ffn_claim, then down units [N1, N1 + N2).  Returns the unit to run or -1.  Producers take the
// NEXT index (atomicAdd on ws->next) as soon as they start a unit and resolve it one unit later,
// so the claim's L2 round trip overlaps the current unit's loads instead of stalling the ring.
__device__ __forceinline__ int resolve_claim(const TileMap& m1, int N2, FfnWorkspace* ws, const volatile int32_t* flag,
                                             int& last_e, int t) {
  const int N1 = m1.total;
  while (true) {
    if (t >= N1) return t - N1 < N2 ? t : -1;
    int local;
    const int e = m1.expert_of(t, local);
    if (flag != nullptr && e != last_e) {
      const int s = *flag;
      if (s != 0) {  // s < 0: the iteration was preempted by an earlier launch -- stop here
        int cand = (s < 0 || local == 0) ? e : e + 1;
        if (cand < s) cand = s;
        atomicMax(&ws->stop_inv, INT_MAX - cand);
      }
    }
    last_e = e;
    const int stop = INT_MAX - ld_acquire(&ws->stop_inv);
    if (e < stop) return t;
    // every later gate_up unit belongs to an expert >= e >= stop: skip straight to the down units
    atomicMax(&ws->next, N1);
    t = atomicAdd(&ws->next, 1);
  }
}

__device__ __forceinline__ int two_phase_claim(const TileMap& m1, int N2, FfnWorkspace* ws,
                                               const volatile int32_t* flag, int& last_e) {
  return resolve_claim(m1, N2, ws, flag, last_e, atomicAdd(&ws->next, 1));
}

// Down unit of expert e: true once all gate_up units of e stored their act rows, false if e can
// no longer complete (the stop fell at or below it).
__device__ __forceinline__ bool expert_ready(const int* done, int e, int need, const FfnWorkspace* ws) {
  while (true) {
    if (ld_acquire(done + e) >= need) return true;
    if (INT_MAX - ld_acquire(&ws->stop_inv) <= e) return false;
    __nanosleep(64);
  }
}

// Extra workspace the bf16 SwiGLU path needs for split-K partials of the down projection.
size_t splitk_bytes(int xp_rows, int d);
// cursor = min(stop of ws, *limit (optional), e_end); written to ws->stop and cursor_out (optional).
// flag (optional): set to -1 when the stop falls before e_end (see ffn_exit).
int ffn_finalize(FfnWorkspace* ws, const int32_t* limit, int e_end, int32_t* cursor_out, cudaStream_t s,
                 const volatile int32_t* flag = nullptr);

int expert_ffn_simt(int variant, int dtype, const void* xp, const int32_t* offsets, const int32_t* perm, int E,
                    int d, int F, const void* w1, const void* w2, int e_begin, int e_end, void* act_ws, void* y,
                    const volatile int32_t* flag, int32_t* cursor_out, FfnWorkspace* ws, cudaStream_t s);
// ---- host helpers of the tcgen05 paths (expert_tc.cu) -----------------------------------
int tc_init_driver();  // cuTensorMapEncodeTiled entry point + SM count; QMOE_OK or error
int tc_num_sms();
// 2D bf16 row-major [rows, cols] -> tensor map with box {64 cols, box_rows}, 128B swizzle.
int tc_make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows);
// Small-batch path (expert_swap.cu): swap-AB tiles, gate_up and down in one persistent launch.
bool use_swap_ab(int xp_rows, int n_experts, int d, int F);
int expert_ffn_swap(const void* xp, const int32_t* offsets, const int32_t* perm, int E, int d, int F,
                    const void* w1, const void* w2, int e_begin, int e_end, void* act_ws, void* y,
                    const volatile int32_t* flag, int32_t* cursor_out, FfnWorkspace* ws, int xp_rows,
                    void* const* y_peers, const void* x, int T, int k, cudaStream_t s,
                    int32_t* progress = nullptr, int seq = 0, int path_rows = -1);

// Mid-size and large batches (expert_fused.cu): 128 x 256 (1 CTA) or 256 x 256 (CTA pair) tiles,
// gate_up and down in one persistent launch.
bool use_fused_tc();
int expert_ffn_fused(const void* xp, const int32_t* offsets, const int32_t* perm, int E, int d, int F,
                     const void* w1, const void* w2, int e_begin, int e_end, void* act_ws, void* y,
                     const volatile int32_t* flag, int32_t* cursor_out, FfnWorkspace* ws, int xp_rows,
                     void* const* y_peers, bool pair, const void* x, int T, int k, cudaStream_t s,
                     int32_t* progress = nullptr, int seq = 0, const void* x_direct = nullptr,
                     int x_first = 0);
// Mid-size batches of fine-grained experts (expert_fused.cu): swap-AB CTA-pair tiles (256 weight
// rows x <= 256 tokens, N sized to the valid rows), gate_up and down in one persistent launch.
bool use_swap_pair(int xp_rows, int n_experts, int d, int F);
int expert_ffn_swap_pair(const void* xp, const int32_t* offsets, const int32_t* perm, int E, int d, int F,
                         const void* w1, const void* w2, int e_begin, int e_end, void* act_ws, void* y,
                         const volatile int32_t* flag, int32_t* cursor_out, FfnWorkspace* ws, int xp_rows,
                         void* const* y_peers, const void* x, int T, int k, cudaStream_t s,
                         int32_t* progress = nullptr, int seq = 0);
// Which bf16 SwiGLU kernel qmoe_expert_ffn runs for this shape (QMOE_PATH_* in qmoe.h).
int expert_ffn_path(int d, int F, int E, int xp_rows);

int expert_ffn_tc(int variant, const void* xp, const int32_t* offsets, const int32_t* perm, int E, int d, int F,
                  const void* w1, const void* w2, int e_begin, int e_end, void* act_ws, void* y,
                  const volatile int32_t* flag, int32_t* cursor_out, FfnWorkspace* ws, int total_rows_hint,
                  void* const* y_peers, cudaStream_t s, int32_t* progress = nullptr, int seq = 0,
                  int path_rows = -1);
// Marks experts [e_begin, e_end) done in progress[] once the stream reaches it (paths whose
// kernels do not signal per expert: SIMT, tanh, two-launch).
int ffn_progress_all(int32_t* progress, int seq, int e_begin, int e_end, cudaStream_t s);

}  // namespace qmoe
