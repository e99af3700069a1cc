// Tile scheduling shared by the SIMT and tcgen05 grouped expert kernels.
//
// Tiles are numbered expert-major (ascending expert id, the reference's drain order,
// model.py:202-204), then by N block, then by M block (M fastest, so consecutive claims reuse the
// same weight block from L2).  They are claimed from one global counter, so at any instant the
// claimed set is a prefix of that order.  The device preempt flag is checked at each claim:
// seeing it at the FIRST tile of expert e stops before e; seeing it inside e lets e finish and
// stops before e+1.  The stop expert is kept as max(INT_MAX - stop) so a zeroed workspace means
// "no stop".  Invariant: every tile of every expert < final stop is executed.
#pragma once

#include <limits.h>

#include "common.cuh"

namespace qmoe {

struct alignas(128) FfnWorkspace {
  int next;      // next tile index to claim
  int stop_inv;  // INT_MAX - stop expert (0 == no stop yet)
  int stop;      // finalized stop (written by ffn_finalize_kernel, read by chained launches)
  int pad[29];
};

constexpr int kFfnWorkspaceSlots = 2;

struct TileMap {
  int e_first;              // absolute id of experts[0]
  int n_exp;                // experts covered
  int total;                // total tiles
  int tile_begin[65];       // prefix over covered experts
  int row_begin[64];        // offsets[e]
  int m_tiles[64];

  __device__ __forceinline__ void locate(int tile, int bm, int n_tiles_n, int bn, int& e, int& m0, int& n0) const {
    int i = 0;
    while (tile >= tile_begin[i + 1]) ++i;
    const int local = tile - tile_begin[i];
    const int nt = local / m_tiles[i];
    const int mt = local - nt * m_tiles[i];
    e = e_first + i;
    m0 = row_begin[i] + mt * bm;
    n0 = nt * bn;
  }
  __device__ __forceinline__ int expert_of(int tile, int& local) const {
    int i = 0;
    while (tile >= tile_begin[i + 1]) ++i;
    local = tile - tile_begin[i];
    return e_first + i;
  }
};

// Called by one thread.  e_limit (optional, device) caps the covered experts (chained launches).
__device__ __forceinline__ void build_tile_map(TileMap& m, const int32_t* offsets, int e_begin, int e_end,
                                               const int32_t* e_limit, int bm, int n_tiles_n) {
  int hi = e_end;
  if (e_limit != nullptr) hi = min(hi, *e_limit);
  if (hi < e_begin) hi = e_begin;
  m.e_first = e_begin;
  m.n_exp = hi - e_begin;
  int acc = 0;
  m.tile_begin[0] = 0;
  for (int i = 0; i < m.n_exp; ++i) {
    const int r0 = offsets[e_begin + i], r1 = offsets[e_begin + i + 1];
    const int mt = (r1 - r0 + bm - 1) / bm;
    m.row_begin[i] = r0;
    m.m_tiles[i] = mt;
    acc += mt * n_tiles_n;
    m.tile_begin[i + 1] = acc;
  }
  m.total = acc;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Claim the next tile or return -1 (no work left, or the preempt boundary was reached).
__device__ __forceinline__ int ffn_claim(const TileMap& m, FfnWorkspace* ws, const volatile int32_t* flag) {
  const int t = atomicAdd(&ws->next, 1);
  if (t >= m.total) return -1;
  int local;
  const int e = m.expert_of(t, local);
  if (flag != nullptr && *flag != 0) {
    const int cand = local == 0 ? e : e + 1;
    atomicMax(&ws->stop_inv, INT_MAX - cand);
  }
  const int stop = INT_MAX - ld_acquire(&ws->stop_inv);
  return e < stop ? t : -1;
}

int ffn_ws_reset(FfnWorkspace* ws, cudaStream_t s);
// cursor = min(stop of ws, *limit (optional), e_end); written to ws->stop and cursor_out (optional).
int ffn_finalize(FfnWorkspace* ws, const int32_t* limit, int e_end, int32_t* cursor_out, cudaStream_t s);

int expert_ffn_simt(int variant, int dtype, const void* xp, const int32_t* offsets, const int32_t* perm, int E,
                    int d, int F, const void* w1, const void* w2, int e_begin, int e_end, void* act_ws, void* y,
                    const volatile int32_t* flag, int32_t* cursor_out, FfnWorkspace* ws, cudaStream_t s);
int expert_ffn_tc(int variant, const void* xp, const int32_t* offsets, const int32_t* perm, int E, int d, int F,
                  const void* w1, const void* w2, int e_begin, int e_end, void* act_ws, void* y,
                  const volatile int32_t* flag, int32_t* cursor_out, FfnWorkspace* ws, int total_rows_hint,
                  cudaStream_t s);

}  // namespace qmoe
