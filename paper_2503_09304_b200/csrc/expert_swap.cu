// Small-batch grouped expert FFN (decode, fine-grained experts): swap-AB tcgen05 tiles with the
// gate_up and down projections in ONE persistent launch.
//
// Replaces the reference's per-expert drain (engine.py:204-215 -> model.py:141-145) for the
// north-star SwiGLU expert (HF MixtralExperts / Qwen2MoeExperts) when an expert sees few rows.
//
// Why a separate kernel.  With a handful of rows per expert (Mixtral decode: ~8, Qwen: ~2) the
// layer is pure weight streaming.  The 128-row token tiles of the large-batch kernel would spend
// most of their MMA work and 1/3 of their L2 traffic on padding rows, and the two launches
// (gate_up, then down) each leave a partial last wave on a 148-SM part.  Here:
//   * swap-AB: the weights are the MMA's M = 128 side (A, from HBM through TMA), the tokens the
//     N = NT side (B, NT in {32, 64, 128} rows from L2).  D[128 weight rows x NT tokens] lives in TMEM.
//   * gate_up unit = (expert, 128 F columns, token tile): two MMAs per K step (gate rows and up
//     rows of the same 128 columns) into two accumulators, so every epilogue thread holds g and u
//     of one column and writes SiLU(g)*u for its tokens to act.
//   * down unit = (expert, 128 output columns, token tile, K split): W2 rows x act rows.  Two K
//     blocks per pipeline stage so a stage always streams 32 KB of weights.  Large-F experts
//     (Mixtral, 3.7 MB per unit) are K-split into ~1 MB units (fp32 partials, fixed-order reduce).
//   * one unit counter covers all gate_up units (expert-major, the reference's drain order) then
//     all down units.  A down unit of expert e waits until every gate_up unit of e has stored its
//     act rows (per-expert completion counter, release/acquire + async-proxy fence before TMA
//     reads act).  The gate_up tail of one expert overlaps the down units of earlier experts, so
//     the layer has a single tail.
// Preemption keeps the expert-boundary contract of expert_common.cuh: the device flag is read
// when a claimer of a gate_up unit moves to a new expert; the stop vote is final for the launch;
// down units run for every expert below the stop and are skipped for experts that will never
// complete their gate_up.
#include <cudaTypedefs.h>

#include <algorithm>

#include "expert_common.cuh"
#include "tc_ptx.cuh"

namespace qmoe {
namespace {

constexpr int kThreadsS = 256;
constexpr int kWRows = 128;  // weight rows per unit (MMA M)
constexpr int kBK = 64;      // K elements per TMA box (128 B rows, 128B swizzle)
constexpr int kRing = 4;
constexpr int kEpi0 = 4;     // first epilogue warp
constexpr int kSwapRowsMax = 512;
constexpr int kMaxSplitS = 8;

struct SwapParams {
  int d, F;
  int e_begin, e_end;
  const int32_t* offsets;
  const int32_t* perm;
  const volatile int32_t* flag;
  FfnWorkspace* ws;
  int* done;
  __nv_bfloat16* act;
  __nv_bfloat16* y;
  float* part;
  int nsplit, kb_per_split, part_rows;
  void* const* peers;  // expert parallel over peer memory: per-rank slot buffers (see out_row)
  int k;               // top-k: gate_up B rows are x[perm[r] / k] when gather != 0
  int gather;          // 1: token rows gathered from X by the producer warp (TMA tile::gather4)
  int32_t* cursor;     // optional cursor_out (written by the last CTA out, ffn_exit)
  int32_t* progress;   // optional host-mapped per-expert progress words (signal_expert_done)
  int seq;
  const __nv_bfloat16* w1;  // gate_up weights [E, 2F, d] (L2 prefetch ahead of griddepcontrol.wait)
  int prefetch_bytes;       // per CTA; 0 = none
};

template <int NT>
struct SwapCfg {
  static constexpr int kABytes = kWRows * kBK * 2;  // 16 KB: one 128-row weight K block
  static constexpr int kBBytes = NT * kBK * 2;      // one NT-row token K block
  // down-projection K blocks per stage: 2 keeps 32 KB of weights per stage for small token tiles;
  // NT = 128 stages one (48 KB stages, 4 in flight)
  static constexpr int kKB2 = NT <= 64 ? 2 : 1;
  static constexpr int kStageBytes = 2 * kABytes + kKB2 * kBBytes;
  static constexpr int kStages = (200 * 1024) / kStageBytes;
  static constexpr int kSmem = kStages * kStageBytes + 1024;
  static constexpr uint32_t kTmemCols = 4 * NT;  // 2 accumulator stages x (gate, up) x NT
};

__device__ __forceinline__ float silu_mul(float g, float u) { return g / (1.f + __expf(-g)) * u; }

template <int NT>
__global__ void __launch_bounds__(kThreadsS, 1)
ffn_swap_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW1,
                const __grid_constant__ CUtensorMap tmAct, const __grid_constant__ CUtensorMap tmW2, SwapParams p) {
  if (threadIdx.x == 0 && p.prefetch_bytes > 0) {
    // The weights are not produced by the kernels this launch depends on, so before
    // griddepcontrol.wait -- while the router and the permute of this layer still run (they
    // trigger their dependents at entry) -- each CTA pulls into L2 the first rows of the gate and
    // up halves of the unit it will most likely claim first (unit = CTA index: expert e_begin +
    // b / nt1, 128-column block b % nt1, one token tile per expert at decode sizes).
    const int nt1 = (p.F + kWRows - 1) / kWRows;
    const int e = p.e_begin + (int)blockIdx.x / nt1, fb = (int)blockIdx.x % nt1;
    if (e < p.e_end) {
      const size_t row_bytes = (size_t)p.d * 2;
      const int rows = min(kWRows, p.F - fb * kWRows);
      const uint32_t half = (uint32_t)min((size_t)p.prefetch_bytes / 2, (size_t)rows * row_bytes) & ~15u;
      const __nv_bfloat16* g = p.w1 + ((size_t)e * 2 * p.F + (size_t)fb * kWRows) * p.d;
      const __nv_bfloat16* u = g + (size_t)p.F * p.d;
      for (uint32_t off = 0; off < half; off += 65536) {
        const uint32_t n = min(65536u, half - off);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<const char*>(g) + off),
                     "r"(n) : "memory");
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<const char*>(u) + off),
                     "r"(n) : "memory");
      }
    }
  }
  pdl_wait();
  pdl_trigger();
  using C = SwapCfg<NT>;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[C::kStages], empty_bar[C::kStages];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ __align__(8) uint64_t ring_full[kRing], ring_empty[kRing];
  __shared__ int ring_tile[kRing];
  __shared__ uint32_t tmem_base_smem;
  __shared__ TileMap map1, map2;

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt1 = (p.F + kWRows - 1) / kWRows;  // F column blocks (gate_up)
  const int nt2 = (p.d + kWRows - 1) / kWRows;  // d column blocks (down)
  const int nkb1 = (p.d + kBK - 1) / kBK;
  const int nkb2 = (p.F + kBK - 1) / kBK;

  if (warp == 0) build_tile_map(map1, p.offsets, p.e_begin, p.e_end, nullptr, NT, nt1);
  if (warp == 3) build_tile_map(map2, p.offsets, p.e_begin, p.e_end, nullptr, NT, nt2 * p.nsplit);
  if (threadIdx.x == 32) {
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull_bar[a], 1);
      ptx::mbar_init(&tempty_bar[a], 4);
    }
    for (int i = 0; i < kRing; ++i) {
      ptx::mbar_init(&ring_full[i], 1);
      ptx::mbar_init(&ring_empty[i], 1 + 4);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<C::kTmemCols>(&tmem_base_smem);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = tmem_base_smem;
  const int N1 = map1.total, N2 = map2.total;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer (warp-wide:
    // lane 0 claims and issues the tile loads; in gather mode lanes [0, NT/4) each issue one
    // tile::gather4 of 4 token rows of X per K block instead of one Xp tile load)
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmX);
      ptx::tma_prefetch_desc(&tmW1);
      ptx::tma_prefetch_desc(&tmAct);
      ptx::tma_prefetch_desc(&tmW2);
    }
    int stage = 0, slot = 0, last_e = -1;
    uint32_t phase = 0, rphase = 0;
    int pending = lane == 0 ? atomicAdd(&p.ws->next, 1) : 0;  // claim one unit ahead (see resolve_claim)
    while (true) {
      int t = -1;
      if (lane == 0) {
        while (true) {
          t = resolve_claim(map1, N2, p.ws, p.flag, last_e, pending);
          if (t >= N1) {
            int e2, m2, n2, s2;
            map2.locate(t - N1, NT, nt2 * p.nsplit, kWRows, e2, m2, n2, p.nsplit, &s2);
            if (!expert_ready(p.done, e2, map1.m_tiles[e2 - map1.e_first] * nt1 * 4, p.ws)) {
              pending = atomicAdd(&p.ws->next, 1);
              continue;
            }
            fence_proxy_async_global();  // act rows written by generic stores, read below by TMA
          }
          break;
        }
        ptx::mbar_wait(&ring_empty[slot], rphase ^ 1);
        ring_tile[slot] = t;
        ptx::mbar_arrive(&ring_full[slot]);
        if (t >= 0) pending = atomicAdd(&p.ws->next, 1);  // in flight while this unit's loads issue
      }
      t = __shfl_sync(0xffffffffu, t, 0);
      if (++slot == kRing) { slot = 0; rphase ^= 1; }
      if (t < 0) break;
      int e = 0, m0 = 0, n0 = 0, split = 0;
      if (t < N1) {
        map1.locate(t, NT, nt1, kWRows, e, m0, n0);
        const bool gather = p.gather != 0;
        int g[4] = {0, 0, 0, 0};
        const bool g_lane = gather && lane < NT / 4;
        if (g_lane) {
          const int row_end = p.offsets[e + 1];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int r = m0 + 4 * lane + j;
            g[j] = r < row_end ? p.perm[r] / p.k : 0;  // rows past the queue read token 0 (never stored)
          }
        }
        const int g_row = e * 2 * p.F + n0, u_row = g_row + p.F;
        for (int kb = 0; kb < nkb1; ++kb) {
          ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::kStageBytes;
          if (lane == 0) {
            ptx::mbar_arrive_expect_tx(&full_bar[stage], 2 * C::kABytes + C::kBBytes);
            ptx::tma_load_2d(&tmW1, &full_bar[stage], sa, kb * kBK, g_row, ptx::kEvictNormal);
            ptx::tma_load_2d(&tmW1, &full_bar[stage], sa + C::kABytes, kb * kBK, u_row, ptx::kEvictNormal);
            if (!gather) ptx::tma_load_2d(&tmX, &full_bar[stage], sa + 2 * C::kABytes, kb * kBK, m0, ptx::kEvictLast);
          }
          if (g_lane)
            ptx::tma_gather4(&tmX, &full_bar[stage], sa + 2 * C::kABytes + lane * 512, kb * kBK, g[0], g[1], g[2], g[3],
                             ptx::kEvictLast);
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      } else {
        map2.locate(t - N1, NT, nt2 * p.nsplit, kWRows, e, m0, n0, p.nsplit, &split);
        const int kb0 = split * p.kb_per_split, kb1 = min(nkb2, kb0 + p.kb_per_split);
        const int w_row = e * p.d + n0;
        for (int kb = kb0; kb < kb1; kb += C::kKB2) {
          const bool two = C::kKB2 == 2 && kb + 1 < kb1;
          ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::kStageBytes;
          if (lane == 0) {
            ptx::mbar_arrive_expect_tx(&full_bar[stage], (two ? 2 : 1) * (C::kABytes + C::kBBytes));
            ptx::tma_load_2d(&tmW2, &full_bar[stage], sa, kb * kBK, w_row, ptx::kEvictNormal);
            ptx::tma_load_2d(&tmAct, &full_bar[stage], sa + 2 * C::kABytes, kb * kBK, m0, ptx::kEvictLast);
            if (two) {
              ptx::tma_load_2d(&tmW2, &full_bar[stage], sa + C::kABytes, (kb + 1) * kBK, w_row, ptx::kEvictNormal);
              ptx::tma_load_2d(&tmAct, &full_bar[stage], sa + 2 * C::kABytes + C::kBBytes, (kb + 1) * kBK, m0,
                               ptx::kEvictLast);
            }
          }
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int stage = 0, slot = 0, acc = 0;
      uint32_t phase = 0, rphase = 0, aphase = 0;
      while (true) {
        ptx::mbar_wait(&ring_full[slot], rphase);
        const int t = ring_tile[slot];
        ptx::mbar_arrive(&ring_empty[slot]);
        if (++slot == kRing) { slot = 0; rphase ^= 1; }
        if (t < 0) break;
        // MMA N = the tile's valid token rows rounded up to 16 (an expert's last token tile is
        // usually partial): the tensor work tracks the real rows instead of NT
        int e, m0, n0, split = 0;
        if (t < N1) map1.locate(t, NT, nt1, kWRows, e, m0, n0);
        else map2.locate(t - N1, NT, nt2 * p.nsplit, kWRows, e, m0, n0, p.nsplit, &split);
        const int rows = min(NT, p.offsets[e + 1] - m0);
        const uint32_t kIdesc = ptx::idesc_bf16_f32(kWRows, max(16, (rows + 15) & ~15));
        ptx::mbar_wait(&tempty_bar[acc], aphase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 2 * NT;
        if (t < N1) {
          for (int kb = 0; kb < nkb1; ++kb) {
            ptx::mbar_wait(&full_bar[stage], phase);
            ptx::tc_fence_after();
            const uint32_t a = ptx::smem_u32(smem + stage * C::kStageBytes);
            const uint32_t b = a + 2 * C::kABytes;
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              const uint32_t accum = (kb | k) != 0;
              const uint64_t db = ptx::sw128_kmajor_desc(b + k * 32);
              ptx::tc_mma_bf16(d_tmem, ptx::sw128_kmajor_desc(a + k * 32), db, kIdesc, accum);
              ptx::tc_mma_bf16(d_tmem + NT, ptx::sw128_kmajor_desc(a + C::kABytes + k * 32), db, kIdesc, accum);
            }
            ptx::tc_commit(&empty_bar[stage]);
            if (++stage == C::kStages) { stage = 0; phase ^= 1; }
          }
        } else {
          const int kb0 = split * p.kb_per_split, kb1 = min(nkb2, kb0 + p.kb_per_split);
          for (int kb = kb0; kb < kb1; kb += C::kKB2) {
            const int nh = C::kKB2 == 2 && kb + 1 < kb1 ? 2 : 1;
            ptx::mbar_wait(&full_bar[stage], phase);
            ptx::tc_fence_after();
            const uint32_t a = ptx::smem_u32(smem + stage * C::kStageBytes);
            const uint32_t b = a + 2 * C::kABytes;
            for (int h = 0; h < nh; ++h) {
#pragma unroll
              for (int k = 0; k < kBK / 16; ++k)
                ptx::tc_mma_bf16(d_tmem, ptx::sw128_kmajor_desc(a + h * C::kABytes + k * 32),
                                 ptx::sw128_kmajor_desc(b + h * C::kBBytes + k * 32), kIdesc,
                                 (kb > kb0 || h > 0 || k > 0) ? 1u : 0u);
            }
            ptx::tc_commit(&empty_bar[stage]);
            if (++stage == C::kStages) { stage = 0; phase ^= 1; }
          }
        }
        ptx::tc_commit(&tfull_bar[acc]);
        if (++acc == 2) { acc = 0; aphase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp >= kEpi0) {
    // ------------------------------------------------------------------ epilogue
    // Thread (ew, lane) owns TMEM lane 32*ew + lane = one weight row (an F column for gate_up,
    // a d column for down) and the NT token columns of that row.
    const int ew = warp - kEpi0;
    int slot = 0, acc = 0;
    uint32_t rphase = 0, aphase = 0;
    while (true) {
      ptx::mbar_wait(&ring_full[slot], rphase);
      const int t = ring_tile[slot];
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&ring_empty[slot]);
      if (++slot == kRing) { slot = 0; rphase ^= 1; }
      if (t < 0) break;
      const bool up_phase = t < N1;
      int e, m0, n0, split = 0;
      if (up_phase) map1.locate(t, NT, nt1, kWRows, e, m0, n0);
      else map2.locate(t - N1, NT, nt2 * p.nsplit, kWRows, e, m0, n0, p.nsplit, &split);
      const int nrows = min(NT, p.offsets[e + 1] - m0);  // warp-uniform
      const int col = n0 + ew * 32 + lane;
      ptx::mbar_wait(&tfull_bar[acc], aphase);
      ptx::tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * 2 * NT;
      if (up_phase) {
        const bool ok = col < p.F;
#pragma unroll 1
        for (int c = 0; c < nrows; c += 32) {
          uint32_t g[32], u[32];
          ptx::tmem_ld32(t_row + c, g);
          ptx::tmem_ld32(t_row + NT + c, u);
          ptx::tmem_ld_wait();
          __nv_bfloat16* dst = p.act + (size_t)(m0 + c) * p.F + col;
          const int n = min(32, nrows - c);
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < n && ok) dst[(size_t)j * p.F] = __float2bfloat16_rn(silu_mul(__uint_as_float(g[j]), __uint_as_float(u[j])));
        }
      } else {
        const bool ok = col < p.d;
#pragma unroll 1
        for (int c = 0; c < nrows; c += 32) {
          uint32_t v[32];
          ptx::tmem_ld32(t_row + c, v);
          ptx::tmem_ld_wait();
          const int n = min(32, nrows - c);
          if (p.nsplit > 1) {
            float* dst = p.part + ((size_t)split * p.part_rows + m0 + c) * p.d + col;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < n && ok) dst[(size_t)j * p.d] = __uint_as_float(v[j]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < n && ok) out_row(p.y, p.peers, p.perm[m0 + c + j], p.d)[col] = __float2bfloat16_rn(__uint_as_float(v[j]));
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) { acc = 0; aphase ^= 1; }
      if (up_phase) {
        // publish this warp's act rows to the down units of expert e (read by TMA: async proxy)
        fence_proxy_async_global();
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(p.done + e, 1);
      } else if (p.progress != nullptr) {
        __syncwarp();
        if (lane == 0)
          signal_expert_done(p.done, e, map2.m_tiles[e - map2.e_first] * nt2 * p.nsplit * 4, p.progress, p.seq);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) ffn_exit(p.ws, p.done, p.e_end, p.cursor, p.flag);
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

// Y[perm[r]] = bf16(sum_s part[s][r]) for the rows of experts [e_begin, stop), splits summed in
// order (deterministic).  One thread per 8 columns of a row, so a decode batch (64 rows x 4096)
// still spreads over ~128 CTAs.
__global__ void __launch_bounds__(256) swap_reduce_kernel(const float* __restrict__ part, int nsplit, int part_rows,
                                                          int N, const int32_t* __restrict__ perm,
                                                          const int32_t* __restrict__ offsets, int e_begin,
                                                          const int32_t* __restrict__ stop,
                                                          __nv_bfloat16* __restrict__ y, void* const* peers) {
  pdl_wait();
  pdl_trigger();
  const int r0 = offsets[e_begin], r1 = offsets[*stop];
  const int per_row = N / 8;
  const long long total = (long long)(r1 - r0) * per_row;
  for (long long i = blockIdx.x * 256ll + threadIdx.x; i < total; i += (long long)gridDim.x * 256) {
    const int r = r0 + (int)(i / per_row), c = (int)(i % per_row) * 8;
    float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int s = 0; s < nsplit; ++s) {
      const float4* src = reinterpret_cast<const float4*>(part + ((size_t)s * part_rows + r) * N + c);
      const float4 u = __ldg(src), w = __ldg(src + 1);
      a[0] += u.x; a[1] += u.y; a[2] += u.z; a[3] += u.w; a[4] += w.x; a[5] += w.y; a[6] += w.z; a[7] += w.w;
    }
    __nv_bfloat162 h[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) h[q] = __floats2bfloat162_rn(a[2 * q], a[2 * q + 1]);
    *reinterpret_cast<uint4*>(out_row(y, peers, perm[r], N) + c) = *reinterpret_cast<const uint4*>(h);
  }
}

template <int NT>
int launch_swap(const CUtensorMap* maps, const SwapParams& p, cudaStream_t s) {
  static uint64_t attr_set = 0;  // devices already configured
  if (!(attr_set & current_device_bit())) {
    QMOE_CUDA_TRY(cudaFuncSetAttribute(ffn_swap_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       SwapCfg<NT>::kSmem));
    attr_set |= current_device_bit();
  }
  return launch_pdl("qmoe_expert_ffn(tcgen05 swap-AB)", ffn_swap_kernel<NT>, dim3(tc_num_sms()), dim3(kThreadsS),
                    SwapCfg<NT>::kSmem, s, maps[0], maps[1], maps[2], maps[3], p);
}

// K splits of a down unit so each streams about 1 MB of weights (Mixtral: 128 x 14336 bf16 =
// 3.7 MB -> 4 splits; Qwen: 0.36 MB -> 1).  A function of the layer shape only, so a resumed
// launch rounds exactly like an uninterrupted one.
int swap_splits(int F) {
  const double unit = (double)kWRows * F * 2;
  int n = (int)(unit / (1 << 20) + 0.5);
  if (n > kMaxSplitS) n = kMaxSplitS;
  const int nkb = (F + kBK - 1) / kBK;
  if (n > nkb / 8) n = nkb / 8;  // >= 8 K blocks per split
  return n < 1 ? 1 : n;
}

}  // namespace

// Small batches: at most ~80 routed rows per expert on average (Mixtral decode up to 320 tokens,
// Qwen up to ~1.2k tokens).  K-split down units need the split-K workspace, which is sized for at
// most kSwapRowsMax rows (qmoe_expert_ffn_workspace_bytes).  QMOE_SWAP_AB=0/1 forces the choice.
bool use_swap_ab(int xp_rows, int n_experts, int d, int F) {
  static int forced = [] {
    const char* v = getenv("QMOE_SWAP_AB");
    return v == nullptr ? -1 : atoi(v);
  }();
  (void)F;
  if (d % kWRows != 0 || F % kBK != 0 || n_experts < 1 || n_experts > kFfnMaxExperts) return false;
  if (forced >= 0) return forced == 1;
  // measured crossover: Qwen (60 experts) 1k tokens (~68 rows per expert) is faster here, Mixtral
  // 512 tokens (~128 per expert) on the 128/256-row tcgen05 tiles
  return xp_rows <= 80 * n_experts;
}

int expert_ffn_swap(const void* xp, const int32_t* offsets, const int32_t* perm, int E, int d, int F,
                    const void* w1, const void* w2, int e_begin, int e_end, void* act_ws, void* y,
                    const volatile int32_t* flag, int32_t* cursor_out, FfnWorkspace* ws, int xp_rows,
                    void* const* y_peers, const void* x, int T, int k, cudaStream_t s, int32_t* progress, int seq,
                    int path_rows) {
  int st;
  // Token tile: 32 rows when experts see ~1-24 rows on average (decode), 64 up to ~64, else 128.
  const double mean_rows = (double)(path_rows < 0 ? xp_rows : path_rows) / (E > 0 ? E : 1);
  const int NT = mean_rows <= 24.0 ? 32 : (mean_rows <= 64.0 ? 64 : 128);
  CUtensorMap maps[4];
  // token rows: NT-row boxes of Xp, or single rows of X for the tile::gather4 loads (x != nullptr)
  if ((st = x != nullptr ? tc_make_map(&maps[0], x, T, d, 1) : tc_make_map(&maps[0], xp, xp_rows, d, NT)) || (st = tc_make_map(&maps[1], w1, (uint64_t)E * 2 * F, d, kWRows)) ||
      (st = tc_make_map(&maps[2], act_ws, xp_rows, F, NT)) || (st = tc_make_map(&maps[3], w2, (uint64_t)E * d, F, kWRows)))
    return st;
  SwapParams p{};
  p.d = d;
  p.F = F;
  p.e_begin = e_begin;
  p.e_end = e_end;
  p.offsets = offsets;
  p.perm = perm;
  p.flag = flag;
  p.ws = ws;
  p.done = ffn_done(ws);
  p.act = (__nv_bfloat16*)act_ws;
  p.y = (__nv_bfloat16*)y;
  p.peers = y_peers;
  p.k = k;
  p.gather = x != nullptr;
  p.cursor = cursor_out;
  p.progress = progress;
  p.seq = seq;
  p.w1 = (const __nv_bfloat16*)w1;
  {
    // L2 prefetch of the first wave's gate_up rows ahead of the dependency wait
    // (QMOE_SWAP_PREFETCH_KB = bytes per CTA / 1024).  Off by default: measured on the Qwen decode
    // layer (tools/qwen_layer_timeline.py 32, CUPTI) with 553 KB per CTA (~80 MB) the layer span
    // stays at 185-187 us while the router it overlaps slows from 10.8 to 12.9 us; the early
    // trigger of the router / permute kernels alone took the span from ~190 to ~186 us.
    static const int kb_env = [] {
      const char* v = getenv("QMOE_SWAP_PREFETCH_KB");
      return v == nullptr ? 0 : atoi(v);
    }();
    p.prefetch_bytes = kb_env > 0 ? kb_env * 1024 : 0;
  }
  const int nkb2 = (F + kBK - 1) / kBK;
  const int want = xp_rows <= kSwapRowsMax ? swap_splits(F) : 1;  // partials sized for <= 512 rows
  p.kb_per_split = (nkb2 + want - 1) / want;
  p.nsplit = (nkb2 + p.kb_per_split - 1) / p.kb_per_split;  // every split non-empty
  p.part = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + kFfnHeaderBytes);
  p.part_rows = xp_rows;
  if ((st = NT == 32 ? launch_swap<32>(maps, p, s)
                     : (NT == 64 ? launch_swap<64>(maps, p, s) : launch_swap<128>(maps, p, s))))
    return st;
  if (p.nsplit > 1) {
    const long long work = (long long)xp_rows * (d / 8);
    const int grid = (int)std::min<long long>((work + 255) / 256, 148 * 8);
    return launch_pdl("qmoe_expert_ffn(swap-AB split-K reduce)", swap_reduce_kernel, dim3(grid), dim3(256), 0, s,
                      (const float*)p.part, p.nsplit, xp_rows, d, perm, offsets, e_begin, (const int32_t*)&ws[0].stop,
                      (__nv_bfloat16*)y, y_peers);
  }
  return QMOE_OK;
}

}  // namespace qmoe
