// Grouped SwiGLU expert FFN with gate_up AND down in ONE persistent launch, 128 x 256 tcgen05
// tiles (1 CTA per SM) -- the mid-size-batch / fine-grained-expert path.
//
// Replaces the reference's per-expert drain (engine.py:204-215 -> model.py:141-145) for the
// north-star SwiGLU expert (HF MixtralExperts / Qwen2MoeExperts).
//
// The two-launch path (expert_tc.cu) ends the gate_up launch with a partial last wave, pays a
// launch + prologue, and ends the down launch with another partial wave.  Here one unit counter
// covers all gate_up tiles (expert-major, the reference's drain order) then all down tiles, and a
// down tile of expert e waits on a per-expert completion counter (release/acquire, then an
// async-proxy fence before TMA reads act) -- the protocol of the swap-AB kernel (expert_swap.cu),
// with token rows on the MMA's M side:
//   gate_up tile = (expert, 128 token rows, 128 F columns): B stacks the gate rows over the up rows
//                  of those columns, so accumulator columns [0,128) = gate, [128,256) = up and the
//                  epilogue writes SiLU(g)*u to act;
//   down tile    = (expert, 128 token rows, 256 output columns), rows scattered to token slots
//                  (or, expert parallel over peer memory, to the source rank's slot buffer).
// Preemption: the device flag is read by gate_up claimers (expert_common.cuh); down tiles run for
// exactly the experts below the stop.
#include <cudaTypedefs.h>

#include <stdlib.h>

#include "expert_common.cuh"
#include "tc_ptx.cuh"

namespace qmoe {
namespace {

constexpr int kBM = 128, kBN = 256, kBKf = 64;
constexpr int kStagesF = 4;
constexpr int kRingF = 4;
constexpr int kThreadsF = 256;
constexpr int kEpiF = 4;
constexpr int kABytesF = kBM * kBKf * 2;                 // 16 KB
constexpr int kStageBytesF = kABytesF + kBN * kBKf * 2;  // 48 KB
constexpr int kSmemF = kStagesF * kStageBytesF + 1024;

struct FusedParams {
  int d, F;
  int e_begin, e_end;
  const int32_t* offsets;
  const int32_t* perm;
  const volatile int32_t* flag;
  FfnWorkspace* ws;
  int* done;
  __nv_bfloat16* act;
  __nv_bfloat16* y;
  void* const* peers;
  int k;       // top-k: gate_up A rows are x[perm[r] / k] when gather != 0
  int gather;  // 1: gate_up A tiles are gathered from X by the producer warp (TMA tile::gather4)
  int32_t* cursor;  // optional cursor_out (written by the last CTA out, ffn_exit)
  int32_t* progress;  // optional host-mapped per-expert progress words (signal_expert_done)
  int seq;
  int merge;  // swap-AB pair: remainder rows (<= merge) folded into an expert's last token tile
  int x_first;  // 1-CTA kernel: experts >= x_first read their A rows straight from X (row m0 -
                // offsets[e]; Qwen's shared sub-experts, whose queues are X's rows in order)
};

// Token rows of one 128-row A tile for the gather: lane l owns rows [4l, 4l+4) of the tile; rows
// past the expert's queue read token 0 (their results are never stored).
__device__ __forceinline__ void gather_rows4(const FusedParams& p, int m0, int row_end, int lane, int (&g)[4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int r = m0 + 4 * lane + j;
    g[j] = r < row_end ? p.perm[r] / p.k : 0;
  }
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__global__ void __launch_bounds__(kThreadsF, 1)
ffn_fused_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW1,
                 const __grid_constant__ CUtensorMap tmAct, const __grid_constant__ CUtensorMap tmW2,
                 const __grid_constant__ CUtensorMap tmXd, FusedParams p) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kStagesF], empty_bar[kStagesF];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ __align__(8) uint64_t ring_full[kRingF], ring_empty[kRingF];
  __shared__ int ring_tile[kRingF];
  __shared__ uint32_t tmem_base_smem;
  __shared__ TileMap map1, map2;
  constexpr uint32_t kIdesc = ptx::idesc_bf16_f32(kBM, kBN);

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt1 = (p.F + kBN / 2 - 1) / (kBN / 2);  // 128 act columns per gate_up tile
  const int nt2 = (p.d + kBN - 1) / kBN;            // 256 output columns per down tile
  const int nkb1 = (p.d + kBKf - 1) / kBKf, nkb2 = (p.F + kBKf - 1) / kBKf;

  if (warp == 0) build_tile_map(map1, p.offsets, p.e_begin, p.e_end, nullptr, kBM, nt1);
  if (warp == 3) build_tile_map(map2, p.offsets, p.e_begin, p.e_end, nullptr, kBM, nt2);
  if (threadIdx.x == 32) {
    for (int s = 0; s < kStagesF; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull_bar[a], 1);
      ptx::mbar_init(&tempty_bar[a], 4);
    }
    for (int i = 0; i < kRingF; ++i) {
      ptx::mbar_init(&ring_full[i], 1);
      ptx::mbar_init(&ring_empty[i], 1 + 4);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<2 * kBN>(&tmem_base_smem);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = tmem_base_smem;
  const int N1 = map1.total, N2 = map2.total;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer (warp-wide:
    // lane 0 claims and issues the tile loads; in gather mode all 32 lanes issue tile::gather4)
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmX);
      ptx::tma_prefetch_desc(&tmW1);
      ptx::tma_prefetch_desc(&tmAct);
      ptx::tma_prefetch_desc(&tmW2);
    }
    int stage = 0, slot = 0, last_e = -1;
    uint32_t phase = 0, rphase = 0;
    int pending = lane == 0 ? atomicAdd(&p.ws->next, 1) : 0;  // claim one unit ahead
    while (true) {
      int t = -1;
      if (lane == 0) {
        while (true) {
          t = resolve_claim(map1, N2, p.ws, p.flag, last_e, pending);
          if (t >= N1) {
            int e2, m2, n2;
            map2.locate(t - N1, kBM, nt2, kBN, e2, m2, n2);
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
      if (++slot == kRingF) { slot = 0; rphase ^= 1; }
      if (t < 0) break;
      const bool up = t < N1;
      int e, m0, n0;
      if (up) map1.locate(t, kBM, nt1, kBN / 2, e, m0, n0);
      else map2.locate(t - N1, kBM, nt2, kBN, e, m0, n0);
      const bool gather = up && p.gather;
      int g[4] = {0, 0, 0, 0};
      if (gather) gather_rows4(p, m0, p.offsets[e + 1], lane, g);
      const bool direct = up && e >= p.x_first;  // A rows = X rows m0 - offsets[e] .. (never with gather)
      const CUtensorMap* ta = up ? (direct ? &tmXd : &tmX) : &tmAct;
      const int arow = direct ? m0 - p.offsets[e] : m0;
      const CUtensorMap* tb = up ? &tmW1 : &tmW2;
      // B rows: gate_up -> gate [n0, +128) over up F + [n0, +128); down -> [n0, +256)
      const int brow0 = up ? e * 2 * p.F + n0 : e * p.d + n0;
      const int brow1 = up ? brow0 + p.F : brow0 + kBN / 2;
      const int nkb = up ? nkb1 : nkb2;
      for (int kb = 0; kb < nkb; ++kb) {
        ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sa = smem + stage * kStageBytesF;
        if (lane == 0) {
          ptx::mbar_arrive_expect_tx(&full_bar[stage], kStageBytesF);
          if (!gather) ptx::tma_load_2d(ta, &full_bar[stage], sa, kb * kBKf, arow, ptx::kEvictNormal);
          ptx::tma_load_2d(tb, &full_bar[stage], sa + kABytesF, kb * kBKf, brow0, ptx::kEvictNormal);
          ptx::tma_load_2d(tb, &full_bar[stage], sa + kABytesF + (kBN / 2) * 128, kb * kBKf, brow1,
                           ptx::kEvictNormal);
        }
        if (gather)
          ptx::tma_gather4(&tmX, &full_bar[stage], sa + lane * 512, kb * kBKf, g[0], g[1], g[2], g[3],
                           ptx::kEvictNormal);
        if (++stage == kStagesF) { stage = 0; phase ^= 1; }
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
        if (++slot == kRingF) { slot = 0; rphase ^= 1; }
        if (t < 0) break;
        const int nkb = t < N1 ? nkb1 : nkb2;
        ptx::mbar_wait(&tempty_bar[acc], aphase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kBN;
        for (int kb = 0; kb < nkb; ++kb) {
          ptx::mbar_wait(&full_bar[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_addr = ptx::smem_u32(smem + stage * kStageBytesF);
          const uint32_t b_addr = a_addr + kABytesF;
#pragma unroll
          for (int k = 0; k < kBKf / 16; ++k)
            ptx::tc_mma_bf16(d_tmem, ptx::sw128_kmajor_desc(a_addr + k * 32), ptx::sw128_kmajor_desc(b_addr + k * 32),
                             kIdesc, (kb | k) != 0);
          ptx::tc_commit(&empty_bar[stage]);
          if (++stage == kStagesF) { stage = 0; phase ^= 1; }
        }
        ptx::tc_commit(&tfull_bar[acc]);
        if (++acc == 2) { acc = 0; aphase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp >= kEpiF) {
    // ------------------------------------------------------------------ epilogue
    const int ew = warp - kEpiF;  // TMEM lanes [32*ew, 32*ew+32) = token rows of the tile
    int slot = 0, acc = 0;
    uint32_t rphase = 0, aphase = 0;
    while (true) {
      ptx::mbar_wait(&ring_full[slot], rphase);
      const int t = ring_tile[slot];
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&ring_empty[slot]);
      if (++slot == kRingF) { slot = 0; rphase ^= 1; }
      if (t < 0) break;
      const bool up = t < N1;
      int e, m0, n0;
      if (up) map1.locate(t, kBM, nt1, kBN / 2, e, m0, n0);
      else map2.locate(t - N1, kBM, nt2, kBN, e, m0, n0);
      const int row = m0 + ew * 32 + lane;
      const bool valid = row < p.offsets[e + 1];
      __nv_bfloat16* dst = nullptr;
      if (valid) dst = up ? p.act + (size_t)row * p.F : out_row(p.y, p.peers, p.perm[row], p.d);
      const int ncols = up ? p.F : p.d;
      ptx::mbar_wait(&tfull_bar[acc], aphase);
      ptx::tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * kBN;
      const int out_cols = up ? kBN / 2 : kBN;
#pragma unroll 1
      for (int c = 0; c < out_cols; c += 32) {
        uint32_t v[32];
        uint32_t packed[16];
        ptx::tmem_ld32(t_row + c, v);
        if (up) {
          uint32_t u[32];
          ptx::tmem_ld32(t_row + kBN / 2 + c, u);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float g0 = __uint_as_float(v[2 * i]), g1 = __uint_as_float(v[2 * i + 1]);
            const float u0 = __uint_as_float(u[2 * i]), u1 = __uint_as_float(u[2 * i + 1]);
            packed[i] = pack2(g0 / (1.f + __expf(-g0)) * u0, g1 / (1.f + __expf(-g1)) * u1);
          }
        } else {
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) packed[i] = pack2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
        }
        if (valid && n0 + c < ncols) {
          uint4* d4 = reinterpret_cast<uint4*>(dst + n0 + c);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            d4[q] = make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) { acc = 0; aphase ^= 1; }
      if (up) {
        // publish this warp's act rows to the down tiles of expert e (read by TMA: async proxy)
        fence_proxy_async_global();
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(p.done + e, 1);
      } else if (p.progress != nullptr) {
        __syncwarp();
        if (lane == 0) signal_expert_done(p.done, e, map2.m_tiles[e - map2.e_first] * nt2 * 4, p.progress, p.seq);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) ffn_exit(p.ws, p.done, p.e_end, p.cursor, p.flag);
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<2 * kBN>(tmem_base);
  }
}

// ================================================================================================
// CTA-pair (cta_group::2) variant: 256 token rows x 256 B rows per tile, one tile per cluster of 2.
// Same protocol as ffn_tc2_kernel (expert_tc.cu): the leader claims tiles (two_phase_claim) and
// publishes them to both CTAs' rings over DSMEM, both CTAs' TMA loads complete on the leader's
// barrier, the leader issues tcgen05.mma.cta_group::2 with multicast commits.  A down tile of
// expert e is published only once the leader saw every gate_up tile of e complete (8 epilogue
// warps per pair tile arrive); the peer re-acquires the counter before its async-proxy fence.
constexpr int kStagesP = 6;
constexpr int kHalfP = 128 * kBKf * 2;  // 16 KB: this CTA's A rows, and separately its B rows
constexpr int kStageBytesP = 2 * kHalfP;
constexpr int kSmemP = kStagesP * kStageBytesP + 1024;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsF, 1)
ffn_fused_pair_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW1,
                      const __grid_constant__ CUtensorMap tmAct, const __grid_constant__ CUtensorMap tmW2,
                      FusedParams p) {
  pdl_wait();
  pdl_trigger();
  constexpr int kBMp = 256;
  constexpr uint32_t kIdesc = ptx::idesc_bf16_f32(kBMp, kBN);
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kStagesP], empty_bar[kStagesP];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ __align__(8) uint64_t ring_full[kRingF], ring_empty[kRingF];
  __shared__ int ring_tile[kRingF];
  __shared__ uint32_t tmem_base_smem;
  __shared__ TileMap map1, map2;

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int nt1 = (p.F + kBN / 2 - 1) / (kBN / 2), nt2 = (p.d + kBN - 1) / kBN;
  const int nkb1 = (p.d + kBKf - 1) / kBKf, nkb2 = (p.F + kBKf - 1) / kBKf;

  if (warp == 0) build_tile_map(map1, p.offsets, p.e_begin, p.e_end, nullptr, kBMp, nt1);
  if (warp == 3) build_tile_map(map2, p.offsets, p.e_begin, p.e_end, nullptr, kBMp, nt2);
  if (threadIdx.x == 32) {
    for (int s = 0; s < kStagesP; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull_bar[a], 1);
      ptx::mbar_init(&tempty_bar[a], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is used)
    }
    for (int i = 0; i < kRingF; ++i) {
      ptx::mbar_init(&ring_full[i], 1);
      ptx::mbar_init(&ring_empty[i], 10);  // leader: MMA + 4 epi; peer: producer + 4 epi
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc_cg2<2 * kBN>(&tmem_base_smem);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  __syncthreads();  // CTA-scope order for the allocator's smem write too (racecheck models this one)
  ptx::tc_fence_after();
  const uint32_t tmem_base = tmem_base_smem;
  const int N1 = map1.total, N2 = map2.total;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer (both CTAs,
    // warp-wide: lane 0 claims / receives tiles; in gather mode all lanes issue tile::gather4)
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmX);
      ptx::tma_prefetch_desc(&tmW1);
      ptx::tma_prefetch_desc(&tmAct);
      ptx::tma_prefetch_desc(&tmW2);
    }
    int stage = 0, slot = 0, last_e = -1;
    uint32_t phase = 0, rphase = 0;
    int pending = (lane == 0 && leader) ? atomicAdd(&p.ws->next, 1) : 0;  // claim one unit ahead
    while (true) {
      int t = -1;
      if (lane == 0) {
        if (leader) {
          while (true) {
            t = resolve_claim(map1, N2, p.ws, p.flag, last_e, pending);
            if (t >= N1) {
              int e2, m2, n2;
              map2.locate(t - N1, kBMp, nt2, kBN, e2, m2, n2);
              if (!expert_ready(p.done, e2, map1.m_tiles[e2 - map1.e_first] * nt1 * 8, p.ws)) {
                pending = atomicAdd(&p.ws->next, 1);
                continue;
              }
              fence_proxy_async_global();
            }
            break;
          }
          ptx::mbar_wait_cluster(&ring_empty[slot], rphase ^ 1);
          ring_tile[slot] = t;
          ptx::st_remote_u32(&ring_tile[slot], 1, (uint32_t)t);
          ptx::mbar_arrive(&ring_full[slot]);
          ptx::mbar_arrive_remote(&ring_full[slot], 1);
          if (t >= 0) pending = atomicAdd(&p.ws->next, 1);  // in flight while this unit's loads issue
        } else {
          ptx::mbar_wait_cluster(&ring_full[slot], rphase);
          t = ring_tile[slot];
          ptx::mbar_arrive_remote(&ring_empty[slot], 0);
          if (t >= N1) {
            int e2, m2, n2;
            map2.locate(t - N1, kBMp, nt2, kBN, e2, m2, n2);
            (void)ld_acquire(p.done + e2);  // the leader saw it complete; acquire it here too
            fence_proxy_async_global();
          }
        }
      }
      t = __shfl_sync(0xffffffffu, t, 0);
      if (++slot == kRingF) { slot = 0; rphase ^= 1; }
      if (t < 0) break;
      const bool up = t < N1;
      int e, m0, n0;
      if (up) map1.locate(t, kBMp, nt1, kBN / 2, e, m0, n0);
      else map2.locate(t - N1, kBMp, nt2, kBN, e, m0, n0);
      const bool gather = up && p.gather;
      int g[4] = {0, 0, 0, 0};
      if (gather) gather_rows4(p, m0 + (int)rank * 128, p.offsets[e + 1], lane, g);
      const CUtensorMap* ta = up ? &tmX : &tmAct;
      const CUtensorMap* tb = up ? &tmW1 : &tmW2;
      const int arow = m0 + (int)rank * 128;
      // this CTA's 128 B rows: gate_up -> CTA0 gate [n0, +128), CTA1 up F + [n0, +128);
      // down -> rows n0 + rank*128 of expert e
      const int brow = up ? e * 2 * p.F + (rank ? p.F : 0) + n0 : e * p.d + n0 + (int)rank * 128;
      const int nkb = up ? nkb1 : nkb2;
      for (int kb = 0; kb < nkb; ++kb) {
        ptx::mbar_wait_cluster(&empty_bar[stage], phase ^ 1);
        uint8_t* sa = smem + stage * kStageBytesP;
        if (lane == 0) {
          if (leader) ptx::mbar_arrive_expect_tx(&full_bar[stage], 2 * kStageBytesP);
          if (!gather) ptx::tma_load_2d_cg2(ta, &full_bar[stage], sa, kb * kBKf, arow, ptx::kEvictNormal);
          ptx::tma_load_2d_cg2(tb, &full_bar[stage], sa + kHalfP, kb * kBKf, brow, ptx::kEvictNormal);
        }
        if (gather)
          ptx::tma_gather4_cg2(&tmX, &full_bar[stage], sa + lane * 512, kb * kBKf, g[0], g[1], g[2], g[3],
                               ptx::kEvictNormal);
        if (++stage == kStagesP) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer (leader only)
    if (leader && lane == 0) {
      int stage = 0, slot = 0, acc = 0;
      uint32_t phase = 0, rphase = 0, aphase = 0;
      while (true) {
        ptx::mbar_wait_cluster(&ring_full[slot], rphase);
        const int t = ring_tile[slot];
        ptx::mbar_arrive(&ring_empty[slot]);
        if (++slot == kRingF) { slot = 0; rphase ^= 1; }
        if (t < 0) break;
        const int nkb = t < N1 ? nkb1 : nkb2;
        ptx::mbar_wait_cluster(&tempty_bar[acc], aphase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kBN;
        for (int kb = 0; kb < nkb; ++kb) {
          ptx::mbar_wait(&full_bar[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_addr = ptx::smem_u32(smem + stage * kStageBytesP);
          const uint32_t b_addr = a_addr + kHalfP;
#pragma unroll
          for (int k = 0; k < kBKf / 16; ++k)
            ptx::tc_mma_bf16_cg2(d_tmem, ptx::sw128_kmajor_desc(a_addr + k * 32),
                                 ptx::sw128_kmajor_desc(b_addr + k * 32), kIdesc, (kb | k) != 0);
          ptx::tc_commit_cg2(&empty_bar[stage], 0x3);
          if (++stage == kStagesP) { stage = 0; phase ^= 1; }
        }
        ptx::tc_commit_cg2(&tfull_bar[acc], 0x3);
        if (++acc == 2) { acc = 0; aphase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp >= kEpiF) {
    // ------------------------------------------------------------------ epilogue (both CTAs)
    const int ew = warp - kEpiF;
    int slot = 0, acc = 0;
    uint32_t rphase = 0, aphase = 0;
    while (true) {
      ptx::mbar_wait_cluster(&ring_full[slot], rphase);
      const int t = ring_tile[slot];
      __syncwarp();
      if (lane == 0) {
        if (leader) ptx::mbar_arrive(&ring_empty[slot]);
        else ptx::mbar_arrive_remote(&ring_empty[slot], 0);
      }
      if (++slot == kRingF) { slot = 0; rphase ^= 1; }
      if (t < 0) break;
      const bool up = t < N1;
      int e, m0, n0;
      if (up) map1.locate(t, kBMp, nt1, kBN / 2, e, m0, n0);
      else map2.locate(t - N1, kBMp, nt2, kBN, e, m0, n0);
      const int row = m0 + (int)rank * 128 + ew * 32 + lane;
      const bool valid = row < p.offsets[e + 1];
      __nv_bfloat16* dst = nullptr;
      if (valid) dst = up ? p.act + (size_t)row * p.F : out_row(p.y, p.peers, p.perm[row], p.d);
      const int ncols = up ? p.F : p.d;
      ptx::mbar_wait_cluster(&tfull_bar[acc], aphase);
      ptx::tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * kBN;
      const int out_cols = up ? kBN / 2 : kBN;
#pragma unroll 1
      for (int c = 0; c < out_cols; c += 32) {
        uint32_t v[32];
        uint32_t packed[16];
        ptx::tmem_ld32(t_row + c, v);
        if (up) {
          uint32_t u[32];
          ptx::tmem_ld32(t_row + kBN / 2 + c, u);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float g0 = __uint_as_float(v[2 * i]), g1 = __uint_as_float(v[2 * i + 1]);
            const float u0 = __uint_as_float(u[2 * i]), u1 = __uint_as_float(u[2 * i + 1]);
            packed[i] = pack2(g0 / (1.f + __expf(-g0)) * u0, g1 / (1.f + __expf(-g1)) * u1);
          }
        } else {
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) packed[i] = pack2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
        }
        if (valid && n0 + c < ncols) {
          uint4* d4 = reinterpret_cast<uint4*>(dst + n0 + c);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            d4[q] = make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) ptx::mbar_arrive(&tempty_bar[acc]);
        else ptx::mbar_arrive_remote(&tempty_bar[acc], 0);
      }
      if (++acc == 2) { acc = 0; aphase ^= 1; }
      if (up) {
        fence_proxy_async_global();
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(p.done + e, 1);
      } else if (p.progress != nullptr) {
        __syncwarp();  // both CTAs' 4 epilogue warps store part of every pair tile
        if (lane == 0) signal_expert_done(p.done, e, map2.m_tiles[e - map2.e_first] * nt2 * 8, p.progress, p.seq);
      }
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (threadIdx.x == 0) ffn_exit(p.ws, p.done, p.e_end, p.cursor, p.flag);
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_cg2<2 * kBN>(tmem_base);
  }
}

// ================================================================================================
// Swap-AB CTA pair (cta_group::2): WEIGHT rows on the MMA's M side (256 per unit, 128 per CTA),
// token rows on N, N = the unit's valid token rows rounded up to 16 (<= 256; each CTA supplies
// N/2 token rows).  For fine-grained experts (Qwen: ~270 rows per expert at 4k tokens) the
// token-row padding of a 256-row M tile (the pair kernel above) or a 128-row one (the 1-CTA
// kernel) wastes 30-50% of the tensor work; here it is < 16 rows per token tile, at the pair's
// operand traffic (each SM stages 128 weight rows + N/2 token rows per K block).
//   gate_up unit = (expert, 128 F columns f0, <= 256 tokens): CTA c stages gate rows
//                  f0 + 64c + [0, 64) over up rows F + f0 + 64c + [0, 64), so its TMEM lanes
//                  [0, 64) hold gate and [64, 128) the matching up rows; the up warps hand their
//                  rows to the gate warps through shared memory for SiLU(g) * u;
//   down unit    = (expert, 256 d columns, <= 256 tokens), CTA c owns d columns + 128c.
// Same claim / ring / completion-counter / preemption protocol as ffn_fused_pair_kernel.
// Wide last tile (QMOE_SP_MERGE=n, off by default, see expert_ffn_swap_pair): an expert whose rows
// leave a remainder of <= p.merge rows after its full
// 256-row tiles runs that remainder in the same unit as its last full tile (up to 256 + merge
// token rows): the unit streams its weight rows ONCE and multiplies them into both TMEM
// accumulators (the first 256 tokens and the remainder), taking two ring stages per K block (the
// second holds only the remainder's token rows) and two accumulator turns.  Without it a
// remainder of a few rows costs a whole extra pass over the expert's weights (Mixtral ~1k tokens:
// about half the experts hold 257-300 rows).  Per-token results are unchanged (same K order per
// accumulator).
constexpr int kStagesSP = 6;
constexpr int kTokSP = 256;                     // token rows per unit
constexpr int kHalfSP = 128 * kBKf * 2;         // 16 KB: this CTA's weight rows, then its token rows
constexpr int kStageBytesSP = 2 * kHalfSP;
constexpr int kSmemSP = kStagesSP * kStageBytesSP + 1024;

__device__ __forceinline__ int sp_ncols(int rows) { return rows < 16 ? 16 : (rows + 15) & ~15; }

// Token-row boxes of 32 / 64 / 128 rows: a CTA stages the smallest box holding its N/2 rows, so a
// short token tile (an expert's remainder rows) does not pay a full 128-row operand load.
struct alignas(64) SpMaps {
  CUtensorMap tok[2][3];  // [Xp (or X for tile::gather4), act][box 32, 64, 128]
  CUtensorMap w1, w2;     // 64-row gate / up boxes, 128-row down boxes
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsF, 1)
ffn_swap_pair_kernel(const __grid_constant__ SpMaps maps, FusedParams p) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kStagesSP], empty_bar[kStagesSP];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ __align__(8) uint64_t ring_full[kRingF], ring_empty[kRingF];
  __shared__ int ring_tile[kRingF];
  __shared__ uint32_t tmem_base_smem;
  __shared__ TileMap map1, map2;
  // gate <-> up halves of a 32-token chunk ([0] gate, [1] up; warp pairs 0/2, 1/3), float4 rows of
  // 20 floats (conflict-free 16-byte accesses); per-warp staging tiles of 32 token rows x 32
  // columns (64-byte rows: the two rows of a paired 32-bit store land 16 banks apart)
  __shared__ __align__(16) float sp_x[2][2][32][20];
  __shared__ __align__(16) __nv_bfloat16 sp_w[4][32][32];

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int nt1 = (p.F + 127) / 128, nt2 = (p.d + 255) / 256;
  const int nkb1 = (p.d + kBKf - 1) / kBKf, nkb2 = (p.F + kBKf - 1) / kBKf;

  if (warp == 0) build_tile_map(map1, p.offsets, p.e_begin, p.e_end, nullptr, kTokSP, nt1, p.merge);
  if (warp == 3) build_tile_map(map2, p.offsets, p.e_begin, p.e_end, nullptr, kTokSP, nt2, p.merge);
  // token rows of the unit starting at row m0 of an expert ending at row_end: a full tile, or the
  // last (possibly wide) one
  auto unit_rows = [&](int m0, int row_end) {
    const int r = row_end - m0;
    return r > kTokSP + p.merge ? kTokSP : r;
  };
  if (threadIdx.x == 32) {
    for (int s = 0; s < kStagesSP; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull_bar[a], 1);
      ptx::mbar_init(&tempty_bar[a], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is used)
    }
    for (int i = 0; i < kRingF; ++i) {
      ptx::mbar_init(&ring_full[i], 1);
      ptx::mbar_init(&ring_empty[i], 10);  // leader: MMA + 4 epi; peer: producer + 4 epi
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc_cg2<2 * kTokSP>(&tmem_base_smem);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = tmem_base_smem;
  const int N1 = map1.total, N2 = map2.total;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      for (int i = 0; i < 6; ++i) ptx::tma_prefetch_desc(&maps.tok[i / 3][i % 3]);
      ptx::tma_prefetch_desc(&maps.w1);
      ptx::tma_prefetch_desc(&maps.w2);
    }
    int stage = 0, slot = 0, last_e = -1;
    uint32_t phase = 0, rphase = 0;
    int pending = (lane == 0 && leader) ? atomicAdd(&p.ws->next, 1) : 0;  // claim one unit ahead
    while (true) {
      int t = -1;
      if (lane == 0) {
        if (leader) {
          while (true) {
            t = resolve_claim(map1, N2, p.ws, p.flag, last_e, pending);
            if (t >= N1) {
              int e2, m2, n2;
              map2.locate(t - N1, kTokSP, nt2, 256, e2, m2, n2);
              if (!expert_ready(p.done, e2, map1.m_tiles[e2 - map1.e_first] * nt1 * 8, p.ws)) {
                pending = atomicAdd(&p.ws->next, 1);
                continue;
              }
              fence_proxy_async_global();
            }
            break;
          }
          ptx::mbar_wait_cluster(&ring_empty[slot], rphase ^ 1);
          ring_tile[slot] = t;
          ptx::st_remote_u32(&ring_tile[slot], 1, (uint32_t)t);
          ptx::mbar_arrive(&ring_full[slot]);
          ptx::mbar_arrive_remote(&ring_full[slot], 1);
          if (t >= 0) pending = atomicAdd(&p.ws->next, 1);
        } else {
          ptx::mbar_wait_cluster(&ring_full[slot], rphase);
          t = ring_tile[slot];
          ptx::mbar_arrive_remote(&ring_empty[slot], 0);
          if (t >= N1) {
            int e2, m2, n2;
            map2.locate(t - N1, kTokSP, nt2, 256, e2, m2, n2);
            (void)ld_acquire(p.done + e2);  // the leader saw it complete; acquire it here too
            fence_proxy_async_global();
          }
        }
      }
      t = __shfl_sync(0xffffffffu, t, 0);
      if (++slot == kRingF) { slot = 0; rphase ^= 1; }
      if (t < 0) break;
      const bool up = t < N1;
      int e, m0, n0;
      if (up) map1.locate(t, kTokSP, nt1, 128, e, m0, n0);
      else map2.locate(t - N1, kTokSP, nt2, 256, e, m0, n0);
      const int row_end = p.offsets[e + 1];
      const int rows = unit_rows(m0, row_end);
      const bool wide = rows > kTokSP;  // (never with gather: the host sets merge = 0 then)
      const int half = sp_ncols(min(kTokSP, rows)) >> 1;
      const int tok = m0 + (int)rank * half;  // this CTA's N/2 token rows
      const int bi = half <= 32 ? 0 : (half <= 64 ? 1 : 2);
      const int box = 32 << bi;
      const CUtensorMap* tm = &maps.tok[up ? 0 : 1][up && p.gather ? 0 : bi];
      // the wide unit's remainder: token rows [m0 + 256, m0 + rows), N2/2 per CTA
      const int half2 = wide ? sp_ncols(rows - kTokSP) >> 1 : 0;
      const int bi2 = half2 <= 32 ? 0 : (half2 <= 64 ? 1 : 2);
      const int box2 = 32 << bi2;
      const CUtensorMap* tm2 = &maps.tok[up ? 0 : 1][bi2];
      const int tok2 = m0 + kTokSP + (int)rank * half2;
      const bool gather = up && p.gather;
      int g[4] = {0, 0, 0, 0};
      if (gather) gather_rows4(p, tok, row_end, lane, g);
      const int wrow = up ? e * 2 * p.F + n0 + (int)rank * 64 : e * p.d + n0 + (int)rank * 128;
      const int nkb = up ? nkb1 : nkb2;
      for (int kb = 0; kb < nkb; ++kb) {
        ptx::mbar_wait_cluster(&empty_bar[stage], phase ^ 1);
        uint8_t* sa = smem + stage * kStageBytesSP;
        if (lane == 0) {
          if (leader) ptx::mbar_arrive_expect_tx(&full_bar[stage], 2 * (kHalfSP + box * kBKf * 2));
          if (up) {  // 64 gate rows over the 64 matching up rows
            ptx::tma_load_2d_cg2(&maps.w1, &full_bar[stage], sa, kb * kBKf, wrow, ptx::kEvictNormal);
            ptx::tma_load_2d_cg2(&maps.w1, &full_bar[stage], sa + kHalfSP / 2, kb * kBKf, wrow + p.F, ptx::kEvictNormal);
          } else {
            ptx::tma_load_2d_cg2(&maps.w2, &full_bar[stage], sa, kb * kBKf, wrow, ptx::kEvictNormal);
          }
          if (!gather) ptx::tma_load_2d_cg2(tm, &full_bar[stage], sa + kHalfSP, kb * kBKf, tok, ptx::kEvictNormal);
        }
        if (gather && lane < box / 4)
          ptx::tma_gather4_cg2(tm, &full_bar[stage], sa + kHalfSP + lane * 512, kb * kBKf, g[0], g[1], g[2], g[3],
                               ptx::kEvictNormal);
        if (++stage == kStagesSP) { stage = 0; phase ^= 1; }
        if (wide) {  // next stage: the remainder's token rows only (its weight half stays unused)
          ptx::mbar_wait_cluster(&empty_bar[stage], phase ^ 1);
          uint8_t* sb = smem + stage * kStageBytesSP;
          if (lane == 0) {
            if (leader) ptx::mbar_arrive_expect_tx(&full_bar[stage], 2 * (box2 * kBKf * 2));
            ptx::tma_load_2d_cg2(tm2, &full_bar[stage], sb + kHalfSP, kb * kBKf, tok2, ptx::kEvictNormal);
          }
          if (++stage == kStagesSP) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer (leader only)
    if (leader && lane == 0) {
      int stage = 0, slot = 0, acc = 0;
      uint32_t phase = 0, rphase = 0, aphase = 0;
      while (true) {
        ptx::mbar_wait_cluster(&ring_full[slot], rphase);
        const int t = ring_tile[slot];
        ptx::mbar_arrive(&ring_empty[slot]);
        if (++slot == kRingF) { slot = 0; rphase ^= 1; }
        if (t < 0) break;
        int e, m0, n0;
        if (t < N1) map1.locate(t, kTokSP, nt1, 128, e, m0, n0);
        else map2.locate(t - N1, kTokSP, nt2, 256, e, m0, n0);
        const int rows = unit_rows(m0, p.offsets[e + 1]);
        const bool wide = rows > kTokSP;
        const uint32_t idesc = ptx::idesc_bf16_f32(256, sp_ncols(min(kTokSP, rows)));
        const uint32_t idesc2 = wide ? ptx::idesc_bf16_f32(256, sp_ncols(rows - kTokSP)) : 0u;
        const int nkb = t < N1 ? nkb1 : nkb2;
        // accumulator turn(s): a wide unit takes this turn and the next one
        const int acc2 = acc ^ 1;
        const uint32_t aphase2 = acc2 == 0 ? aphase ^ 1 : aphase;
        ptx::mbar_wait_cluster(&tempty_bar[acc], aphase ^ 1);
        if (wide) ptx::mbar_wait_cluster(&tempty_bar[acc2], aphase2 ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kTokSP;
        const uint32_t d_tmem2 = tmem_base + acc2 * kTokSP;
        for (int kb = 0; kb < nkb; ++kb) {
          ptx::mbar_wait(&full_bar[stage], phase);
          ptx::tc_fence_after();
          const int stage_a = stage;
          const uint32_t a_addr = ptx::smem_u32(smem + stage * kStageBytesSP);
          const uint32_t b_addr = a_addr + kHalfSP;
#pragma unroll
          for (int k = 0; k < kBKf / 16; ++k)
            ptx::tc_mma_bf16_cg2(d_tmem, ptx::sw128_kmajor_desc(a_addr + k * 32),
                                 ptx::sw128_kmajor_desc(b_addr + k * 32), idesc, (kb | k) != 0);
          if (++stage == kStagesSP) { stage = 0; phase ^= 1; }
          if (wide) {
            ptx::mbar_wait(&full_bar[stage], phase);
            ptx::tc_fence_after();
            const uint32_t b2_addr = ptx::smem_u32(smem + stage * kStageBytesSP) + kHalfSP;
#pragma unroll
            for (int k = 0; k < kBKf / 16; ++k)
              ptx::tc_mma_bf16_cg2(d_tmem2, ptx::sw128_kmajor_desc(a_addr + k * 32),
                                   ptx::sw128_kmajor_desc(b2_addr + k * 32), idesc2, (kb | k) != 0);
            ptx::tc_commit_cg2(&empty_bar[stage], 0x3);
            if (++stage == kStagesSP) { stage = 0; phase ^= 1; }
          }
          ptx::tc_commit_cg2(&empty_bar[stage_a], 0x3);  // after the MMAs reading its weights
        }
        ptx::tc_commit_cg2(&tfull_bar[acc], 0x3);
        if (++acc == 2) { acc = 0; aphase ^= 1; }
        if (wide) {
          ptx::tc_commit_cg2(&tfull_bar[acc], 0x3);
          if (++acc == 2) { acc = 0; aphase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp >= kEpiF) {
    // ------------------------------------------------------------------ epilogue (both CTAs)
    // Thread (ew, lane) owns TMEM lane 32 ew + lane = one weight row, columns = the unit's tokens.
    const int ew = warp - kEpiF;
    int slot = 0, acc = 0;
    uint32_t rphase = 0, aphase = 0;
    while (true) {
      ptx::mbar_wait_cluster(&ring_full[slot], rphase);
      const int t = ring_tile[slot];
      __syncwarp();
      if (lane == 0) {
        if (leader) ptx::mbar_arrive(&ring_empty[slot]);
        else ptx::mbar_arrive_remote(&ring_empty[slot], 0);
      }
      if (++slot == kRingF) { slot = 0; rphase ^= 1; }
      if (t < 0) break;
      const bool up = t < N1;
      int e, m0, n0;
      if (up) map1.locate(t, kTokSP, nt1, 128, e, m0, n0);
      else map2.locate(t - N1, kTokSP, nt2, 256, e, m0, n0);
      const int unit = unit_rows(m0, p.offsets[e + 1]);  // uniform over the CTA
      const int m_unit = m0;
#pragma unroll 1
      for (int sub = 0; sub < (unit > kTokSP ? 2 : 1); ++sub) {  // a wide unit's two accumulators
        const int m0 = m_unit + sub * kTokSP;
        const int rows = sub ? unit - kTokSP : min(kTokSP, unit);
        ptx::mbar_wait_cluster(&tfull_bar[acc], aphase);
        ptx::tc_fence_after();
        const uint32_t t_row = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * kTokSP;
        __nv_bfloat16 (*stg)[32] = sp_w[ew];  // this warp's staging tile (token rows x 32 columns)
#pragma unroll 1
        for (int c = 0; c < rows; c += 32) {
          uint32_t v[32];
          ptx::tmem_ld32(t_row + c, v);
          ptx::tmem_ld_wait();
          if (up) {
            // warp pair q = ew & 1 holds gate (ew = q) and up (ew = q + 2) of the same 32 features:
            // the gate warp finishes tokens [0, 16) of the chunk, the up warp tokens [16, 32); the
            // halves cross through shared memory under a barrier of the pair only
            const int q = ew & 1;
            const bool gate = ew < 2;
            float4* xs = reinterpret_cast<float4*>(&sp_x[gate ? 0 : 1][q][lane][0]);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              float e4[4];
#pragma unroll
              for (int c4 = 0; c4 < 4; ++c4) e4[c4] = __uint_as_float(gate ? v[16 + 4 * i + c4] : v[4 * i + c4]);
              xs[i] = make_float4(e4[0], e4[1], e4[2], e4[3]);
            }
            asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
            const float4* xr = reinterpret_cast<const float4*>(&sp_x[gate ? 1 : 0][q][lane][0]);
            float h[16];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float4 t4 = xr[i];
              const float tv[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
              for (int c4 = 0; c4 < 4; ++c4) {
                const int j = 4 * i + c4;
                const float gv = gate ? __uint_as_float(v[j]) : tv[c4];
                const float uv = gate ? tv[c4] : __uint_as_float(v[16 + j]);
                h[j] = gv / (1.f + __expf(-gv)) * uv;
              }
            }
            asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");  // sp_x is rewritten by the next chunk
            // transpose through the warp's staging tile: lane pairs (2m, 2m+1) swap one value per
            // token pair so each lane stores one 32-bit word (rows j, j+1 land 16 banks apart)
#pragma unroll
            for (int j = 0; j < 16; j += 2) {
              const float recv = __shfl_xor_sync(0xffffffffu, (lane & 1) ? h[j] : h[j + 1], 1);
              *reinterpret_cast<uint32_t*>(&stg[j + (lane & 1)][lane & ~1]) =
                  (lane & 1) ? pack2(recv, h[j + 1]) : pack2(h[j], recv);
            }
            __syncwarp();
            // 16 token rows x 32 features (64 B) of act, 16-byte stores
            const int t0 = c + (gate ? 0 : 16);
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int idx = lane + 32 * i, r = idx >> 2, vq = idx & 3;
              if (t0 + r < rows)
                *reinterpret_cast<uint4*>(p.act + (size_t)(m0 + t0 + r) * p.F + n0 + (int)rank * 64 + 32 * q + 8 * vq) =
                    *reinterpret_cast<const uint4*>(&stg[r][8 * vq]);
            }
          } else {
            const int pr = c + lane < rows ? p.perm[m0 + c + lane] : 0;  // slot of token c + lane
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              const float a0 = __uint_as_float(v[j]), a1 = __uint_as_float(v[j + 1]);
              const float recv = __shfl_xor_sync(0xffffffffu, (lane & 1) ? a0 : a1, 1);
              *reinterpret_cast<uint32_t*>(&stg[j + (lane & 1)][lane & ~1]) = (lane & 1) ? pack2(recv, a1) : pack2(a0, recv);
            }
            __syncwarp();
            // 32 token rows x 32 output columns (64 B) scattered to the token slots, 16-byte stores
            const int col = n0 + (int)rank * 128 + 32 * ew;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int idx = lane + 32 * i, r = idx >> 2, vq = idx & 3;
              const int slot = __shfl_sync(0xffffffffu, pr, r);
              if (c + r < rows)
                *reinterpret_cast<uint4*>(out_row(p.y, p.peers, slot, p.d) + col + 8 * vq) =
                    *reinterpret_cast<const uint4*>(&stg[r][8 * vq]);
            }
          }
          __syncwarp();  // the staging tile is rewritten by the next chunk
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (leader) ptx::mbar_arrive(&tempty_bar[acc]);
          else ptx::mbar_arrive_remote(&tempty_bar[acc], 0);
        }
        if (++acc == 2) { acc = 0; aphase ^= 1; }
      }
      if (up) {
        fence_proxy_async_global();
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(p.done + e, 1);
      } else if (p.progress != nullptr) {
        __syncwarp();  // both CTAs' 4 epilogue warps store part of every pair tile
        if (lane == 0) signal_expert_done(p.done, e, map2.m_tiles[e - map2.e_first] * nt2 * 8, p.progress, p.seq);
      }
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (threadIdx.x == 0) ffn_exit(p.ws, p.done, p.e_end, p.cursor, p.flag);
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_cg2<2 * kTokSP>(tmem_base);
  }
}

}  // namespace

// The single-launch path for the 1-CTA tile shape (mid-size batches and fine-grained experts);
// QMOE_FUSED=0/1 forces it off/on (tests compare the paths).
bool use_fused_tc() {
  static int forced = [] {
    const char* v = getenv("QMOE_FUSED");
    return v == nullptr ? -1 : atoi(v);
  }();
  return forced != 0;
}

int expert_ffn_fused(const void* xp, const int32_t* offsets, const int32_t* perm, int E, int d, int F,
                     const void* w1, const void* w2, int e_begin, int e_end, void* act_ws, void* y,
                     const volatile int32_t* flag, int32_t* cursor_out, FfnWorkspace* ws, int xp_rows,
                     void* const* y_peers, bool pair, const void* x, int T, int k, cudaStream_t s,
                     int32_t* progress, int seq, const void* x_direct, int x_first) {
  int st;
  CUtensorMap maps[5];
  QMOE_REQUIRE(x_direct == nullptr || (!pair && x == nullptr), "qmoe_expert_ffn_xs: direct-X rows need the 1-CTA tiles");
  if (x_direct != nullptr && (st = tc_make_map(&maps[4], x_direct, T, d, kBM))) return st;
  // A boxes: 128 token rows (each CTA of a pair loads its own 128), or single rows of X for the
  // tile::gather4 loads (x != nullptr); B boxes: 128 weight rows
  if ((st = x != nullptr ? tc_make_map(&maps[0], x, T, d, 1) : tc_make_map(&maps[0], xp, xp_rows, d, kBM)) ||
      (st = tc_make_map(&maps[1], w1, (uint64_t)E * 2 * F, d, kBN / 2)) ||
      (st = tc_make_map(&maps[2], act_ws, xp_rows, F, kBM)) ||
      (st = tc_make_map(&maps[3], w2, (uint64_t)E * d, F, kBN / 2)))
    return st;
  FusedParams p{};
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
  p.x_first = x_direct != nullptr ? x_first : INT_MAX;
  if (x_direct == nullptr) maps[4] = maps[0];  // unused
  static uint64_t attr_set = 0;  // devices already configured
  if (!(attr_set & current_device_bit())) {
    QMOE_CUDA_TRY(cudaFuncSetAttribute(ffn_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemF));
    QMOE_CUDA_TRY(cudaFuncSetAttribute(ffn_fused_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemP));
    attr_set |= current_device_bit();
  }
  if (pair)
    return launch_pdl("qmoe_expert_ffn(tcgen05 single launch, pair)", ffn_fused_pair_kernel,
                      dim3((tc_num_sms() / 2) * 2), dim3(kThreadsF), kSmemP, s, maps[0], maps[1], maps[2], maps[3], p);
  return launch_pdl("qmoe_expert_ffn(tcgen05 single launch)", ffn_fused_kernel, dim3(tc_num_sms()), dim3(kThreadsF),
                    kSmemF, s, maps[0], maps[1], maps[2], maps[3], maps[4], p);
}

// Batches past the swap-AB range (checked first) of coarse experts: the swap-AB CTA-pair kernel,
// whose token tiles pad to 16 rows instead of 256.  Same-box eager A/B on B200 (tools/ffn_ab.py,
// FFN alone, L2 flushed): Mixtral 768/1k/2k tokens 0.54/0.72/1.18 ms vs 0.58/0.80/1.25 on the
// 256-row pair tiles, tied (+-2%) at 4k-16k.  Fine-grained experts (Qwen, 60 experts) lose 3-10%
// at 1.5k-16k tokens except at 2k (+6%), and a single expert (Qwen's shared expert) loses 5-9%
// (the transposing epilogue, DESIGN 2.3b), so the path is used for 4..16 experts, and for more
// experts only where the token-row tiles would pad by > 30%.  QMOE_SWAP_PAIR=0/1 forces it off/on (when
// the shape allows it: d % 256 == 0, F % 128 == 0).
bool use_swap_pair(int xp_rows, int n_experts, int d, int F) {
  static int forced = [] {
    const char* v = getenv("QMOE_SWAP_PAIR");
    return v == nullptr ? -1 : atoi(v);
  }();
  if (d % 256 != 0 || F % 128 != 0 || n_experts < 1 || n_experts > kFfnMaxExperts) return false;
  if (forced >= 0) return forced == 1;
  if (n_experts >= 4 && n_experts <= 16) return true;
  // one to three experts (Qwen's shared expert) up to 256 rows: the alternative is the two-launch
  // split-K path (0.057 / 0.061 / 0.070 ms vs 0.084 / 0.071 / 0.073 at 96 / 128 / 256 tokens;
  // behind from 384)
  if (n_experts < 4) return xp_rows <= 256;
  // fine-grained experts: only where the 128-row token tiles would waste > 30% of the tensor
  // work on padding (mean rows per expert just above a multiple of 128: Qwen 2k tokens, ~137
  // rows, 0.22 vs 0.23 ms); elsewhere the token-row tiles are 3-10% faster (epilogue, §2.3b)
  const double rows = (double)xp_rows / n_experts;
  const double padded = 128.0 * (double)(long long)((rows + 127.0) / 128.0);
  return rows > 128.0 && rows / padded < 0.7;
}

int expert_ffn_swap_pair(const void* xp, const int32_t* offsets, const int32_t* perm, int E, int d, int F,
                         const void* w1, const void* w2, int e_begin, int e_end, void* act_ws, void* y,
                         const volatile int32_t* flag, int32_t* cursor_out, FfnWorkspace* ws, int xp_rows,
                         void* const* y_peers, const void* x, int T, int k, cudaStream_t s,
                         int32_t* progress, int seq) {
  int st;
  SpMaps maps;
  // tokens: 32/64/128-row boxes of Xp / act (each CTA loads its N/2 rows from the box start), or
  // single rows of X for tile::gather4; weights: 64-row gate / up boxes, 128-row down boxes
  for (int b = 0; b < 3; ++b) {
    if ((st = x != nullptr ? tc_make_map(&maps.tok[0][b], x, T, d, 1)
                           : tc_make_map(&maps.tok[0][b], xp, xp_rows, d, 32 << b)) ||
        (st = tc_make_map(&maps.tok[1][b], act_ws, xp_rows, F, 32 << b)))
      return st;
  }
  if ((st = tc_make_map(&maps.w1, w1, (uint64_t)E * 2 * F, d, 64)) ||
      (st = tc_make_map(&maps.w2, w2, (uint64_t)E * d, F, 128)))
    return st;
  FusedParams p{};
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
  // remainder rows folded into an expert's last token tile (wide unit): off by default.  Same-box
  // A/B (profiles/ffn_wide_ab_r02.json, FFN alone, L2 flushed): QMOE_SP_MERGE=128 is 7-12% faster
  // where experts hold 270-320 rows (Mixtral 1.1-1.3k tokens) but 2-9% slower at 1k, 2k, 3k and
  // 16k tokens -- consecutive wide units cannot overlap one unit's epilogue with the next unit's
  // MMAs (both TMEM accumulators busy), which costs more than the saved weight pass.
  static const int merge_env = [] {
    const char* v = getenv("QMOE_SP_MERGE");
    return v == nullptr ? 0 : atoi(v);
  }();
  p.merge = p.gather ? 0 : std::max(0, std::min(merge_env, kTokSP));
  static uint64_t attr_set = 0;  // devices already configured
  if (!(attr_set & current_device_bit())) {
    QMOE_CUDA_TRY(cudaFuncSetAttribute(ffn_swap_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemSP));
    attr_set |= current_device_bit();
  }
  return launch_pdl("qmoe_expert_ffn(tcgen05 swap-AB pair)", ffn_swap_pair_kernel, dim3((tc_num_sms() / 2) * 2),
                    dim3(kThreadsF), kSmemSP, s, maps, p);
}

}  // namespace qmoe
