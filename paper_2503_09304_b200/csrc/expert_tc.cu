// Grouped expert FFN on 5th-gen tensor cores (tcgen05 + TMEM), TMA-fed, persistent and
// warp-specialised — the production bf16 path of qmoe_expert_ffn.
//
// Replaces the reference's per-expert drain (engine.py:204-215 → model.py:141-145) and, for the
// north-star SwiGLU expert, HF MixtralExperts.forward (gate_up → SiLU(g)*u → down).
//
// One CTA per SM, 256 threads:
//   warp 0  TMA producer: claims tiles (expert-major, device preempt flag checked at each claim),
//           streams A (gathered token rows) and B (expert weights) 128x64 / BNx64 bf16 tiles into
//           a kStages-deep 128B-swizzled smem ring (mbarrier complete_tx).
//   warp 1  MMA issuer: one thread issues tcgen05.mma.cta_group::1.kind::f16 (M=128, N=BN, K=16)
//           into a double-buffered fp32 TMEM accumulator (2 x BN columns of 512).
//   warp 2  TMEM allocator.
//   warps 4-7 epilogue: tcgen05.ld 32 lanes x 32 columns, fused SiLU(g)*u / bias+tanh / plain,
//           bf16 pack, 16-byte stores to act rows (expert order) or Y slot rows (perm scatter).
// The TMEM double buffer lets the epilogue of tile i overlap the MMAs of tile i+1.
#include <cudaTypedefs.h>

#include <stdlib.h>

#include <cmath>

#include <mutex>

#include "expert_common.cuh"
#include "tc_ptx.cuh"

namespace qmoe {
namespace {

constexpr int BM = 128, BK = 64;
constexpr int kStages = 4;
constexpr int kAccStages = 2;
constexpr int kTileRing = 4;
constexpr int kThreads = 256;
constexpr int kEpiWarp0 = 4;

enum { EPI_TANH = 0, EPI_SWIGLU = 1, EPI_DOWN = 2, EPI_DOWN_PART = 3 };

// Small-batch down projection: split the K loop so a launch with few (expert, N-block) tiles
// still spreads over every SM.  Partials are fp32 [split][row][N], reduced in fixed split order
// (deterministic) by splitk_reduce_kernel, which also scatters rows to their token slots.
constexpr int kMaxSplit = 8;
constexpr int kSplitRowsMax = 512;
}  // namespace
int down_splits(int xp_rows, int n_experts, int d, int F);
float* splitk_buffer(FfnWorkspace* ws);
bool use_cta_pair(int xp_rows, int n_experts);
namespace {

struct TcParams {
  int N;         // output columns of this GEMM (act columns F for the SwiGLU gate_up pass)
  int K;         // reduction length
  int b_rows;    // rows of the B operand per expert (N, or 2F for gate_up)
  int e_begin, e_end;
  const int32_t* offsets;
  const int32_t* perm;
  const int32_t* e_limit;
  const __nv_bfloat16* bias;  // [E, N] for the tanh expert
  __nv_bfloat16* out;
  int out_ld;
  const volatile int32_t* flag;
  FfnWorkspace* ws;
  int nsplit;         // K splits per (M, N) tile (EPI_DOWN_PART), else 1
  int kb_per_split;
  float* part;        // [nsplit][part_rows][N] fp32 partials
  int part_rows;
  void* const* peers;  // down projection: per-rank slot buffers (expert parallel over peer memory)
};

template <int BN>
constexpr int stage_bytes() { return BM * BK * 2 + BN * BK * 2; }
template <int BN>
constexpr int smem_bytes() { return kStages * stage_bytes<BN>() + 1024; }

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <int BN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
ffn_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages];
  __shared__ __align__(8) uint64_t tfull_bar[kAccStages], tempty_bar[kAccStages];
  __shared__ __align__(8) uint64_t ring_full[kTileRing], ring_empty[kTileRing];
  __shared__ int ring_tile[kTileRing];
  __shared__ uint32_t tmem_base_smem;
  __shared__ TileMap map;

  constexpr int BN_OUT = (EPI == EPI_SWIGLU) ? BN / 2 : BN;  // output columns per tile
  const int nsplit = (EPI == EPI_DOWN_PART) ? p.nsplit : 1;
  constexpr int kStageBytes = stage_bytes<BN>();
  constexpr int kABytes = BM * BK * 2;
  constexpr uint32_t kIdesc = ptx::idesc_bf16_f32(BM, BN);

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles_n = (p.N + BN_OUT - 1) / BN_OUT;
  const int nkb = (p.K + BK - 1) / BK;

  if (warp == 0) build_tile_map(map, p.offsets, p.e_begin, p.e_end, p.e_limit, BM, n_tiles_n * nsplit);
  if (threadIdx.x == 32) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < kAccStages; ++a) {
      ptx::mbar_init(&tfull_bar[a], 1);
      ptx::mbar_init(&tempty_bar[a], 4);
    }
    for (int i = 0; i < kTileRing; ++i) {
      ptx::mbar_init(&ring_full[i], 1);
      ptx::mbar_init(&ring_empty[i], 1 + 4);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<2 * BN>(&tmem_base_smem);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = tmem_base_smem;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmA);
      ptx::tma_prefetch_desc(&tmB);
      int stage = 0, slot = 0, last_e = -1;
      uint32_t phase = 0, rphase = 0;
      while (true) {
        const int tile = ffn_claim(map, p.ws, p.flag, last_e);
        ptx::mbar_wait(&ring_empty[slot], rphase ^ 1);
        ring_tile[slot] = tile;
        ptx::mbar_arrive(&ring_full[slot]);
        if (++slot == kTileRing) { slot = 0; rphase ^= 1; }
        if (tile < 0) break;
        int e, m0, n0, split;
        map.locate(tile, BM, n_tiles_n * nsplit, BN_OUT, e, m0, n0, nsplit, &split);
        // B rows of this tile: two halves of BN/2 rows each.  gate_up: gate rows [n0, n0+BN/2),
        // up rows F + [n0, n0+BN/2) so accumulator columns [0,BN/2) = gate, [BN/2,BN) = up.
        const int brow0 = e * p.b_rows + n0;
        const int brow1 = (EPI == EPI_SWIGLU) ? e * p.b_rows + p.N + n0 : brow0 + BN / 2;
        const int kb0 = split * (nsplit > 1 ? p.kb_per_split : nkb);
        const int kb1 = min(nkb, kb0 + (nsplit > 1 ? p.kb_per_split : nkb));
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * kStageBytes;
          uint8_t* sb = sa + kABytes;
          ptx::mbar_arrive_expect_tx(&full_bar[stage], kStageBytes);
          ptx::tma_load_2d(&tmA, &full_bar[stage], sa, kb * BK, m0, ptx::kEvictNormal);
          ptx::tma_load_2d(&tmB, &full_bar[stage], sb, kb * BK, brow0, ptx::kEvictNormal);
          ptx::tma_load_2d(&tmB, &full_bar[stage], sb + (BN / 2) * 128, kb * BK, brow1, ptx::kEvictNormal);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int stage = 0, slot = 0, acc = 0;
      uint32_t phase = 0, rphase = 0, aphase = 0;
      while (true) {
        ptx::mbar_wait(&ring_full[slot], rphase);
        const int tile = ring_tile[slot];
        ptx::mbar_arrive(&ring_empty[slot]);
        if (++slot == kTileRing) { slot = 0; rphase ^= 1; }
        if (tile < 0) break;
        int e_, m0_, n0_, split;
        map.locate(tile, BM, n_tiles_n * nsplit, BN_OUT, e_, m0_, n0_, nsplit, &split);
        const int kb0 = split * (nsplit > 1 ? p.kb_per_split : nkb);
        const int kb1 = min(nkb, kb0 + (nsplit > 1 ? p.kb_per_split : nkb));
        ptx::mbar_wait(&tempty_bar[acc], aphase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&full_bar[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_addr = ptx::smem_u32(smem + stage * kStageBytes);
          const uint32_t b_addr = a_addr + kABytes;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            ptx::tc_mma_bf16(d_tmem, ptx::sw128_kmajor_desc(a_addr + k * 32), ptx::sw128_kmajor_desc(b_addr + k * 32),
                             kIdesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          ptx::tc_commit(&empty_bar[stage]);  // smem slot free once these MMAs retire
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        ptx::tc_commit(&tfull_bar[acc]);  // accumulator ready for the epilogue
        if (++acc == kAccStages) { acc = 0; aphase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp >= kEpiWarp0) {
    // ------------------------------------------------------------------ epilogue
    const int ew = warp - kEpiWarp0;  // TMEM lanes [32*ew, 32*ew+32)
    int slot = 0, acc = 0;
    uint32_t rphase = 0, aphase = 0;
    while (true) {
      ptx::mbar_wait(&ring_full[slot], rphase);
      const int tile = ring_tile[slot];
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&ring_empty[slot]);
      if (++slot == kTileRing) { slot = 0; rphase ^= 1; }
      if (tile < 0) break;
      int e, m0, n0, split;
      map.locate(tile, BM, n_tiles_n * nsplit, BN_OUT, e, m0, n0, nsplit, &split);
      const int row = m0 + ew * 32 + lane;
      const bool valid = row < p.offsets[e + 1];
      __nv_bfloat16* dst_row = nullptr;
      float* part_row = nullptr;
      if (valid) {
        if constexpr (EPI == EPI_DOWN_PART) {
          part_row = p.part + ((size_t)split * p.part_rows + row) * p.N;
        } else {
          dst_row = (EPI == EPI_SWIGLU) ? p.out + (size_t)row * p.out_ld
                                        : out_row(p.out, p.peers, p.perm[row], p.out_ld);
        }
      }
      ptx::mbar_wait(&tfull_bar[acc], aphase);
      ptx::tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < BN_OUT; c += 32) {
        uint32_t v[32];
        ptx::tmem_ld32(t_row + c, v);
        uint32_t packed[16];
        if constexpr (EPI == EPI_DOWN_PART) {
          ptx::tmem_ld_wait();
          if (valid && n0 + c < p.N) {
            uint4* d4 = reinterpret_cast<uint4*>(part_row + n0 + c);
#pragma unroll
            for (int q = 0; q < 8; ++q) d4[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          }
          continue;
        } else if constexpr (EPI == EPI_SWIGLU) {
          uint32_t u[32];
          ptx::tmem_ld32(t_row + BN / 2 + c, u);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float g0 = __uint_as_float(v[2 * i]), g1 = __uint_as_float(v[2 * i + 1]);
            const float u0 = __uint_as_float(u[2 * i]), u1 = __uint_as_float(u[2 * i + 1]);
            packed[i] = pack_bf16(g0 / (1.f + __expf(-g0)) * u0, g1 / (1.f + __expf(-g1)) * u1);
          }
        } else if constexpr (EPI == EPI_TANH) {
          ptx::tmem_ld_wait();
          const __nv_bfloat16* b = p.bias + (size_t)e * p.N + n0 + c;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float x0 = __uint_as_float(v[2 * i]) + __bfloat162float(b[2 * i]);
            const float x1 = __uint_as_float(v[2 * i + 1]) + __bfloat162float(b[2 * i + 1]);
            packed[i] = pack_bf16(tanhf(x0), tanhf(x1));
          }
        } else {
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) packed[i] = pack_bf16(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
        }
        if (valid && n0 + c < p.N) {
          uint4* d4 = reinterpret_cast<uint4*>(dst_row + n0 + c);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            d4[q] = make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty_bar[acc]);
      if (++acc == kAccStages) { acc = 0; aphase ^= 1; }
    }
  }
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<2 * BN>(tmem_base);
  }
}

// Y[perm[r]] = bf16(sum_s part[s][r]) for the rows of experts [e_begin, stop); one warp per row.
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float* __restrict__ part, int nsplit, int part_rows,
                                                            int N, const int32_t* __restrict__ perm,
                                                            const int32_t* __restrict__ offsets, int e_begin,
                                                            const int32_t* __restrict__ stop,
                                                            __nv_bfloat16* __restrict__ y, void* const* peers) {
  const int r0 = offsets[e_begin], r1 = offsets[*stop];
  const int lane = threadIdx.x & 31;
  for (int r = r0 + blockIdx.x * 8 + (threadIdx.x >> 5); r < r1; r += gridDim.x * 8) {
    __nv_bfloat16* dst = out_row(y, peers, perm[r], N);
    for (int c = lane * 8; c < N; c += 256) {
      float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int s = 0; s < nsplit; ++s) {
        const float4* src = reinterpret_cast<const float4*>(part + ((size_t)s * part_rows + r) * N + c);
        const float4 u = __ldg(src), w = __ldg(src + 1);
        a[0] += u.x; a[1] += u.y; a[2] += u.z; a[3] += u.w; a[4] += w.x; a[5] += w.y; a[6] += w.z; a[7] += w.w;
      }
      uint4 o = make_uint4(pack_bf16(a[0], a[1]), pack_bf16(a[2], a[3]), pack_bf16(a[4], a[5]), pack_bf16(a[6], a[7]));
      *reinterpret_cast<uint4*>(dst + c) = o;
    }
  }
}


// ================================================================================================
// CTA-pair variant (cta_group::2) for large batches: one M=256 x N=256 tile per CTA pair.  Each
// CTA stages its 128 rows of A and its 128 rows of B (gate_up: CTA0 the gate rows, CTA1 the up
// rows), so per-SM operand traffic per MMA drops by a third versus the 1-CTA kernel.  The leader
// (cluster rank 0) claims tiles and publishes them to both CTAs' tile rings over DSMEM; both
// CTAs' TMA loads complete on the leader's full barrier; the leader alone issues
// tcgen05.mma.cta_group::2 and its commits multicast to both CTAs' smem-empty / TMEM-full
// barriers; both CTAs' epilogue warps release the accumulator on the leader's TMEM-empty barrier.
constexpr int kStages2 = 6;
constexpr int kBM2 = 256;  // rows per pair tile (128 per CTA)

template <int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
ffn_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcParams p) {
  constexpr int BN = 256;
  constexpr int BN_OUT = (EPI == EPI_SWIGLU) ? BN / 2 : BN;
  constexpr int kHalfA = 128 * BK * 2;         // 16 KB: this CTA's A rows
  constexpr int kHalfB = (BN / 2) * BK * 2;    // 16 KB: this CTA's B rows
  constexpr int kStageBytes = kHalfA + kHalfB;
  constexpr uint32_t kIdesc = ptx::idesc_bf16_f32(kBM2, BN);
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kStages2], empty_bar[kStages2];
  __shared__ __align__(8) uint64_t tfull_bar[kAccStages], tempty_bar[kAccStages];
  __shared__ __align__(8) uint64_t ring_full[kTileRing], ring_empty[kTileRing];
  __shared__ int ring_tile[kTileRing];
  __shared__ uint32_t tmem_base_smem;
  __shared__ TileMap map;

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int n_tiles_n = (p.N + BN_OUT - 1) / BN_OUT;
  const int nkb = (p.K + BK - 1) / BK;

  if (warp == 0) build_tile_map(map, p.offsets, p.e_begin, p.e_end, p.e_limit, kBM2, n_tiles_n);
  if (threadIdx.x == 32) {
    for (int s = 0; s < kStages2; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < kAccStages; ++a) {
      ptx::mbar_init(&tfull_bar[a], 1);
      ptx::mbar_init(&tempty_bar[a], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is used)
    }
    for (int i = 0; i < kTileRing; ++i) {
      ptx::mbar_init(&ring_full[i], 1);
      ptx::mbar_init(&ring_empty[i], 10);  // leader: MMA + 4 epi; peer: producer + 4 epi
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc_cg2<2 * BN>(&tmem_base_smem);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  __syncthreads();  // CTA-scope order for the allocator's smem write too (racecheck models this one)
  ptx::tc_fence_after();
  const uint32_t tmem_base = tmem_base_smem;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmA);
      ptx::tma_prefetch_desc(&tmB);
      int stage = 0, slot = 0, last_e = -1;
      uint32_t phase = 0, rphase = 0;
      while (true) {
        int tile;
        if (leader) {
          tile = ffn_claim(map, p.ws, p.flag, last_e);
          ptx::mbar_wait_cluster(&ring_empty[slot], rphase ^ 1);
          ring_tile[slot] = tile;
          ptx::st_remote_u32(&ring_tile[slot], 1, (uint32_t)tile);
          ptx::mbar_arrive(&ring_full[slot]);
          ptx::mbar_arrive_remote(&ring_full[slot], 1);
        } else {
          ptx::mbar_wait_cluster(&ring_full[slot], rphase);
          tile = ring_tile[slot];
          ptx::mbar_arrive_remote(&ring_empty[slot], 0);
        }
        if (++slot == kTileRing) { slot = 0; rphase ^= 1; }
        if (tile < 0) break;
        int e, m0, n0;
        map.locate(tile, kBM2, n_tiles_n, BN_OUT, e, m0, n0);
        const int arow = m0 + (int)rank * 128;
        // B rows of this CTA: gate_up -> CTA0 gate [n0, +128), CTA1 up F + [n0, +128);
        // plain -> rows n0 + rank*128 of expert e.
        const int brow = (EPI == EPI_SWIGLU) ? e * p.b_rows + (rank ? p.N : 0) + n0 : e * p.b_rows + n0 + (int)rank * 128;
        for (int kb = 0; kb < nkb; ++kb) {
          ptx::mbar_wait_cluster(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * kStageBytes;
          uint8_t* sb = sa + kHalfA;
          if (leader) ptx::mbar_arrive_expect_tx(&full_bar[stage], 2 * kStageBytes);
          ptx::tma_load_2d_cg2(&tmA, &full_bar[stage], sa, kb * BK, arow, ptx::kEvictNormal);
          ptx::tma_load_2d_cg2(&tmB, &full_bar[stage], sb, kb * BK, brow, ptx::kEvictNormal);
          if (++stage == kStages2) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer (leader only)
    if (leader && lane == 0) {
      int stage = 0, slot = 0, acc = 0;
      uint32_t phase = 0, rphase = 0, aphase = 0;
      while (true) {
        ptx::mbar_wait_cluster(&ring_full[slot], rphase);
        const int tile = ring_tile[slot];
        ptx::mbar_arrive(&ring_empty[slot]);
        if (++slot == kTileRing) { slot = 0; rphase ^= 1; }
        if (tile < 0) break;
        ptx::mbar_wait_cluster(&tempty_bar[acc], aphase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < nkb; ++kb) {
          ptx::mbar_wait(&full_bar[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_addr = ptx::smem_u32(smem + stage * kStageBytes);
          const uint32_t b_addr = a_addr + kHalfA;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            ptx::tc_mma_bf16_cg2(d_tmem, ptx::sw128_kmajor_desc(a_addr + k * 32), ptx::sw128_kmajor_desc(b_addr + k * 32),
                                 kIdesc, (kb | k) != 0);
          ptx::tc_commit_cg2(&empty_bar[stage], 0x3);  // both CTAs' smem slots free
          if (++stage == kStages2) { stage = 0; phase ^= 1; }
        }
        ptx::tc_commit_cg2(&tfull_bar[acc], 0x3);  // both CTAs' accumulators ready
        if (++acc == kAccStages) { acc = 0; aphase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp >= kEpiWarp0) {
    // ------------------------------------------------------------------ epilogue (both CTAs)
    const int ew = warp - kEpiWarp0;
    int slot = 0, acc = 0;
    uint32_t rphase = 0, aphase = 0;
    while (true) {
      ptx::mbar_wait_cluster(&ring_full[slot], rphase);
      const int tile = ring_tile[slot];
      __syncwarp();
      if (lane == 0) {
        if (leader) ptx::mbar_arrive(&ring_empty[slot]);
        else ptx::mbar_arrive_remote(&ring_empty[slot], 0);
      }
      if (++slot == kTileRing) { slot = 0; rphase ^= 1; }
      if (tile < 0) break;
      int e, m0, n0;
      map.locate(tile, kBM2, n_tiles_n, BN_OUT, e, m0, n0);
      const int row = m0 + (int)rank * 128 + ew * 32 + lane;
      const bool valid = row < p.offsets[e + 1];
      __nv_bfloat16* dst_row = nullptr;
      if (valid) {
        dst_row = (EPI == EPI_SWIGLU) ? p.out + (size_t)row * p.out_ld
                                      : out_row(p.out, p.peers, p.perm[row], p.out_ld);
      }
      ptx::mbar_wait_cluster(&tfull_bar[acc], aphase);
      ptx::tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < BN_OUT; c += 32) {
        uint32_t v[32];
        ptx::tmem_ld32(t_row + c, v);
        uint32_t packed[16];
        if constexpr (EPI == EPI_SWIGLU) {
          uint32_t u[32];
          ptx::tmem_ld32(t_row + BN / 2 + c, u);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float g0 = __uint_as_float(v[2 * i]), g1 = __uint_as_float(v[2 * i + 1]);
            const float u0 = __uint_as_float(u[2 * i]), u1 = __uint_as_float(u[2 * i + 1]);
            packed[i] = pack_bf16(g0 / (1.f + __expf(-g0)) * u0, g1 / (1.f + __expf(-g1)) * u1);
          }
        } else {
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) packed[i] = pack_bf16(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
        }
        if (valid && n0 + c < p.N) {
          uint4* d4 = reinterpret_cast<uint4*>(dst_row + n0 + c);
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
      if (++acc == kAccStages) { acc = 0; aphase ^= 1; }
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_cg2<2 * BN>(tmem_base);
  }
}

constexpr int smem_bytes2() { return kStages2 * (128 * BK * 2 + 128 * BK * 2) + 1024; }

// ---- host side --------------------------------------------------------------------------

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
int g_num_sms = 0;
std::once_flag g_once;
int g_init_status = QMOE_OK;

int init_driver() {
  std::call_once(g_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || fn == nullptr) {
      set_error("qmoe_expert_ffn: cuTensorMapEncodeTiled unavailable");
      g_init_status = QMOE_ERR_CUDA;
      return;
    }
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (major != 10) {
      set_error("qmoe_expert_ffn: tcgen05 path needs sm_100 (found sm_%d%d)", major, minor);
      g_init_status = QMOE_ERR_UNSUPPORTED;
    }
  });
  return g_init_status;
}

// 2D bf16 row-major [rows, cols] -> tensor map with box {64 cols, box_rows}, 128B swizzle.
int make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) rows=%llu cols=%llu", (int)r, (unsigned long long)rows,
              (unsigned long long)cols);
    return QMOE_ERR_CUDA;
  }
  return QMOE_OK;
}

}  // namespace

int tc_init_driver() { return init_driver(); }
int tc_num_sms() {
  // per device (g_num_sms is the count of the device current at driver init)
  static int per_dev[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int& n = per_dev[dev & 63];
  if (n == 0) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : g_num_sms;
}
int tc_make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  return make_map(m, base, rows, cols, box_rows);
}

namespace {

template <int BN, int EPI>
int launch_tc(const CUtensorMap& a, const CUtensorMap& b, const TcParams& p, cudaStream_t s) {
  static uint64_t attr_set = 0;  // devices already configured
  if (!(attr_set & current_device_bit())) {
    QMOE_CUDA_TRY(cudaFuncSetAttribute(ffn_tc_kernel<BN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem_bytes<BN>()));
    attr_set |= current_device_bit();
  }
  ffn_tc_kernel<BN, EPI><<<tc_num_sms(), kThreads, smem_bytes<BN>(), s>>>(a, b, p);
  return check_launch("qmoe_expert_ffn(tcgen05)");
}

template <int EPI>
int launch_tc2(const CUtensorMap& a, const CUtensorMap& b, const TcParams& p, cudaStream_t s) {
  static uint64_t attr_set = 0;  // devices already configured
  if (!(attr_set & current_device_bit())) {
    QMOE_CUDA_TRY(cudaFuncSetAttribute(ffn_tc2_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes2()));
    attr_set |= current_device_bit();
  }
  ffn_tc2_kernel<EPI><<<(tc_num_sms() / 2) * 2, kThreads, smem_bytes2(), s>>>(a, b, p);
  return check_launch("qmoe_expert_ffn(tcgen05 cta pair)");
}

}  // namespace

int expert_ffn_tc(int variant, const void* xp, const int32_t* offsets, const int32_t* perm, int E, int d, int F,
                  const void* w1, const void* w2, int e_begin, int e_end, void* act_ws, void* y,
                  const volatile int32_t* flag, int32_t* cursor_out, FfnWorkspace* ws, int xp_rows,
                  void* const* y_peers, cudaStream_t s, int32_t* progress, int seq, int path_rows) {
  int st = init_driver();
  // path_rows: the row count the kernel-path heuristics see (expert parallel: xp_rows is the
  // receive buffer's capacity, the received count is only on the device); buffers use xp_rows
  if (path_rows < 0) path_rows = xp_rows;
  if (st) return st;
  QMOE_REQUIRE(d % 64 == 0, "qmoe_expert_ffn(bf16): d must be a multiple of 64 (d=%d)", d);
  QMOE_REQUIRE(variant != QMOE_EXPERT_SWIGLU || F % 64 == 0, "qmoe_expert_ffn(bf16): F must be a multiple of 64");
  QMOE_REQUIRE(((uintptr_t)xp | (uintptr_t)w1 | (uintptr_t)y | (uintptr_t)(act_ws ? act_ws : y)) % 16 == 0,
               "qmoe_expert_ffn(bf16): buffers must be 16-byte aligned");
  if (variant == QMOE_EXPERT_SWIGLU && use_swap_ab(path_rows, E, d, F))
    return expert_ffn_swap(xp, offsets, perm, E, d, F, w1, w2, e_begin, e_end, act_ws, y, flag, cursor_out, ws,
                           xp_rows, y_peers, nullptr, 0, 0, s, progress, seq, path_rows);
  if (variant == QMOE_EXPERT_SWIGLU && use_swap_pair(path_rows, E, d, F))
    return expert_ffn_swap_pair(xp, offsets, perm, E, d, F, w1, w2, e_begin, e_end, act_ws, y, flag, cursor_out, ws,
                                xp_rows, y_peers, nullptr, 0, 0, s, progress, seq);
  constexpr int BN = 256;
  TcParams p{};
  p.e_begin = e_begin;
  p.e_end = e_end;
  p.offsets = offsets;
  p.perm = perm;
  p.flag = flag;
  p.peers = y_peers;
  CUtensorMap ta, tb;
  if (variant == QMOE_EXPERT_TANH_AFFINE) {
    if ((st = make_map(&ta, xp, xp_rows, d, BM)) || (st = make_map(&tb, w1, (uint64_t)E * d, d, BN / 2))) return st;
    p.N = d; p.K = d; p.b_rows = d;
    p.bias = (const __nv_bfloat16*)w2;
    p.out = (__nv_bfloat16*)y; p.out_ld = d;
    p.ws = ws;
    if ((st = launch_tc<BN, EPI_TANH>(ta, tb, p, s))) return st;
    return ffn_finalize(ws, nullptr, e_end, cursor_out, s, flag);
  }
  const bool pair = use_cta_pair(path_rows, e_end - e_begin);
  if (down_splits(xp_rows, e_end - e_begin, d, F) == 1 && use_fused_tc())
    return expert_ffn_fused(xp, offsets, perm, E, d, F, w1, w2, e_begin, e_end, act_ws, y, flag, cursor_out, ws,
                            xp_rows, y_peers, pair, nullptr, 0, 0, s, progress, seq);
  // gate_up: act[r, :F] = SiLU(x W1^T) * (x W3^T), expert order rows
  if ((st = make_map(&ta, xp, xp_rows, d, BM)) || (st = make_map(&tb, w1, (uint64_t)E * 2 * F, d, BN / 2))) return st;
  p.N = F; p.K = d; p.b_rows = 2 * F;
  p.out = (__nv_bfloat16*)act_ws; p.out_ld = F;
  p.ws = ws + 0;
  if ((st = pair ? launch_tc2<EPI_SWIGLU>(ta, tb, p, s) : launch_tc<BN, EPI_SWIGLU>(ta, tb, p, s))) return st;
  if ((st = ffn_finalize(ws + 0, nullptr, e_end, nullptr, s))) return st;
  // down: Y[perm[r], :d] = act[r] W2^T, only experts whose gate_up completed
  CUtensorMap ta2, tb2;
  if ((st = make_map(&ta2, act_ws, xp_rows, F, BM)) || (st = make_map(&tb2, w2, (uint64_t)E * d, F, BN / 2))) return st;
  TcParams p2 = p;
  p2.N = d; p2.K = F; p2.b_rows = d;
  p2.out = (__nv_bfloat16*)y; p2.out_ld = d;
  p2.e_limit = &ws[0].stop;
  p2.ws = ws + 1;
  const int nsplit = down_splits(xp_rows, e_end - e_begin, d, F);
  if (nsplit > 1) {
    const int nkb = (F + BK - 1) / BK;
    p2.kb_per_split = (nkb + nsplit - 1) / nsplit;
    p2.nsplit = (nkb + p2.kb_per_split - 1) / p2.kb_per_split;  // every split non-empty
    p2.part = splitk_buffer(ws);
    p2.part_rows = xp_rows;
    if ((st = launch_tc<BN, EPI_DOWN_PART>(ta2, tb2, p2, s))) return st;
    if ((st = ffn_finalize(ws + 1, &ws[0].stop, e_end, cursor_out, s, flag))) return st;
    const int grid = xp_rows / 8 + 1 < 148 * 4 ? xp_rows / 8 + 1 : 148 * 4;
    splitk_reduce_kernel<<<grid, 256, 0, s>>>(p2.part, p2.nsplit, xp_rows, d, perm, offsets, e_begin, &ws[1].stop,
                                               (__nv_bfloat16*)y, y_peers);
    return check_launch("qmoe_expert_ffn(split-K reduce)");
  }
  p2.nsplit = 1;
  if ((st = pair ? launch_tc2<EPI_DOWN>(ta2, tb2, p2, s) : launch_tc<BN, EPI_DOWN>(ta2, tb2, p2, s))) return st;
  return ffn_finalize(ws + 1, &ws[0].stop, e_end, cursor_out, s, flag);
}

int expert_ffn_path(int d, int F, int E, int xp_rows) {
  if (d % 64 != 0 || F % 64 != 0) return QMOE_PATH_UNSUPPORTED;
  if (use_swap_ab(xp_rows, E, d, F)) return QMOE_PATH_SWAP_AB;
  if (use_swap_pair(xp_rows, E, d, F)) return QMOE_PATH_SWAP_PAIR;
  const bool pair = use_cta_pair(xp_rows, E);
  if (down_splits(xp_rows, E, d, F) == 1 && use_fused_tc()) return pair ? QMOE_PATH_FUSED_PAIR : QMOE_PATH_FUSED_1CTA;
  return pair ? QMOE_PATH_TWO_LAUNCH_PAIR : QMOE_PATH_TWO_LAUNCH_1CTA;
}

// Large batches use the CTA-pair kernel (M = 256 rows per tile) unless its row padding would
// cost more than the 1-CTA kernel's (M = 128): with many fine-grained experts (Qwen: 60 experts,
// ~550 rows each at 8k tokens) a 256-row tile wastes ~30% of the tensor work on padding rows.
// The host does not know the per-expert counts (they stay on the device), so the padding is
// estimated from the mean rows per covered expert.  QMOE_CTA_PAIR=0/1 forces either path.
bool use_cta_pair(int xp_rows, int n_experts) {
  static int forced = [] {
    const char* v = getenv("QMOE_CTA_PAIR");
    return v == nullptr ? -1 : atoi(v);
  }();
  if (forced >= 0) return forced == 1 && xp_rows > kSplitRowsMax;
  if (xp_rows < 1536) return false;  // measured crossover (Mixtral: pair faster from ~768 tokens)
  // fine-grained experts (Qwen's 60 routed + 4 shared sub-experts): the mean is inflated by the
  // shared sub-experts' T rows while the routed experts see ~T/15 -- the 1-CTA tiles measured
  // 0-7% faster at 1k-16k tokens (tools/qwen_ab.py, profiles/qwen_paths_r02.jsonl)
  if (n_experts > 16) return false;
  const double r = (double)xp_rows / (n_experts > 0 ? n_experts : 1);
  auto eff = [r](int m) { return r / (m * std::ceil(r / m)); };
  return eff(256) >= eff(128) - 0.02;
}

int down_splits(int xp_rows, int n_experts, int d, int F) {
  // Small batches (<= 512 routed rows) run the down projection K-split so launches covering few
  // experts (a resume after an expert-boundary preemption, or a batch hitting 1-2 experts) still
  // fill every SM.  The split count depends only on the problem shape — never on the expert
  // range — so a resumed launch rounds exactly like an uninterrupted one (bit-identical resume).
  (void)n_experts;
  (void)d;
  if (xp_rows > kSplitRowsMax) return 1;
  int want = 4;
  if (want > (F / BK) / 16) want = (F / BK) / 16;  // >= 16 K blocks (1024) per split
  if (want > kMaxSplit) want = kMaxSplit;
  return want < 1 ? 1 : want;
}

size_t splitk_bytes(int xp_rows, int d) {
  return xp_rows > kSplitRowsMax ? 0 : (size_t)kMaxSplit * xp_rows * d * sizeof(float);
}

float* splitk_buffer(FfnWorkspace* ws) {
  return reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + kFfnHeaderBytes);
}

}  // namespace qmoe
