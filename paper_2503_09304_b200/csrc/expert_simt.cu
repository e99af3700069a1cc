// Grouped expert FFN, SIMT path (f32 / f64) — the parity build.
//
// Replaces the drain loop of the reference (engine.py:204-215) and MoEModel.expert_forward_many
// (model.py:141-145): for every expert e in [e_begin, e_end) the rows Xp[offsets[e]:offsets[e+1]]
// go through tanh(A_e x + b_e) (or the SwiGLU FFN) and land in their slot rows of Y.
// Tensor cores have no f64/f32 kind with the reference's rounding, so parity builds use CUDA
// cores; production bf16 runs on tcgen05 (expert_tc.cu).  Tiles are claimed dynamically in
// expert-major order from a global counter, which makes the expert boundary well defined for
// the device preempt flag (see ffn_claim below and DESIGN.md).
#include "expert_common.cuh"

namespace qmoe {
namespace {

constexpr int BM = 32, BN = 64, BK = 32, kThreads = 256;

template <typename T> __device__ __forceinline__ T tanh_t(T v);
template <> __device__ __forceinline__ float tanh_t<float>(float v) { return tanhf(v); }
template <> __device__ __forceinline__ double tanh_t<double>(double v) { return tanh(v); }
template <typename T> __device__ __forceinline__ T silu_t(T v);
template <> __device__ __forceinline__ float silu_t<float>(float v) { return v / (1.f + expf(-v)); }
template <> __device__ __forceinline__ double silu_t<double>(double v) { return v / (1.0 + exp(-v)); }

// EPI_TANH  : N = d,  K = d,  B = A_e [d, d],          out = tanh(acc + b_e)   -> Y[perm[r]]
// EPI_SWIGLU: N = F,  K = d,  B = gate_up_e [2F, d],   out = silu(g) * u       -> act[r]
// EPI_DOWN  : N = d,  K = F,  B = down_e [d, F],       out = acc               -> Y[perm[r]]
enum { EPI_TANH = 0, EPI_SWIGLU = 1, EPI_DOWN = 2 };

template <typename T, int EPI>
__global__ void __launch_bounds__(kThreads)
ffn_simt_kernel(const T* __restrict__ a_rows, const int32_t* __restrict__ offsets,
                const int32_t* __restrict__ perm, int E, int N, int K, const T* __restrict__ wB,
                const T* __restrict__ bias, int e_begin, int e_end, const int32_t* __restrict__ e_limit,
                T* __restrict__ out, const volatile int32_t* flag, FfnWorkspace* ws) {
  __shared__ T As[BK][BM + 1];
  __shared__ T Bs[BK][BN + 1];
  __shared__ T Bu[EPI == EPI_SWIGLU ? BK : 1][BN + 1];
  __shared__ TileMap map;
  __shared__ int s_tile;
  const int tid = threadIdx.x;
  const int n_tiles_n = (N + BN - 1) / BN;
  if (tid < 32) build_tile_map(map, offsets, e_begin, e_end, e_limit, BM, n_tiles_n);
  __syncthreads();
  const int ty = tid >> 5, tx = tid & 31;  // rows ty*4.., cols tx, tx+32
  int last_e = -1;

  while (true) {
    if (tid == 0) s_tile = ffn_claim(map, ws, flag, last_e);
    __syncthreads();
    const int tile = s_tile;
    __syncthreads();
    if (tile < 0) break;
    int e, m0, n0;
    map.locate(tile, BM, n_tiles_n, BN, e, m0, n0);
    const int r_end = offsets[e + 1];
    const T* W = wB + (size_t)e * (EPI == EPI_SWIGLU ? 2 * (size_t)N : (size_t)N) * K;

    T acc[4][2], accu[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) acc[i][j] = accu[i][j] = T(0);

    for (int k0 = 0; k0 < K; k0 += BK) {
      for (int i = tid; i < BM * BK; i += kThreads) {
        const int r = i / BK, kk = i % BK;
        const int row = m0 + r;
        As[kk][r] = (row < r_end && k0 + kk < K) ? a_rows[(size_t)row * K + k0 + kk] : T(0);
      }
      for (int i = tid; i < BN * BK; i += kThreads) {
        const int n = i / BK, kk = i % BK;
        const bool ok = n0 + n < N && k0 + kk < K;
        Bs[kk][n] = ok ? W[(size_t)(n0 + n) * K + k0 + kk] : T(0);
        if constexpr (EPI == EPI_SWIGLU) Bu[kk][n] = ok ? W[(size_t)(N + n0 + n) * K + k0 + kk] : T(0);
      }
      __syncthreads();
#pragma unroll 8
      for (int kk = 0; kk < BK; ++kk) {
        T av[4], bv[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
        bv[0] = Bs[kk][tx];
        bv[1] = Bs[kk][tx + 32];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) acc[i][j] += av[i] * bv[j];
        if constexpr (EPI == EPI_SWIGLU) {
          const T u0 = Bu[kk][tx], u1 = Bu[kk][tx + 32];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            accu[i][0] += av[i] * u0;
            accu[i][1] += av[i] * u1;
          }
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = m0 + ty * 4 + i;
      if (row >= r_end) continue;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int n = n0 + tx + 32 * j;
        if (n >= N) continue;
        if constexpr (EPI == EPI_TANH) {
          out[(size_t)perm[row] * N + n] = tanh_t<T>(acc[i][j] + bias[(size_t)e * N + n]);
        } else if constexpr (EPI == EPI_SWIGLU) {
          out[(size_t)row * N + n] = silu_t<T>(acc[i][j]) * accu[i][j];
        } else {
          out[(size_t)perm[row] * N + n] = acc[i][j];
        }
      }
    }
  }
}

template <typename T>
int run_simt(int variant, const void* xp, const int32_t* offsets, const int32_t* perm, int E, int d, int F,
             const void* w1, const void* w2, int e_begin, int e_end, void* act_ws, void* y,
             const volatile int32_t* flag, int32_t* cursor_out, FfnWorkspace* ws, cudaStream_t s) {
  const int grid = 148 * 4;
  int st;
  if (variant == QMOE_EXPERT_TANH_AFFINE) {
    ffn_simt_kernel<T, EPI_TANH><<<grid, kThreads, 0, s>>>((const T*)xp, offsets, perm, E, d, d, (const T*)w1,
                                                          (const T*)w2, e_begin, e_end, nullptr, (T*)y, flag,
                                                          ws + 0);
    if ((st = check_launch("qmoe_expert_ffn(simt tanh)"))) return st;
    return ffn_finalize(ws + 0, nullptr, e_end, cursor_out, s, flag);
  }
  ffn_simt_kernel<T, EPI_SWIGLU><<<grid, kThreads, 0, s>>>((const T*)xp, offsets, perm, E, F, d, (const T*)w1,
                                                          nullptr, e_begin, e_end, nullptr, (T*)act_ws, flag,
                                                          ws + 0);
  if ((st = check_launch("qmoe_expert_ffn(simt gate_up)"))) return st;
  if ((st = ffn_finalize(ws + 0, nullptr, e_end, nullptr, s))) return st;
  // down projection only for experts whose gate_up completed (stop of launch 1)
  ffn_simt_kernel<T, EPI_DOWN><<<grid, kThreads, 0, s>>>((const T*)act_ws, offsets, perm, E, d, F, (const T*)w2,
                                                        nullptr, e_begin, e_end, &ws[0].stop, (T*)y, flag, ws + 1);
  if ((st = check_launch("qmoe_expert_ffn(simt down)"))) return st;
  return ffn_finalize(ws + 1, &ws[0].stop, e_end, cursor_out, s, flag);
}

}  // namespace

int expert_ffn_simt(int variant, int dtype, const void* xp, const int32_t* offsets, const int32_t* perm, int E,
                    int d, int F, const void* w1, const void* w2, int e_begin, int e_end, void* act_ws, void* y,
                    const volatile int32_t* flag, int32_t* cursor_out, FfnWorkspace* ws, cudaStream_t s) {
  if (dtype == QMOE_F64)
    return run_simt<double>(variant, xp, offsets, perm, E, d, F, w1, w2, e_begin, e_end, act_ws, y, flag,
                            cursor_out, ws, s);
  return run_simt<float>(variant, xp, offsets, perm, E, d, F, w1, w2, e_begin, e_end, act_ws, y, flag, cursor_out,
                         ws, s);
}

}  // namespace qmoe
