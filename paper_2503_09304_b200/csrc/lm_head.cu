// Device-side greedy emission: LM head GEMV + argmax (lowest id on ties) in one launch.
//
// Replaces MoEModel.emit_token (reference model.py:166-169: argmax over w_out h + b_out, numpy's
// first maximal index) for the decoder plugins, where it was a cuBLAS GEMM writing [T, V] fp32
// logits, torch.argmax and a host read of the logits' argmax.  At decode this is weight streaming
// (Mixtral: 32000 x 4096 bf16 = 262 MB per iteration; Qwen: 622 MB), so the kernel is built like
// the streaming router: one warp per 8 vocabulary rows over the whole of d, the rows streamed from
// HBM with 16-byte loads straight into mma.sync B fragments (k permuted identically in A and B),
// the <= 64 token rows (A) read from L1/L2.  Each warp reduces its 8 logits per token to a
// (value, id) key ordered by value then lowest id, the CTA folds its warps' keys with shared-memory
// atomicMax, one global atomicMax per token per CTA, and the last CTA out converts the keys into
// token ids and re-zeroes the workspace (zeroed once at allocation, like the expert FFN's).
#include "common.cuh"

namespace qmoe {
namespace {

constexpr int kLmWarps = 8;

__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <bool NOALLOC>
__device__ __forceinline__ uint4 ldv4(const uint4* p) {
  uint4 v;
  if constexpr (NOALLOC)
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// (value, id) -> key: larger value first, then the LOWER id (numpy argmax's first maximum).
__device__ __forceinline__ unsigned long long argmax_key(float v, int id) {
  uint32_t u = __float_as_uint(v);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((unsigned long long)u << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)id);
}

struct LmWorkspace {
  unsigned long long keys[64];
  int exits;
};

template <int MT, int U>
__global__ void __launch_bounds__(kLmWarps * 32)
lm_head_argmax_kernel(const __nv_bfloat16* __restrict__ h, const __nv_bfloat16* __restrict__ w, int T, int d, int V,
                      int32_t* __restrict__ tokens_out, LmWorkspace* ws) {
  pdl_wait();
  pdl_trigger();
  __shared__ unsigned long long s_key[16 * MT];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  for (int i = threadIdx.x; i < 16 * MT; i += blockDim.x) s_key[i] = 0ull;
  __syncthreads();
  const int tile = blockIdx.x * kLmWarps + warp;  // 8 vocabulary rows
  const int v0 = tile * 8;
  if (v0 < V) {
    const uint4* wp = reinterpret_cast<const uint4*>(w + (size_t)min(v0 + g, V - 1) * d) + t4;
    const uint4* xp[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
        xp[mt][hh] = reinterpret_cast<const uint4*>(h + (size_t)min(16 * mt + g + 8 * hh, T - 1) * d) + t4;
    float acc[MT][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
    const int nsteps = d / 32;  // 32-wide k steps; a multiple of U (host-checked)
    uint4 a[2][U][MT][2], b[2][U];
    auto load = [&](int buf, int s0) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        b[buf][u] = ldv4<true>(wp + 4 * (s0 + u));
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          a[buf][u][mt][0] = ldv4<false>(xp[mt][0] + 4 * (s0 + u));
          a[buf][u][mt][1] = ldv4<false>(xp[mt][1] + 4 * (s0 + u));
        }
      }
    };
    auto mma = [&](int buf) {
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const uint4& x0 = a[buf][u][mt][0];
          const uint4& x1 = a[buf][u][mt][1];
          mma16816(acc[mt], x0.x, x1.x, x0.y, x1.y, b[buf][u].x, b[buf][u].y);
          mma16816(acc[mt], x0.z, x1.z, x0.w, x1.w, b[buf][u].z, b[buf][u].w);
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
    // lane (g, t4) holds tokens 16mt+g (c0, c1) and 16mt+g+8 (c2, c3) at vocab v0+2t4, v0+2t4+1
    const int c0 = v0 + 2 * t4;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const float x = acc[mt][2 * hh], y = acc[mt][2 * hh + 1];
        unsigned long long key = 0ull;
        if (c0 < V) key = argmax_key(x, c0);
        if (c0 + 1 < V) {
          const unsigned long long k1 = argmax_key(y, c0 + 1);
          key = k1 > key ? k1 : key;
        }
#pragma unroll
        for (int o = 1; o < 4; o <<= 1) {
          const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
          key = other > key ? other : key;
        }
        const int tok = 16 * mt + g + 8 * hh;
        if (t4 == 0 && tok < T && key != 0ull) atomicMax(&s_key[tok], key);
      }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < T; i += blockDim.x)
    if (s_key[i] != 0ull) atomicMax(&ws->keys[i], s_key[i]);
  // last CTA out: keys -> token ids, workspace back to zero
  __threadfence();
  __syncthreads();
  __shared__ int last;
  if (threadIdx.x == 0) last = atomicAdd(&ws->exits, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int i = threadIdx.x; i < T; i += blockDim.x) {
    const unsigned long long key = atomicExch(&ws->keys[i], 0ull);
    tokens_out[i] = (int32_t)(0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull));
  }
  if (threadIdx.x == 0) ws->exits = 0;
}

template <int MT>
int launch_lm(const void* h, const void* w, int T, int d, int V, int32_t* out, LmWorkspace* ws, cudaStream_t s) {
  const int tiles = (V + 7) / 8;
  return launch_pdl("qmoe_lm_head_argmax", lm_head_argmax_kernel<MT, 2>, dim3((tiles + kLmWarps - 1) / kLmWarps),
                    dim3(kLmWarps * 32), 0, s, (const __nv_bfloat16*)h, (const __nv_bfloat16*)w, T, d, V, out, ws);
}

}  // namespace
}  // namespace qmoe

extern "C" size_t qmoe_lm_head_argmax_workspace_bytes(void) { return sizeof(qmoe::LmWorkspace); }

extern "C" int qmoe_lm_head_argmax(const void* h, const void* w_out, int T, int d, int V, int32_t* tokens_out,
                                   void* workspace, size_t workspace_bytes, void* stream) {
  using namespace qmoe;
  QMOE_REQUIRE(T >= 0 && T <= 64 && V >= 1 && d >= 32 && d % 128 == 0,
               "qmoe_lm_head_argmax: need 0 <= T <= 64, V >= 1, d %% 128 == 0 (T=%d d=%d V=%d)", T, d, V);
  QMOE_REQUIRE(workspace != nullptr && workspace_bytes >= sizeof(LmWorkspace),
               "qmoe_lm_head_argmax: workspace too small");
  if (T == 0) return QMOE_OK;
  QMOE_REQUIRE(h && w_out && tokens_out, "qmoe_lm_head_argmax: null pointer");
  QMOE_REQUIRE(((uintptr_t)h | (uintptr_t)w_out) % 16 == 0, "qmoe_lm_head_argmax: buffers must be 16-byte aligned");
  auto ws = reinterpret_cast<LmWorkspace*>(workspace);
  cudaStream_t s = as_stream(stream);
  if (T <= 16) return launch_lm<1>(h, w_out, T, d, V, tokens_out, ws, s);
  if (T <= 32) return launch_lm<2>(h, w_out, T, d, V, tokens_out, ws, s);
  return launch_lm<4>(h, w_out, T, d, V, tokens_out, ws, s);
}
