// Weighted combine + small state-movement kernels (restore gather, cursor advance, paged KV).
//
// combine replaces InferenceEngine._finish_layer (reference engine.py:330-365):
//   acc = residual; for j in ascending expert id: acc = acc + w[:, j] * out[:, j]
// One warp per token, 16-byte vector loads of the k slot rows; the sum is taken in the same j
// order, and the fp64/fp32 variants round product and sum separately (no FMA contraction) so
// the result is bit-identical to the reference's numpy expression on identical inputs.
#include <stdarg.h>

#include "common.cuh"

namespace qmoe {

static thread_local char g_last_error[512] = {0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

namespace {

constexpr int kCombWarps = 8;

__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }

// Exact-order variant for f32 / f64 (parity builds).
template <typename T>
__global__ void __launch_bounds__(kCombWarps * 32)
combine_exact_kernel(const T* __restrict__ y, const T* __restrict__ w, const T* __restrict__ residual,
                     int ntok, int k, int d, T* __restrict__ out) {
  const int tok = blockIdx.x * kCombWarps + warp_id();
  if (tok >= ntok) return;
  const int lane = lane_id();
  const T* yt = y + (size_t)tok * k * d;
  for (int i = lane; i < d; i += 32) {
    T acc = residual != nullptr ? residual[(size_t)tok * d + i] : T(0);
    for (int j = 0; j < k; ++j) acc = add_rn(acc, mul_rn(w[(size_t)tok * k + j], yt[(size_t)j * d + i]));
    out[(size_t)tok * d + i] = acc;
  }
}

// bf16 Y/residual/out, fp32 weights and accumulation, 8 elements (16 B) per lane per step.
// `parts` warps share one token (each a contiguous slice of the row) so small decode batches
// still put enough warps in flight.
template <int K>
__global__ void __launch_bounds__(kCombWarps * 32)
combine_bf16_kernel(const __nv_bfloat16* __restrict__ y, const float* __restrict__ w,
                    const __nv_bfloat16* __restrict__ residual, int ntok, int k, int d, int parts,
                    __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int gw = blockIdx.x * kCombWarps + warp_id();
  const int tok = gw / parts, part = gw - tok * parts;
  if (tok >= ntok) return;
  const int lane = lane_id();
  float wt[8];
  const int kk = K > 0 ? K : k;
#pragma unroll
  for (int j = 0; j < 8; ++j) wt[j] = j < kk ? w[(size_t)tok * kk + j] : 0.f;
  const uint4* y4 = reinterpret_cast<const uint4*>(y + (size_t)tok * kk * d);
  const int nv = d >> 3;  // uint4 per row
  const int per = (nv + parts - 1) / parts;
  const int v_end = min(nv, (part + 1) * per);
#pragma unroll 2
  for (int v = part * per + lane; v < v_end; v += 32) {
    float acc[8];
    if (residual != nullptr) {
      uint4 r = __ldg(reinterpret_cast<const uint4*>(residual + (size_t)tok * d) + v);
      const __nv_bfloat162* r2 = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float2 f = __bfloat1622float2(r2[q]);
        acc[2 * q] = f.x;
        acc[2 * q + 1] = f.y;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < (K > 0 ? K : 8); ++j) {
      if (K == 0 && j >= kk) break;
      uint4 u = __ldg(y4 + (size_t)j * nv + v);
      const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float2 f = __bfloat1622float2(u2[q]);
        acc[2 * q] = fmaf(wt[j], f.x, acc[2 * q]);
        acc[2 * q + 1] = fmaf(wt[j], f.y, acc[2 * q + 1]);
      }
    }
    uint4 o;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int q = 0; q < 4; ++q) o2[q] = __floats2bfloat162_rn(acc[2 * q], acc[2 * q + 1]);
    reinterpret_cast<uint4*>(out + (size_t)tok * d)[v] = o;
  }
}

// src_stride: bytes between consecutive source rows in scatter mode (row_bytes when dense; e.g. the
// K|V part of packed qkv rows for the KV append)
__global__ void gather_rows_kernel(const uint8_t* __restrict__ src, const int32_t* __restrict__ idx,
                                   int rows, size_t row_bytes, uint8_t* __restrict__ dst, int scatter,
                                   const volatile int32_t* guard, size_t src_stride) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x * 8 + warp_id();
  if (r >= rows) return;
  if (guard != nullptr && *guard < 0) return;  // voided iteration (qmoe_kv_append_guarded)
  const int lane = lane_id();
  const uint8_t* s = scatter ? src + (size_t)r * src_stride : src + (size_t)idx[r] * row_bytes;
  uint8_t* d = scatter ? dst + (size_t)idx[r] * row_bytes : dst + (size_t)r * row_bytes;
  if ((row_bytes & 15) == 0 && ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d)) & 15) == 0) {
    const uint4* s4 = reinterpret_cast<const uint4*>(s);
    uint4* d4 = reinterpret_cast<uint4*>(d);
    for (int i = lane; i < (int)(row_bytes >> 4); i += 32) d4[i] = __ldg(s4 + i);
  } else {
    for (size_t i = lane; i < row_bytes; i += 32) d[i] = s[i];
  }
}

__global__ void cursor_advance_kernel(int32_t* cursor, int ntok, const int32_t* stop) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < ntok) {
    const int s = *stop;
    if (cursor[t] < s) cursor[t] = s;
  }
}

// Preemption at an expert boundary: cursors advance to the stop (as cursor_advance_kernel) and the
// launch's queue offsets are rewritten so experts below the stop are empty: out[e] = in[max(e,
// stop)].  The resumed launch then reuses the first launch's perm / Xp (a stable sort of the
// pending slots gives the same per-expert order), so a resume needs no re-permute.
__global__ void resume_point_kernel(int32_t* cursor, int ntok, const int32_t* stop, const int32_t* offsets, int E,
                                    int32_t* offsets_out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = *stop;
  if (t < ntok && cursor[t] < s) cursor[t] = s;
  if (offsets != nullptr && t <= E) offsets_out[t] = offsets[t < s ? s : t];
}

int launch_rows(const void* src, const int32_t* idx, int rows, size_t row_bytes, void* dst, int scatter,
                cudaStream_t s, const char* what, const int32_t* guard = nullptr, size_t src_stride = 0) {
  QMOE_REQUIRE(rows >= 0 && row_bytes > 0, "%s: bad sizes", what);
  if (src_stride == 0) src_stride = row_bytes;
  QMOE_REQUIRE(src_stride >= row_bytes, "%s: source row stride %zu < row bytes %zu", what, src_stride, row_bytes);
  if (rows == 0) return QMOE_OK;
  QMOE_REQUIRE(src && idx && dst, "%s: null pointer", what);
  return launch_pdl(what, gather_rows_kernel, dim3((rows + 7) / 8), dim3(256), 0, s, (const uint8_t*)src, idx, rows,
                    row_bytes, (uint8_t*)dst, scatter, (const volatile int32_t*)guard, src_stride);
}

}  // namespace
}  // namespace qmoe

extern "C" int qmoe_version(void) { return 1; }

extern "C" const char* qmoe_status_string(int status) {
  switch (status) {
    case QMOE_OK: return "ok";
    case QMOE_ERR_INVALID: return "invalid argument";
    case QMOE_ERR_STATE: return "state corruption";
    case QMOE_ERR_PARTIAL: return "partial token";
    case QMOE_ERR_CAPACITY: return "cache capacity exceeded";
    case QMOE_ERR_CUDA: return "cuda error";
    case QMOE_ERR_UNSUPPORTED: return "unsupported";
    default: return "unknown status";
  }
}

extern "C" const char* qmoe_last_error(void) { return qmoe::g_last_error; }

extern "C" int qmoe_combine(int dtype, const void* y, const void* w, const void* residual, int T, int k, int d,
                            void* out, void* stream) {
  using namespace qmoe;
  QMOE_REQUIRE(T >= 0 && k >= 1 && k <= 8 && d >= 1, "qmoe_combine: bad sizes T=%d k=%d d=%d", T, k, d);
  if (T == 0) return QMOE_OK;
  QMOE_REQUIRE(y && w && out, "qmoe_combine: null pointer");
  cudaStream_t s = as_stream(stream);
  const dim3 grid((T + kCombWarps - 1) / kCombWarps), block(kCombWarps * 32);
  switch (dtype) {
    case QMOE_F64:
      combine_exact_kernel<double><<<grid, block, 0, s>>>((const double*)y, (const double*)w,
                                                          (const double*)residual, T, k, d, (double*)out);
      break;
    case QMOE_F32:
      combine_exact_kernel<float><<<grid, block, 0, s>>>((const float*)y, (const float*)w, (const float*)residual,
                                                         T, k, d, (float*)out);
      break;
    case QMOE_BF16: {
      QMOE_REQUIRE(d % 8 == 0, "qmoe_combine: bf16 path needs d %% 8 == 0 (d=%d)", d);
      QMOE_REQUIRE(((uintptr_t)y | (uintptr_t)out | (uintptr_t)(residual ? residual : out)) % 16 == 0,
                   "qmoe_combine: bf16 buffers must be 16-byte aligned");
      auto yb = (const __nv_bfloat16*)y;
      auto rb = (const __nv_bfloat16*)residual;
      auto ob = (__nv_bfloat16*)out;
      // enough warps to cover the SMs: split each row over up to d/256 warps for small T
      int parts = (148 * kCombWarps + T - 1) / T;
      const int max_parts = d / 256 > 0 ? d / 256 : 1;
      parts = parts < 1 ? 1 : (parts > max_parts ? max_parts : parts);
      const dim3 g2((T * parts + kCombWarps - 1) / kCombWarps);
      if (k == 2)
        return launch_pdl("qmoe_combine", combine_bf16_kernel<2>, g2, block, 0, s, yb, (const float*)w, rb, T, k, d,
                          parts, ob);
      if (k == 4)
        return launch_pdl("qmoe_combine", combine_bf16_kernel<4>, g2, block, 0, s, yb, (const float*)w, rb, T, k, d,
                          parts, ob);
      if (k == 8)  // Qwen: 4 routed + 4 shared sub-expert slots (generic k: 79 us at 8k tokens, 4.2 TB/s)
        return launch_pdl("qmoe_combine", combine_bf16_kernel<8>, g2, block, 0, s, yb, (const float*)w, rb, T, k, d,
                          parts, ob);
      return launch_pdl("qmoe_combine", combine_bf16_kernel<0>, g2, block, 0, s, yb, (const float*)w, rb, T, k, d,
                        parts, ob);
    }
    default:
      set_error("qmoe_combine: unknown dtype %d", dtype);
      return QMOE_ERR_INVALID;
  }
  return check_launch("qmoe_combine");
}

extern "C" int qmoe_gather_rows(const void* src, const int32_t* idx, int rows, size_t row_bytes, void* dst,
                                void* stream) {
  return qmoe::launch_rows(src, idx, rows, row_bytes, dst, 0, qmoe::as_stream(stream), "qmoe_gather_rows");
}

extern "C" int qmoe_scatter_rows(const void* src, const int32_t* idx, int rows, size_t row_bytes, void* dst,
                                 void* stream) {
  return qmoe::launch_rows(src, idx, rows, row_bytes, dst, 1, qmoe::as_stream(stream), "qmoe_scatter_rows");
}

extern "C" int qmoe_cursor_advance(int32_t* cursor, int T, const int32_t* stop_expert_dev, void* stream) {
  using namespace qmoe;
  QMOE_REQUIRE(T >= 0, "qmoe_cursor_advance: bad T");
  if (T == 0) return QMOE_OK;
  QMOE_REQUIRE(cursor && stop_expert_dev, "qmoe_cursor_advance: null pointer");
  cursor_advance_kernel<<<(T + 255) / 256, 256, 0, as_stream(stream)>>>(cursor, T, stop_expert_dev);
  return check_launch("qmoe_cursor_advance");
}

extern "C" int qmoe_resume_point(int32_t* cursor, int T, const int32_t* stop_expert_dev, const int32_t* offsets, int E,
                                 int32_t* offsets_out, void* stream) {
  using namespace qmoe;
  QMOE_REQUIRE(T >= 0 && E >= 1 && E <= 64, "qmoe_resume_point: bad sizes T=%d E=%d", T, E);
  QMOE_REQUIRE(stop_expert_dev && (T == 0 || cursor) && (offsets == nullptr || offsets_out),
               "qmoe_resume_point: null pointer");
  const int n = T > E + 1 ? T : E + 1;
  resume_point_kernel<<<(n + 255) / 256, 256, 0, as_stream(stream)>>>(cursor, T, stop_expert_dev, offsets, E,
                                                                       offsets_out);
  return check_launch("qmoe_resume_point");
}

extern "C" int qmoe_kv_append(void* pool, const int32_t* slot_mapping, const void* rows, int n_rows,
                              size_t row_bytes, void* stream) {
  return qmoe::launch_rows(rows, slot_mapping, n_rows, row_bytes, pool, 1, qmoe::as_stream(stream),
                           "qmoe_kv_append");
}

extern "C" int qmoe_kv_append_guarded(void* pool, const int32_t* slot_mapping, const void* rows, int n_rows,
                                      size_t row_bytes, const int32_t* guard, void* stream) {
  return qmoe::launch_rows(rows, slot_mapping, n_rows, row_bytes, pool, 1, qmoe::as_stream(stream),
                           "qmoe_kv_append_guarded", guard);
}

extern "C" int qmoe_kv_append_strided(void* pool, const int32_t* slot_mapping, const void* rows, int n_rows,
                                      size_t row_bytes, size_t row_stride, const int32_t* guard, void* stream) {
  return qmoe::launch_rows(rows, slot_mapping, n_rows, row_bytes, pool, 1, qmoe::as_stream(stream),
                           "qmoe_kv_append_strided", guard, row_stride);
}

extern "C" int qmoe_kv_gather(const void* pool, const int32_t* slot_mapping, int n_rows, size_t row_bytes,
                              void* dst, void* stream) {
  return qmoe::launch_rows(pool, slot_mapping, n_rows, row_bytes, dst, 0, qmoe::as_stream(stream),
                           "qmoe_kv_gather");
}
