// Shared helpers for libqmoe: status plumbing, element-type traits, small device utilities.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include "../../include/qmoe.h"

namespace qmoe {

// Thread-local text of the last failure; surfaced by qmoe_last_error().
void set_error(const char* fmt, ...);

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return QMOE_ERR_CUDA;
  }
  return QMOE_OK;
}

#define QMOE_REQUIRE(cond, ...)            \
  do {                                     \
    if (!(cond)) {                         \
      ::qmoe::set_error(__VA_ARGS__);      \
      return QMOE_ERR_INVALID;             \
    }                                      \
  } while (0)

#define QMOE_CUDA_TRY(expr)                                                       \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess) {                                                      \
      ::qmoe::set_error("%s failed: %s", #expr, cudaGetErrorString(_e));          \
      return QMOE_ERR_CUDA;                                                       \
    }                                                                             \
  } while (0)

inline size_t dtype_bytes(int dtype) {
  switch (dtype) {
    case QMOE_F64: return 8;
    case QMOE_F32: return 4;
    case QMOE_BF16: return 2;
    default: return 0;
  }
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Bit of the current device in a per-call-site mask: function attributes such as
// cudaFuncAttributeMaxDynamicSharedMemorySize are per device, so a process driving several GPUs
// must set them once on each.
inline uint64_t current_device_bit() {
  int dev = 0;
  cudaGetDevice(&dev);
  return 1ull << (dev & 63);
}

// ---- programmatic dependent launch (PDL) -----------------------------------------------
// The hot-path kernels (router, permute, expert FFN, split-K reduce, combine) are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization: a kernel may be scheduled while its
// predecessor in the stream is still running, and blocks in pdl_wait() -- its first statement,
// before any global memory access -- until the predecessor grid has completed and its writes are
// visible.  pdl_trigger() right after lets this kernel's own successor be scheduled as soon as all
// of this grid's CTAs are resident, so a layer's 5-7 dependent launches do not pay a full
// launch latency each.  Launched without the attribute both are no-ops.  QMOE_PDL=0 disables it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("QMOE_PDL");
    return v == nullptr || atoi(v) != 0;
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline int launch_pdl(const char* what, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                      Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    set_error("%s: %s", what, cudaGetErrorString(e));
    return QMOE_ERR_CUDA;
  }
  return QMOE_OK;
}

// ---- element conversion ---------------------------------------------------------------
template <typename T> __device__ __forceinline__ float to_f32(T v);
template <> __device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// Accumulator-precision load: bf16/f32 inputs accumulate in f32, f64 in f64.
template <typename T> struct AccOf { using type = float; };
template <> struct AccOf<double> { using type = double; };

template <typename T, typename A> __device__ __forceinline__ A load_as(const T* p) {
  return static_cast<A>(to_f32<T>(*p));
}
template <> __device__ __forceinline__ double load_as<double, double>(const double* p) { return *p; }

template <typename T, typename A> __device__ __forceinline__ void store_from(T* p, A v) {
  *p = from_f32<T>(static_cast<float>(v));
}
template <> __device__ __forceinline__ void store_from<double, double>(double* p, double v) { *p = v; }

__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

}  // namespace qmoe
