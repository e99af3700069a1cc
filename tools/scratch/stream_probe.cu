// Read-bandwidth probe for the router's access pattern (X: T x d bf16, 16-token CTAs, d split over
// 8 warps): how fast can 512 CTAs stream 67 MB when (0) a CTA just loads its rows and xor-reduces,
// (1) it also reads W_router rows (8 x d) from L2 per k step, (2) it grid-strides 4 tiles per CTA
// (148 x 4 persistent CTAs).  Isolates the memory pattern from the MMA / selection work.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/stream_probe tools/scratch/stream_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>

__device__ __forceinline__ uint4 ldg_nc(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

template <int MODE, int U>
__global__ void __launch_bounds__(256) probe(const __nv_bfloat16* x, const __nv_bfloat16* w, int T, int d,
                                             unsigned* sink) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int dq = d / 8, k0 = warp * dq;
  unsigned acc = 0;
  const int ntiles = (T + 15) / 16;
  const int step = MODE == 2 ? gridDim.x : ntiles;
  for (int tile = blockIdx.x; tile < ntiles; tile += step) {
    const uint4* r0 = reinterpret_cast<const uint4*>(x + (size_t)(tile * 16 + g) * d + k0) + t4;
    const uint4* r1 = reinterpret_cast<const uint4*>(x + (size_t)(tile * 16 + g + 8) * d + k0) + t4;
    const uint4* wr = reinterpret_cast<const uint4*>(w + (size_t)g * d + k0) + t4;
    for (int s = 0; s < dq / 32; s += U) {
      uint4 a[U], b[U], c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        a[u] = ldg_nc(r0 + 4 * (s + u));
        b[u] = ldg_nc(r1 + 4 * (s + u));
        if (MODE >= 1) c[u] = __ldg(wr + 4 * (s + u));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        acc ^= a[u].x ^ a[u].y ^ a[u].z ^ a[u].w ^ b[u].x ^ b[u].w;
        if (MODE >= 1) acc ^= c[u].x ^ c[u].w;
      }
    }
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

template <int MODE, int U>
float run(const __nv_bfloat16* x, const __nv_bfloat16* w, int T, int d, unsigned* sink, int grid) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) probe<MODE, U><<<grid, 256>>>(x, w, T, d, sink);
  float best = 1e9f;
  for (int i = 0; i < 10; ++i) {
    cudaEventRecord(a);
    probe<MODE, U><<<grid, 256>>>(x, w, T, d, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  const int T = 8192, d = 4096;
  __nv_bfloat16 *x, *w;
  unsigned* sink;
  cudaMalloc(&x, (size_t)T * d * 2);
  cudaMalloc(&w, (size_t)8 * d * 2);
  cudaMalloc(&sink, 4);
  cudaMemset(x, 1, (size_t)T * d * 2);
  cudaMemset(w, 1, (size_t)8 * d * 2);
  const double gb = (double)T * d * 2 / 1e9;
  const int tiles = T / 16;
  float t;
  t = run<0, 2>(x, w, T, d, sink, tiles); printf("loads only, U=2, %d CTAs: %.1f us  %.0f GB/s\n", tiles, t * 1e3, gb / t * 1e3);
  t = run<0, 4>(x, w, T, d, sink, tiles); printf("loads only, U=4, %d CTAs: %.1f us  %.0f GB/s\n", tiles, t * 1e3, gb / t * 1e3);
  t = run<1, 2>(x, w, T, d, sink, tiles); printf("+W rows,   U=2, %d CTAs: %.1f us  %.0f GB/s\n", tiles, t * 1e3, gb / t * 1e3);
  t = run<1, 4>(x, w, T, d, sink, tiles); printf("+W rows,   U=4, %d CTAs: %.1f us  %.0f GB/s\n", tiles, t * 1e3, gb / t * 1e3);
  t = run<2, 4>(x, w, T, d, sink, 148 * 4); printf("+W rows, persistent 592 CTAs, U=4: %.1f us  %.0f GB/s\n", t * 1e3, gb / t * 1e3);
  t = run<2, 4>(x, w, T, d, sink, 148 * 2); printf("+W rows, persistent 296 CTAs, U=4: %.1f us  %.0f GB/s\n", t * 1e3, gb / t * 1e3);
  return 0;
}
