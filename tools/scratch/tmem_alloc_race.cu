// Minimal repro for the compute-sanitizer racecheck reports at tmem_alloc_cg2 (tc_ptx.cuh): a CTA
// pair allocates TMEM with tcgen05.alloc.cta_group::2 (the instruction writes the TMEM address to
// shared memory), orders it with tcgen05.fence::before_thread_sync + barrier.cluster + __syncthreads
// + tcgen05.fence::after_thread_sync, and every thread reads the address -- the handoff the
// expert kernels use.  Variant 1 (relay): warp 2 lane 0 re-stores the address with a plain st.shared
// into a second variable before the barriers and the other threads read that one.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tmem_race tools/scratch/tmem_alloc_race.cu
//   compute-sanitizer --tool racecheck /tmp/tmem_race 0   (direct read)
//   compute-sanitizer --tool racecheck /tmp/tmem_race 1   (relay)
#include <cstdio>
#include <cstdlib>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __cluster_dims__(2, 1, 1) alloc_kernel(uint32_t* out, int relay) {
  __shared__ uint32_t tmem_base_smem;
  __shared__ uint32_t tmem_base_relay;
  const int warp = threadIdx.x >> 5;
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base_smem))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    if (relay && (threadIdx.x & 31) == 0) {
      uint32_t v;
      asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(&tmem_base_smem)) : "memory");
      tmem_base_relay = v;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t base = relay ? tmem_base_relay : tmem_base_smem;
  out[blockIdx.x * blockDim.x + threadIdx.x] = base;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(base) : "memory");
  }
}

int main(int argc, char** argv) {
  const int relay = argc > 1 ? atoi(argv[1]) : 0;
  uint32_t* out = nullptr;
  cudaMalloc(&out, 2 * 256 * sizeof(uint32_t));
  alloc_kernel<<<2, 256>>>(out, relay);
  cudaError_t e = cudaDeviceSynchronize();
  uint32_t h[512];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  bool same = true;
  for (int i = 0; i < 512; ++i) same = same && h[i] == h[(i / 256) * 256];
  printf("relay=%d status=%s base0=%u base1=%u uniform=%d\n", relay, cudaGetErrorString(e), h[0], h[256], same);
  return e == cudaSuccess && same ? 0 : 1;
}
