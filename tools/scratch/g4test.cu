// gather4 semantics probe: load rows {r0..r3} x 64 bf16 cols with 128B swizzle; dump smem.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <vector>
__global__ void k(const __grid_constant__ CUtensorMap m, const int* rows, uint16_t* out) {
  __shared__ __align__(1024) uint16_t buf[8 * 64];
  __shared__ __align__(8) uint64_t bar;
  uint32_t s = (uint32_t)__cvta_generic_to_shared(buf);
  uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(2 * 4 * 128));
    for (int g = 0; g < 2; ++g)
      asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                   :: "r"(s + g * 512), "l"(&m), "r"(0), "r"(rows[4*g]), "r"(rows[4*g+1]), "r"(rows[4*g+2]), "r"(rows[4*g+3]), "r"(b) : "memory");
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" :: "r"(b) : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 8 * 64; i += blockDim.x) out[i] = buf[i];
}
int main(int argc, char** argv) {
  int box_rows = atoi(argv[1]);
  const int R = 64, C = 64;
  std::vector<uint16_t> h(R * C);
  for (int r = 0; r < R; ++r) for (int c = 0; c < C; ++c) h[r * C + c] = r * 256 + c;  // tag
  uint16_t* d; cudaMalloc(&d, R * C * 2); cudaMemcpy(d, h.data(), R * C * 2, cudaMemcpyHostToDevice);
  int hr[8] = {5, 17, 3, 40, 63, 0, 22, 9}; int* dr; cudaMalloc(&dr, 32); cudaMemcpy(dr, hr, 32, cudaMemcpyHostToDevice);
  uint16_t* o; cudaMalloc(&o, 8 * 64 * 2);
  void* fn; cudaDriverEntryPointQueryResult q; cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap m; cuuint64_t dims[2] = {C, R}; cuuint64_t str[1] = {C * 2}; cuuint32_t box[2] = {64, (cuuint32_t)box_rows}; cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode box_rows=%d -> %d\n", box_rows, (int)r);
  k<<<1, 128>>>(m, dr, o);
  cudaError_t e = cudaDeviceSynchronize(); printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<uint16_t> ho(8 * 64); cudaMemcpy(ho.data(), o, 8 * 64 * 2, cudaMemcpyDeviceToHost);
  // expected: smem row i holds gmem row hr[i], 16B chunk j stored at chunk j ^ (i % 8)
  int bad = 0;
  for (int i = 0; i < 8; ++i) for (int c = 0; c < 64; ++c) {
    int chunk = c / 8, within = c % 8; int pos = i * 64 + ((chunk ^ (i % 8)) * 8) + within;
    if (ho[pos] != hr[i] * 256 + c) ++bad;
  }
  printf("row0 first 8: "); for (int c = 0; c < 8; ++c) printf("%d ", ho[c]); printf("\nmismatches vs swizzled expectation: %d\n", bad);
  return 0;
}
