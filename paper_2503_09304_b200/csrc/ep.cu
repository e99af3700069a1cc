// Expert parallelism over NVLink peer memory (one process per GPU, one node).
//
// The NCCL path (ep.py, transport "nccl") moves tokens with two all-to-all-v collectives per MoE
// layer plus a regroup gather and a return scatter.  This path fuses them into the producing and
// consuming kernels instead, the B200-native way for an NVSwitch box where every peer is one
// load/store away:
//   dispatch  qmoe_ep_dispatch: one kernel gathers each routed row of the local tokens (expert-major
//             queue order from qmoe_permute) and stores it straight into the OWNING rank's receive
//             buffer at its final position (owner's local-expert-major order, source ranks in order,
//             so the owner's grouped GEMM consumes it with no regroup), together with a 32-bit return
//             address (source rank << 24 | source slot).
//   combine   the grouped expert FFN's down-projection epilogue (qmoe_expert_ffn_peer) writes every
//             output row directly into the source rank's slot buffer through that return address,
//             tile by tile as the tensor cores finish it, so the return transfer overlaps the GEMM.
//   ordering  qmoe_ep_barrier: a device-side flag barrier over peer memory (release/acquire at
//             system scope), stream-ordered, no host round trip.
// Peer buffers are exchanged once with CUDA IPC handles (qmoe_ipc_export / qmoe_ipc_import).
#include <cudaTypedefs.h>

#include <map>
#include <mutex>
#include <string>

#include "common.cuh"

namespace qmoe {
namespace {

// dst_x[g] row (dest_base[e] + i) = x[perm[r] / k] for the i-th pending row r of expert e;
// dst_ret[g][same row] = me << 24 | perm[r].  One warp per row, 16-byte vector copies.
__global__ void __launch_bounds__(256) ep_dispatch_kernel(const uint8_t* __restrict__ x, const int32_t* __restrict__ perm,
                                                          const int32_t* __restrict__ offsets, int k, int E,
                                                          size_t row_bytes, int me,
                                                          const int32_t* __restrict__ dest_rank,
                                                          const int32_t* __restrict__ dest_base,
                                                          void* const* __restrict__ x_peers,
                                                          int32_t* const* __restrict__ ret_peers) {
  __shared__ int s_off[65];
  for (int i = threadIdx.x; i <= E; i += blockDim.x) s_off[i] = offsets[i];
  __syncthreads();
  const int R = s_off[E];
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < R; r += warps) {
    int lo = 0, hi = E - 1;  // expert owning queue position r: last e with s_off[e] <= r
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= r) lo = mid; else hi = mid - 1;
    }
    const int e = lo;
    const int slot = perm[r];
    const int g = dest_rank[e];
    const size_t row = (size_t)dest_base[e] + (r - s_off[e]);
    const uint4* src = reinterpret_cast<const uint4*>(x + (size_t)(slot / k) * row_bytes);
    uint4* dst = reinterpret_cast<uint4*>(static_cast<uint8_t*>(x_peers[g]) + row * row_bytes);
    for (size_t c = lane; c < row_bytes / 16; c += 32) dst[c] = __ldg(src + c);
    if (lane == 0) ret_peers[g][row] = (me << 24) | slot;
  }
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// flags[g] = this rank's view of rank g's last barrier epoch (flags live in each rank's memory,
// flag_peers[g] = rank g's flag array).  Lane g releases `epoch` into rank g's slot `me`, then
// waits for rank g's release into our slot g.  Times out (error_out = 1) instead of hanging.
__global__ void ep_barrier_kernel(int32_t* const* flag_peers, int me, int world, int epoch, long long timeout_ns,
                                  int32_t* error_out) {
  const int g = threadIdx.x;
  __threadfence_system();  // this rank's earlier peer stores (dispatch / epilogue) before the release
  if (g < world) {
    int32_t* remote = flag_peers[g] + me;
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(remote), "r"(epoch) : "memory");
    const int32_t* mine = flag_peers[me] + g;
    const uint64_t t0 = globaltimer_ns();
    while (true) {
      int v;
      asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
      if (v - epoch >= 0) break;
      if ((long long)(globaltimer_ns() - t0) > timeout_ns) {
        if (error_out != nullptr) atomicExch(error_out, 1);
        break;
      }
      __nanosleep(256);
    }
  }
  __syncwarp();
}

// Device-side count exchange (replaces offsets D2H + host all-gather + host dispatch tables + H2D,
// the NCCL transport's per-layer host round trip): lane e < E of warp 0 reads this rank's queue
// length of expert e and stores it into row `me` of every peer's counts[world][E]; then the flag
// barrier of ep_barrier_kernel (system-scope release of the stores, acquire of every peer's).
__global__ void ep_exchange_counts_kernel(const int32_t* __restrict__ offsets, int E, int me, int world,
                                          int32_t* const* counts_peers, int32_t* const* flag_peers, int epoch,
                                          long long timeout_ns, int32_t* error_out) {
  const int t = threadIdx.x;
  for (int i = t; i < world * E; i += blockDim.x) {
    const int g = i / E, e = i - g * E;
    counts_peers[g][me * E + e] = offsets[e + 1] - offsets[e];
  }
  __syncthreads();
  if (t < 32) {
    __threadfence_system();
    if (t < world) {
      asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(flag_peers[t] + me), "r"(epoch) : "memory");
      const int32_t* mine = flag_peers[me] + t;
      const uint64_t t0 = globaltimer_ns();
      while (true) {
        int v;
        asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
        if (v - epoch >= 0) break;
        if ((long long)(globaltimer_ns() - t0) > timeout_ns) {
          if (error_out != nullptr) atomicExch(error_out, 1);
          break;
        }
        __nanosleep(128);
      }
    }
  }
}

// Dispatch with tables built on the device from the exchanged counts (counts[s][e]: rows of expert e
// rank s sends).  Owner g of expert e (bounds[g] <= e < bounds[g+1]) lays its receive buffer out
// local-expert-major, then source rank, then queue order (ep.py dispatch_tables / regroup_index),
// so the first row of this rank's expert-e block there is
//   sum_{bounds[g] <= e' < e} sum_s counts[s][e']  +  sum_{s < me} counts[s][e].
// Block 0 also writes this rank's own local offsets (its experts' received row ranges) for the
// grouped GEMM.
__global__ void __launch_bounds__(256) ep_dispatch_dev_kernel(const uint8_t* __restrict__ x,
                                                              const int32_t* __restrict__ perm,
                                                              const int32_t* __restrict__ offsets, int k, int E,
                                                              size_t row_bytes, int me, int world,
                                                              const int32_t* __restrict__ counts,
                                                              const int32_t* __restrict__ bounds,
                                                              void* const* __restrict__ x_peers,
                                                              int32_t* const* __restrict__ ret_peers,
                                                              int32_t* __restrict__ loc_offsets) {
  __shared__ int s_off[65], s_rank[64], s_base[64];
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int i = lane; i <= E; i += 32) s_off[i] = offsets[i];
    if (lane == 0) {
      for (int g = 0; g < world; ++g) {
        int base = 0;
        for (int e = bounds[g]; e < bounds[g + 1]; ++e) {
          int before = 0, all = 0;
          for (int s2 = 0; s2 < world; ++s2) {
            const int c = counts[s2 * E + e];
            all += c;
            if (s2 < me) before += c;
          }
          s_rank[e] = g;
          s_base[e] = base + before;
          if (g == me && blockIdx.x == 0) loc_offsets[e - bounds[g]] = base;
          base += all;
        }
        if (g == me && blockIdx.x == 0) loc_offsets[bounds[g + 1] - bounds[g]] = base;
      }
    }
  }
  __syncthreads();
  const int R = s_off[E];
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < R; r += warps) {
    int lo = 0, hi = E - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= r) lo = mid; else hi = mid - 1;
    }
    const int e = lo;
    const int slot = perm[r];
    const int g = s_rank[e];
    const size_t row = (size_t)s_base[e] + (r - s_off[e]);
    const uint4* src = reinterpret_cast<const uint4*>(x + (size_t)(slot / k) * row_bytes);
    uint4* dst = reinterpret_cast<uint4*>(static_cast<uint8_t*>(x_peers[g]) + row * row_bytes);
    for (size_t c = lane; c < row_bytes / 16; c += 32) dst[c] = __ldg(src + c);
    if (lane == 0) ret_peers[g][row] = (me << 24) | slot;
  }
}

// Replicated-attention expert parallelism (ep_serving.py): every rank holds the whole batch (the
// attention stage is replicated) and runs the grouped GEMM on its own experts only.  Afterwards
// each rank pushes the output rows of its experts -- queue positions [offsets[e_lo],
// offsets[e_hi]) of the launch, slot perm[r] -- into the same slot of every peer's receive buffer
// (one warp per row, 16-byte stores over NVLink), a flag barrier orders the pushes, and each rank
// copies the rows of the other ranks' experts in the launch range from its receive buffer into its
// own slot-ordered y (ep_collect).  Slots outside the launch's queues (completed before a
// preemption, or not routed) are never touched.
__global__ void __launch_bounds__(256) ep_share_kernel(const uint8_t* __restrict__ y, const int32_t* __restrict__ perm,
                                                       const int32_t* __restrict__ offsets, int e_lo, int e_hi,
                                                       size_t row_bytes, void* const* __restrict__ recv_peers,
                                                       int me, int world) {
  const int r0 = offsets[e_lo], r1 = offsets[e_hi];
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int r = r0 + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < r1; r += warps) {
    const size_t off = (size_t)perm[r] * row_bytes;
    const uint4* src = reinterpret_cast<const uint4*>(y + off);
    for (size_t c = lane; c < row_bytes / 16; c += 32) {
      const uint4 v = src[c];
      for (int g = 0; g < world; ++g)
        if (g != me) reinterpret_cast<uint4*>(static_cast<uint8_t*>(recv_peers[g]) + off)[c] = v;
    }
  }
}

__global__ void __launch_bounds__(256) ep_collect_kernel(const uint8_t* __restrict__ recv, uint8_t* __restrict__ y,
                                                         const int32_t* __restrict__ perm,
                                                         const int32_t* __restrict__ offsets, int e_begin, int e_end,
                                                         int skip_lo, int skip_hi, size_t row_bytes) {
  const int r0 = offsets[e_begin], r1 = offsets[e_end];
  const int s0 = offsets[skip_lo], s1 = offsets[skip_hi];
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int r = r0 + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < r1; r += warps) {
    if (r >= s0 && r < s1) continue;  // this rank's own experts: computed in place
    const size_t off = (size_t)perm[r] * row_bytes;
    const uint4* src = reinterpret_cast<const uint4*>(recv + off);
    uint4* dst = reinterpret_cast<uint4*>(y + off);
    for (size_t c = lane; c < row_bytes / 16; c += 32) dst[c] = src[c];
  }
}

PFN_cuMemGetAddressRange_v3020 g_range = nullptr;
std::once_flag g_range_once;
std::mutex g_ipc_mu;
std::map<std::string, void*> g_opened;  // full 64-byte IPC handle -> mapped base

}  // namespace
}  // namespace qmoe

extern "C" int qmoe_ipc_export(const void* ptr, void* handle_out, size_t* offset_out) {
  using namespace qmoe;
  QMOE_REQUIRE(ptr && handle_out && offset_out, "qmoe_ipc_export: null pointer");
  std::call_once(g_range_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
  });
  QMOE_REQUIRE(g_range != nullptr, "qmoe_ipc_export: cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (g_range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS) {
    set_error("qmoe_ipc_export: cuMemGetAddressRange failed");
    return QMOE_ERR_CUDA;
  }
  cudaIpcMemHandle_t h;
  QMOE_CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  memcpy(handle_out, &h, sizeof(h));
  *offset_out = reinterpret_cast<uintptr_t>(ptr) - static_cast<uintptr_t>(base);
  return QMOE_OK;
}

extern "C" int qmoe_ipc_import(const void* handle, size_t offset, void** ptr_out) {
  using namespace qmoe;
  QMOE_REQUIRE(handle && ptr_out, "qmoe_ipc_import: null pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  const std::string key(reinterpret_cast<const char*>(&h), sizeof(h));
  std::lock_guard<std::mutex> lock(g_ipc_mu);
  auto it = g_opened.find(key);
  void* base = nullptr;
  if (it != g_opened.end()) {
    base = it->second;
  } else {
    QMOE_CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    g_opened[key] = base;
  }
  *ptr_out = static_cast<uint8_t*>(base) + offset;
  return QMOE_OK;
}

extern "C" int qmoe_ep_dispatch(const void* x, const int32_t* perm, const int32_t* offsets, int T, int k, int E,
                                size_t row_bytes, int me, const int32_t* dest_rank, const int32_t* dest_base,
                                void* const* x_peers, int32_t* const* ret_peers, void* stream) {
  using namespace qmoe;
  QMOE_REQUIRE(T >= 0 && k >= 1 && E >= 1 && E <= 64, "qmoe_ep_dispatch: bad sizes T=%d k=%d E=%d", T, k, E);
  QMOE_REQUIRE(me >= 0 && me < 256, "qmoe_ep_dispatch: rank %d outside [0, 256)", me);
  QMOE_REQUIRE(T * k < (1 << 24), "qmoe_ep_dispatch: %d slots exceed the 24-bit return address", T * k);
  QMOE_REQUIRE(row_bytes % 16 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0,
               "qmoe_ep_dispatch: rows must be 16-byte multiples and aligned");
  if (T == 0) return QMOE_OK;
  QMOE_REQUIRE(x && perm && offsets && dest_rank && dest_base && x_peers && ret_peers, "qmoe_ep_dispatch: null pointer");
  const int rows = T * k;
  const int grid = rows / 8 + 1 < 148 * 4 ? rows / 8 + 1 : 148 * 4;
  ep_dispatch_kernel<<<grid, 256, 0, as_stream(stream)>>>(static_cast<const uint8_t*>(x), perm, offsets, k, E,
                                                          row_bytes, me, dest_rank, dest_base, x_peers, ret_peers);
  return check_launch("qmoe_ep_dispatch");
}

extern "C" int qmoe_ep_barrier(int32_t* const* flag_peers, int me, int world, int epoch, long long timeout_ns,
                               int32_t* error_out, void* stream) {
  using namespace qmoe;
  QMOE_REQUIRE(world >= 1 && world <= 32 && me >= 0 && me < world, "qmoe_ep_barrier: bad rank %d / world %d", me,
               world);
  QMOE_REQUIRE(flag_peers != nullptr, "qmoe_ep_barrier: null flag table");
  ep_barrier_kernel<<<1, 32, 0, as_stream(stream)>>>(flag_peers, me, world, epoch, timeout_ns, error_out);
  return check_launch("qmoe_ep_barrier");
}

extern "C" int qmoe_ep_exchange_counts(const int32_t* offsets, int E, int me, int world, int32_t* const* counts_peers,
                                       int32_t* const* flag_peers, int epoch, long long timeout_ns,
                                       int32_t* error_out, void* stream) {
  using namespace qmoe;
  QMOE_REQUIRE(E >= 1 && E <= 64 && world >= 1 && world <= 32 && me >= 0 && me < world,
               "qmoe_ep_exchange_counts: bad sizes E=%d me=%d world=%d", E, me, world);
  QMOE_REQUIRE(offsets && counts_peers && flag_peers, "qmoe_ep_exchange_counts: null pointer");
  ep_exchange_counts_kernel<<<1, 256, 0, as_stream(stream)>>>(offsets, E, me, world, counts_peers, flag_peers, epoch,
                                                              timeout_ns, error_out);
  return check_launch("qmoe_ep_exchange_counts");
}

extern "C" int qmoe_ep_dispatch_dev(const void* x, const int32_t* perm, const int32_t* offsets, int T, int k, int E,
                                    size_t row_bytes, int me, int world, const int32_t* counts, const int32_t* bounds,
                                    void* const* x_peers, int32_t* const* ret_peers, int32_t* loc_offsets,
                                    void* stream) {
  using namespace qmoe;
  QMOE_REQUIRE(T >= 0 && k >= 1 && E >= 1 && E <= 64, "qmoe_ep_dispatch_dev: bad sizes T=%d k=%d E=%d", T, k, E);
  QMOE_REQUIRE(world >= 1 && world <= 32 && me >= 0 && me < world, "qmoe_ep_dispatch_dev: bad rank %d/%d", me, world);
  QMOE_REQUIRE((long long)T * k < (1 << 24), "qmoe_ep_dispatch_dev: %d slots exceed the 24-bit return address", T * k);
  QMOE_REQUIRE(row_bytes % 16 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0,
               "qmoe_ep_dispatch_dev: rows must be 16-byte multiples and aligned");
  QMOE_REQUIRE(offsets && counts && bounds && loc_offsets && x_peers && ret_peers && (T == 0 || (x && perm)),
               "qmoe_ep_dispatch_dev: null pointer");
  const int rows = T * k;
  const int grid = rows / 8 + 1 < 148 * 4 ? rows / 8 + 1 : 148 * 4;
  ep_dispatch_dev_kernel<<<grid, 256, 0, as_stream(stream)>>>(static_cast<const uint8_t*>(x), perm, offsets, k, E,
                                                              row_bytes, me, world, counts, bounds, x_peers,
                                                              ret_peers, loc_offsets);
  return check_launch("qmoe_ep_dispatch_dev");
}

extern "C" int qmoe_ep_share_rows(const void* y, const int32_t* perm, const int32_t* offsets, int E, int e_lo, int e_hi,
                                  int max_rows, size_t row_bytes, void* const* recv_peers, int me, int world,
                                  void* stream) {
  using namespace qmoe;
  QMOE_REQUIRE(E >= 1 && 0 <= e_lo && e_lo <= e_hi && e_hi <= E, "qmoe_ep_share_rows: bad expert range [%d, %d) of %d",
               e_lo, e_hi, E);
  QMOE_REQUIRE(world >= 1 && world <= 32 && me >= 0 && me < world, "qmoe_ep_share_rows: bad rank %d/%d", me, world);
  QMOE_REQUIRE(row_bytes % 16 == 0 && reinterpret_cast<uintptr_t>(y) % 16 == 0,
               "qmoe_ep_share_rows: rows must be 16-byte multiples and aligned");
  if (e_lo == e_hi || max_rows <= 0 || world == 1) return QMOE_OK;
  QMOE_REQUIRE(y && perm && offsets && recv_peers, "qmoe_ep_share_rows: null pointer");
  const int grid = max_rows / 8 + 1 < 148 * 4 ? max_rows / 8 + 1 : 148 * 4;
  ep_share_kernel<<<grid, 256, 0, as_stream(stream)>>>(static_cast<const uint8_t*>(y), perm, offsets, e_lo, e_hi,
                                                       row_bytes, recv_peers, me, world);
  return check_launch("qmoe_ep_share_rows");
}

extern "C" int qmoe_ep_collect_rows(const void* recv, void* y, const int32_t* perm, const int32_t* offsets, int E,
                                    int e_begin, int e_end, int skip_lo, int skip_hi, int max_rows, size_t row_bytes,
                                    void* stream) {
  using namespace qmoe;
  QMOE_REQUIRE(E >= 1 && 0 <= e_begin && e_begin <= e_end && e_end <= E && 0 <= skip_lo && skip_lo <= skip_hi &&
                   skip_hi <= E,
               "qmoe_ep_collect_rows: bad expert ranges [%d, %d) / [%d, %d) of %d", e_begin, e_end, skip_lo, skip_hi,
               E);
  QMOE_REQUIRE(row_bytes % 16 == 0 && reinterpret_cast<uintptr_t>(y) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(recv) % 16 == 0,
               "qmoe_ep_collect_rows: rows must be 16-byte multiples and aligned");
  if (e_begin == e_end || max_rows <= 0) return QMOE_OK;
  QMOE_REQUIRE(recv && y && perm && offsets, "qmoe_ep_collect_rows: null pointer");
  const int grid = max_rows / 8 + 1 < 148 * 4 ? max_rows / 8 + 1 : 148 * 4;
  ep_collect_kernel<<<grid, 256, 0, as_stream(stream)>>>(static_cast<const uint8_t*>(recv), static_cast<uint8_t*>(y),
                                                         perm, offsets, e_begin, e_end, skip_lo, skip_hi, row_bytes);
  return check_launch("qmoe_ep_collect_rows");
}
