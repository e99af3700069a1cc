// qmoe_expert_ffn entry point: validation, workspace reset/finalize, SIMT vs tcgen05 dispatch.
#include "expert_common.cuh"

namespace qmoe {
namespace {

__global__ void ffn_finalize_kernel(FfnWorkspace* ws, const int32_t* limit, int e_end, int32_t* cursor_out,
                                    volatile int32_t* flag) {
  int c = INT_MAX - ws->stop_inv;
  if (c > e_end) c = e_end;
  if (limit != nullptr && *limit < c) c = *limit;
  ws->stop = c;
  if (cursor_out != nullptr) *cursor_out = c;
  if (flag != nullptr && c < e_end) *flag = -1;  // the iteration is void from here (ffn_exit)
  ws->next = 0;  // leave the slot zeroed for the next launch (workspace invariant, expert_common.cuh)
  ws->stop_inv = 0;
}

__global__ void ffn_progress_all_kernel(int32_t* progress, int seq, int e_begin, int e_end) {
  const int e = e_begin + (int)threadIdx.x;
  if (e < e_end) asm volatile("st.release.sys.b32 [%0], %1;" ::"l"(progress + e), "r"(seq) : "memory");
}

}  // namespace

int ffn_progress_all(int32_t* progress, int seq, int e_begin, int e_end, cudaStream_t s) {
  if (progress == nullptr || e_end <= e_begin) return QMOE_OK;
  ffn_progress_all_kernel<<<1, kFfnMaxExperts, 0, s>>>(progress, seq, e_begin, e_end);
  return check_launch("qmoe_expert_ffn(progress)");
}

int ffn_finalize(FfnWorkspace* ws, const int32_t* limit, int e_end, int32_t* cursor_out, cudaStream_t s,
                 const volatile int32_t* flag) {
  ffn_finalize_kernel<<<1, 1, 0, s>>>(ws, limit, e_end, cursor_out, const_cast<volatile int32_t*>(flag));
  return check_launch("qmoe_expert_ffn(finalize)");
}

}  // namespace qmoe

extern "C" size_t qmoe_expert_ffn_workspace_bytes(int variant, int dtype, int d, int xp_rows) {
  size_t n = qmoe::kFfnHeaderBytes;
  if (variant == QMOE_EXPERT_SWIGLU && dtype == QMOE_BF16) n += qmoe::splitk_bytes(xp_rows, d);
  return n;
}

static int expert_ffn_entry(int variant, int dtype, const void* xp, const int32_t* offsets,
                               const int32_t* perm, int E, int d, int F, const void* w1, const void* w2,
                               int e_begin, int e_end, int xp_rows, void* act_ws, void* y,
                               const volatile int32_t* preempt_flag, int32_t* cursor_out, void* workspace,
                               size_t workspace_bytes, void* const* y_peers, void* stream,
                               int32_t* progress = nullptr, int progress_seq = 0, int path_rows = -1) {
  using namespace qmoe;
  QMOE_REQUIRE(variant == QMOE_EXPERT_TANH_AFFINE || variant == QMOE_EXPERT_SWIGLU,
               "qmoe_expert_ffn: unknown variant %d", variant);
  QMOE_REQUIRE(E >= 1 && E <= 64 && d >= 1, "qmoe_expert_ffn: bad sizes E=%d d=%d", E, d);
  QMOE_REQUIRE(variant == QMOE_EXPERT_TANH_AFFINE || F >= 1, "qmoe_expert_ffn: SwiGLU needs F >= 1");
  QMOE_REQUIRE(0 <= e_begin && e_begin <= e_end && e_end <= E, "qmoe_expert_ffn: bad expert range [%d, %d)",
               e_begin, e_end);
  QMOE_REQUIRE(workspace != nullptr && workspace_bytes >= qmoe_expert_ffn_workspace_bytes(variant, dtype, d, xp_rows),
               "qmoe_expert_ffn: workspace too small (%zu < %zu)", workspace_bytes,
               qmoe_expert_ffn_workspace_bytes(variant, dtype, d, xp_rows));
  QMOE_REQUIRE(offsets && w1 && y && (xp_rows == 0 || (xp && perm)), "qmoe_expert_ffn: null pointer");
  QMOE_REQUIRE(variant != QMOE_EXPERT_SWIGLU || act_ws != nullptr, "qmoe_expert_ffn: SwiGLU needs act_ws");
  QMOE_REQUIRE(variant != QMOE_EXPERT_TANH_AFFINE || w2 != nullptr, "qmoe_expert_ffn: tanh expert needs bias");
  FfnWorkspace* ws = reinterpret_cast<FfnWorkspace*>(workspace);
  cudaStream_t s = as_stream(stream);
  if (xp_rows == 0 || e_begin == e_end) {
    const int st = ffn_finalize(ws, nullptr, e_end, cursor_out, s);
    return st ? st : ffn_progress_all(progress, progress_seq, e_begin, e_end, s);
  }
  QMOE_REQUIRE(y_peers == nullptr || (dtype == QMOE_BF16 && variant == QMOE_EXPERT_SWIGLU),
               "qmoe_expert_ffn_peer: peer-memory outputs need the bf16 SwiGLU path");
  switch (dtype) {
    case QMOE_F64:
    case QMOE_F32: {
      const int st = expert_ffn_simt(variant, dtype, xp, offsets, perm, E, d, F, w1, w2, e_begin, e_end, act_ws, y,
                                     preempt_flag, cursor_out, ws, s);
      return st ? st : ffn_progress_all(progress, progress_seq, e_begin, e_end, s);
    }
    case QMOE_BF16: {
      // the single-launch kernels signal each expert as its last down unit is stored; the others
      // mark the launch's experts done when the stream reaches the end of the launch
      const int path = variant == QMOE_EXPERT_SWIGLU ? expert_ffn_path(d, F, E, path_rows < 0 ? xp_rows : path_rows)
                                                     : QMOE_PATH_UNSUPPORTED;
      const bool signals = path == QMOE_PATH_SWAP_AB || path == QMOE_PATH_SWAP_PAIR || path == QMOE_PATH_FUSED_1CTA ||
                           path == QMOE_PATH_FUSED_PAIR;
      const int st = expert_ffn_tc(variant, xp, offsets, perm, E, d, F, w1, w2, e_begin, e_end, act_ws, y,
                                   preempt_flag, cursor_out, ws, xp_rows, y_peers, s, signals ? progress : nullptr,
                                   progress_seq, path_rows);
      return st || signals ? st : ffn_progress_all(progress, progress_seq, e_begin, e_end, s);
    }
    default:
      set_error("qmoe_expert_ffn: unknown dtype %d", dtype);
      return QMOE_ERR_INVALID;
  }
}

extern "C" int qmoe_expert_ffn(int variant, int dtype, const void* xp, const int32_t* offsets,
                               const int32_t* perm, int E, int d, int F, const void* w1, const void* w2,
                               int e_begin, int e_end, int xp_rows, void* act_ws, void* y,
                               const volatile int32_t* preempt_flag, int32_t* cursor_out, void* workspace,
                               size_t workspace_bytes, void* stream) {
  return expert_ffn_entry(variant, dtype, xp, offsets, perm, E, d, F, w1, w2, e_begin, e_end, xp_rows, act_ws, y,
                          preempt_flag, cursor_out, workspace, workspace_bytes, nullptr, stream);
}

extern "C" int qmoe_expert_ffn_ex(int variant, int dtype, const void* xp, const int32_t* offsets, const int32_t* perm,
                                  int E, int d, int F, const void* w1, const void* w2, int e_begin, int e_end,
                                  int xp_rows, void* act_ws, void* y, const volatile int32_t* preempt_flag,
                                  int32_t* cursor_out, int32_t* progress, int32_t progress_seq, void* workspace,
                                  size_t workspace_bytes, void* stream) {
  return expert_ffn_entry(variant, dtype, xp, offsets, perm, E, d, F, w1, w2, e_begin, e_end, xp_rows, act_ws, y,
                          preempt_flag, cursor_out, workspace, workspace_bytes, nullptr, stream, progress,
                          progress_seq);
}

extern "C" int qmoe_expert_ffn_peer(const void* xp, const int32_t* offsets, const int32_t* ret, int E, int d, int F,
                                    const void* gate_up, const void* down, int xp_rows, void* act_ws,
                                    void* const* y_peers, void* workspace, size_t workspace_bytes, void* stream) {
  QMOE_REQUIRE(y_peers != nullptr, "qmoe_expert_ffn_peer: y_peers is null");
  return expert_ffn_entry(QMOE_EXPERT_SWIGLU, QMOE_BF16, xp, offsets, ret, E, d, F, gate_up, down, 0, E, xp_rows,
                          act_ws, const_cast<void*>(static_cast<const void*>(y_peers)), nullptr, nullptr, workspace,
                          workspace_bytes, y_peers, stream);
}

extern "C" int qmoe_expert_ffn_peer_ex(const void* xp, const int32_t* offsets, const int32_t* ret, int E, int d, int F,
                                       const void* gate_up, const void* down, int capacity_rows, int rows_hint,
                                       int e_begin, int e_end, void* act_ws, void* const* y_peers,
                                       const volatile int32_t* preempt_flag, int32_t* cursor_out, void* workspace,
                                       size_t workspace_bytes, void* stream) {
  QMOE_REQUIRE(y_peers != nullptr, "qmoe_expert_ffn_peer_ex: y_peers is null");
  QMOE_REQUIRE(rows_hint >= 0, "qmoe_expert_ffn_peer_ex: bad rows_hint %d", rows_hint);
  return expert_ffn_entry(QMOE_EXPERT_SWIGLU, QMOE_BF16, xp, offsets, ret, E, d, F, gate_up, down, e_begin, e_end,
                          capacity_rows, act_ws, const_cast<void*>(static_cast<const void*>(y_peers)), preempt_flag,
                          cursor_out, workspace, workspace_bytes, y_peers, stream, nullptr, 0,
                          rows_hint > 0 ? rows_hint : 1);
}

extern "C" int qmoe_expert_ffn_path(int d, int F, int E, int xp_rows) { return qmoe::expert_ffn_path(d, F, E, xp_rows); }

extern "C" int qmoe_expert_ffn_gather(const void* x, int T, int k, const int32_t* offsets, const int32_t* perm, int E,
                                      int d, int F, const void* gate_up, const void* down, int e_begin, int e_end,
                                      void* act_ws, void* y, const volatile int32_t* preempt_flag,
                                      int32_t* cursor_out, void* workspace, size_t workspace_bytes, void* stream) {
  using namespace qmoe;
  QMOE_REQUIRE(T >= 0 && k >= 1 && k <= 8 && E >= 1 && E <= 64 && d >= 1 && F >= 1,
               "qmoe_expert_ffn_gather: bad sizes T=%d k=%d E=%d d=%d F=%d", T, k, E, d, F);
  QMOE_REQUIRE(0 <= e_begin && e_begin <= e_end && e_end <= E, "qmoe_expert_ffn_gather: bad expert range [%d, %d)",
               e_begin, e_end);
  const int rows = T * k;
  QMOE_REQUIRE(workspace != nullptr &&
                   workspace_bytes >= qmoe_expert_ffn_workspace_bytes(QMOE_EXPERT_SWIGLU, QMOE_BF16, d, rows),
               "qmoe_expert_ffn_gather: workspace too small");
  FfnWorkspace* ws = reinterpret_cast<FfnWorkspace*>(workspace);
  cudaStream_t s = as_stream(stream);
  if (rows == 0 || e_begin == e_end) {
    return ffn_finalize(ws, nullptr, e_end, cursor_out, s);
  }
  QMOE_REQUIRE(x && offsets && perm && gate_up && down && act_ws && y, "qmoe_expert_ffn_gather: null pointer");
  QMOE_REQUIRE(((uintptr_t)x | (uintptr_t)gate_up | (uintptr_t)y | (uintptr_t)act_ws) % 16 == 0,
               "qmoe_expert_ffn_gather: buffers must be 16-byte aligned");
  const int path = expert_ffn_path(d, F, E, rows);
  if (path != QMOE_PATH_SWAP_AB && path != QMOE_PATH_SWAP_PAIR && path != QMOE_PATH_FUSED_1CTA &&
      path != QMOE_PATH_FUSED_PAIR) {
    set_error("qmoe_expert_ffn_gather: path %d has no fused row gather (use qmoe_permute's gather)", path);
    return QMOE_ERR_UNSUPPORTED;
  }
  int st = tc_init_driver();
  if (st) return st;
  if (path == QMOE_PATH_SWAP_AB)
    return expert_ffn_swap(nullptr, offsets, perm, E, d, F, gate_up, down, e_begin, e_end, act_ws, y, preempt_flag,
                           cursor_out, ws, rows, nullptr, x, T, k, s);
  if (path == QMOE_PATH_SWAP_PAIR)
    return expert_ffn_swap_pair(nullptr, offsets, perm, E, d, F, gate_up, down, e_begin, e_end, act_ws, y,
                                preempt_flag, cursor_out, ws, rows, nullptr, x, T, k, s);
  return expert_ffn_fused(nullptr, offsets, perm, E, d, F, gate_up, down, e_begin, e_end, act_ws, y, preempt_flag,
                          cursor_out, ws, rows, nullptr, path == QMOE_PATH_FUSED_PAIR, x, T, k, s);
}

extern "C" int qmoe_expert_ffn_xs(const void* xp, const int32_t* offsets, const int32_t* perm, int E, int d, int F,
                                  const void* gate_up, const void* down, int e_begin, int e_end, int xp_rows,
                                  void* act_ws, void* y, const volatile int32_t* preempt_flag, int32_t* cursor_out,
                                  int32_t* progress, int32_t progress_seq, const void* x, int T, int x_first,
                                  void* workspace, size_t workspace_bytes, void* stream) {
  using namespace qmoe;
  QMOE_REQUIRE(E >= 1 && E <= 64 && d >= 1 && F >= 1, "qmoe_expert_ffn_xs: bad sizes E=%d d=%d F=%d", E, d, F);
  QMOE_REQUIRE(0 <= e_begin && e_begin <= e_end && e_end <= E, "qmoe_expert_ffn_xs: bad expert range [%d, %d)",
               e_begin, e_end);
  QMOE_REQUIRE(0 <= x_first && x_first <= E && T >= 0, "qmoe_expert_ffn_xs: bad x_first %d / T %d", x_first, T);
  QMOE_REQUIRE(workspace != nullptr &&
                   workspace_bytes >= qmoe_expert_ffn_workspace_bytes(QMOE_EXPERT_SWIGLU, QMOE_BF16, d, xp_rows),
               "qmoe_expert_ffn_xs: workspace too small");
  FfnWorkspace* ws = reinterpret_cast<FfnWorkspace*>(workspace);
  cudaStream_t s = as_stream(stream);
  if (xp_rows == 0 || e_begin == e_end) {
    const int st = ffn_finalize(ws, nullptr, e_end, cursor_out, s);
    return st ? st : ffn_progress_all(progress, progress_seq, e_begin, e_end, s);
  }
  QMOE_REQUIRE(xp && x && offsets && perm && gate_up && down && act_ws && y, "qmoe_expert_ffn_xs: null pointer");
  QMOE_REQUIRE(((uintptr_t)xp | (uintptr_t)x | (uintptr_t)gate_up | (uintptr_t)y | (uintptr_t)act_ws) % 16 == 0,
               "qmoe_expert_ffn_xs: buffers must be 16-byte aligned");
  if (expert_ffn_path(d, F, E, xp_rows) != QMOE_PATH_FUSED_1CTA || !use_fused_tc()) {
    set_error("qmoe_expert_ffn_xs: direct-X rows need the single-launch 1-CTA path (this shape takes path %d)",
              expert_ffn_path(d, F, E, xp_rows));
    return QMOE_ERR_UNSUPPORTED;
  }
  int st = tc_init_driver();
  if (st) return st;
  return expert_ffn_fused(xp, offsets, perm, E, d, F, gate_up, down, e_begin, e_end, act_ws, y, preempt_flag,
                          cursor_out, ws, xp_rows, nullptr, false, nullptr, T, 0, s, progress, progress_seq, x,
                          x_first);
}
