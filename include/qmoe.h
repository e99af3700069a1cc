/*
 * qmoe.h — C ABI of libqmoe.so, the B200 (sm_100a) expert-level preemptive MoE path.
 *
 * Every entry point:
 *   - takes raw DEVICE pointers plus sizes and a cudaStream_t (passed as void*),
 *   - enqueues asynchronously on that stream, never allocates (workspace is caller-provided),
 *   - never synchronises the host (no hidden cudaDeviceSynchronize / D2H copies),
 *   - returns an int status (QMOE_OK == 0).  The Python host maps the codes onto the
 *     reference's exception classes (core.py:20-37 in the reference):
 *       QMOE_ERR_INVALID   -> ValueError
 *       QMOE_ERR_STATE     -> StateCorruptionError
 *       QMOE_ERR_PARTIAL   -> PartialTokenError
 *       QMOE_ERR_CAPACITY  -> CacheCapacityError
 *       QMOE_ERR_CUDA / QMOE_ERR_UNSUPPORTED -> RuntimeError
 *
 * The reference (moesim, pure Python/numpy) has no native boundary: these functions replace
 * the numeric calls the engine makes into its model plugin.  Each declaration cites the
 * reference call site it replaces (paths relative to /root/reference/pkg/src/moesim/).
 *
 * Layouts (all row-major, contiguous):
 *   X        [T, d]            token hidden states of one batch, member-major then token order
 *                              (engine.py:204-209 walks members -> tokens in this order)
 *   W_router [E, d]            gate weight (model.py:99 w_router[l]; HF gate.weight)
 *   ids      [T, k] int32      routed experts per token, ascending id (model.py:129)
 *   w        [T, k]            routing weights, same order as ids
 *   cursor   [T] int32         per-token resume cursor: slot (t,j) is pending iff ids[t,j] >= cursor[t]
 *                              (Checkpoint.pending_experts, core.py:101, compressed: experts drain
 *                              in ascending id so pending == routed ∩ {e >= cursor})
 *   perm     [R] int32         slot index s = t*k + j of the r-th entry in (expert, slot) order
 *   offsets  [E+1] int32       expert e owns perm rows [offsets[e], offsets[e+1])
 *   Xp       [R, d]            X rows gathered in perm order (Xp[r] = X[perm[r] / k])
 *   Y        [T*k, d]          expert outputs in SLOT order (Checkpoint.completed_expert_outputs)
 */
#ifndef QMOE_H_
#define QMOE_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define QMOE_API __attribute__((visibility("default")))
#else
#define QMOE_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---------------------------------------------------------------------- */
#define QMOE_OK 0
#define QMOE_ERR_INVALID 1
#define QMOE_ERR_STATE 2
#define QMOE_ERR_PARTIAL 3
#define QMOE_ERR_CAPACITY 4
#define QMOE_ERR_CUDA 5
#define QMOE_ERR_UNSUPPORTED 6

/* ---- element types --------------------------------------------------------------------- */
#define QMOE_F64 0  /* reference precision (model.py:7-9 computes in fp64) */
#define QMOE_F32 1
#define QMOE_BF16 2 /* production precision: bf16 operands, fp32 accumulation */

/* ---- router weight modes --------------------------------------------------------------- */
#define QMOE_ROUTE_TOPK_SOFTMAX 0 /* softmax over the k picked logits (model.py:122-134; == HF Mixtral) */
#define QMOE_ROUTE_SOFTMAX_TOPK 1 /* softmax over all E, keep top-k probs, no renorm (HF Qwen2-MoE,
                                     norm_topk_prob=False; no reference counterpart) */

/* ---- expert variants ------------------------------------------------------------------- */
#define QMOE_EXPERT_TANH_AFFINE 0 /* y = tanh(A_e x + b_e)          (model.py:141-145)        */
#define QMOE_EXPERT_SWIGLU 1      /* y = W2_e (SiLU(W1_e x) * W3_e x) (HF MixtralExperts)      */

/* ---- bf16 SwiGLU kernel paths (qmoe_expert_ffn_path) ----------------------------------- */
#define QMOE_PATH_UNSUPPORTED 0       /* d or F not a multiple of 64                              */
#define QMOE_PATH_SWAP_AB 1           /* decode-size batches: swap-AB, gate_up+down in one launch  */
#define QMOE_PATH_FUSED_1CTA 2        /* 128x256 tcgen05 tiles, gate_up+down in one launch         */
#define QMOE_PATH_FUSED_PAIR 3        /* 256x256 CTA-pair tiles, gate_up+down in one launch        */
#define QMOE_PATH_TWO_LAUNCH_1CTA 4   /* 128x256 tiles, one launch per projection (split-K small)  */
#define QMOE_PATH_TWO_LAUNCH_PAIR 5   /* 256x256 CTA-pair tiles, one launch per projection         */
#define QMOE_PATH_SWAP_PAIR 6         /* swap-AB CTA pair: 256 weight rows x <=256 tokens, 1 launch */

QMOE_API int qmoe_version(void);
QMOE_API const char* qmoe_status_string(int status);
/* Text of the last error raised on the calling thread (CUDA error string or validation msg). */
QMOE_API const char* qmoe_last_error(void);

/*
 * Router (replaces MoEModel.route / route_many, model.py:115-134, called from
 * InferenceEngine._router_stage, engine.py:303-310).
 * logits = W_router · x per token, accumulated in fp32 (fp64 when dtype == QMOE_F64);
 * top-k by (logit desc, id asc) — lower id wins ties (model.py:71-75) — ids written ascending.
 * w_out has dtype F64 when dtype == QMOE_F64, else F32.  logits_out (optional, same float type
 * as w_out) receives the raw [T, E] logits.  Requires 1 <= k <= E <= 64, k <= 8.
 */
QMOE_API int qmoe_router(const void* x, const void* w_router, int T, int d, int E, int k, int dtype,
                int route_mode, int32_t* ids_out, void* w_out, void* logits_out, void* stream);
/*
 * Router with a sigmoid-gated shared expert folded into the routing (HF Qwen2MoeSparseMoeBlock:
 * out = sum_j w_j expert_j(h) + sigmoid(shared_expert_gate . h) * shared_expert(h)), for running
 * the shared expert as n_shared extra "experts" of the routed width in the same grouped launch
 * (a SwiGLU of width F*n_shared is the sum of n_shared SwiGLUs over its F-wide column blocks).
 * w_router has E + 1 rows when n_shared > 0: the E routed experts, then the shared gate.
 * ids_out / w_out are [T, k + n_shared]: the k routed picks (as qmoe_router), then ids
 * E .. E+n_shared-1 with weight sigmoid(gate logit).  logits_out (optional) is [T, E + 1].
 * n_shared = 0 is qmoe_router.  Requires k + n_shared <= 8 and E + 1 <= 64.
 */
QMOE_API int qmoe_router_shared(const void* x, const void* w_router, int T, int d, int E, int k, int n_shared,
                                int dtype, int route_mode, int32_t* ids_out, void* w_out, void* logits_out,
                                void* stream);

/*
 * Permute (replaces _enqueue_expert_work + ExpertQueues.enqueue/drain, engine.py:312-328,
 * model.py:195-214, and the per-expert gather engine.py:207-209).
 * Stable counting sort of the pending slots s = t*k + j by expert id: entries of one expert
 * keep flat (member, token, j) order — exactly the FIFO order of the reference's (expert, layer)
 * queue.  Writes perm, offsets[E+1] (offsets[E] = R), and, when x/xp are given, the gathered
 * rows Xp (row_bytes = d * element size).  cursor may be NULL (all slots pending).
 * workspace: qmoe_permute_workspace_bytes(T, k, E) bytes of device memory.
 */
QMOE_API size_t qmoe_permute_workspace_bytes(int T, int k, int E);
QMOE_API int qmoe_permute(const int32_t* ids, const int32_t* cursor, int T, int k, int E,
                 int32_t* perm_out, int32_t* offsets_out, void* workspace, size_t workspace_bytes,
                 const void* x, void* xp, size_t row_bytes, void* stream);

/*
 * Grouped expert FFN over experts [e_begin, e_end) (replaces the drain loop body
 * engine.py:205-215 → MoEModel.expert_forward_many, model.py:141-145).
 * Reads Xp rows [offsets[e], offsets[e+1]) for each expert, writes Y[perm[r]] (slot order).
 *   TANH_AFFINE: w1 = A [E, d, d] ([out, in]), w2 = b [E, d]; F ignored.
 *   SWIGLU     : w1 = gate_up [E, 2F, d] (rows [0,F) gate, [F,2F) up), w2 = down [E, d, F];
 *                act_ws = [R, F] scratch of the input dtype.
 * dtype QMOE_BF16 runs on tcgen05/TMEM tensor cores (TMA-fed); F32/F64 run the SIMT path used
 * for bit-faithful parity builds.
 * preempt_flag (optional, device-visible, e.g. mapped host memory): 0 = run on; s > 0 requests a
 * stop at the first expert boundary >= s (experts < s always complete).  Polled at every tile
 * claim, so the launch stops at the next expert boundary without a host round trip.  cursor_out (optional, device
 * int32[1]) receives the first expert NOT completed (== e_end when the launch ran to completion).
 * xp_rows = allocated rows of Xp / act_ws (>= offsets[E]; bounds the TMA tensor maps).
 * workspace: qmoe_expert_ffn_workspace_bytes(variant, dtype, d, xp_rows) bytes of device memory
 * (tile claim counters; for small bf16 SwiGLU batches also the fp32 split-K partials of the down
 * projection, which is then K-split so few-expert launches still fill every SM).  ZERO it once
 * when it is allocated (cudaMemset): every launch leaves its counter header zeroed again, so no
 * launch needs a memset in front of it.  Launches sharing a workspace must be stream-ordered.
 */
QMOE_API size_t qmoe_expert_ffn_workspace_bytes(int variant, int dtype, int d, int xp_rows);
QMOE_API int qmoe_expert_ffn(int variant, int dtype, const void* xp, const int32_t* offsets,
                    const int32_t* perm, int E, int d, int F, const void* w1, const void* w2,
                    int e_begin, int e_end, int xp_rows, void* act_ws, void* y,
                    const volatile int32_t* preempt_flag, int32_t* cursor_out, void* workspace,
                    size_t workspace_bytes, void* stream);

/*
 * qmoe_expert_ffn plus expert-boundary progress signals (wall-clock serving: the host answers
 * expert e's report when the GPU has drained expert e, reference engine.py:204-219).
 * progress (optional): int32[E] in pinned host memory (device-accessible, e.g. cudaHostAlloc under
 * UVA).  When the last down-projection output of expert e in [e_begin, e_end) is stored, the kernel
 * writes progress_seq into progress[e] (system-scope release).  Experts at or past a preemption
 * stop are never signalled.  Paths whose kernels cannot signal per expert (f32/f64 SIMT, the tanh
 * expert, the two-launch bf16 paths) write every progress[e] of the launch when the stream reaches
 * its end.  Use a fresh progress_seq per launch (the words are never reset).
 * Same arguments as qmoe_expert_ffn otherwise.
 */
QMOE_API int qmoe_expert_ffn_ex(int variant, int dtype, const void* xp, const int32_t* offsets, const int32_t* perm,
                                int E, int d, int F, const void* w1, const void* w2, int e_begin, int e_end,
                                int xp_rows, void* act_ws, void* y, const volatile int32_t* preempt_flag,
                                int32_t* cursor_out, int32_t* progress, int32_t progress_seq, void* workspace,
                                size_t workspace_bytes, void* stream);

/*
 * Kernel path qmoe_expert_ffn takes for a bf16 SwiGLU launch over all E experts of xp_rows routed
 * rows (QMOE_PATH_*).  Host-only, no device work.
 */
QMOE_API int qmoe_expert_ffn_path(int d, int F, int E, int xp_rows);
/*
 * Grouped bf16 SwiGLU experts reading the token rows straight from X (no gathered Xp): the i-th
 * row of expert e is X[perm[offsets[e] + i] / k], loaded by the GEMM's producer warp with TMA
 * tile::gather4 (4 arbitrary rows per instruction) -- the permute's row gather fused into the
 * A-operand (token-row) load.  For the single-launch paths (QMOE_PATH_SWAP_AB / _SWAP_PAIR /
 * _FUSED_1CTA / _FUSED_PAIR for xp_rows = T*k); other paths return QMOE_ERR_UNSUPPORTED (callers gather with
 * qmoe_permute).  Measured on B200 it does not pay: on the 128/256-row tiles it is ~2x slower
 * than qmoe_permute's gather + qmoe_expert_ffn (32 gather4 instructions per 64-wide K step per CTA
 * saturate the TMA issue path, where an Xp tile is one instruction); on the swap-AB decode path it
 * is neutral at 1-32 tokens and slower beyond.  The host paths therefore keep the Xp gather; this
 * entry serves callers that cannot afford the T*k*d Xp buffer.
 * Same outputs, preemption flag, cursor and workspace as qmoe_expert_ffn (xp_rows = T*k).
 */
QMOE_API int qmoe_expert_ffn_gather(const void* x, int T, int k, const int32_t* offsets, const int32_t* perm, int E,
                                    int d, int F, const void* gate_up, const void* down, int e_begin, int e_end,
                                    void* act_ws, void* y, const volatile int32_t* preempt_flag, int32_t* cursor_out,
                                    void* workspace, size_t workspace_bytes, void* stream);

/*
 * Combine (replaces InferenceEngine._finish_layer, engine.py:330-365, and MoEModel.combine,
 * model.py:147-164): out[t] = residual[t] + sum_j w[t,j] * Y[t*k+j], j in ascending expert id
 * (the order ids are stored in).  residual may be NULL (HF MoE-block semantics: the residual is
 * added by the caller).  F64 mode rounds each product and each sum separately, matching the
 * reference's `acc = acc + w*y` bit for bit given identical inputs.
 * The caller must have checked that no slot is pending (PartialTokenError, engine.py:344-348).
 */
QMOE_API int qmoe_combine(int dtype, const void* y, const void* w, const void* residual, int T, int k, int d,
                 void* out, void* stream);

/*
 * Row gather (restore of preempted state, engine.py:151-164 + _init_state engine.py:242-250):
 * dst[i] = src[idx[i]] for i < rows.  Used to rebuild a merged resume batch's device state from
 * per-sequence checkpoint rows without a host round trip.
 */
QMOE_API int qmoe_gather_rows(const void* src, const int32_t* idx, int rows, size_t row_bytes, void* dst,
                     void* stream);

/* Row scatter: dst[idx[i]] = src[i] for i < rows (expert-parallel return path: outputs received
 * in expert-major order go back to their token slots). */
QMOE_API int qmoe_scatter_rows(const void* src, const int32_t* idx, int rows, size_t row_bytes, void* dst,
                               void* stream);

/*
 * Cursor advance after a (possibly partial) expert launch: for every token, the next pending
 * expert becomes max(cursor[t], stop_expert) (pending = routed ∩ {e >= cursor}).  stop_expert is
 * read from device memory (the grouped GEMM's cursor_out) so no host sync is needed.
 */
QMOE_API int qmoe_cursor_advance(int32_t* cursor, int T, const int32_t* stop_expert_dev, void* stream);
/*
 * Resume point of a preempted expert stage (replaces the copy-everything checkpoint of
 * engine.py:401-423 plus the re-enqueue of pending experts at restore, engine.py:151-164,
 * 312-328): qmoe_cursor_advance, and offsets_out[e] = offsets[max(e, stop)] for e in [0, E] --
 * the preempted launch's queues with every expert below the stop emptied.  A resumed launch over
 * the same batch passes offsets_out with the first launch's perm and Xp: the pending slots of
 * experts >= stop are exactly its rows there, in the same (stable) order, so no re-permute, no
 * re-gather.  offsets may be NULL (cursor advance only).
 */
QMOE_API int qmoe_resume_point(int32_t* cursor, int T, const int32_t* stop_expert_dev, const int32_t* offsets, int E,
                               int32_t* offsets_out, void* stream);

/*
 * Paged KV ownership (replaces UnifiedDynamicCache storage, model.py:231-329).
 * pool: [n_pages, page_size, row_elems] of the given dtype; slot_mapping[i] = page*page_size +
 * offset for the i-th new row; append copies rows[i] into that slot.  The page allocator and the
 * byte ledger (reference units, entry = 2*d*8 bytes, model.py:277) live on the host.
 */
QMOE_API int qmoe_kv_append(void* pool, const int32_t* slot_mapping, const void* rows, int n_rows,
                   size_t row_bytes, void* stream);
/*
 * qmoe_kv_append that does nothing when *guard < 0 at the time it runs.  guard is the iteration's
 * expert preempt flag: a grouped expert launch that stopped early leaves it at -1, so the K/V
 * rows of the layers a run-ahead host already enqueued behind the preemption point are not
 * appended (the preempted batch resumes at the expert boundary, engine.py:401-423).
 */
QMOE_API int qmoe_kv_append_guarded(void* pool, const int32_t* slot_mapping, const void* rows, int n_rows,
                                    size_t row_bytes, const int32_t* guard, void* stream);
/*
 * qmoe_kv_append(_guarded) with source rows row_stride bytes apart (>= row_bytes): the K|V part of
 * packed qkv projection rows goes to the pool with no staging copy.  guard may be null.
 */
QMOE_API int qmoe_kv_append_strided(void* pool, const int32_t* slot_mapping, const void* rows, int n_rows,
                                    size_t row_bytes, size_t row_stride, const int32_t* guard, void* stream);
/* dst[i] = pool[slot_mapping[i]] (one sequence's entries, ascending entry order). */
QMOE_API int qmoe_kv_gather(const void* pool, const int32_t* slot_mapping, int n_rows, size_t row_bytes,
                   void* dst, void* stream);

/*
 * Expert parallelism over NVLink peer memory (no reference counterpart: the reference is a
 * single process; BASELINE north_star asks for expert-parallel dispatch/combine
 * across the GPUs of one node).  One process per GPU; peer buffers are exchanged once through
 * CUDA IPC.  Per MoE layer: qmoe_permute (no gather) -> counts all-gather (host, the same E ints
 * the scheduler's boundary timestamps need) -> qmoe_ep_dispatch -> qmoe_ep_barrier ->
 * qmoe_expert_ffn_peer -> qmoe_ep_barrier -> qmoe_combine on the local slot buffer.
 *
 * qmoe_ipc_export: 64-byte cudaIpcMemHandle of the allocation containing ptr + ptr's offset in it.
 * qmoe_ipc_import: map a peer's exported buffer (opened once per allocation, then cached).
 */
QMOE_API int qmoe_ipc_export(const void* ptr, void* handle_out, size_t* offset_out);
QMOE_API int qmoe_ipc_import(const void* handle, size_t offset, void** ptr_out);
/*
 * Fused gather + all-to-all dispatch (replaces the Xp gather of qmoe_permute, the dispatch
 * all-to-all and the owner-side regroup): the i-th pending row of expert e (queue order) is
 * stored, over peer memory, to row dest_base[e] + i of rank dest_rank[e]'s receive buffer
 * x_peers[dest_rank[e]], and ret_peers[dest_rank[e]][that row] = me << 24 | slot.
 * dest_rank / dest_base: device int32[E]; x_peers / ret_peers: device arrays of world pointers.
 */
QMOE_API int qmoe_ep_dispatch(const void* x, const int32_t* perm, const int32_t* offsets, int T, int k, int E,
                              size_t row_bytes, int me, const int32_t* dest_rank, const int32_t* dest_base,
                              void* const* x_peers, int32_t* const* ret_peers, void* stream);
/*
 * Stream-ordered device barrier over peer memory: flag_peers[g] = rank g's int32[world] flag
 * array.  Releases `epoch` to every rank (system scope, after a system fence so this rank's
 * earlier peer stores are visible) and waits until every rank released it to us.  After
 * timeout_ns the wait gives up and writes 1 to error_out (device int32, optional) instead of hanging.
 */
QMOE_API int qmoe_ep_barrier(int32_t* const* flag_peers, int me, int world, int epoch, long long timeout_ns,
                             int32_t* error_out, void* stream);
/*
 * Grouped SwiGLU expert FFN (bf16, tcgen05) over the rows a rank received: the combine
 * all-to-all is fused into the down-projection epilogue, which stores output row r straight
 * into row (ret[r] & 0xFFFFFF) of rank (ret[r] >> 24)'s slot buffer y_peers[ret[r] >> 24].
 * Same tiling, preemption-free (whole expert range), workspace as qmoe_expert_ffn.
 */
QMOE_API int qmoe_expert_ffn_peer(const void* xp, const int32_t* offsets, const int32_t* ret, int E, int d, int F,
                                  const void* gate_up, const void* down, int xp_rows, void* act_ws,
                                  void* const* y_peers, void* workspace, size_t workspace_bytes, void* stream);
/*
 * qmoe_expert_ffn_peer with the received row count left on the device and the preemption
 * contract of qmoe_expert_ffn: offsets (device, [E+1], e.g. from qmoe_ep_dispatch_dev) delimit the
 * received rows; capacity_rows bounds the receive / act buffers (TMA maps); rows_hint is the row
 * count the kernel-path heuristics assume (e.g. the rank's own T*k: with balanced routing a rank
 * receives about what it sends); experts [e_begin, e_end); preempt_flag / cursor_out as in
 * qmoe_expert_ffn.  Workspace: qmoe_expert_ffn_workspace_bytes(SWIGLU, BF16, d, capacity_rows).
 */
QMOE_API int qmoe_expert_ffn_peer_ex(const void* xp, const int32_t* offsets, const int32_t* ret, int E, int d, int F,
                                     const void* gate_up, const void* down, int capacity_rows, int rows_hint,
                                     int e_begin, int e_end, void* act_ws, void* const* y_peers,
                                     const volatile int32_t* preempt_flag, int32_t* cursor_out, void* workspace,
                                     size_t workspace_bytes, void* stream);
/*
 * Per-layer queue-length exchange over peer memory, no host round trip: every rank stores its E
 * queue lengths (from its qmoe_permute offsets) into row `me` of every peer's counts[world][E]
 * (counts_peers[g] = rank g's buffer), then the flag barrier of qmoe_ep_barrier (epoch, timeout,
 * error_out as there).  Afterwards every rank holds all ranks' counts.
 */
QMOE_API int qmoe_ep_exchange_counts(const int32_t* offsets, int E, int me, int world, int32_t* const* counts_peers,
                                     int32_t* const* flag_peers, int epoch, long long timeout_ns, int32_t* error_out,
                                     void* stream);
/*
 * qmoe_ep_dispatch with the dispatch tables computed on the device from the exchanged counts
 * (counts: this rank's [world][E] copy; bounds: device int32 [world+1], rank g owns experts
 * [bounds[g], bounds[g+1])), plus loc_offsets (device int32 [local experts + 1]): the received
 * row ranges of this rank's own experts, for qmoe_expert_ffn_peer_ex.
 */
QMOE_API int qmoe_ep_dispatch_dev(const void* x, const int32_t* perm, const int32_t* offsets, int T, int k, int E,
                                  size_t row_bytes, int me, int world, const int32_t* counts, const int32_t* bounds,
                                  void* const* x_peers, int32_t* const* ret_peers, int32_t* loc_offsets, void* stream);

/*
 * Replicated-attention expert parallelism (ep_serving.py; replaces nothing in the reference, which
 * is single-process -- SURVEY.md §8(e)): every rank holds the same batch, permutes it over all E
 * experts (identical perm / offsets on every rank) and runs the grouped GEMM on its own experts
 * [e_lo, e_hi) only, writing y in slot order.  qmoe_ep_share_rows then stores the rows of queue
 * positions [offsets[e_lo], offsets[e_hi]) into the same slot perm[r] of every peer's receive
 * buffer (recv_peers[g], [slots, row_bytes]; recv_peers[me] is not written), NVLink stores, no
 * host round trip.  After a qmoe_ep_barrier, qmoe_ep_collect_rows copies the rows of queue
 * positions [offsets[e_begin], offsets[e_end]) minus [offsets[skip_lo], offsets[skip_hi]) (the
 * rank's own experts) from the local receive buffer into y.  offsets: device [E+1]; max_rows: an
 * upper bound of the queue rows (grid sizing).  A receive buffer must not be re-written before
 * every rank collected from it (ep_serving.py alternates two, one barrier apart).
 */
QMOE_API int qmoe_ep_share_rows(const void* y, const int32_t* perm, const int32_t* offsets, int E, int e_lo, int e_hi,
                                int max_rows, size_t row_bytes, void* const* recv_peers, int me, int world,
                                void* stream);
QMOE_API int qmoe_ep_collect_rows(const void* recv, void* y, const int32_t* perm, const int32_t* offsets, int E,
                                  int e_begin, int e_end, int skip_lo, int skip_hi, int max_rows, size_t row_bytes,
                                  void* stream);

/*
 * qmoe_permute with the row gather limited to the queues of experts [0, gather_e_end) (Xp rows of
 * later experts are left unwritten), for qmoe_expert_ffn_xs.
 */
QMOE_API int qmoe_permute_ex(const int32_t* ids, const int32_t* cursor, int T, int k, int E, int gather_e_end,
                             int32_t* perm_out, int32_t* offsets_out, void* workspace, size_t workspace_bytes,
                             const void* x, void* xp, size_t row_bytes, void* stream);
/*
 * qmoe_expert_ffn_ex (bf16 SwiGLU) where experts [x_first, E) read their token rows straight from
 * x [T, d] instead of Xp: each such expert's queue must hold every token once in token order
 * (Qwen's shared sub-experts -- every token has one slot per sub-expert, and the stable permute
 * keeps token order), so queue row r of expert e is x row r - offsets[e] and the permute need not
 * gather it (qmoe_permute_ex with gather_e_end = x_first).  Same tiles and MMA order as the
 * gathered path (identical results).  Only the single-launch 1-CTA path
 * (QMOE_PATH_FUSED_1CTA for these d, F, E, xp_rows) supports it; otherwise QMOE_ERR_UNSUPPORTED.
 */
QMOE_API int qmoe_expert_ffn_xs(const void* xp, const int32_t* offsets, const int32_t* perm, int E, int d, int F,
                                const void* gate_up, const void* down, int e_begin, int e_end, int xp_rows,
                                void* act_ws, void* y, const volatile int32_t* preempt_flag, int32_t* cursor_out,
                                int32_t* progress, int32_t progress_seq, const void* x, int T, int x_first,
                                void* workspace, size_t workspace_bytes, void* stream);

/*
 * Decoder-side fused helpers (outside the north-star path; used by the Mixtral/Qwen serving
 * plugin to cut per-layer launch counts).  bf16 only.
 * qmoe_rmsnorm: out = rmsnorm(x [+ residual_add]) * weight (HF MixtralRMSNorm rounding);
 *               when residual_add is given, sum_out = x + residual_add (bf16) is written too.
 * qmoe_rope:    in-place rotate-half RoPE of q [T, n_heads, hd] and k [T, n_kv_heads, hd] (row
 *               strides q_stride / k_stride elements) at positions[T], cos/sin tables fp32 [P, hd].
 */
QMOE_API int qmoe_rmsnorm(const void* x, const void* residual_add, const void* weight, float eps, int T, int d,
                          void* out, void* sum_out, void* stream);
QMOE_API int qmoe_rope(void* q, void* k, const int64_t* positions, const float* cos_table, const float* sin_table,
                       int T, int n_heads, int n_kv_heads, int head_dim, int q_stride, int k_stride, void* stream);

/*
 * Greedy emission on the device (replaces MoEModel.emit_token, model.py:166-169, for the bf16
 * decoders): tokens_out[t] = argmax_v (w_out[v] . h[t]), lowest id on ties (numpy's first
 * maximum), fp32 accumulation; the [T, V] logits are never written.  h: [T, d] bf16 (final-normed
 * hidden rows), w_out: [V, d] bf16.  T <= 64, d % 128 == 0.  workspace:
 * qmoe_lm_head_argmax_workspace_bytes() bytes of device memory, ZEROED once at allocation (each
 * launch leaves it zeroed).  One launch; launches sharing a workspace must be stream-ordered.
 */
/*
 * Paged GQA decode attention over the engine's KV page pool (the decoders' attention stage at
 * decode; reference counterpart: the attention stage engine.py:252-301, a toy single-head
 * attention).  q: B rows of [H, head_dim] bf16, q_stride elements apart (one query token per
 * sequence, RoPE applied; e.g. rows of a packed qkv projection);
 * pool: [n_pages, page_size, 2, KV, head_dim] bf16 (K then V); block_table: [B, max_pages] int32;
 * seq_lens: [B] cached tokens incl. the new one (the query attends all of them); max_len >=
 * max(seq_lens) (host-known); scale: softmax scale.  out: [B, H, head_dim] bf16.  fp32 scores,
 * online softmax and accumulation; one CTA per (sequence, KV head, page), pages merged in order
 * by the last CTA (deterministic).  head_dim 64 or 128, H / KV in {1, 2, 4}, B * KV <= 8192.  workspace:
 * qmoe_paged_decode_attention_workspace_bytes(B, KV, max_pages) bytes, ZEROED once at allocation;
 * the arrival counters sit at its head at a fixed offset and each launch leaves them zeroed, so one
 * workspace (of the largest size needed) serves calls of any shape, stream-ordered.
 */
QMOE_API size_t qmoe_paged_decode_attention_workspace_bytes(int B, int KV, int max_pages);
QMOE_API int qmoe_paged_decode_attention(const void* q, int q_stride, const void* pool, const int32_t* block_table,
                                         const int32_t* seq_lens, int B, int H, int KV, int head_dim, int page_size,
                                         int max_pages, int max_len, float scale, void* out, void* workspace,
                                         size_t workspace_bytes, void* stream);
/*
 * Causal varlen GQA prefill attention (the decoders' attention stage on prefill passes; reference
 * counterpart: _prefill_attention, engine.py:252-301 / attend, model.py:58-68, a toy single-head
 * attention; replaces flash-attn's varlen kernel).  Sequence b owns rows [cu_seqlens[b],
 * cu_seqlens[b+1]) of q / k / v (bf16; rows q_stride / kv_stride elements apart, heads dense:
 * e.g. views into a packed qkv projection); query i of a sequence attends its keys 0..i.  max_len
 * >= the longest sequence (host-known).  out: [rows, out_stride] bf16, head h at columns
 * h*head_dim.  fp32 scores, online softmax and accumulation (P rounded to bf16 for P.V).  head_dim
 * 64 or 128, H a multiple of KV; q / k / v 16-byte aligned.
 */
QMOE_API int qmoe_prefill_attention(const void* q, const void* k, const void* v, int q_stride, int kv_stride,
                                    const int32_t* cu_seqlens, int B, int max_len, int H, int KV, int head_dim,
                                    float scale, void* out, int out_stride, void* stream);
QMOE_API size_t qmoe_lm_head_argmax_workspace_bytes(void);
QMOE_API int qmoe_lm_head_argmax(const void* h, const void* w_out, int T, int d, int V, int32_t* tokens_out,
                                 void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* QMOE_H_ */
