"""CPU oracle for the preemptive MoE hot path — TEST INFRASTRUCTURE ONLY.

A plain-numpy restatement of the reference algorithm (moesim, /root/reference/pkg/src/moesim),
used exclusively as the checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs.  The product path (paper_2503_09304_b200) never imports this module.

Parity pinning: the toy-model functions below are pinned against the reference's own golden
fixtures (reference tests/test_model.py:21-23) and against outputs of the reference itself,
generated in this container by tests/golden/gen_golden.py and committed under tests/golden/.
The SwiGLU / Qwen functions have NO counterpart in the reference: they restate the named
third-party source, HF transformers 5.5.0 (MixtralTopKRouter / MixtralExperts /
MixtralSparseMoeBlock, modeling_mixtral.py; Qwen2MoeTopKRouter / Qwen2MoeMLP /
Qwen2MoeSparseMoeBlock, modeling_qwen2_moe.py), and are pinned against those installed modules
run in fp64 on CPU (tests/test_hf_parity.py).

Every function cites the reference file:line it restates (paths relative to pkg/src/moesim/).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

NORM_EPS = 1e-9          # model.py:21
EOS_LOGIT_PENALTY = 0.5  # model.py:30
EOS_TOKEN = 0            # core.py:17


@dataclass(frozen=True)
class ToyConfig:
    """model.py:33-50 (ModelConfig)."""

    num_layers: int = 8
    hidden_dim: int = 16
    num_experts: int = 8
    top_k: int = 2
    vocab_size: int = 256
    seed: int = 0


class ToyParams:
    """Seeded parameters in the reference's exact draw order (model.py:86-102):
    embedding; w_key[l] for all l; w_value[l]; w_router[l]; expert_weight[l]; expert_bias[l];
    w_out; b_out — all standard_normal from one default_rng(seed), all but the embedding scaled
    by 1/sqrt(d); then b_out[0] -= EOS_LOGIT_PENALTY."""

    def __init__(self, cfg: ToyConfig):
        d, e, v, L = cfg.hidden_dim, cfg.num_experts, cfg.vocab_size, cfg.num_layers
        rng = np.random.default_rng(cfg.seed)
        s = 1.0 / math.sqrt(d)
        self.cfg = cfg
        self.embedding = rng.standard_normal((v, d))
        self.w_key = [rng.standard_normal((d, d)) * s for _ in range(L)]
        self.w_value = [rng.standard_normal((d, d)) * s for _ in range(L)]
        self.w_router = [rng.standard_normal((e, d)) * s for _ in range(L)]
        self.expert_weight = [rng.standard_normal((e, d, d)) * s for _ in range(L)]
        self.expert_bias = [rng.standard_normal((e, d)) * s for _ in range(L)]
        self.w_out = rng.standard_normal((v, d)) * s
        self.b_out = rng.standard_normal(v) * s
        self.b_out[0] -= EOS_LOGIT_PENALTY


# ---------------------------------------------------------------------------------------------
# router (model.py:71-80, 112-134)

def topk_lower_id(scores: np.ndarray, k: int) -> list[int]:
    """k largest by (score desc, id asc), returned ascending (model.py:71-75)."""
    vals = scores.tolist()
    order = sorted(range(len(vals)), key=lambda e: (-vals[e], e))
    return sorted(order[:k])


def softmax(v: np.ndarray) -> np.ndarray:
    """model.py:78-80."""
    z = np.exp(v - v.max())
    return z / z.sum()


def route(w_router: np.ndarray, h: np.ndarray, k: int) -> tuple[list[int], np.ndarray]:
    """One token: logits = W_r h, top-k, softmax over the picked logits (model.py:115-120)."""
    scores = w_router @ h
    ids = topk_lower_id(scores, k)
    return ids, softmax(scores[ids])


def route_many(w_router: np.ndarray, H: np.ndarray, k: int) -> tuple[np.ndarray, np.ndarray]:
    """Row-wise route (model.py:122-134): ids [T,k] ascending, weights [T,k]."""
    T = H.shape[0]
    ids = np.zeros((T, k), dtype=np.int64)
    w = np.zeros((T, k))
    scores = H @ w_router.T
    for t in range(T):
        sel = topk_lower_id(scores[t], k)
        ids[t] = sel
        w[t] = softmax(scores[t, sel])
    return ids, w


def route_many_qwen(w_router: np.ndarray, H: np.ndarray, k: int) -> tuple[np.ndarray, np.ndarray]:
    """HF Qwen2-MoE with norm_topk_prob=False (parity unpinned): p = softmax over all experts,
    top-k of p (lower id wins ties), weights = p[ids] without renormalisation, ids ascending."""
    scores = H @ w_router.T
    T = H.shape[0]
    ids = np.zeros((T, k), dtype=np.int64)
    w = np.zeros((T, k))
    for t in range(T):
        p = softmax(scores[t])
        sel = topk_lower_id(p, k)
        ids[t] = sel
        w[t] = p[sel]
    return ids, w


# ---------------------------------------------------------------------------------------------
# per-expert queues (engine.py:312-328, model.py:195-214)

def expert_queues(ids: np.ndarray, cursor: np.ndarray | None, num_experts: int) -> list[list[int]]:
    """FIFO of slot indices s = t*k + j per expert: members -> tokens -> sorted pending experts
    (engine.py:314-318) appended to the expert's deque, drained in ascending expert id."""
    T, k = ids.shape
    queues: list[list[int]] = [[] for _ in range(num_experts)]
    for t in range(T):
        for j in range(k):
            e = int(ids[t, j])
            if cursor is not None and e < int(cursor[t]):
                continue  # completed before the preemption: not pending (engine.py:315-317)
            queues[e].append(t * k + j)
    return queues


def permute(ids: np.ndarray, cursor: np.ndarray | None, num_experts: int) -> tuple[np.ndarray, np.ndarray]:
    """(perm, offsets[E+1]) — the concatenation of expert_queues in ascending expert id."""
    q = expert_queues(ids, cursor, num_experts)
    perm = np.array([s for lst in q for s in lst], dtype=np.int64)
    offsets = np.zeros(num_experts + 1, dtype=np.int64)
    offsets[1:] = np.cumsum([len(lst) for lst in q])
    return perm, offsets


# ---------------------------------------------------------------------------------------------
# experts (model.py:136-145) and the HF SwiGLU expert (parity unpinned)

def expert_tanh(A: np.ndarray, b: np.ndarray, X: np.ndarray) -> np.ndarray:
    """tanh(A x + b) row-wise (model.py:141-145); A is [out, in]."""
    return np.tanh(X @ A.T + b)


def silu(x: np.ndarray) -> np.ndarray:
    return x / (1.0 + np.exp(-x))


def expert_swiglu(gate_up: np.ndarray, down: np.ndarray, X: np.ndarray) -> np.ndarray:
    """HF MixtralExperts.forward per expert: gate, up = (x W13^T).chunk(2); down(silu(gate)*up)."""
    F = gate_up.shape[0] // 2
    h = X @ gate_up.T
    return (silu(h[:, :F]) * h[:, F:]) @ down.T


def sigmoid(x: np.ndarray) -> np.ndarray:
    return 1.0 / (1.0 + np.exp(-x))


def sparse_moe_block(w_router: np.ndarray, gate_up: np.ndarray, down: np.ndarray, H: np.ndarray, k: int,
                     qwen: bool = False, shared_gate_up: np.ndarray | None = None,
                     shared_down: np.ndarray | None = None, shared_gate: np.ndarray | None = None):
    """HF MixtralSparseMoeBlock.forward (qwen=False: softmax over the k picked logits == HF's
    softmax -> top-k -> renormalise) or Qwen2MoeSparseMoeBlock.forward with norm_topk_prob=False
    (qwen=True: weights are the full softmax at the picked ids), plus the sigmoid-gated shared
    expert when its weights are given: out = sum_j w_j expert_{id_j}(h) + sigmoid(g.h) shared(h).
    Routed terms are summed in ascending expert id (reference engine.py:358-360).
    Returns (ids, w, out)."""
    ids, w = (route_many_qwen if qwen else route_many)(w_router, H, k)
    T = H.shape[0]
    Y = np.zeros((T, k, H.shape[1]))
    for e, q in enumerate(expert_queues(ids, None, gate_up.shape[0])):
        if q:
            rows = np.array(q)
            Y.reshape(T * k, -1)[rows] = expert_swiglu(gate_up[e], down[e], H[rows // k])
    out = combine(None, w, Y)
    if shared_gate_up is not None:
        out = out + sigmoid(H @ shared_gate.reshape(-1))[:, None] * expert_swiglu(shared_gate_up, shared_down, H)
    return ids, w, out


# ---------------------------------------------------------------------------------------------
# combine (engine.py:330-365, model.py:147-164)

def combine(residual: np.ndarray | None, w: np.ndarray, Y: np.ndarray) -> np.ndarray:
    """acc = residual; acc = acc + w[:, j] * Y[:, j] for j ascending expert id (engine.py:358-360).
    Y is [T, k, d] in the same j order as w."""
    acc = np.zeros(Y[:, 0].shape) if residual is None else residual.copy()
    for j in range(w.shape[1]):
        acc = acc + w[:, j][:, None] * Y[:, j]
    return acc


def moe_layer_tanh(A: np.ndarray, b: np.ndarray, w_router: np.ndarray, H: np.ndarray, k: int,
                   residual: np.ndarray | None = None):
    """Router -> queues -> experts -> combine for one layer of the toy model."""
    ids, w = route_many(w_router, H, k)
    T = H.shape[0]
    Y = np.zeros((T, k, H.shape[1]))
    for e, q in enumerate(expert_queues(ids, None, A.shape[0])):
        if q:
            rows = np.array(q)
            Y.reshape(T * k, -1)[rows] = expert_tanh(A[e], b[e], H[rows // k])
    return ids, w, Y, combine(H if residual is None else residual, w, Y)


# ---------------------------------------------------------------------------------------------
# toy attention / emission and the straight-line generator (model.py:53-68, 104-110, 166-169;
# tests/reference.py:18-49)

def normalize(v: np.ndarray) -> np.ndarray:
    return v / (math.sqrt(float(v @ v)) + NORM_EPS)


def attend(h: np.ndarray, keys: np.ndarray, values: np.ndarray) -> np.ndarray:
    s = keys @ h
    z = np.exp(s - s.max())
    return normalize(h + (z / z.sum()) @ values)


def emit_token(p: ToyParams, h: np.ndarray) -> int:
    return int(np.argmax(p.w_out @ h + p.b_out))


def _run_tokens(p: ToyParams, kv: list[tuple[list, list]], tokens: list[int]) -> np.ndarray:
    cfg = p.cfg
    hidden = [p.embedding[t] for t in tokens]
    for layer in range(cfg.num_layers):
        keys, values = kv[layer]
        att = []
        for h in hidden:
            keys.append(p.w_key[layer] @ h)
            values.append(p.w_value[layer] @ h)
            att.append(attend(h, np.stack(keys), np.stack(values)))
        nxt = []
        for h in att:
            ids, w = route(p.w_router[layer], h, cfg.top_k)
            out = h.copy()
            for j, e in enumerate(ids):
                out = out + w[j] * expert_tanh(p.expert_weight[layer][e], p.expert_bias[layer][e], h[None])[0]
            nxt.append(out)
        hidden = nxt
    return hidden[-1]


def reference_generate(p: ToyParams, prompt: list[int], max_new_tokens: int) -> list[int]:
    """Zero-preemption straight-line generation (tests/reference.py:41-49)."""
    kv = [([], []) for _ in range(p.cfg.num_layers)]
    out = [emit_token(p, _run_tokens(p, kv, list(prompt)))]
    while len(out) < max_new_tokens and out[-1] != EOS_TOKEN:
        out.append(emit_token(p, _run_tokens(p, kv, [out[-1]])))
    return out


# ---------------------------------------------------------------------------------------------
# virtual clock arithmetic (engine.py:71-85)

@dataclass(frozen=True)
class Costs:
    attn_base: float = 1.2
    attn_per_token: float = 0.001
    attn_per_cached: float = 0.0003
    router_cost: float = 0.8
    expert_base: float = 0.85
    expert_per_entry: float = 0.0005
    checkpoint_cost: float = 2.0
    restore_cost: float = 2.0

    def attention(self, tokens: int, cached: int) -> float:
        return self.attn_base + self.attn_per_token * tokens + self.attn_per_cached * cached

    def expert(self, entries: int) -> float:
        return self.expert_base + self.expert_per_entry * entries
