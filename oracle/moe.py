"""MoE routing, index compaction, expert FFN and layer -- oracle (TEST INFRASTRUCTURE).

Paper:
  * "Within the MoE layer, a routing mechanism selects appropriate experts for
    each token ... The outputs of these experts are then propagated to the
    final output through a weighted sum."                   (§2.1)
  * "the input tensor for expert E_i contains all the tokens that have been
    routed to E_i"; Samoyeds replaces that permuted copy by a selection array
    (SEL) of token ids                          (§3.1)
  * "a typical expert layer consists of three linear layers: gate_proj,
    up_proj, and down_proj ... aggregates the outputs from all experts with
    weighted accumulation"                                   (§4.5)
  * shared experts: "all tokens ... processed by all these shared experts in
    addition to their assigned routed experts"               (§6.2)
Readings: R9 gate normalisation (RENORM_TOPK default, SOFTMAX_ALL preset),
R10 top-k ties -> lower expert id, R10b a NaN logit ranks as -inf, R11 SiLU gated MLP, R12 bf16 intermediate,
R15 shared experts weight 1; R15b (Qwen2-MoE's gated shared expert, beyond the
paper's ungated "isolated shared experts") weight sigmoid(z) of a per-token
shared-gate logit z.
"""
from __future__ import annotations

import numpy as np

from . import bf16
from .fmt import Encoded, dense_f64

RENORM_TOPK = 0
SOFTMAX_ALL = 1


def route(logits: np.ndarray, top_k: int, mode: int = RENORM_TOPK):
    """Top-k experts per token (ties -> lower id, R10) and gate weights (fp64).

    logits: fp32 [T x E].  Returns ids int32 [T x k] (descending logit, then
    ascending id) and weights fp64 [T x k]."""
    lg = np.asarray(logits, dtype=np.float32).astype(np.float64)
    lg = np.where(np.isnan(lg), -np.inf, lg)     # reading R10b: a NaN logit ranks as -inf
    T, E = lg.shape
    if not 1 <= top_k <= E:
        raise ValueError("need 1 <= top_k <= E")
    ids = np.zeros((T, top_k), dtype=np.int32)
    w = np.zeros((T, top_k))
    for t in range(T):
        order = sorted(range(E), key=lambda e: (-lg[t, e], e))[:top_k]
        ids[t] = order
        sel = lg[t, order]
        if mode == RENORM_TOPK:                    # softmax over the selected logits
            z = np.exp(sel - sel.max())
            w[t] = z / z.sum()
        elif mode == SOFTMAX_ALL:                  # softmax over all E, no renormalisation
            z = np.exp(lg[t] - lg[t].max())
            w[t] = z[order] / z.sum()
        else:
            raise ValueError("unknown gating mode")
    return ids, w


def compact(ids: np.ndarray, weights: np.ndarray, num_experts: int):
    """Per-expert selection arrays: token ids ascending.

    Returns counts [E], offsets [E+1] (exclusive scan), sel [T*k] (expert-major,
    ascending token id within an expert), gw [T*k] aligned with sel."""
    T, k = ids.shape
    counts = np.zeros(num_experts, dtype=np.int64)
    sel_lists = [[] for _ in range(num_experts)]
    gw_lists = [[] for _ in range(num_experts)]
    for t in range(T):                               # ascending token id
        for j in range(k):
            e = int(ids[t, j])
            sel_lists[e].append(t)
            gw_lists[e].append(weights[t, j])
            counts[e] += 1
    offsets = np.zeros(num_experts + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(counts)
    sel = np.array([t for e in range(num_experts) for t in sel_lists[e]], dtype=np.int32)
    gw = np.array([g for e in range(num_experts) for g in gw_lists[e]], dtype=np.float64)
    return counts, offsets, sel, gw


def expert_ffn(wg: Encoded, wu: Encoded, wd: Encoded, x_bits: np.ndarray, sel: np.ndarray):
    """y = Wd . bf16( silu(Wg x) * (Wu x) ) for the selected tokens (R11, R12).

    Returns (y [n x d] fp64, a_bits [n x f] bf16 intermediate, S [n x d] error
    scale sum |Wd| |a|)."""
    xs = bf16.to_f64(np.asarray(x_bits)[np.asarray(sel, dtype=np.int64)])
    g = xs @ dense_f64(wg).T
    u = xs @ dense_f64(wu).T
    a_bits = bf16.from_f64(g / (1.0 + np.exp(-g)) * u)
    a = bf16.to_f64(a_bits)
    wdd = dense_f64(wd)
    return a @ wdd.T, a_bits, np.abs(a) @ np.abs(wdd).T


def moe_layer(experts, x_bits: np.ndarray, logits: np.ndarray, top_k: int,
              mode: int = RENORM_TOPK, shared=(), shared_logits=None):
    """out[t] = sum_{(e,g) in route(t)} g * y_e[t]  (+ sum_s c_s[t] y_s[t]).

    experts: list of (wg, wu, wd) Encoded; shared: same for shared experts.
    c_s[t] = 1 (R15), or, when shared_logits [T x len(shared)] fp32 is given,
    c_s[t] = 1 / (1 + exp(-shared_logits[t, s])) (R15b, computed in fp64).
    Returns (out [T x d] fp64, S [T x d] error scale)."""
    x_bits = np.asarray(x_bits)
    T = x_bits.shape[0]
    d = experts[0][2].rows
    ids, w = route(logits, top_k, mode)
    counts, offsets, sel, gw = compact(ids, w, len(experts))
    out = np.zeros((T, d))
    scale = np.zeros((T, d))
    for e, (wg, wu, wd) in enumerate(experts):
        s = sel[offsets[e]:offsets[e + 1]]
        if len(s) == 0:
            continue
        y, _, S = expert_ffn(wg, wu, wd, x_bits, s)
        g = gw[offsets[e]:offsets[e + 1]]
        for i, t in enumerate(s):
            out[t] += g[i] * y[i]
            scale[t] += abs(g[i]) * S[i]
    all_t = np.arange(T)
    for si, (wg, wu, wd) in enumerate(shared):
        y, _, S = expert_ffn(wg, wu, wd, x_bits, all_t)
        if shared_logits is None:
            c = np.ones(T)
        else:
            z = np.asarray(shared_logits, dtype=np.float32)[:, si].astype(np.float64)
            c = 1.0 / (1.0 + np.exp(-z))
        out += c[:, None] * y
        scale += np.abs(c)[:, None] * S
    return out, scale


def moe_layer_textbook(experts_dense, x_bits, logits, top_k, mode=RENORM_TOPK):
    """The permute -> dense GEMM -> un-permute formulation the paper replaces
    (P:187-189): per expert, physically copy the routed tokens, run dense
    fp64 GEMMs on decoded weights, then scatter back with the gate weight.
    Used to pin moe_layer."""
    x = bf16.to_f64(np.asarray(x_bits))
    T = x.shape[0]
    ids, w = route(logits, top_k, mode)
    d = experts_dense[0][2].shape[0]
    out = np.zeros((T, d))
    for e, (g, u, dn) in enumerate(experts_dense):
        rows = [(t, j) for t in range(T) for j in range(top_k) if ids[t, j] == e]
        if not rows:
            continue
        xp = np.stack([x[t] for t, _ in rows])                      # permuted copy
        h = xp @ g.T
        a = bf16.round_f64(h / (1.0 + np.exp(-h)) * (xp @ u.T))
        y = a @ dn.T
        for i, (t, j) in enumerate(rows):                         # un-permute
            out[t] += w[t, j] * y[i]
    return out


# ------------------------------------------------------------- EP simulation

def ep_owner(e: int, num_experts: int, world: int) -> int:
    """Contiguous expert ranges: rank r owns [r*E/P, (r+1)*E/P)."""
    return e // (num_experts // world)


def ep_dispatch_plan(ids_per_rank, weights_per_rank, num_experts: int, world: int):
    """Which token rows each rank sends where (one copy per destination rank).

    ids_per_rank[s]: [T_s x k] expert ids of rank s's tokens.  Returns
    recv[d] = list of (src, token, [(local_expert, weight), ...]) ordered by
    (source rank, token id), i.e. the receive-buffer order."""
    recv = [[] for _ in range(world)]
    for s in range(world):
        ids = ids_per_rank[s]
        ws = weights_per_rank[s]
        for t in range(ids.shape[0]):
            per_dst = {}
            for j in range(ids.shape[1]):
                e = int(ids[t, j])
                d = ep_owner(e, num_experts, world)
                per_dst.setdefault(d, []).append((e - d * (num_experts // world), float(ws[t, j])))
            for d in sorted(per_dst):
                recv[d].append((s, t, sorted(per_dst[d])))
    return recv
