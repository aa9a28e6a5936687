"""CPU oracle for the FlashBias hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module, and only as the checker or the timed
CPU baseline; the product path (paper_2505_12044_b200) never calls it.

A float64 numpy restatement of the reference algorithm
(/root/reference/pkg/src/flashbias, referred to as ``ref:`` below), batched
over leading [B, H] dims.  Parity pin: tests/test_oracle_golden.py checks it
against golden vectors produced by the reference package itself
(tests/golden/make_golden.py imports /root/reference and records outputs),
so the restatement is pinned, not merely self-consistent.  The backward has
no reference counterpart (ref: SPEC.md:183); it is the analytic gradient of
the forward, cross-checked by central finite differences in the tests.
"""

from __future__ import annotations

import math
from typing import Optional

import numpy as np

MASK_FILL = float(np.finfo(np.float64).min)  # ref: attention.py:35


def rel_max_err(got, want) -> float:
    """max|got - want| / max|want| (SURVEY §7.1 tolerance metric)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    den = np.abs(want).max()
    return float(np.abs(got - want).max() / (den if den > 0 else 1.0))


def _logits(q, k, fq, fk, premul, bias, scale):
    """scale * [q | premul fq] [k | fk]^T + bias  (ref: attention.py:186-190, 225-230)."""
    s = np.einsum("...nc,...mc->...nm", q, k) * scale
    if fq is not None:
        s = s + np.einsum("...nr,...mr->...nm", premul * fq, fk) * scale
    if bias is not None:
        s = s + bias
    return s


def materialized_attention(q, k, v, fq=None, fk=None, premul=1.0, bias=None, mask="none", scale=None):
    """softmax(logits) v with the full logit matrix (ref: attention.py:111-137)."""
    q, k, v = (np.asarray(x, dtype=np.float64) for x in (q, k, v))
    scale = 1.0 / math.sqrt(q.shape[-1]) if scale is None else scale
    s = _logits(q, k, fq, fk, premul, bias, scale)
    n, m = s.shape[-2:]
    if mask == "causal":
        s = np.where(np.triu(np.ones((n, m), dtype=bool), k=1), MASK_FILL, s)
    s = s - s.max(axis=-1, keepdims=True)  # ref: core.py:41-51
    e = np.exp(s)
    return (e / e.sum(axis=-1, keepdims=True)) @ v


def streaming_attention(q, k, v, fq=None, fk=None, premul=1.0, bias=None, mask="none", scale=None,
                        block_q=128, block_kv=128, row0=0):
    """Online-softmax streaming loop (ref: attention.py:140-202, hot loop 174-201).

    Returns (O, LSE) with LSE = logsumexp of the masked logits per row.
    Causal key blocks entirely above the diagonal are skipped (ref: 184-185).
    ``row0``: global index of q's first row (a row sample of a causal head).
    """
    q, k, v = (np.asarray(x, dtype=np.float64) for x in (q, k, v))
    fq = None if fq is None else np.asarray(fq, dtype=np.float64)
    fk = None if fk is None else np.asarray(fk, dtype=np.float64)
    bias = None if bias is None else np.asarray(bias, dtype=np.float64)
    scale = 1.0 / math.sqrt(q.shape[-1]) if scale is None else scale
    n, m = q.shape[-2], k.shape[-2]
    lead = np.broadcast_shapes(q.shape[:-2], k.shape[:-2])
    out = np.empty(lead + (n, v.shape[-1]))
    lse = np.empty(lead + (n,))
    cols = np.arange(m)
    for q0 in range(0, n, block_q):
        q1 = min(q0 + block_q, n)
        rows = np.arange(q0, q1) + row0
        mx = np.full(lead + (q1 - q0,), -np.inf)
        den = np.zeros(lead + (q1 - q0,))
        acc = np.zeros(lead + (q1 - q0, v.shape[-1]))
        for k0 in range(0, m, block_kv):
            k1 = min(k0 + block_kv, m)
            if mask == "causal" and k0 > row0 + q1 - 1:
                break
            s = np.einsum("...nc,...mc->...nm", q[..., q0:q1, :], k[..., k0:k1, :]) * scale
            if fq is not None:
                s = s + np.einsum("...nr,...mr->...nm", premul * fq[..., q0:q1, :], fk[..., k0:k1, :]) * scale
            if bias is not None:
                s = s + bias[..., q0:q1, k0:k1]
            if mask == "causal" and k1 - 1 > row0 + q0:
                s = np.where(cols[None, k0:k1] > rows[:, None], MASK_FILL, s)
            m_new = np.maximum(mx, s.max(axis=-1))
            p = np.exp(s - m_new[..., None])
            alpha = np.exp(mx - m_new)
            den = alpha * den + p.sum(axis=-1)
            acc = alpha[..., None] * acc + p @ v[..., k0:k1, :]
            mx = m_new
        out[..., q0:q1, :] = acc / den[..., None]
        lse[..., q0:q1] = mx + np.log(den)
    return out, lse


def flashbias_attention(q, k, v, fq, fk, mask="none"):
    """Widened contraction with the original 1/sqrt(C) scale (ref: attention.py:205-230)."""
    c = np.asarray(q).shape[-1]
    o, _ = streaming_attention(q, k, v, fq=fq, fk=fk, premul=math.sqrt(c), mask=mask, scale=1.0 / math.sqrt(c))
    return o


def attention_bwd(q, k, v, do, fq=None, fk=None, premul=1.0, bias=None, mask="none", scale=None):
    """Analytic backward of streaming_attention (no reference counterpart:
    ref SPEC.md:183).  With s = scale*(q k^T + premul fq fk^T) + bias,
    P = softmax(s), dP = dO V^T, dS = P (dP - rowsum(dO*O)):
      dq = scale dS k, dk = scale dS^T q, dv = P^T dO,
      dfq = scale*premul dS fk, dfk = scale*premul dS^T fq, dbias = dS
    (factor and bias gradients are summed over broadcast leading dims)."""
    q, k, v, do = (np.asarray(x, dtype=np.float64) for x in (q, k, v, do))
    scale = 1.0 / math.sqrt(q.shape[-1]) if scale is None else scale
    s = _logits(q, k, None if fq is None else np.asarray(fq, np.float64),
                None if fk is None else np.asarray(fk, np.float64), premul,
                None if bias is None else np.asarray(bias, np.float64), scale)
    n, m = s.shape[-2:]
    if mask == "causal":
        s = np.where(np.triu(np.ones((n, m), dtype=bool), k=1), -np.inf, s)
    s = s - s.max(axis=-1, keepdims=True)
    p = np.exp(s)
    p /= p.sum(axis=-1, keepdims=True)
    o = p @ v
    dp = do @ np.swapaxes(v, -1, -2)
    delta = (do * o).sum(axis=-1, keepdims=True)
    ds = p * (dp - delta)
    res = {
        "o": o,
        "dq": scale * ds @ k,
        "dk": scale * np.swapaxes(ds, -1, -2) @ q,
        "dv": np.swapaxes(p, -1, -2) @ do,
    }
    if bias is not None:  # the bias enters the logits unscaled: dlogits/dbias = dS (summed where it broadcasts)
        res["dbias"] = _reduce_to(ds, np.shape(bias))
    if fq is not None:
        fq = np.asarray(fq, np.float64)
        fk = np.asarray(fk, np.float64)
        dfq = scale * premul * ds @ fk
        dfk = scale * premul * np.swapaxes(ds, -1, -2) @ fq
        res["dfq"] = _reduce_to(dfq, fq.shape)
        res["dfk"] = _reduce_to(dfk, fk.shape)
    return res


def blocked_attention_fwd_bwd(q, k, v, do, fq=None, fk=None, premul=1.0, mask="none", scale=None,
                              block=1024, row0=0):
    """attention_bwd for ONE 2-D head at full config size, streamed over query
    blocks so memory stays O(block * M) (a 16384^2 float64 logit matrix would
    be 2 GiB per array).  Same arithmetic as attention_bwd (its analytic
    gradient of ref attention.py:111-137 / 205-230), row block by row block:
    each block sees all the keys it can attend to, so its softmax, O rows, dS
    rows, dq rows and dfq rows are final and its dK, dV, dfk contributions are
    summed.  ``row0``: global index of q's first row (q, do, fq may be a row
    sample of the head; dk, dv, dfk are then that sample's contributions).
    Returns dict(o, lse, dq, dk, dv[, dfq, dfk])."""
    q, k, v, do = (np.asarray(x, dtype=np.float64) for x in (q, k, v, do))
    scale = 1.0 / math.sqrt(q.shape[-1]) if scale is None else scale
    n, m = q.shape[0], k.shape[0]
    if fq is not None:
        fq = np.asarray(fq, np.float64) * premul
        fk = np.asarray(fk, np.float64)
    res = {"o": np.empty((n, v.shape[1])), "lse": np.empty(n), "dq": np.empty_like(q),
           "dk": np.zeros_like(k), "dv": np.zeros_like(v)}
    if fq is not None:
        res["dfq"], res["dfk"] = np.empty_like(fq), np.zeros_like(fk)
    for q0 in range(0, n, block):
        q1 = min(q0 + block, n)
        m1 = min(m, row0 + q1) if mask == "causal" else m  # keys any row of the block can see
        s = (q[q0:q1] @ k[:m1].T) * scale
        if fq is not None:
            s += (fq[q0:q1] @ fk[:m1].T) * scale
        if mask == "causal":
            s[np.arange(m1)[None, :] > np.arange(row0 + q0, row0 + q1)[:, None]] = -np.inf
        mx = s.max(axis=1, keepdims=True)
        p = np.exp(s - mx)
        den = p.sum(axis=1, keepdims=True)
        p /= den
        o = p @ v[:m1]
        dp = do[q0:q1] @ v[:m1].T
        ds = p * (dp - (do[q0:q1] * o).sum(axis=1, keepdims=True))
        res["o"][q0:q1] = o
        res["lse"][q0:q1] = (mx + np.log(den))[:, 0]
        res["dq"][q0:q1] = scale * ds @ k[:m1]
        res["dk"][:m1] += scale * ds.T @ q[q0:q1]
        res["dv"][:m1] += p.T @ do[q0:q1]
        if fq is not None:
            res["dfq"][q0:q1] = scale * premul * ds @ fk[:m1]
            res["dfk"][:m1] += scale * premul * ds.T @ (fq[q0:q1] / premul)
    return res


def chunk_attention_bwd(q, k, v, do, o, lse, fq=None, fk=None, premul=1.0, mask="none", scale=None):
    """The backward of one (query chunk, key chunk) pair of a sequence split
    across ranks (ring attention), given the GLOBAL output rows ``o`` and
    log-sum-exps ``lse`` of the query chunk: P = exp(S - lse) is then the
    exact slice of the global softmax, so the pair's dq / dk / dv / dfq / dfk
    are the exact contributions of that slice to attention_bwd's gradients."""
    q, k, v, do, o = (np.asarray(x, dtype=np.float64) for x in (q, k, v, do, o))
    scale = 1.0 / math.sqrt(q.shape[-1]) if scale is None else scale
    s = _logits(q, k, None if fq is None else np.asarray(fq, np.float64),
                None if fk is None else np.asarray(fk, np.float64), premul, None, scale)
    if mask == "causal":
        n, m = s.shape[-2:]
        s = np.where(np.triu(np.ones((n, m), dtype=bool), k=1), -np.inf, s)
    p = np.exp(s - np.asarray(lse, np.float64)[..., None])
    ds = p * (do @ np.swapaxes(v, -1, -2) - (do * o).sum(axis=-1, keepdims=True))
    res = {"dq": scale * ds @ k, "dk": scale * np.swapaxes(ds, -1, -2) @ q, "dv": np.swapaxes(p, -1, -2) @ do}
    if fq is not None:
        res["dfq"] = scale * premul * ds @ np.asarray(fk, np.float64)
        res["dfk"] = scale * premul * np.swapaxes(ds, -1, -2) @ np.asarray(fq, np.float64)
    return res


def _reduce_to(x, shape):
    """Sum x over dims where ``shape`` broadcasts (size 1 / missing)."""
    while x.ndim > len(shape):
        x = x.sum(axis=0)
    for ax, sz in enumerate(shape):
        if sz == 1 and x.shape[ax] != 1:
            x = x.sum(axis=ax, keepdims=True)
    return x


# ---------------------------------------------------------------- decomposers
def decompose_alibi(n: int, m: int, slope: float = 1.0):
    """fq_i = slope [1, i], fk_j = [-j, 1], 1-based (ref: decompose.py:37-52)."""
    i = np.arange(1, n + 1, dtype=np.float64)
    j = np.arange(1, m + 1, dtype=np.float64)
    return slope * np.column_stack([np.ones(n), i]), np.column_stack([-j, np.ones(m)])


def decompose_spatial(pos_q, pos_k, row_weights=None):
    """Rank-9 squared-distance factors (ref: decompose.py:55-81)."""
    pq = np.asarray(pos_q, np.float64)
    pk = np.asarray(pos_k, np.float64)
    fq = np.column_stack([c for d in range(3) for c in (pq[:, d] ** 2, np.ones(len(pq)), -2.0 * pq[:, d])])
    fk = np.column_stack([c for d in range(3) for c in (np.ones(len(pk)), pk[:, d] ** 2, pk[:, d])])
    if row_weights is not None:
        fq = np.asarray(row_weights, np.float64).reshape(-1)[:, None] * fq
    return fq, fk


def alibi_dense(n: int, m: int, slope: float = 1.0):
    """slope (i - j) (ref: bias.py:160-165)."""
    i = np.arange(1, n + 1, dtype=np.float64)
    j = np.arange(1, m + 1, dtype=np.float64)
    return slope * (i[:, None] - j[None, :])


def spatial_dense(pos_q, pos_k, row_weights=None):
    """(weighted) squared distance (ref: bias.py:167-178)."""
    pq = np.asarray(pos_q, np.float64)
    pk = np.asarray(pos_k, np.float64)
    d = pq[:, None, :] - pk[None, :, :]
    b = (d * d).sum(-1)
    if row_weights is not None:
        b = np.asarray(row_weights, np.float64).reshape(-1)[:, None] * b
    return b


def energy_profile(s):
    """Cumulative energy fractions (ref: decompose.py:84-95)."""
    s2 = np.asarray(s, np.float64) ** 2
    cum = np.cumsum(s2)
    tot = cum[-1] if cum.size else 0.0
    return np.ones_like(cum) if tot == 0.0 else cum / tot


def svd_decompose(b, rank: Optional[int] = None, energy: Optional[float] = None):
    """Truncated SVD factors + report dict (ref: decompose.py:98-138)."""
    b = np.asarray(b, np.float64)
    u, s, vt = np.linalg.svd(b, full_matrices=False)
    prof = energy_profile(s)
    k = int(rank) if rank is not None else min(int(np.searchsorted(prof, energy) + 1), len(s))
    root = np.sqrt(s[:k])
    fq, fk = u[:, :k] * root, vt[:k].T * root
    diff = fq @ fk.T - b
    nb = np.linalg.norm(b)
    rep = {"rank_used": k, "energy_retained": float(prof[k - 1]), "max_abs_err": float(np.abs(diff).max()),
           "rel_fro_err": float(np.linalg.norm(diff) / nb) if nb > 0 else 0.0}
    return fq, fk, rep


# ---------------------------------------------------------------- head splitting
def split_heads_by_rank(biases, energy_threshold: float, max_rank: int):
    """Rank-based head partition (ref: decompose.py:179-225): a head is "low"
    when the smallest rank retaining ``energy_threshold`` of its energy is
    <= max_rank; low heads share the subset's maximum rank rounded up to a
    multiple of 8, with factors U sqrt(s), V sqrt(s) zero-padded to it.
    Returns (low_indices, [(fq, fk)], dense_indices, common_rank)."""
    mats = [np.asarray(b, np.float64) for b in biases]
    svds = [np.linalg.svd(b, full_matrices=False) for b in mats]
    ranks = [int(np.searchsorted(energy_profile(s), energy_threshold) + 1) for _, s, _ in svds]
    low = [i for i, r in enumerate(ranks) if r <= max_rank]
    dense = [i for i in range(len(mats)) if i not in low]
    if not low:
        return [], [], dense, 0
    common = (max(ranks[i] for i in low) + 7) // 8 * 8
    factors = []
    for i in low:
        u, s, vt = svds[i]
        k_eff = min(common, len(s))
        root = np.sqrt(s[:k_eff])
        fq, fk = u[:, :k_eff] * root, vt[:k_eff].T * root
        if k_eff < common:
            fq = np.hstack([fq, np.zeros((fq.shape[0], common - k_eff))])
            fk = np.hstack([fk, np.zeros((fk.shape[0], common - k_eff))])
        factors.append((fq, fk))
    return low, factors, dense, common


# ---------------------------------------------------------------- neural factor networks
def mlp_forward(params, x):
    """Three linear layers, tanh after the first two (ref: neural.py:44-47).
    params = [w1, w2, w3, b1, b2, b3]."""
    w1, w2, w3, b1, b2, b3 = params
    h1 = np.tanh(x @ w1 + b1)
    h2 = np.tanh(h1 @ w2 + b2)
    return h2 @ w3 + b3, (x, h1, h2)


def factor_loss_and_grads(q_params, k_params, xq, xk, target):
    """MSE of yq yk^T against target and its gradients (ref: neural.py:49-60, 88-98)."""
    def back(params, cache, dy):
        w1, w2, w3 = params[:3]
        x, h1, h2 = cache
        dh2 = (dy @ w3.T) * (1.0 - h2 * h2)
        dh1 = (dh2 @ w2.T) * (1.0 - h1 * h1)
        return [x.T @ dh1, h1.T @ dh2, h2.T @ dy, dh1.sum(0), dh2.sum(0), dy.sum(0)]
    yq, cq = mlp_forward(q_params, xq)
    yk, ck = mlp_forward(k_params, xk)
    diff = yq @ yk.T - target
    g = (2.0 / diff.size) * diff
    return float(np.mean(diff * diff)), back(q_params, cq, g @ yk) + back(k_params, ck, g.T @ yq)


def glorot_params(rng, dims):
    """Reference initialisation (ref: neural.py:31-40) from an Rng-like stream."""
    ws, bs = [], []
    for fan_in, fan_out in zip(dims[:-1], dims[1:]):
        limit = np.sqrt(6.0 / (fan_in + fan_out))
        ws.append((rng.uniform(fan_in, fan_out) * 2.0 - 1.0) * limit)
        bs.append(np.zeros(fan_out))
    return ws + bs
