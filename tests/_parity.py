"""Shared helpers of the GPU parity tests (oracle on the values the device holds).

Protocol: the oracle (oracle/moe_oracle.c, fp64) is fed the
weights downloaded from the device after RNE rounding and the tokens rounded
to fp32, so a tolerance measures kernel arithmetic, not quantisation.  Ids
must be equal wherever the 2nd-3rd logit margin exceeds 1e-5 * max|logit|.
"""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

MARGIN = 1e-5


def normwise(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300))


def f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


def margin(logits, k):
    s = np.sort(np.asarray(logits, np.float64))[::-1]
    return (s[k - 1] - s[k]) / max(np.abs(logits).max(), 1e-30) if k < len(s) else np.inf


def oracle_route(orc, router, X, k):
    """gate_topk (model.cpp:69-101) of every row of X: ids, gates, logits, margins."""
    X = np.atleast_2d(X)
    ids = np.zeros((len(X), k), np.int32)
    gates = np.zeros((len(X), k))
    logits = np.zeros((len(X), router.shape[0]))
    for t, x in enumerate(X):
        ids[t], gates[t], logits[t] = orc.gate_topk(router, x, k)
    marg = np.array([margin(lg, k) for lg in logits])
    return ids, gates, logits, marg


def oracle_deltas(orc, get_expert, X, ids, gates, threads=8):
    """delta[t] = sum_j gates[t,j] * expert_ffn(ids[t,j], X[t]) in ascending
    id order (model.cpp:128-147), fp64.  get_expert(e) -> (w_in, w_gate,
    w_out) fp64; each expert is fetched once and its tokens run through the
    batched oracle in `threads` parallel chunks (ctypes releases the GIL)."""
    X = np.atleast_2d(np.asarray(X, np.float64))
    delta = np.zeros_like(X)
    for e in sorted(set(int(v) for v in np.asarray(ids).ravel())):
        rows = [(t, j) for t in range(len(X)) for j in range(ids.shape[1]) if ids[t, j] == e]
        wi, wg, wo = get_expert(e)
        toks = np.array([t for t, _ in rows])
        chunks = np.array_split(np.arange(len(rows)), min(threads, len(rows)))
        with ThreadPoolExecutor(len(chunks)) as ex:
            ys = list(ex.map(lambda c: orc.expert_ffn_batch(wi, wg, wo, X[toks[c]]), chunks))
        Y = np.concatenate(ys)
        for (t, j), y in zip(rows, Y):
            delta[t] += gates[t, j] * y
        del wi, wg, wo
    return delta


def assemble_expert(ws, l, e, mode, owner=None):
    """The full device-held expert (l, e) of a sharded model: expert
    parallelism downloads it from its owner rank; tensor parallelism
    assembles every rank's ffn slice into one set of arrays."""
    if mode == "ep":
        return ws[int(owner[l, e])].download_expert(l, e)
    d, f = ws[0].shape.hidden_dim, ws[0].shape.ffn_dim
    out = (np.zeros((f, d)), np.zeros((f, d)), np.zeros((d, f)))
    for w in ws:
        w.download_expert(l, e, out=out)
    return out
