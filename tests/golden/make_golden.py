"""Generate the golden vectors in tests/golden/ from the REFERENCE itself.

Runs the reference's own code (oracle/_ref/libmoe_ref.so, compiled from
/root/reference/proj/src by oracle/Makefile) on the cases its own tests use
(proj/tests/test_model.cpp, test_placement.cpp, acceptance.cpp criteria 8/9)
plus the SURVEY §8c probe configs, and stores inputs + outputs as
tests/golden/golden.npz.  The GPU box has no /root/reference, so the
committed fixture is what travels.

    python tests/golden/make_golden.py [--mixtral]

--mixtral also records the Mixtral-8x7B-shaped layer (d=4096, f=14336,
seed 0, token mt19937_64(1)); it needs ~12 GB RAM and ~1 min.
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mixtral", action="store_true")
    args = ap.parse_args()
    O.build(ref=True)
    ref = O.Reference()
    orc = O.Oracle()  # only its mt19937_64/normal stream, for reproducible inputs
    g = {}

    # -- random_model / model_forward on the toy shape (test_model.cpp:217-231)
    toy = O.Shape(4, 8, 2, 32, 64, 2)
    for name, seed, tok_seed, n_tok in (("toy_s3", 3, 5, 4), ("crit8", 8, 1008, 6),
                                        ("crit9", 9, 1009, 16)):
        w = ref.random_model(toy, seed)
        toks = orc.normal(tok_seed, n_tok * toy.hidden_dim).reshape(n_tok, toy.hidden_dim)
        out, cnt, gate, kind, sink = ref.model_forward(toy, w, toks, with_sink=True,
                                                       sink_cap=n_tok * 4 * 2 * 64)
        g[f"{name}_tokens"] = toks
        g[f"{name}_out"] = out
        g[f"{name}_count"] = cnt
        g[f"{name}_gate"] = gate
        g[f"{name}_kind"] = np.int32(kind)
        g[f"{name}_sink"] = sink
        g[f"{name}_w_in0"] = w.w_in[0]
        g[f"{name}_router3"] = w.router[3]
        g[f"{name}_wsum"] = np.array([sum(float(m.sum()) for m in w.w_in),
                                      sum(float(m.sum()) for m in w.w_gate),
                                      sum(float(m.sum()) for m in w.w_out),
                                      sum(float(m.sum()) for m in w.router)])
    thr = np.array([0.001, 0.01, 0.1, 1.0])
    per_layer = []
    sink = g["crit9_sink"].reshape(16, 4, 2, 64)  # token -> layer -> expert-asc calls
    for l in range(4):
        per_layer.append(ref.sparsity_histogram(sink[:, l].reshape(-1), thr))
    g["crit9_hist"] = np.array(per_layer)
    g["hand_hist"] = ref.sparsity_histogram(np.array([0.0005, 0.05, 0.5, 2.0]), thr)

    # -- single-layer hand-composed case (test_model.cpp:193-215)
    s1 = O.Shape(1, 2, 2, 3, 4, 2)
    w = ref.random_model(s1, 42)
    x = np.array([[0.3, -0.7, 1.1]])
    out, cnt, gate, kind = ref.model_forward(s1, w, x)
    g["s42_out"] = out
    g["s42_w"] = np.concatenate([w.w_in[0].ravel(), w.w_gate[0].ravel(), w.w_out[0].ravel(),
                                 w.w_in[1].ravel(), w.w_gate[1].ravel(), w.w_out[1].ravel(),
                                 w.router[0].ravel()])
    g["s42_count"] = cnt
    g["s42_gate"] = gate

    # -- expert_ffn random instances (shape ranges of test_model.cpp:92-107)
    rs = np.random.RandomState(7)
    inst = []
    for _ in range(100):
        d, f = 2 + rs.randint(5), 2 + rs.randint(7)
        wi, wg, wo = rs.randn(f, d), rs.randn(f, d), rs.randn(d, f)
        xx = rs.randn(d)
        inst.append(np.concatenate([[d, f], wi.ravel(), wg.ravel(), wo.ravel(), xx,
                                    ref.expert_ffn(wi, wg, wo, xx)]))
    g["ffn_inst"] = np.concatenate([[len(i)] for i in inst] + inst)

    # -- gate_topk known answers (test_model.cpp:132-180) via the reference
    cases = [([3.0, 1.0, 1.0, 1.0], 2), ([2.0, 2.0, 2.0, 2.0], 2), ([1.0, 2.0, 3.0], 3)]
    rs = np.random.RandomState(11)
    for _ in range(50):
        cases.append((list(rs.randn(6) * 2.0), 3))
    topk = []
    for logits, k in cases:
        r = np.array(logits)[:, None]
        ids, wts = ref.gate_topk(r, np.array([1.0]), k)
        topk.append(np.concatenate([[len(logits), k], logits, ids, wts]))
    g["topk"] = np.concatenate([[len(t)] for t in topk] + topk)

    # -- tiny config T (SURVEY §8c probe): d=512 f=1792 E=8 L=1 seed 0, token mt(1)
    T = O.Shape(1, 8, 2, 512, 1792, 4)
    w = ref.random_model(T, 0)
    x = orc.normal(1, 512)[None]
    out, cnt, gate, kind = ref.model_forward(T, w, x)
    g["T_token"] = x
    g["T_out"] = out
    g["T_count"] = cnt
    g["T_gate"] = gate
    g["T_router"] = w.router[0]
    g["T_samples"] = np.array([[w.w_in[e][0, :4], w.w_gate[e][5, :4], w.w_out[e][7, :4]]
                               for e in range(8)])
    g["T_wsum"] = np.array([[float(w.w_in[e].sum()), float(w.w_gate[e].sum()),
                             float(w.w_out[e].sum())] for e in range(8)])

    # -- placement (test_placement.cpp:93-193, acceptance.cpp:116-183)
    rs = np.random.RandomState(21)
    pl = []
    for _ in range(60):
        L, E = 1 + rs.randint(4), 2 + rs.randint(6)
        counts = rs.randint(0, 6, size=(L, E)).astype(np.int64)
        if counts.sum() == 0:
            counts[0, 0] = 1
        cap = rs.randint(0, L * E + 2)
        res = ref.greedy_place(counts, cap)
        resq = ref.greedy_place(counts, cap, per_layer_quota=True)
        hr = ref.expected_hit_rate(res, counts, int(counts.sum()))
        b = ref.hit_rate_bounds(counts, int(counts.sum()), cap)
        pl.append(np.concatenate([[L, E, cap], counts.ravel(), res.ravel(), resq.ravel(),
                                  [hr], b]))
    g["placement"] = np.concatenate([[len(p)] for p in pl] + pl)

    if args.mixtral:
        M = O.Shape(1, 8, 2, 4096, 14336, 2)
        w = ref.random_model(M, 0)
        x = orc.normal(1, 4096)[None]
        out, cnt, gate, kind = ref.model_forward(M, w, x)
        g["M_token"] = x
        g["M_out"] = out
        g["M_count"] = cnt
        g["M_gate"] = gate
        g["M_router"] = w.router[0]
        g["M_samples"] = np.array([[w.w_in[e][0, :4], w.w_gate[e][5, :4], w.w_out[e][7, :4]]
                                   for e in range(8)])
    elif os.path.exists(OUT):
        old = np.load(OUT)
        for k in old.files:
            if k.startswith("M_"):
                g[k] = old[k]

    np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT), "bytes;", len(g), "arrays")


if __name__ == "__main__":
    main()
