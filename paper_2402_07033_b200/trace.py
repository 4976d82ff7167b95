"""RoutingTrace JSONL emission for GPU runs.

The reference's on-disk trace format (trace.cpp:90-108, save_trace_jsonl):
one JSON object per step, keys in nlohmann's (sorted) order and compact
separators — {"kind":"prefill"|"decode","layers":[[[expert,tokens,gate],...],...]}
— with one [expert, token_count, mean gate] triple per selected expert of
a layer, ascending expert (model.cpp:151-158).  Steps built here come from
the device routing record of moe_forward (Ctx.routing_trace_step), so a GPU
run can be replayed through the reference's loader / validator
(load_trace_jsonl, trace.cpp:110-141) and its placement / simulator tools.
"""
from __future__ import annotations

import json

import numpy as np


def step_from_counts(token_count: np.ndarray, gate_weight: np.ndarray, n_tok: int) -> dict:
    """One TraceStep as the reference serialises it."""
    layers = []
    for l in range(token_count.shape[0]):
        layers.append([[int(e), int(token_count[l, e]), float(gate_weight[l, e])]
                       for e in range(token_count.shape[1]) if token_count[l, e] > 0])
    return {"kind": "decode" if n_tok == 1 else "prefill", "layers": layers}


def device_step(ctx, ids, gates, n_experts: int) -> dict:
    """TraceStep of one forward from its device routing record [L x n x k]."""
    cnt, gw = ctx.routing_trace_step(ids, gates, n_experts)
    return step_from_counts(cnt, gw, int(ids.shape[1]))


def dumps_step(step: dict) -> str:
    return json.dumps({"kind": step["kind"], "layers": step["layers"]}, separators=(",", ":"))


def save_trace_jsonl(steps: list, path: str) -> None:
    with open(path, "w") as f:
        for st in steps:
            f.write(dumps_step(st) + "\n")
