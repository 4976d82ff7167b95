"""oracle — TEST INFRASTRUCTURE ONLY.

ctypes front-ends for
  * ``Oracle``    : the plain-C fp64 restatement (oracle/moe_oracle.c), and
  * ``Reference`` : the reference itself compiled from /root/reference sources
                    (oracle/_ref/libmoe_ref.so, built by oracle/Makefile).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this package.  The product package
``paper_2402_07033_b200`` never does; it fails loudly without its CUDA library.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libmoe_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmoe_ref.so")
REF_SRC = "/root/reference/proj"

_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)


def build(ref: bool | None = None) -> None:
    """Compile the oracle (always) and oracle/_ref (when the reference tree is here)."""
    targets = ["oracle"]
    if ref or (ref is None and os.path.isdir(REF_SRC)):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


@dataclass(frozen=True)
class Shape:
    """Mirrors ModelShape (reference include/moe_orch/shape.hpp:9-35)."""

    num_layers: int = 4
    experts_per_layer: int = 8
    top_k: int = 2
    hidden_dim: int = 32
    ffn_dim: int = 64
    bytes_per_param: int = 2

    def arr(self):
        return (C.c_int32 * 6)(self.num_layers, self.experts_per_layer, self.top_k,
                                self.hidden_dim, self.ffn_dim, self.bytes_per_param)


def _p(a: np.ndarray, t=_dp):
    return a.ctypes.data_as(t)


class Weights:
    """Flat fp64 weights in the reference layout (model.hpp:14-49)."""

    def __init__(self, shape: Shape, experts=None):
        L, E, d, f = shape.num_layers, shape.experts_per_layer, shape.hidden_dim, shape.ffn_dim
        self.shape = shape
        keep = set(range(L * E)) if experts is None else set(experts)
        self.w_in = [np.zeros((f, d)) if i in keep else None for i in range(L * E)]
        self.w_gate = [np.zeros((f, d)) if i in keep else None for i in range(L * E)]
        self.w_out = [np.zeros((d, f)) if i in keep else None for i in range(L * E)]
        self.router = [np.zeros((E, d)) for _ in range(L)]

    @staticmethod
    def _ptrs(mats):
        arr = (_dp * max(1, len(mats)))()
        for i, m in enumerate(mats):
            arr[i] = m.ctypes.data_as(_dp) if m is not None else _dp()
        return arr

    def ptrs(self):
        return (self._ptrs(self.w_in), self._ptrs(self.w_gate), self._ptrs(self.w_out),
                self._ptrs(self.router))

    def expert(self, l, e):
        i = l * self.shape.experts_per_layer + e
        return self.w_in[i], self.w_gate[i], self.w_out[i]


class _Base:
    so_path = ""

    def __init__(self):
        if not os.path.exists(self.so_path):
            raise FileNotFoundError(f"{self.so_path} missing: run `make -C oracle`")
        self.lib = C.CDLL(self.so_path)


class Oracle(_Base):
    """The C restatement (oracle/moe_oracle.c)."""

    so_path = ORACLE_SO

    def __init__(self):
        super().__init__()
        L = self.lib
        L.oracle_random_model.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p]
        L.oracle_expert_ffn.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp]
        L.oracle_expert_ffn_batch.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, C.c_int, _dp, _dp]
        L.oracle_gate_topk.argtypes = [C.c_int, C.c_int, _dp, _dp, C.c_int, _i32p, _dp, _dp]
        L.oracle_model_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_int, _dp, _i32p, _dp, _i32p, _dp,
                                           C.c_void_p, C.c_void_p]
        L.oracle_normal_fill.argtypes = [C.c_void_p, C.c_double, _dp, C.c_int64]
        L.oracle_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
        L.oracle_rng_next.argtypes = [C.c_void_p]
        L.oracle_rng_next.restype = C.c_uint64
        L.oracle_silu.argtypes = [C.c_double]
        L.oracle_silu.restype = C.c_double
        L.oracle_greedy_place.argtypes = [C.c_int, C.c_int, _i64p, C.c_int, C.c_int, _u8p]
        L.oracle_expected_hit_rate.argtypes = [C.c_int, C.c_int, _i64p, C.c_int64, _u8p, _dp]
        L.oracle_hit_rate_bounds.argtypes = [C.c_int, C.c_int, _i64p, C.c_int64, C.c_int, _dp]
        L.oracle_sparsity_histogram.argtypes = [_dp, C.c_int64, _dp, C.c_int, _dp]
        L.oracle_shape_validate.argtypes = [C.c_void_p]

    # -- rng --------------------------------------------------------------
    def normal(self, seed: int, n: int, stddev: float = 1.0) -> np.ndarray:
        """n draws of N(0,stddev) from mt19937_64(seed) with ONE distribution
        object (the token convention of moe_orch_cli.cpp:251-256)."""
        st = (C.c_uint8 * (312 * 8 + 16))()
        self.lib.oracle_rng_seed(st, seed)
        out = np.empty(n)
        self.lib.oracle_normal_fill(st, stddev, _p(out), n)
        return out

    def shape_validate(self, shape: Shape) -> int:
        return self.lib.oracle_shape_validate(shape.arr())

    def random_model(self, shape: Shape, seed: int, experts=None) -> Weights:
        w = Weights(shape, experts)
        a, b, c, r = w.ptrs()
        rc = self.lib.oracle_random_model(shape.arr(), seed, a, b, c, r)
        if rc:
            raise ValueError("ShapeError")
        return w

    def silu(self, x: float) -> float:
        return self.lib.oracle_silu(x)

    def expert_ffn(self, w_in, w_gate, w_out, x) -> np.ndarray:
        f, d = w_in.shape
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(d)
        self.lib.oracle_expert_ffn(d, f, _p(np.ascontiguousarray(w_in)),
                                   _p(np.ascontiguousarray(w_gate)),
                                   _p(np.ascontiguousarray(w_out)), _p(x), _p(y))
        return y

    def expert_ffn_batch(self, w_in, w_gate, w_out, X) -> np.ndarray:
        """expert_ffn for every row of X [n x d] (each row bit-identical to
        expert_ffn); releases the GIL, so threads can run experts in parallel."""
        f, d = w_in.shape
        X = np.ascontiguousarray(X, dtype=np.float64).reshape(-1, d)
        Y = np.empty_like(X)
        self.lib.oracle_expert_ffn_batch(d, f, _p(np.ascontiguousarray(w_in)),
                                         _p(np.ascontiguousarray(w_gate)),
                                         _p(np.ascontiguousarray(w_out)), X.shape[0], _p(X), _p(Y))
        return Y

    def random_model_stream(self, shape: Shape, seed: int):
        """random_model (model.cpp:34-53) one matrix group at a time, so a
        Mixtral-shaped layer (11.3 GB of fp64) never sits in host memory at
        once.  Yields ("expert", l, e, w_in, w_gate, w_out) and ("router", l,
        R) in the reference's draw order — the same values as random_model."""
        L, E, d, f = shape.num_layers, shape.experts_per_layer, shape.hidden_dim, shape.ffn_dim
        st = (C.c_uint8 * (312 * 8 + 16))()
        self.lib.oracle_rng_seed(st, seed)
        scale = 1.0 / np.sqrt(d)
        for l in range(L):
            for e in range(E):
                mats = []
                for rows, cols in ((f, d), (f, d), (d, f)):
                    m = np.empty((rows, cols))
                    self.lib.oracle_normal_fill(st, scale, _p(m), m.size)
                    mats.append(m)
                yield ("expert", l, e, *mats)
            r = np.empty((E, d))
            self.lib.oracle_normal_fill(st, scale, _p(r), r.size)
            yield ("router", l, r)

    def gate_topk(self, router_l, x, k):
        E, d = router_l.shape
        ids = np.empty(k, np.int32)
        w = np.empty(k)
        logits = np.empty(E)
        rc = self.lib.oracle_gate_topk(E, d, _p(np.ascontiguousarray(router_l)),
                                       _p(np.ascontiguousarray(x, dtype=np.float64)), k,
                                       _p(ids, _i32p), _p(w), _p(logits))
        if rc:
            raise ValueError("ShapeError")
        return ids, w, logits

    def model_forward(self, shape: Shape, w: Weights, tokens: np.ndarray, sink=None):
        """Returns (outputs [n,d], tally [L,E], gate_sum [L,E], ids [n,L,k], gates [n,L,k])."""
        L, E, k = shape.num_layers, shape.experts_per_layer, shape.top_k
        toks = np.array(tokens, dtype=np.float64, copy=True).reshape(-1, shape.hidden_dim)
        n = toks.shape[0]
        tally = np.zeros(max(1, L * E), np.int32)
        gsum = np.zeros(max(1, L * E))
        ids = np.zeros(max(1, n * L * k), np.int32)
        gates = np.zeros(max(1, n * L * k))
        a, b, c, r = w.ptrs()
        cb = C.c_void_p()
        keep = None
        if sink is not None:
            SINK = C.CFUNCTYPE(None, C.c_int, _dp, C.c_int, C.c_void_p)
            keep = SINK(lambda layer, vals, cnt, ctx: sink(layer, np.ctypeslib.as_array(vals, (cnt,)).copy()))
            cb = C.cast(keep, C.c_void_p)
        rc = self.lib.oracle_model_forward(shape.arr(), a, b, c, r, n, _p(toks), _p(tally, _i32p),
                                           _p(gsum), _p(ids, _i32p), _p(gates), cb, None)
        if rc:
            raise ValueError("ShapeError")
        return (toks, tally[:L * E].reshape(L, E), gsum[:L * E].reshape(L, E),
                ids[:n * L * k].reshape(n, L, k), gates[:n * L * k].reshape(n, L, k))

    # -- placement ----------------------------------------------------------
    def greedy_place(self, counts: np.ndarray, capacity: int, per_layer_quota=False):
        counts = np.ascontiguousarray(counts, dtype=np.int64)
        L, E = counts.shape
        res = np.zeros(L * E, np.uint8)
        rc = self.lib.oracle_greedy_place(L, E, _p(counts, _i64p), capacity, int(per_layer_quota),
                                          _p(res, _u8p))
        if rc:
            raise ValueError("ValidationError")
        return res.reshape(L, E)

    def expected_hit_rate(self, resident, counts, total):
        counts = np.ascontiguousarray(counts, dtype=np.int64)
        L, E = counts.shape
        out = C.c_double()
        rc = self.lib.oracle_expected_hit_rate(L, E, _p(counts, _i64p), total,
                                               _p(np.ascontiguousarray(resident, np.uint8), _u8p),
                                               C.byref(out))
        if rc:
            raise ValueError("ValidationError")
        return out.value

    def hit_rate_bounds(self, counts, total, capacity):
        counts = np.ascontiguousarray(counts, dtype=np.int64)
        L, E = counts.shape
        out = np.zeros(3)
        rc = self.lib.oracle_hit_rate_bounds(L, E, _p(counts, _i64p), total, capacity, _p(out))
        if rc:
            raise ValueError("ValidationError")
        return tuple(out)

    def sparsity_histogram(self, acts, thr):
        acts = np.ascontiguousarray(acts, np.float64)
        thr = np.ascontiguousarray(thr, np.float64)
        out = np.zeros(len(thr))
        rc = self.lib.oracle_sparsity_histogram(_p(acts), len(acts), _p(thr), len(thr), _p(out))
        if rc:
            raise ValueError("ValidationError")
        return out


class Reference(_Base):
    """The reference's own code (oracle/_ref/libmoe_ref.so)."""

    so_path = REF_SO

    def __init__(self):
        super().__init__()
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_random_model.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p]
        L.ref_expert_ffn.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, _dp, C.c_int, _dp]
        L.ref_gate_topk.argtypes = [C.c_int, C.c_int, _dp, _dp, C.c_int, _i32p, _dp]
        L.ref_model_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_int, C.c_int, _dp, _dp, _i32p, _dp,
                                        _i32p, _dp, C.c_int64, _i64p]
        L.ref_time_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_int, _dp, _dp, _dp]
        L.ref_greedy_place.argtypes = [C.c_int, C.c_int, _i64p, C.c_int64, C.c_int, C.c_int, _u8p]
        L.ref_expected_hit_rate.argtypes = [C.c_int, C.c_int, _i64p, C.c_int64, _u8p, _dp]
        L.ref_hit_rate_bounds.argtypes = [C.c_int, C.c_int, _i64p, C.c_int64, C.c_int, _dp]
        L.ref_sparsity_histogram.argtypes = [_dp, C.c_int64, _dp, C.c_int, _dp]
        L.ref_model_create.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_model_create.restype = C.c_void_p
        L.ref_model_destroy.argtypes = [C.c_void_p]
        L.ref_model_forward_timed.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp]
        L.ref_shape_validate.argtypes = [C.c_void_p]
        L.ref_shape_preset.argtypes = [C.c_char_p, _i32p]
        L.ref_load_trace_jsonl.argtypes = [C.c_char_p, C.c_void_p, _i32p]
        L.ref_fit_records.argtypes = [C.c_char_p, C.c_double, _dp]

    def _check(self, rc):
        if rc == 1:
            raise ValueError("ShapeError: " + self.lib.ref_last_error().decode())
        if rc == 2:
            raise ValueError("ValidationError: " + self.lib.ref_last_error().decode())
        if rc:
            raise RuntimeError(self.lib.ref_last_error().decode())

    def fit_records(self, path: str, nonexpert_ms: float = 2.0) -> dict:
        """The reference's load_records_csv + CostModel fit (cost_model.cpp:57-156)."""
        out = np.zeros(6)
        rc = self.lib.ref_fit_records(path.encode(), nonexpert_ms, _p(out))
        if rc not in (0, 100):
            self._check(rc)
        keys = ["weight_copy_ms", "activation_copy_ms", "fast_exec_ms", "slow_ms_per_token",
                "slow_intercept_ms", "nonexpert_ms_per_step"]
        d = dict(zip(keys, out.tolist()))
        d["decode_assumption_check"] = rc == 0
        return d

    def load_trace_jsonl(self, path: str, shape: Shape) -> int:
        """The reference's loader + validator (trace.cpp:110-141); returns the step count."""
        n = C.c_int()
        self._check(self.lib.ref_load_trace_jsonl(path.encode(), shape.arr(), C.byref(n)))
        return n.value

    def random_model(self, shape: Shape, seed: int, experts=None) -> Weights:
        w = Weights(shape, experts)
        a, b, c, r = w.ptrs()
        self._check(self.lib.ref_random_model(shape.arr(), seed, a, b, c, r))
        return w

    def expert_ffn(self, w_in, w_gate, w_out, x):
        f, d = w_in.shape
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(w_out.shape[0])
        self._check(self.lib.ref_expert_ffn(d, f, _p(np.ascontiguousarray(w_in)),
                                            _p(np.ascontiguousarray(w_gate)),
                                            _p(np.ascontiguousarray(w_out)), _p(x), len(x), _p(y)))
        return y

    def expert_ffn_batch(self, w_in, w_gate, w_out, X) -> np.ndarray:
        """expert_ffn for every row of X [n x d] (each row bit-identical to
        expert_ffn); releases the GIL, so threads can run experts in parallel."""
        f, d = w_in.shape
        X = np.ascontiguousarray(X, dtype=np.float64).reshape(-1, d)
        Y = np.empty_like(X)
        self.lib.oracle_expert_ffn_batch(d, f, _p(np.ascontiguousarray(w_in)),
                                         _p(np.ascontiguousarray(w_gate)),
                                         _p(np.ascontiguousarray(w_out)), X.shape[0], _p(X), _p(Y))
        return Y

    def random_model_stream(self, shape: Shape, seed: int):
        """random_model (model.cpp:34-53) one matrix group at a time, so a
        Mixtral-shaped layer (11.3 GB of fp64) never sits in host memory at
        once.  Yields ("expert", l, e, w_in, w_gate, w_out) and ("router", l,
        R) in the reference's draw order — the same values as random_model."""
        L, E, d, f = shape.num_layers, shape.experts_per_layer, shape.hidden_dim, shape.ffn_dim
        st = (C.c_uint8 * (312 * 8 + 16))()
        self.lib.oracle_rng_seed(st, seed)
        scale = 1.0 / np.sqrt(d)
        for l in range(L):
            for e in range(E):
                mats = []
                for rows, cols in ((f, d), (f, d), (d, f)):
                    m = np.empty((rows, cols))
                    self.lib.oracle_normal_fill(st, scale, _p(m), m.size)
                    mats.append(m)
                yield ("expert", l, e, *mats)
            r = np.empty((E, d))
            self.lib.oracle_normal_fill(st, scale, _p(r), r.size)
            yield ("router", l, r)

    def gate_topk(self, router_l, x, k):
        E, d = router_l.shape
        ids = np.empty(k, np.int32)
        w = np.empty(k)
        self._check(self.lib.ref_gate_topk(E, d, _p(np.ascontiguousarray(router_l)),
                                           _p(np.ascontiguousarray(x, dtype=np.float64)), k,
                                           _p(ids, _i32p), _p(w)))
        return ids, w

    def model_forward(self, shape: Shape, w: Weights, tokens, with_sink=False, sink_cap=0):
        L, E = shape.num_layers, shape.experts_per_layer
        toks = np.ascontiguousarray(tokens, dtype=np.float64)
        n = toks.shape[0] if toks.ndim == 2 else 0
        width = toks.shape[1] if toks.ndim == 2 else shape.hidden_dim
        out = np.zeros_like(toks)
        cnt = np.zeros(max(1, L * E), np.int32)
        gate = np.zeros(max(1, L * E))
        kind = np.zeros(1, np.int32)
        sink = np.zeros(max(1, sink_cap)) if with_sink else None
        sink_n = np.zeros(1, np.int64)
        a, b, c, r = w.ptrs()
        self._check(self.lib.ref_model_forward(shape.arr(), a, b, c, r, n, width, _p(toks),
                                               _p(out), _p(cnt, _i32p), _p(gate), _p(kind, _i32p),
                                               _p(sink) if with_sink else _dp(), sink_cap,
                                               _p(sink_n, _i64p)))
        res = (out, cnt[:L * E].reshape(L, E), gate[:L * E].reshape(L, E), int(kind[0]))
        if with_sink:
            return res + (sink[:int(sink_n[0])],)
        return res

    def time_forward(self, shape: Shape, w: Weights, tokens):
        toks = np.ascontiguousarray(tokens, dtype=np.float64)
        out = np.zeros_like(toks)
        secs = C.c_double()
        a, b, c, r = w.ptrs()
        self._check(self.lib.ref_time_forward(shape.arr(), a, b, c, r, toks.shape[0], _p(toks),
                                              _p(out), C.byref(secs)))
        return out, secs.value

    def model_create(self, shape: Shape, w: Weights):
        """Persistent reference ModelWeights (built once, shared by threads)."""
        a, b, c, r = w.ptrs()
        h = self.lib.ref_model_create(shape.arr(), a, b, c, r)
        if not h:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return h

    def model_destroy(self, h):
        self.lib.ref_model_destroy(h)

    def model_forward_timed(self, h, tokens):
        """model_forward on the shared model; releases the GIL (ctypes)."""
        toks = np.ascontiguousarray(tokens, dtype=np.float64)
        secs = C.c_double()
        self._check(self.lib.ref_model_forward_timed(h, toks.shape[0], _p(toks), _dp(), C.byref(secs)))
        return secs.value

    def greedy_place(self, counts, capacity, per_layer_quota=False, total=None):
        counts = np.ascontiguousarray(counts, dtype=np.int64)
        L, E = counts.shape
        total = int(counts.sum()) if total is None else total
        res = np.zeros(L * E, np.uint8)
        self._check(self.lib.ref_greedy_place(L, E, _p(counts, _i64p), total, capacity,
                                              int(per_layer_quota), _p(res, _u8p)))
        return res.reshape(L, E)

    def expected_hit_rate(self, resident, counts, total):
        counts = np.ascontiguousarray(counts, dtype=np.int64)
        L, E = counts.shape
        out = C.c_double()
        self._check(self.lib.ref_expected_hit_rate(
            L, E, _p(counts, _i64p), total, _p(np.ascontiguousarray(resident, np.uint8), _u8p),
            C.byref(out)))
        return out.value

    def hit_rate_bounds(self, counts, total, capacity):
        counts = np.ascontiguousarray(counts, dtype=np.int64)
        L, E = counts.shape
        out = np.zeros(3)
        self._check(self.lib.ref_hit_rate_bounds(L, E, _p(counts, _i64p), total, capacity, _p(out)))
        return tuple(out)

    def sparsity_histogram(self, acts, thr):
        acts = np.ascontiguousarray(acts, np.float64)
        thr = np.ascontiguousarray(thr, np.float64)
        out = np.zeros(len(thr))
        self._check(self.lib.ref_sparsity_histogram(_p(acts), len(acts), _p(thr), len(thr), _p(out)))
        return out


def reference_available() -> bool:
    return os.path.exists(REF_SO)
