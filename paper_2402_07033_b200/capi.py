"""ctypes bindings for include/moe_b200.h (the C-ABI of libmoe_b200.so)."""
from __future__ import annotations

import ctypes as C
import os
import re
from dataclasses import dataclass

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
BUILD = os.path.join(PKG, "_build")
HEADER = os.path.join(ROOT, "include", "moe_b200.h")

DTYPE_BF16 = 0
DTYPE_F32 = 1

ERR_NAMES = {1: "ShapeError", 2: "ValidationError", 3: "CudaError", 4: "NcclError",
             5: "OutOfMemory", 6: "ArgumentError", 7: "Unsupported", 8: "NoDevice"}

_lib = None


def lib_path() -> str:
    # MOE_B200_LIB: an alternative in-tree build (A/B experiments)
    return os.environ.get("MOE_B200_LIB") or os.path.join(BUILD, "libmoe_b200.so")


class MoeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERR_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERR_NAMES.get(code, str(code))


def declared_symbols() -> list[str]:
    """Every function the C-ABI header declares."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(moe_\w+)\s*\(", txt, re.M)))


class _Shape(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("experts_per_layer", C.c_int32),
                ("top_k", C.c_int32), ("hidden_dim", C.c_int32), ("ffn_dim", C.c_int32),
                ("bytes_per_param", C.c_int32)]


@dataclass(frozen=True)
class Shape:
    """moe_orch::ModelShape (shape.hpp:9-35)."""

    num_layers: int = 4
    experts_per_layer: int = 8
    top_k: int = 2
    hidden_dim: int = 32
    ffn_dim: int = 64
    bytes_per_param: int = 2

    def c(self):
        return _Shape(self.num_layers, self.experts_per_layer, self.top_k, self.hidden_dim,
                      self.ffn_dim, self.bytes_per_param)


_vp = C.c_void_p
_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)


def lib():
    """Load libmoe_b200.so; raises if it was not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    p = lib_path()
    if not os.path.exists(p):
        raise ImportError(f"{p} not built — run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(p)
    sig = {
        "moe_version": ([], C.c_int),
        "moe_last_error": ([], C.c_char_p),
        "moe_shape_validate": ([C.POINTER(_Shape)], C.c_int),
        "moe_ctx_create": ([C.c_int, C.POINTER(_vp)], C.c_int),
        "moe_ctx_destroy": ([_vp], C.c_int),
        "moe_ctx_stream": ([_vp], _vp),
        "moe_ctx_synchronize": ([_vp], C.c_int),
        "moe_ctx_sm_count": ([_vp], C.c_int),
        "moe_ep_unique_id": ([_vp], C.c_int),
        "moe_ctx_init_ep": ([_vp, C.c_int, C.c_int, _vp], C.c_int),
        "moe_ctx_world": ([_vp, C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
        "moe_ctx_set_virtual_rank": ([_vp, C.c_int, C.c_int], C.c_int),
        "moe_ctx_peer_window": ([_vp, C.c_int, C.c_int, _vp], C.c_int),
        "moe_ctx_open_peers": ([_vp, C.c_int, C.c_int, _vp], C.c_int),
        "moe_ctx_link_peers": ([C.POINTER(_vp), C.c_int, C.c_int], C.c_int),
        "moe_ctx_peer_check": ([_vp], C.c_int),
        "moe_ctx_peer_window_tokens": ([_vp, C.c_int, C.c_int, C.c_int, _vp], C.c_int),
        "moe_ctx_link_peers_tokens": ([C.POINTER(_vp), C.c_int, C.c_int, C.c_int], C.c_int),
        "moe_weights_create": ([_vp, C.POINTER(_Shape), C.c_int, _vp, C.POINTER(_vp)], C.c_int),
        "moe_weights_create_tp": ([_vp, C.POINTER(_Shape), C.c_int, C.POINTER(_vp)], C.c_int),
        "moe_weights_create_ep": ([_vp, C.POINTER(_Shape), C.c_int, _vp, _vp, C.POINTER(_vp)], C.c_int),
        "moe_weights_set_replica_cost": ([_vp, C.c_int64, C.c_int64, C.c_int64], C.c_int),
        "moe_debug_kernel_timing": ([_vp, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int64)], C.c_int),
        "moe_weights_replica_cost": ([_vp] + [C.POINTER(C.c_int64)] * 3, C.c_int),
        "moe_replica_plan": ([_vp, C.c_int, _vp, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                              C.c_int, _vp, _vp, C.POINTER(C.c_int64)], C.c_int),
        "moe_ep_shard_map_coselect": ([_vp, _vp, C.c_int, C.c_int, C.c_int, _vp, _vp], C.c_int),
        "moe_routing_pair_histogram": ([_vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _vp], C.c_int),
        "moe_weights_reserve": ([_vp, C.c_int], C.c_int),
        "moe_weights_tp": ([_vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
        "moe_weights_destroy": ([_vp], C.c_int),
        "moe_weights_device_bytes": ([_vp], C.c_int64),
        "moe_weights_upload_expert": ([_vp, C.c_int, C.c_int, _dp, _dp, _dp], C.c_int),
        "moe_weights_upload_router": ([_vp, C.c_int, _dp], C.c_int),
        "moe_weights_random": ([_vp, C.c_uint64], C.c_int),
        "moe_weights_download_expert": ([_vp, C.c_int, C.c_int, _dp, _dp, _dp], C.c_int),
        "moe_weights_download_router": ([_vp, C.c_int, _dp], C.c_int),
        "moe_router_topk": ([_vp, C.c_int, _vp, C.c_int, _vp, _vp, _vp], C.c_int),
        "moe_routing_histogram": ([_vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _vp], C.c_int),
        "moe_routing_trace_step": ([_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, _i32p, _dp], C.c_int),
        "moe_permute": ([_vp, _vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp], C.c_int),
        "moe_experts_forward": ([_vp, C.c_int, _vp, C.c_int, _vp, _vp, _vp, _vp, _vp], C.c_int),
        "moe_decode_experts_partial": ([_vp, C.c_int, _vp, _vp, _vp, _vp, _vp], C.c_int),
        "moe_layer_forward": ([_vp, C.c_int, _vp, _vp, C.c_int, _vp, _vp, _vp], C.c_int),
        "moe_forward": ([_vp, _vp, C.c_int, _vp, _vp, _vp], C.c_int),
        "moe_forward_sparsity": ([_vp, _vp, C.c_int, _vp, _vp, _dp, C.c_int, _vp, _vp], C.c_int),
        "moe_forward_host": ([_vp, _dp, C.c_int, _dp, _i32p, _dp, _dp], C.c_int),
        "moe_forward_host_async": ([_vp, C.c_int, _vp, C.c_int, _vp, _vp, _vp, C.POINTER(C.c_int64)], C.c_int),
        "moe_host_wait": ([_vp, C.c_int64], C.c_int),
        "moe_expert_ffn_host": ([_vp, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp], C.c_int),
        "moe_gate_topk_host": ([_vp, C.c_int, C.c_int, _dp, _dp, C.c_int, _i32p, _dp], C.c_int),
        "moe_expert_path": ([_vp, C.c_int], C.c_int),
        "moe_forward_launches": ([_vp, C.c_int], C.c_int),
        "moe_layer_launches": ([_vp, C.c_int], C.c_int),
        "moe_debug_trace_forward": ([_vp, _vp, _vp, _vp, C.POINTER(C.c_uint64), C.c_int64], C.c_int),
        "moe_forward_logits": ([_vp, _vp, _vp, _vp, _vp, _vp], C.c_int),
        "moe_debug_set_option": ([C.c_char_p, C.c_int64], C.c_int),
        "moe_debug_get_option": ([C.c_char_p, C.POINTER(C.c_int64)], C.c_int),
        "moe_debug_set_trace_path": ([C.c_char_p], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def check(rc: int):
    if rc != 0:
        raise MoeError(rc, lib().moe_last_error().decode())


def get_option(name: str) -> int:
    v = C.c_int64()
    check(lib().moe_debug_get_option(name.encode(), C.byref(v)))
    return v.value


def set_option(name: str, value: int) -> None:
    """Debug / A-B switch of the library (moe_debug_set_option)."""
    check(lib().moe_debug_set_option(name.encode(), int(value)))


class options:
    """Context manager: ``with options(stack=0): ...`` sets library debug
    options and restores the previous values on exit."""

    def __init__(self, **kw):
        self.kw = kw
        self.old = {}

    def __enter__(self):
        for k, v in self.kw.items():
            self.old[k] = get_option(k)
            set_option(k, v)
        return self

    def __exit__(self, *a):
        for k, v in self.old.items():
            set_option(k, v)


def set_trace_path(path: str | None) -> None:
    check(lib().moe_debug_set_trace_path((path or "").encode()))


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _hptr(a):
    """Host pointer of a CPU torch tensor or numpy array (contiguous)."""
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return C.c_void_p(a.ctypes.data)
    assert not a.is_cuda and a.is_contiguous()
    return C.c_void_p(a.data_ptr())


def _ptr(t):
    """Device pointer of a torch tensor (or None)."""
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy: the explicit handle of the legacy default stream


def _stream(stream, *tensors):
    """Default for device-pointer calls on torch tensors: torch's current
    stream on the tensors' device, so the kernels are ordered after the
    torch ops that produced their inputs.  torch's default stream is the
    legacy default stream, whose handle is 0 — and a NULL stream means "the
    context's own (non-blocking) stream" in the C-ABI, which would race with
    the torch kernels that produced the inputs — so it is passed as
    cudaStreamLegacy."""
    if stream is not None:
        return stream
    for t in tensors:
        if t is not None and hasattr(t, "device") and getattr(t.device, "type", "") == "cuda":
            import torch

            h = torch.cuda.current_stream(t.device).cuda_stream
            return C.c_void_p(h if h else CUDA_STREAM_LEGACY)
    return None


class Ctx:
    def __init__(self, device: int = 0):
        import weakref

        h = _vp()
        check(lib().moe_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device
        self._weights = weakref.WeakSet()  # closed before the context (C-ABI order)

    def close(self):
        if self.h:
            for w in list(self._weights):
                w.close()
            lib().moe_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self):
        return lib().moe_ctx_stream(self.h)

    @property
    def sm_count(self):
        return lib().moe_ctx_sm_count(self.h)

    def synchronize(self):
        check(lib().moe_ctx_synchronize(self.h))

    def init_ep(self, world: int, rank: int, uid: bytes):
        buf = C.create_string_buffer(bytes(uid), 128)
        check(lib().moe_ctx_init_ep(self.h, world, rank, buf))

    def set_virtual_rank(self, world: int, rank: int):
        check(lib().moe_ctx_set_virtual_rank(self.h, world, rank))

    # ---- peer-memory combine (NVLink P2P / CUDA IPC) ----
    def peer_window(self, world: int, max_hidden: int, max_tokens: int = 0) -> bytes:
        """Allocate this rank's exchange window (max_tokens > 0 adds the
        multi-token area); returns its 64-byte IPC handle."""
        buf = C.create_string_buffer(64)
        check(lib().moe_ctx_peer_window_tokens(self.h, world, max_hidden, max_tokens, buf))
        return buf.raw

    def open_peers(self, world: int, rank: int, handles: list):
        """handles: every rank's peer_window() bytes, in rank order."""
        blob = C.create_string_buffer(b"".join(bytes(h) for h in handles), 64 * world)
        check(lib().moe_ctx_open_peers(self.h, world, rank, blob))

    @staticmethod
    def link_peers(ctxs: list, max_hidden: int, max_tokens: int = 0):
        """In-process peers (several contexts, same or peer-capable GPUs)."""
        arr = (_vp * len(ctxs))(*[c.h for c in ctxs])
        check(lib().moe_ctx_link_peers_tokens(arr, len(ctxs), max_hidden, max_tokens))

    def peer_check(self):
        check(lib().moe_ctx_peer_check(self.h))

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().moe_ep_unique_id(buf))
        return buf.raw

    def permute(self, ids, n_tok, top_k, n_experts, counts, offsets, perm, inv_perm=None,
                stream=None):
        check(lib().moe_permute(self.h, _ptr(ids), n_tok, top_k, n_experts, _ptr(counts),
                                _ptr(offsets), _ptr(perm), _ptr(inv_perm), _stream(stream, ids)))

    def routing_histogram(self, ids, counts, stream=None):
        """counts[l][e] += selections in ids [L x n_tok x k] (int64 device tensor [L x E])."""
        L, n, k = ids.shape
        check(lib().moe_routing_histogram(self.h, _ptr(ids), L, n, k, counts.shape[1], _ptr(counts),
                                          _stream(stream, ids)))

    def routing_pair_histogram(self, ids, pairs, stream=None):
        """pairs[l][a][b] (a < b) += tokens whose top-k holds a and b (int64 device [L x E x E])."""
        L, n, k = ids.shape
        check(lib().moe_routing_pair_histogram(self.h, _ptr(ids), L, n, k, pairs.shape[1], _ptr(pairs),
                                               _stream(stream, ids)))

    def routing_trace_step(self, ids, gates, n_experts):
        """(token_count [L x E] int32, gate_weight [L x E] fp64) of one step."""
        L, n, k = ids.shape
        cnt = np.zeros((L, n_experts), np.int32)
        gw = np.zeros((L, n_experts), np.float64)
        check(lib().moe_routing_trace_step(self.h, _ptr(ids), _ptr(gates), L, n, k, n_experts,
                                           cnt.ctypes.data_as(_i32p), _dptr(gw)))
        return cnt, gw

    def expert_ffn_host(self, dtype, w_in, w_gate, w_out, x):
        f, d = w_in.shape
        y = np.empty(d)
        args = [np.ascontiguousarray(a, np.float64) for a in (w_in, w_gate, w_out, x)]
        check(lib().moe_expert_ffn_host(self.h, dtype, d, f, *[_dptr(a) for a in args], _dptr(y)))
        return y

    def gate_topk_host(self, router, x, k):
        E, d = router.shape
        ids = np.empty(k, np.int32)
        g = np.empty(k)
        r = np.ascontiguousarray(router, np.float64)
        xx = np.ascontiguousarray(x, np.float64)
        check(lib().moe_gate_topk_host(self.h, E, d, _dptr(r), _dptr(xx), k,
                                       ids.ctypes.data_as(_i32p), _dptr(g)))
        return ids, g


class Weights:
    def __init__(self, ctx: Ctx, shape: Shape, dtype: int = DTYPE_BF16, owner=None, tp=False,
                 replicas=None):
        """owner: expert-parallel [L x E] shard map; tp=True: tensor-parallel
        shard (ffn rows of every expert) over the context's (world, rank);
        replicas: [L x E] rank bitmasks of extra holders of each expert (the
        prefill path splits a hot expert's tokens over its holders)."""
        self.ctx = ctx
        self.shape = shape
        self.dtype = dtype
        h = _vp()
        sh = shape.c()
        if tp:
            check(lib().moe_weights_create_tp(ctx.h, C.byref(sh), dtype, C.byref(h)))
        else:
            own = None
            if owner is not None:
                self._owner = np.ascontiguousarray(owner, np.int32).ravel()
                own = self._owner.ctypes.data_as(_vp)
            if replicas is not None:
                self._replicas = np.ascontiguousarray(replicas, np.uint32).ravel()
                check(lib().moe_weights_create_ep(ctx.h, C.byref(sh), dtype, own,
                                                  self._replicas.ctypes.data_as(_vp), C.byref(h)))
            else:
                check(lib().moe_weights_create(ctx.h, C.byref(sh), dtype, own, C.byref(h)))
        self.h = h
        ctx._weights.add(self)

    @property
    def replica_cost(self):
        """(weight_ps, row_ps, part_ps) of the replica split's cost model."""
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().moe_weights_replica_cost(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    @replica_cost.setter
    def replica_cost(self, v):
        check(lib().moe_weights_set_replica_cost(self.h, int(v[0]), int(v[1]), int(v[2])))

    def kernel_timing(self, enable: bool):
        """Live CUDA-event timing of the grouped prefill kernel launches:
        kernel_timing(True) starts; kernel_timing(False) returns
        (total_us, launches)."""
        t, n = C.c_double(), C.c_int64()
        check(lib().moe_debug_kernel_timing(self.h, 1 if enable else 0, C.byref(t), C.byref(n)))
        return t.value, n.value

    def reserve(self, max_tokens: int):
        """Allocate all scratch for calls of up to max_tokens tokens now."""
        check(lib().moe_weights_reserve(self.h, max_tokens))

    @property
    def tp(self):
        """(tp_world, tp_rank, ffn rows resident on this rank)."""
        a, b, c = C.c_int(), C.c_int(), C.c_int()
        check(lib().moe_weights_tp(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def close(self):
        if self.h:
            lib().moe_weights_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def device_bytes(self):
        return lib().moe_weights_device_bytes(self.h)

    def upload_expert(self, layer, expert, w_in, w_gate, w_out):
        a = [np.ascontiguousarray(m, np.float64) for m in (w_in, w_gate, w_out)]
        check(lib().moe_weights_upload_expert(self.h, layer, expert, *[_dptr(m) for m in a]))

    def upload_router(self, layer, router):
        r = np.ascontiguousarray(router, np.float64)
        check(lib().moe_weights_upload_router(self.h, layer, _dptr(r)))

    def upload_oracle(self, ow):
        """Upload an oracle.Weights (reference layout, fp64)."""
        s = self.shape
        for l in range(s.num_layers):
            for e in range(s.experts_per_layer):
                wi, wg, wo = ow.expert(l, e)
                if wi is not None:
                    self.upload_expert(l, e, wi, wg, wo)
            self.upload_router(l, ow.router[l])

    def random(self, seed: int):
        check(lib().moe_weights_random(self.h, seed))

    def download_expert(self, layer, expert, out=None):
        """Device-held values of one expert in the reference layout (fp64).
        out=(w_in, w_gate, w_out) fills given arrays: a tensor-parallel rank
        writes only its slice, so the ranks' downloads into one set of
        arrays assemble the full expert."""
        d, f = self.shape.hidden_dim, self.shape.ffn_dim
        if out is not None:
            wi, wg, wo = out
            assert wi.shape == (f, d) and wg.shape == (f, d) and wo.shape == (d, f)
            assert all(m.dtype == np.float64 and m.flags.c_contiguous for m in out)
        else:
            wi, wg, wo = np.empty((f, d)), np.empty((f, d)), np.empty((d, f))
        check(lib().moe_weights_download_expert(self.h, layer, expert, _dptr(wi), _dptr(wg),
                                                _dptr(wo)))
        return wi, wg, wo

    def download_router(self, layer):
        r = np.empty((self.shape.experts_per_layer, self.shape.hidden_dim))
        check(lib().moe_weights_download_router(self.h, layer, _dptr(r)))
        return r

    # -- device-pointer API (torch tensors) ----------------------------------
    def router_topk(self, layer, x, ids, gates, stream=None):
        check(lib().moe_router_topk(self.h, layer, _ptr(x), x.shape[0], _ptr(ids), _ptr(gates),
                                    _stream(stream, x)))

    def experts_forward(self, layer, x, ids, gates, x_out, post_silu=None, stream=None):
        check(lib().moe_experts_forward(self.h, layer, _ptr(x), x.shape[0], _ptr(ids), _ptr(gates),
                                        _ptr(x_out), _ptr(post_silu), _stream(stream, x)))

    def decode_experts_partial(self, layer, x, ids, gates, ypart, stream=None):
        check(lib().moe_decode_experts_partial(self.h, layer, _ptr(x), _ptr(ids), _ptr(gates),
                                               _ptr(ypart), _stream(stream, x)))

    def layer_forward(self, layer, x, x_out, ids, gates, stream=None):
        check(lib().moe_layer_forward(self.h, layer, _ptr(x), _ptr(x_out), x.shape[0], _ptr(ids),
                                      _ptr(gates), _stream(stream, x)))

    def forward(self, x, ids, gates, stream=None):
        check(lib().moe_forward(self.h, _ptr(x), x.shape[0], _ptr(ids), _ptr(gates),
                                _stream(stream, x)))

    # -- host-buffer API ------------------------------------------------------
    def forward_sparsity(self, x, ids, gates, thresholds, counts, stream=None):
        """forward + fused sparsity counters: counts [L x n_thr] int64 device tensor."""
        thr = np.ascontiguousarray(thresholds, np.float64)
        check(lib().moe_forward_sparsity(self.h, _ptr(x), x.shape[0], _ptr(ids), _ptr(gates), _dptr(thr),
                                         len(thr), _ptr(counts), _stream(stream, x)))

    def forward_host_async(self, layer, x_host, out_host, ids_host, gates_host) -> int:
        """Pipelined host-buffer step (moe_forward_host_async): fp32 host
        tensors/arrays (pinned for overlap) [n x hidden]; layer -1 = the whole
        stack.  Returns the ticket for host_wait()."""
        t = C.c_int64()
        n = x_host.shape[0]
        check(lib().moe_forward_host_async(self.h, layer, _hptr(x_host), n, _hptr(out_host), _hptr(ids_host),
                                           _hptr(gates_host), C.byref(t)))
        return t.value

    def host_wait(self, ticket: int = -1):
        check(lib().moe_host_wait(self.h, ticket))

    def forward_host(self, tokens: np.ndarray, with_post=False):
        s = self.shape
        toks = np.ascontiguousarray(tokens, np.float64).reshape(-1, s.hidden_dim)
        n = toks.shape[0]
        out = np.empty_like(toks)
        ids = np.zeros((max(1, s.num_layers), n, s.top_k), np.int32)
        gates = np.zeros((max(1, s.num_layers), n, s.top_k))
        post = np.zeros(max(1, n * s.num_layers * s.top_k * s.ffn_dim)) if with_post else None
        check(lib().moe_forward_host(self.h, _dptr(toks), n, _dptr(out), ids.ctypes.data_as(_i32p),
                                     _dptr(gates), _dptr(post) if with_post else _dp()))
        res = (out, ids[:s.num_layers], gates[:s.num_layers])
        if with_post:
            return res + (post[:n * s.num_layers * s.top_k * s.ffn_dim],)
        return res

    def debug_trace_forward(self, x, ids, gates):
        n = self.shape.num_layers * self.ctx.sm_count * 16
        tr = np.zeros(n, np.uint64)
        check(lib().moe_debug_trace_forward(self.h, _ptr(x), _ptr(ids), _ptr(gates),
                                            tr.ctypes.data_as(C.POINTER(C.c_uint64)), n))
        return tr.reshape(self.shape.num_layers, self.ctx.sm_count, 16)

    def forward_logits(self, x, ids, gates, logits, stream=None):
        """Batch-1 forward through the persistent kernel that also records
        every layer's router logits (logits: device fp32 [L x E])."""
        check(lib().moe_forward_logits(self.h, _ptr(x), _ptr(ids), _ptr(gates), _ptr(logits),
                                       _stream(stream, x)))

    def expert_path(self, n_tok: int) -> int:
        return lib().moe_expert_path(self.h, n_tok)

    def forward_launches(self, n_tok: int) -> int:
        return lib().moe_forward_launches(self.h, n_tok)

    def layer_launches(self, n_tok: int) -> int:
        return lib().moe_layer_launches(self.h, n_tok)


def ep_shard_map_coselect(counts, pairs, world):
    """Co-selection-aware EP shard map (moe_ep_shard_map_coselect): counts
    [L x E] selections, pairs [L x E x E] co-selections (host) -> (owner
    [L x E] int32, exact [L] bool)."""
    c = np.ascontiguousarray(counts, np.int64)
    p = np.ascontiguousarray(pairs, np.int64)
    L, E = c.shape
    if p.shape != (L, E, E):
        raise MoeError(-1, f"pairs must be [L x E x E] = {(L, E, E)}, got {p.shape}")
    owner = np.zeros((L, E), np.int32)
    exact = np.zeros(L, np.int32)
    check(lib().moe_ep_shard_map_coselect(c.ctypes.data_as(_vp), p.ctypes.data_as(_vp), L, E, world,
                                          owner.ctypes.data_as(_vp), exact.ctypes.data_as(_vp)))
    return owner, exact.astype(bool)


def replica_plan(counts, holders, world, weight_ps, row_ps, part_ps, chunk, rank):
    """Host mirror of the device replica planner (moe_replica_plan): rank
    `rank`'s rows (lo[e], hi[e]) of every expert and the plan's makespan."""
    c = np.ascontiguousarray(counts, np.int32)
    hm = np.ascontiguousarray(holders, np.uint32)
    E = c.size
    lo = np.zeros(E, np.int32)
    hi = np.zeros(E, np.int32)
    mk = C.c_int64()
    check(lib().moe_replica_plan(c.ctypes.data_as(_vp), E, hm.ctypes.data_as(_vp), world,
                                 int(weight_ps), int(row_ps), int(part_ps), chunk, rank,
                                 lo.ctypes.data_as(_vp), hi.ctypes.data_as(_vp), C.byref(mk)))
    return lo, hi, mk.value
