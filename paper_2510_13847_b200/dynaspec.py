"""Thin ctypes binding of libdynaspec.so (include/dynaspec.h).

Argument marshalling only: every step of the DynaSpec head runs in the CUDA library.
PyTorch provides device memory, streams and events.  There is no CPU fallback: if the
library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import c_int32, c_int64, c_size_t, c_uint64, c_void_p, POINTER

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DS_LIB_PATH") or os.path.join(_HERE, "lib", "libdynaspec.so")  # override: A/B builds

DS_BF16, DS_F32 = 0, 1
_DTYPE = {torch.bfloat16: DS_BF16, torch.float32: DS_F32}

STATUS = {
    0: "DS_OK", 1: "DS_ERR_SHAPE", 2: "DS_ERR_DTYPE", 3: "DS_ERR_INVALID_BUDGET",
    4: "DS_ERR_INVALID_CLUSTER_COUNT", 5: "DS_ERR_INVALID_CLUSTER_ID", 6: "DS_ERR_INVALID_TOKEN",
    7: "DS_ERR_DEGENERATE_COLUMN", 8: "DS_ERR_EMPTY_SHORTLIST", 9: "DS_ERR_WORKSPACE", 10: "DS_ERR_CUDA",
    11: "DS_ERR_UNSUPPORTED", 12: "DS_ERR_DEVICE_TIMEOUT",
}


class DynaspecError(RuntimeError):
    def __init__(self, code, what=""):
        self.code = code
        self.name = STATUS.get(code, str(code))
        super().__init__(f"{what}: {self.name} ({_lib.dynaspec_status_string(code).decode()})")


class DsClusters(ctypes.Structure):
    _fields_ = [("V", c_int64), ("d", c_int32), ("M", c_int32), ("dtype", c_int32), ("min_size", c_int32),
                ("max_size", c_int32), ("tau", c_void_p), ("perm", c_void_p), ("offsets", c_void_p),
                ("W_perm", c_void_p)]


class DsRouter(ctypes.Structure):
    _fields_ = [("d", c_int32), ("h_r", c_int32), ("M", c_int32), ("dtype", c_int32), ("W1", c_void_p),
                ("b1", c_void_p), ("W2", c_void_p), ("b2", c_void_p)]


class DsStepOutputs(ctypes.Structure):
    _fields_ = [("scores", c_void_p), ("sel", c_void_p), ("sel_count", c_void_p), ("sl_offsets", c_void_p),
                ("top_ids", c_void_p), ("top_logits", c_void_p), ("top_logp", c_void_p), ("lse", c_void_p),
                ("z_out", c_void_p), ("z_stride", c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`. "
                          "There is no CPU fallback for the DynaSpec head.")
    lib = ctypes.CDLL(LIB_PATH)
    P = c_void_p
    sig = {
        "dynaspec_status_string": (ctypes.c_char_p, [c_int32]),
        "dynaspec_budget": (c_int32, [c_int32, c_int32, c_int32]),
        "dynaspec_pa_fr_budget": (c_int32, [c_int32, c_int32]),
        "dynaspec_gather_rows": (c_int32, [P, c_int32, c_int64, c_int32, P, c_int64, P, P]),
        "dynaspec_max_shortlist": (c_int64, [POINTER(DsClusters), c_int32]),
        "dynaspec_ws_init": (c_int32, [P, c_size_t, P]),
        "dynaspec_ws_error": (c_int32, [P, c_size_t, P, P]),
        "dynaspec_build_clusters_ws": (c_size_t, [c_int64, c_int32, c_int32]),
        "dynaspec_build_clusters": (c_int32, [P, c_int32, c_int64, c_int32, c_int32, c_uint64, c_int32, P, P, P, P,
                                              P, P, P, P, c_size_t, P]),
        "dynaspec_layout_ws": (c_size_t, [c_int64, c_int32]),
        "dynaspec_layout": (c_int32, [P, P, c_int32, c_int64, c_int32, c_int32, P, P, P, P, P, c_size_t, P]),
        "dynaspec_meta_score_ws": (c_size_t, [POINTER(DsRouter), c_int32]),
        "dynaspec_meta_score": (c_int32, [POINTER(DsRouter), P, P, c_int32, P, P, c_size_t, P]),
        "dynaspec_select": (c_int32, [P, c_int32, POINTER(DsClusters), c_int32, P, c_int32, P, P, P, P]),
        "dynaspec_head_forward_ws": (c_size_t, [POINTER(DsClusters), c_int32, c_int32]),
        "dynaspec_head_forward": (c_int32, [POINTER(DsClusters), P, c_int32, P, P, P, c_int32, c_int32, c_int64, P,
                                            P, P, P, P, c_int64, P, c_size_t, P]),
        "dynaspec_draft_step_ws": (c_size_t, [POINTER(DsClusters), POINTER(DsRouter), c_int32, c_int32]),
        "dynaspec_draft_step": (c_int32, [POINTER(DsClusters), POINTER(DsRouter), P, P, P, c_int32, c_int32,
                                          c_int32, c_int32, c_int32, c_int32, POINTER(DsStepOutputs), P, c_size_t,
                                          P, P, P, P, P, P]),
        "dynaspec_debug_set_trace": (c_int32, [P]),
        "dynaspec_step_route": (c_int32, [POINTER(DsClusters), POINTER(DsRouter), P, P, c_int32, c_int32, c_int32,
                                          c_int32, c_int32, POINTER(DsStepOutputs), P, c_size_t, P]),
        "dynaspec_step_head": (c_int32, [POINTER(DsClusters), P, c_int32, c_int32, c_int32, c_int32, c_int32, c_int32,
                                         POINTER(DsStepOutputs), P, c_size_t, P]),
        "dynaspec_tree_step": (c_int32, [P, P, c_int32, c_int32, P, P, c_int32, c_int32, P, P, P, P, P, P, P, P, P]),
        "dynaspec_tree_rerank": (c_int32, [P, P, c_int32, c_int32, P, P]),
        "dynaspec_restrict_selection": (c_int32, [P, P, P, c_int32, POINTER(DsClusters), c_int32, c_int32, P, P, P, P]),
        "dynaspec_head_partial": (c_int32, [POINTER(DsClusters), P, c_int32, P, P, P, c_int32, c_int32, c_int64, P, P,
                                            c_size_t, P]),
        "dynaspec_merge_records": (c_int32, [P, c_int32, c_int32, c_int32, P, P, P, P, P]),
        "dynaspec_shortlist_ids": (c_int32, [POINTER(DsClusters), c_int32, P, P, P, c_int64, P, P]),
        "dynaspec_verify_ws": (c_size_t, [c_int64, c_int32, c_int32]),
        "dynaspec_verify_chain": (c_int32, [P, c_int32, c_int64, c_int32, c_int32, P, P, c_int64, P, P, P, P, P, P,
                                            P, P, P, c_size_t, P]),
        "dynaspec_draft_step_launches": (c_int32, [POINTER(DsClusters), POINTER(DsRouter), c_int32, c_int32,
                                                   c_int32, c_int32, c_int32]),
        "dynaspec_draft_step_kernel": (ctypes.c_char_p, [POINTER(DsClusters), POINTER(DsRouter), c_int32, c_int32,
                                                         c_int32, c_int32, c_int32]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = _load()

EXPORTED = [
    "dynaspec_status_string", "dynaspec_budget", "dynaspec_pa_fr_budget", "dynaspec_gather_rows",
    "dynaspec_max_shortlist", "dynaspec_ws_init", "dynaspec_ws_error",
    "dynaspec_build_clusters_ws", "dynaspec_build_clusters", "dynaspec_layout_ws", "dynaspec_layout",
    "dynaspec_meta_score_ws", "dynaspec_meta_score", "dynaspec_select", "dynaspec_head_forward_ws",
    "dynaspec_head_forward", "dynaspec_draft_step_ws", "dynaspec_draft_step", "dynaspec_draft_step_launches",
    "dynaspec_draft_step_kernel",
    "dynaspec_debug_set_trace", "dynaspec_restrict_selection", "dynaspec_head_partial", "dynaspec_merge_records",
    "dynaspec_tree_step", "dynaspec_tree_rerank", "dynaspec_step_route", "dynaspec_step_head",
    "dynaspec_shortlist_ids", "dynaspec_verify_ws", "dynaspec_verify_chain",
]


def lib():
    return _lib


def _check(code, what):
    if code != 0:
        raise DynaspecError(code, what)


def _ptr(t):
    return None if t is None else c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return c_void_p(s.cuda_stream)


def _need_cuda(*ts):
    for t in ts:
        if t is not None:
            if not t.is_cuda:
                raise ValueError("DynaSpec head tensors must be CUDA tensors (no CPU path)")
            if not t.is_contiguous():
                raise ValueError("DynaSpec head tensors must be contiguous")


# ---------------------------------------------------------------------------- host helpers

def debug_set_trace(buf):
    """buf: int64 CUDA tensor of >= #SM*16 entries, or None (fused-step phase timestamps)."""
    _check(_lib.dynaspec_debug_set_trace(_ptr(buf)), "dynaspec_debug_set_trace")


def budget(t, k_max, k_min=1):
    """k_c(t) (R1).  Returns -1 on invalid arguments."""
    return _lib.dynaspec_budget(t, k_max, k_min)


class Workspace:
    """Caller-provided scratch (zero-filled once, reused across calls on one stream)."""

    def __init__(self, nbytes, device="cuda"):
        self.nbytes = max(int(nbytes), 256)
        self.buf = torch.empty(self.nbytes, dtype=torch.uint8, device=device)
        _check(_lib.dynaspec_ws_init(_ptr(self.buf), self.nbytes, _stream()), "ws_init")

    def ptr(self):
        return _ptr(self.buf)

    def error(self, stream=None):
        """Read and clear the device error word (dynaspec_ws_error; synchronises the stream).
        Returns the status name, "DS_OK" if no kernel raised one."""
        code = c_int32(0)
        _check(_lib.dynaspec_ws_error(self.ptr(), self.nbytes, ctypes.cast(ctypes.pointer(code), c_void_p),
                                      _stream(stream)), "dynaspec_ws_error")
        return STATUS.get(code.value, str(code.value))

    def ensure(self, nbytes):
        if nbytes > self.nbytes:
            self.__init__(nbytes, self.buf.device)
        return self


# ---------------------------------------------------------------------------- S0 partition

class Clusters:
    """Cluster-permuted LM head (ds_clusters)."""

    def __init__(self, tau, perm, offsets, W_perm, min_size, max_size):
        self.tau, self.perm, self.offsets, self.W_perm = tau, perm, offsets, W_perm
        self.min_size, self.max_size = int(min_size), int(max_size)
        self.V, self.d = W_perm.shape
        self.M = offsets.numel() - 1
        self.dtype = W_perm.dtype
        self._s = DsClusters(self.V, self.d, self.M, _DTYPE[self.dtype], self.min_size, self.max_size,
                             _ptr(tau), _ptr(perm), _ptr(offsets), _ptr(W_perm))

    def struct(self):
        return ctypes.byref(self._s)

    def max_shortlist(self, k):
        return _lib.dynaspec_max_shortlist(self.struct(), k)

    def shard(self, m_lo, m_hi, copy=True):
        """View of this partition holding only W_perm rows of clusters [m_lo, m_hi) (cluster
        sharding): W_perm is a (copied) slice, addressed through a base pointer
        offsets[m_lo] rows before it, so global row indices keep working for owned clusters."""
        off = self.offsets.cpu()
        r0, r1 = int(off[m_lo]), int(off[m_hi])
        sl = self.W_perm[r0:r1].clone() if copy else self.W_perm[r0:r1]
        v = Clusters.__new__(Clusters)
        v.tau, v.perm, v.offsets, v.W_perm = self.tau, self.perm, self.offsets, sl
        v.min_size, v.max_size, v.V, v.d, v.M, v.dtype = self.min_size, self.max_size, self.V, self.d, self.M, self.dtype
        v.m_lo, v.m_hi, v.row0 = m_lo, m_hi, r0
        base = sl.data_ptr() - r0 * self.d * sl.element_size()
        v._s = DsClusters(self.V, self.d, self.M, _DTYPE[self.dtype], self.min_size, self.max_size, _ptr(self.tau),
                          _ptr(self.perm), _ptr(self.offsets), c_void_p(base))
        return v

    @classmethod
    def from_tau(cls, W, tau, M):
        """dynaspec_layout: perm / offsets / W_perm from a given partition tau."""
        _need_cuda(W, tau)
        V, d = W.shape
        tau = tau.to(torch.int32).contiguous()
        perm = torch.empty(V, dtype=torch.int32, device=W.device)
        offsets = torch.empty(M + 1, dtype=torch.int32, device=W.device)
        W_perm = torch.empty_like(W)
        sizes = (c_int32 * 2)()
        ws = Workspace(_lib.dynaspec_layout_ws(V, M), W.device)
        _check(_lib.dynaspec_layout(_ptr(tau), _ptr(W), _DTYPE[W.dtype], V, d, M, _ptr(perm), _ptr(offsets),
                                    _ptr(W_perm), ctypes.cast(sizes, c_void_p), ws.ptr(), ws.nbytes, _stream()),
               "dynaspec_layout")
        return cls(tau, perm, offsets, W_perm, sizes[0], sizes[1])

    @classmethod
    def build(cls, W, M, seed=2, max_iters=20, init_ids=None):
        """dynaspec_build_clusters: offline spherical k-means (R12) + layout."""
        _need_cuda(W)
        V, d = W.shape
        tau = torch.empty(V, dtype=torch.int32, device=W.device)
        perm = torch.empty(V, dtype=torch.int32, device=W.device)
        offsets = torch.empty(M + 1, dtype=torch.int32, device=W.device)
        W_perm = torch.empty_like(W)
        iters = c_int32(0)
        sizes = (c_int32 * 2)()
        init = None
        if init_ids is not None:
            init = (c_int32 * M)(*[int(x) for x in init_ids])
        ws = Workspace(_lib.dynaspec_build_clusters_ws(V, d, M), W.device)
        _check(_lib.dynaspec_build_clusters(_ptr(W), _DTYPE[W.dtype], V, d, M, seed, max_iters,
                                            None if init is None else ctypes.cast(init, c_void_p),
                                            _ptr(tau), _ptr(perm), _ptr(offsets), _ptr(W_perm),
                                            ctypes.cast(ctypes.pointer(iters), c_void_p),
                                            ctypes.cast(sizes, c_void_p), ws.ptr(), ws.nbytes, _stream()),
               "dynaspec_build_clusters")
        c = cls(tau, perm, offsets, W_perm, sizes[0], sizes[1])
        c.iters = iters.value
        return c


# ---------------------------------------------------------------------------- S1 router

class Router:
    def __init__(self, W1, b1, W2=None, b2=None):
        _need_cuda(W1, b1, W2, b2)
        self.W1, self.b1, self.W2, self.b2 = W1, b1, W2, b2
        self.h_r = 0 if W2 is None else W1.shape[0]
        self.M = W1.shape[0] if W2 is None else W2.shape[0]
        self.d = W1.shape[1] // 2
        self._s = DsRouter(self.d, self.h_r, self.M, _DTYPE[W1.dtype], _ptr(W1), _ptr(b1), _ptr(W2), _ptr(b2))

    def struct(self):
        return ctypes.byref(self._s)


def meta_score(router, h_prev, e, ws=None):
    _need_cuda(h_prev, e)
    B = h_prev.shape[0]
    scores = torch.empty((B, router.M), dtype=torch.float32, device=h_prev.device)
    ws = (ws or Workspace(256, h_prev.device)).ensure(_lib.dynaspec_meta_score_ws(router.struct(), B))
    _check(_lib.dynaspec_meta_score(router.struct(), _ptr(h_prev), _ptr(e), B, _ptr(scores), ws.ptr(), ws.nbytes,
                                    _stream()), "dynaspec_meta_score")
    return scores


# ---------------------------------------------------------------------------- S3/S4 select

def select(scores, clusters, k, shared=False, k_per_row=None):
    _need_cuda(scores, k_per_row)
    B, M = scores.shape
    rows = 1 if shared else B
    dev = scores.device
    sel = torch.empty((rows, M), dtype=torch.int32, device=dev)
    cnt = torch.empty(rows, dtype=torch.int32, device=dev)
    off = torch.empty((rows, M + 1), dtype=torch.int32, device=dev)
    _check(_lib.dynaspec_select(_ptr(scores), B, clusters.struct(), k, _ptr(k_per_row), int(shared), _ptr(sel),
                                _ptr(cnt), _ptr(off), _stream()), "dynaspec_select")
    return sel, cnt, off


# ---------------------------------------------------------------------------- S5/S6 head

def head_forward(clusters, h_new, sel, sel_count, sl_offsets, k_t, shared=False, max_shortlist=0, z_out=False,
                 ws=None):
    _need_cuda(h_new, sel, sel_count, sl_offsets)
    B = h_new.shape[0]
    dev = h_new.device
    out = {
        "top_ids": torch.empty((B, k_t), dtype=torch.int32, device=dev),
        "top_logits": torch.empty((B, k_t), dtype=torch.float32, device=dev),
        "top_logp": torch.empty((B, k_t), dtype=torch.float32, device=dev),
        "lse": torch.empty(B, dtype=torch.float32, device=dev),
    }
    zs = 0
    z = None
    if z_out:
        zs = max_shortlist if max_shortlist > 0 else clusters.V
        z = torch.full((B, zs), float("nan"), dtype=torch.float32, device=dev)
    ws = (ws or Workspace(256, dev)).ensure(_lib.dynaspec_head_forward_ws(clusters.struct(), B, k_t))
    _check(_lib.dynaspec_head_forward(clusters.struct(), _ptr(h_new), B, _ptr(sel), _ptr(sel_count),
                                      _ptr(sl_offsets), int(shared), k_t, max_shortlist, _ptr(out["top_ids"]),
                                      _ptr(out["top_logits"]), _ptr(out["top_logp"]), _ptr(out["lse"]), _ptr(z), zs,
                                      ws.ptr(), ws.nbytes, _stream()), "dynaspec_head_forward")
    out["z"] = z
    return out


# ---------------------------------------------------------------------------- draft tree (NEXT-1)

class DraftTree:
    """Device-resident draft list d (Alg. 1 lines 12-18) for up to `capacity` nodes."""

    def __init__(self, k_t, capacity, device="cuda"):
        self.k_t, self.capacity = k_t, capacity
        z = lambda dt: torch.zeros(capacity, dtype=dt, device=device)
        self.tok, self.score, self.parent, self.depth = z(torch.int32), z(torch.float32), z(torch.int32), z(torch.int32)
        self.next_tok = torch.zeros(k_t, dtype=torch.int32, device=device)
        self.next_score = torch.zeros(k_t, dtype=torch.float32, device=device)
        self.next_node = torch.zeros(k_t, dtype=torch.int32, device=device)
        self.next_beam = torch.zeros(k_t, dtype=torch.int32, device=device)
        self.n = 0

    def step(self, top_ids, top_logp, j):
        """Fold the head outputs [R][k_t] of draft step j into the tree (R = 1 at j = 0)."""
        R = top_ids.shape[0]
        if self.n + R * self.k_t > self.capacity:
            raise ValueError(f"DraftTree capacity {self.capacity} exceeded")
        first = j == 0
        last_s = None if first else self.next_score.clone()
        last_n = None if first else self.next_node.clone()
        _check(_lib.dynaspec_tree_step(_ptr(top_ids), _ptr(top_logp), R, self.k_t, _ptr(last_s), _ptr(last_n), j,
                                       self.n, _ptr(self.tok), _ptr(self.score), _ptr(self.parent), _ptr(self.depth),
                                       _ptr(self.next_tok), _ptr(self.next_score), _ptr(self.next_node),
                                       _ptr(self.next_beam), _stream()), "dynaspec_tree_step")
        self.n += R * self.k_t
        return self

    def rerank(self, n_out):
        out = torch.empty(n_out, dtype=torch.int32, device=self.tok.device)
        _check(_lib.dynaspec_tree_rerank(_ptr(self.score), _ptr(self.tok), self.n, n_out, _ptr(out), _stream()),
               "dynaspec_tree_rerank")
        return out


# ---------------------------------------------------------------------------- cluster sharding

def restrict_selection(sel, sel_count, sl_offsets, clusters, m_lo, m_hi):
    rows, M = sel.shape
    o_sel = torch.zeros_like(sel)
    o_cnt = torch.zeros_like(sel_count)
    o_off = torch.zeros_like(sl_offsets)
    _check(_lib.dynaspec_restrict_selection(_ptr(sel), _ptr(sel_count), _ptr(sl_offsets), rows, clusters.struct(),
                                            m_lo, m_hi, _ptr(o_sel), _ptr(o_cnt), _ptr(o_off), _stream()),
           "dynaspec_restrict_selection")
    return o_sel, o_cnt, o_off


def head_partial(clusters, h_new, sel, sel_count, sl_offsets, k_t, shared=False, max_shortlist=0, ws=None,
                 records=None):
    """Per-row records {max, sum exp, top-k_t (z, id)} of this shard (dynaspec_head_partial)."""
    B = h_new.shape[0]
    rec = 2 + 2 * k_t
    if records is None:
        records = torch.empty((B, rec), dtype=torch.float32, device=h_new.device)
    ws = (ws or Workspace(256, h_new.device)).ensure(_lib.dynaspec_head_forward_ws(clusters.struct(), B, k_t))
    _check(_lib.dynaspec_head_partial(clusters.struct(), _ptr(h_new), B, _ptr(sel), _ptr(sel_count),
                                      _ptr(sl_offsets), int(shared), k_t, max_shortlist, _ptr(records), ws.ptr(),
                                      ws.nbytes, _stream()), "dynaspec_head_partial")
    return records


def merge_records(records, k_t):
    """records: [G][B][2 + 2 k_t] (rank-major) -> dict(top_ids, top_logits, top_logp, lse)."""
    G, B, _ = records.shape
    dev = records.device
    out = {"top_ids": torch.empty((B, k_t), dtype=torch.int32, device=dev),
           "top_logits": torch.empty((B, k_t), dtype=torch.float32, device=dev),
           "top_logp": torch.empty((B, k_t), dtype=torch.float32, device=dev),
           "lse": torch.empty(B, dtype=torch.float32, device=dev)}
    _check(_lib.dynaspec_merge_records(_ptr(records.contiguous()), G, B, k_t, _ptr(out["top_ids"]),
                                       _ptr(out["top_logits"]), _ptr(out["top_logp"]), _ptr(out["lse"]), _stream()),
           "dynaspec_merge_records")
    return out


# ---------------------------------------------------------------------------- S7 draft step

def make_event(enable_timing=False):
    """torch.cuda.Event created eagerly (torch creates the CUDA event lazily on first record)."""
    ev = torch.cuda.Event(enable_timing=enable_timing)
    ev.record()
    return ev


class DraftStep:
    """Pre-allocated outputs + workspace + events for repeated dynaspec_draft_step calls
    (graph-capturable: no allocation, no host sync inside __call__)."""

    def __init__(self, clusters, router, B, k_t, shared=False, z_out=False, two_streams=False, device="cuda"):
        """two_streams=False: one fused launch per step (router + select + head + epilogue);
        two_streams=True: router + select on a side stream S_m joined before the head."""
        self.c, self.r, self.B, self.k_t, self.shared = clusters, router, B, k_t, bool(shared)
        M = clusters.M
        rows = 1 if shared else B
        dev = device
        self.scores = torch.zeros((B, M), dtype=torch.float32, device=dev)
        self.sel = torch.zeros((rows, M), dtype=torch.int32, device=dev)
        self.sel_count = torch.zeros(rows, dtype=torch.int32, device=dev)
        self.sl_offsets = torch.zeros((rows, M + 1), dtype=torch.int32, device=dev)
        self.top_ids = torch.empty((B, k_t), dtype=torch.int32, device=dev)
        self.top_logits = torch.empty((B, k_t), dtype=torch.float32, device=dev)
        self.top_logp = torch.empty((B, k_t), dtype=torch.float32, device=dev)
        self.lse = torch.empty(B, dtype=torch.float32, device=dev)
        self.z_stride = clusters.V if z_out else 0
        self.z = torch.full((B, clusters.V), float("nan"), dtype=torch.float32, device=dev) if z_out else None
        self._o = DsStepOutputs(_ptr(self.scores), _ptr(self.sel), _ptr(self.sel_count), _ptr(self.sl_offsets),
                                _ptr(self.top_ids), _ptr(self.top_logits), _ptr(self.top_logp), _ptr(self.lse),
                                _ptr(self.z), self.z_stride)
        self.ws = Workspace(_lib.dynaspec_draft_step_ws(clusters.struct(), router.struct(), B, k_t), dev)
        self.two_streams = two_streams
        self.s_meta = torch.cuda.Stream(device=dev) if two_streams else None
        self.ev_fork = make_event() if two_streams else None
        self.ev_join = make_event() if two_streams else None
        self.launches = _lib.dynaspec_draft_step_launches(clusters.struct(), router.struct(), B, k_t, int(shared),
                                                          int(two_streams), int(bool(z_out)))
        self.kernel = _lib.dynaspec_draft_step_kernel(clusters.struct(), router.struct(), B, k_t, int(shared),
                                                      int(two_streams), int(bool(z_out))).decode()

    def __call__(self, h_prev, e, h_new, t, k_max, k_min, head_events=None, stream=None):
        sd = _stream(stream)
        hb, he = (head_events if head_events is not None else (None, None))
        _check(_lib.dynaspec_draft_step(self.c.struct(), self.r.struct(), _ptr(h_prev), _ptr(e), _ptr(h_new), self.B,
                                        t, k_max, k_min, self.k_t, int(self.shared), ctypes.byref(self._o),
                                        self.ws.ptr(), self.ws.nbytes, sd,
                                        c_void_p(self.s_meta.cuda_stream) if self.s_meta is not None else None,
                                        self.ev_fork, self.ev_join, hb, he), "dynaspec_draft_step")
        return self

    def route(self, h_prev, e, t, k_max, k_min, stream):
        """Router + TopK half of the step (Alg. 1 line 8) on `stream` (S_m)."""
        if not hasattr(self, "ws_head"):
            self.ws_head = Workspace(_lib.dynaspec_head_forward_ws(self.c.struct(), self.B, self.k_t),
                                     self.ws.buf.device)
        _check(_lib.dynaspec_step_route(self.c.struct(), self.r.struct(), _ptr(h_prev), _ptr(e), self.B, t, k_max,
                                        k_min, int(self.shared), ctypes.byref(self._o), self.ws.ptr(), self.ws.nbytes,
                                        _stream(stream)), "dynaspec_step_route")

    def head(self, h_new, t, k_max, k_min, stream):
        """Head + epilogue half of the step (Alg. 1 lines 10-11) on `stream` (S_d)."""
        if not hasattr(self, "ws_head"):
            self.ws_head = Workspace(_lib.dynaspec_head_forward_ws(self.c.struct(), self.B, self.k_t),
                                     self.ws.buf.device)
        _check(_lib.dynaspec_step_head(self.c.struct(), _ptr(h_new), self.B, t, k_max, k_min, self.k_t,
                                       int(self.shared), ctypes.byref(self._o), self.ws_head.ptr(),
                                       self.ws_head.nbytes, _stream(stream)), "dynaspec_step_head")

    def bind_outputs(self, top_ids=None, top_logp=None):
        """Write the token top-k ids / log-probs into caller tensors (contiguous (B, k_t) int32 /
        float32 on the step's device, e.g. slices of one buffer read back with a single copy)."""
        for name, t, dt in (("top_ids", top_ids, torch.int32), ("top_logp", top_logp, torch.float32)):
            if t is None:
                continue
            if t.dtype != dt or tuple(t.shape) != (self.B, self.k_t) or not t.is_contiguous():
                raise ValueError(f"{name}: need a contiguous ({self.B}, {self.k_t}) {dt} tensor")
            setattr(self, name, t)
        self._o.top_ids = _ptr(self.top_ids)
        self._o.top_logp = _ptr(self.top_logp)
        return self

    def outputs(self):
        return {k: getattr(self, k) for k in ("scores", "sel", "sel_count", "sl_offsets", "top_ids", "top_logits",
                                               "top_logp", "lse", "z")}


# ---------------------------------------------------------------------------- static heads (NEXT-3)

class FrequencyHead:
    """FR-Spec / PA-FR static shortlist heads (App. A.1) on the same kernels:
    W is stored in frequency order (a drafter-side copy, like W_perm) and the shortlist of step t
    is the prefix [0, K) — one contiguous run, expressed as a one-cluster partition."""

    def __init__(self, W, pi_f):
        _need_cuda(W)
        self.V, self.d = W.shape
        self.perm = torch.as_tensor(pi_f, dtype=torch.int32, device=W.device).contiguous()
        self.W_freq = torch.empty_like(W)  # W_freq[i] = W[pi_f[i]] (dynaspec_gather_rows)
        _check(_lib.dynaspec_gather_rows(_ptr(W.contiguous()), _DTYPE[W.dtype], self.V, self.d, _ptr(self.perm),
                                         self.V, _ptr(self.W_freq), _stream()), "dynaspec_gather_rows")
        self._views = {}

    def _view(self, K):
        if K not in self._views:
            dev = self.W_freq.device
            off = torch.tensor([0, K], dtype=torch.int32, device=dev)
            sel = torch.zeros((1, 1), dtype=torch.int32, device=dev)
            cnt = torch.ones(1, dtype=torch.int32, device=dev)
            sl = torch.tensor([[0, K]], dtype=torch.int32, device=dev)
            c = Clusters.__new__(Clusters)
            c.tau, c.perm, c.offsets, c.W_perm = None, self.perm, off, self.W_freq
            c.min_size = c.max_size = K
            c.V, c.d, c.M, c.dtype = self.V, self.d, 1, self.W_freq.dtype
            c._s = DsClusters(self.V, self.d, 1, _DTYPE[c.dtype], K, K, None, _ptr(self.perm), _ptr(off),
                              _ptr(self.W_freq))
            self._views[K] = (c, sel, cnt, sl, off)
        return self._views[K]

    def forward(self, h_new, K, k_t, z_out=False, ws=None):
        """Top-k_t / lse / logp over the K most frequent tokens (ids are vocabulary ids)."""
        c, sel, cnt, sl, _ = self._view(int(K))
        return head_forward(c, h_new, sel, cnt, sl, k_t, shared=True, max_shortlist=int(K), z_out=z_out, ws=ws)

    def forward_pa_fr(self, h_new, t, K_max, k_t, z_out=False, ws=None):
        """PA-FR: the prefix length shrinks with the draft position, K_fr(t) (App. A.1)."""
        return self.forward(h_new, pa_fr_budget(t, K_max), k_t, z_out=z_out, ws=ws)


def pa_fr_budget(t, K_max):
    """K_fr(t) = K_max for t < 2, else max(1, floor(K_max / (t + 1))) (App. A.1):
    dynaspec_pa_fr_budget."""
    k = _lib.dynaspec_pa_fr_budget(int(t), int(K_max))
    if k < 1:
        raise ValueError("pa_fr_budget: t >= 0 and K_max >= 1 required")
    return k


# ---------------------------------------------------------------------------- verification (NEXT-4)

def shortlist_ids(clusters, sel, sel_count, sl_offsets, stride, rows=None):
    """dynaspec_shortlist_ids: V_S as vocabulary ids in shortlist order, [rows][stride] (-1 padded)."""
    _need_cuda(sel, sel_count, sl_offsets)
    rows = sel_count.shape[0] if rows is None else rows
    ids = torch.full((rows, stride), -1, dtype=torch.int32, device=sel.device)
    _check(_lib.dynaspec_shortlist_ids(clusters.struct(), rows, _ptr(sel), _ptr(sel_count), _ptr(sl_offsets), stride,
                                       _ptr(ids), _stream()), "dynaspec_shortlist_ids")
    return ids


class Verifier:
    """dynaspec_verify_chain with a persistent (self-zeroing) workspace (Eq. 3; R25)."""

    def __init__(self, V, B, gamma, device="cuda"):
        self.V, self.B, self.gamma = V, B, gamma
        self.ws = Workspace(_lib.dynaspec_verify_ws(V, B, gamma), device)
        self.accepted = torch.zeros(B, dtype=torch.int32, device=device)
        self.committed = torch.full((B, gamma + 1), -1, dtype=torch.int32, device=device)

    def __call__(self, p_logits, q_ids, q_logits, q_count, q_lse, x, x_slot, u_acc, u_res):
        _need_cuda(p_logits, u_res)
        B, g1, V = p_logits.shape
        if (B, g1 - 1, V) != (self.B, self.gamma, self.V):
            raise ValueError("shape does not match the Verifier")
        g = self.gamma
        stride = q_ids.shape[-1] if g > 0 else 1
        _check(_lib.dynaspec_verify_chain(_ptr(p_logits), _DTYPE[p_logits.dtype], V, B, g,
                                          _ptr(q_ids) if g else None, _ptr(q_logits) if g else None, stride,
                                          _ptr(q_count) if g else None, _ptr(q_lse) if g else None,
                                          _ptr(x) if g else None, _ptr(x_slot) if g else None,
                                          _ptr(u_acc) if g else None, _ptr(u_res), _ptr(self.accepted),
                                          _ptr(self.committed), self.ws.ptr(), self.ws.nbytes, _stream()),
               "dynaspec_verify_chain")
        return self.accepted, self.committed
