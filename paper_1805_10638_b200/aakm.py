"""Thin Python binding of libaakm.so (include/aakm.h).  Argument marshalling
only: every step of the hot path runs in the library's sm_100a kernels.
PyTorch provides device memory (the workspace and outputs), the CUDA stream
and, for nranks > 1, the process group used to broadcast the NCCL id.

There is no CPU fallback: :func:`lib` raises if the shared library is missing.
"""
from __future__ import annotations

import ctypes as ct
import dataclasses
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libaakm.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "aakm.h")
_lib = None
_lock = threading.Lock()

KMEANS_M_MAX = 30
PATHS = {"auto": 0, "simt": 1, "tc": 2, "tc16": 3}
STATUS = {0: "OK", 1: "INVALID", 2: "CUDA", 3: "NCCL", 4: "NOMEM", 5: "STATE"}


class AAKMError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"kmeans status {STATUS.get(status, status)}: {msg}")
        self.status = status


class Config(ct.Structure):
    _fields_ = [("m0", ct.c_int32), ("m_max", ct.c_int32), ("eps1", ct.c_double), ("eps2", ct.c_double),
                ("dynamic_m", ct.c_int32), ("max_iters", ct.c_int32), ("ridge", ct.c_double),
                ("assign_path", ct.c_int32), ("timing", ct.c_int32), ("bounded", ct.c_int32),
                ("x_refresh", ct.c_int32), ("comm_always", ct.c_int32), ("fused_comm", ct.c_int32)]


class Report(ct.Structure):
    _fields_ = [("iters", ct.c_int64), ("n_assign", ct.c_int64), ("n_accepted", ct.c_int64),
                ("n_rejected", ct.c_int64), ("converged", ct.c_int32), ("m_final", ct.c_int32),
                ("energy", ct.c_double), ("mse", ct.c_double), ("seconds", ct.c_double)]


class StepInfo(ct.Structure):
    _fields_ = [("t", ct.c_int64), ("m", ct.c_int32), ("m_t", ct.c_int32), ("accepted", ct.c_int32),
                ("rejected", ct.c_int32), ("converged", ct.c_int32), ("lloyd", ct.c_int32),
                ("energy_cand", ct.c_double), ("energy", ct.c_double), ("changed", ct.c_int64)]


class State(ct.Structure):
    _fields_ = [("C", ct.c_void_p), ("fallback", ct.c_void_p), ("Ghist", ct.c_void_p), ("Fhist", ct.c_void_p),
                ("labels_prev", ct.c_void_p), ("hist_count", ct.c_int32), ("m", ct.c_int32),
                ("lloyd", ct.c_int32), ("done", ct.c_int32), ("t", ct.c_int64), ("E1", ct.c_double),
                ("E2", ct.c_double), ("n_accepted", ct.c_int64), ("n_rejected", ct.c_int64),
                ("n_assign", ct.c_int64), ("gram", ct.c_void_p)]


def _struct(s):
    return {k: getattr(s, k) for k, _ in s._fields_}


def lib():
    """Load libaakm.so (built by ``__graft_entry__.build()``); raise if absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                                  "(there is no CPU fallback)")
            L = ct.CDLL(LIB_PATH)
            P, I64, I32, D, S = ct.c_void_p, ct.c_int64, ct.c_int32, ct.c_double, ct.c_size_t
            sig = {
                "kmeans_abi_version": ([], I32),
                "kmeans_config_default": ([ct.POINTER(Config)], I32),
                "kmeans_workspace_size": ([I64, I32, I32, ct.POINTER(Config), ct.POINTER(S)], I32),
                "kmeans_nccl_unique_id": ([P], I32),
                "kmeans_create": ([ct.POINTER(P), P, I64, I64, I32, I32, ct.POINTER(Config), P, S, I32, I32, P, P], I32),
                "kmeans_assign": ([P, P, P, P, ct.POINTER(D), ct.POINTER(I64)], I32),
                "kmeans_update": ([P, P, P, P, P], I32),
                "kmeans_aa_step": ([P, P, ct.POINTER(StepInfo), P], I32),
                "kmeans_run": ([P, P, P, P, ct.POINTER(Report)], I32),
                "kmeans_get_centroids": ([P, P, P], I32),
                "kmeans_state_export": ([P, ct.POINTER(State)], I32),
                "kmeans_state_import": ([P, ct.POINTER(State)], I32),
                "kmeans_update_partials": ([P, P, P, P, P], I32),
                "kmeans_assign_timing": ([P, ct.POINTER(D), ct.POINTER(I64)], I32),
                "kmeans_launch_count": ([P], I64),
                "kmeans_last_flagged": ([P, ct.POINTER(I64)], I32),
                "kmeans_bounded_stats": ([P, ct.POINTER(I64), ct.POINTER(I64)], I32),
                "kmeans_update_stats": ([P, ct.POINTER(I64), ct.POINTER(I64), ct.POINTER(I64)], I32),
                "kmeans_seed_pp": ([P, P, P, P], I32),
                "kmeans_aa_step_host": ([P, P, I32, P, P], I32),
                "kmeans_update_timing": ([P, ct.POINTER(D), ct.POINTER(I64)], I32),
                "kmeans_assign_path_name": ([P], ct.c_char_p),
                "kmeans_debug_scores": ([P, P, P, ct.POINTER(I32), ct.POINTER(D)], I32),
                "kmeans_bounds_export": ([P, P, P, P, P], I32),
                "kmeans_trace_export": ([P, P, I64, ct.POINTER(I64)], I32),
                "kmeans_comm_info": ([P, ct.POINTER(I32), ct.POINTER(I32)], I32),
                "kmeans_debug_check_canaries": ([P, ct.POINTER(I64), ct.POINTER(I64)], I32),
                "kmeans_bounds_repeat": ([P, P, P, P, ct.POINTER(I32)], I32),
                "kmeans_destroy": ([P], I32),
                "kmeans_last_error": ([P], ct.c_char_p),
            }
            for name, (args, res) in sig.items():
                f = getattr(L, name)
                f.argtypes = args
                f.restype = res
            _lib = L
    return _lib


def header_symbols():
    """Entry points declared in include/aakm.h (for the ABI export test)."""
    import re
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(kmeans_[a-z0-9_]+)\s*\(", txt)))


def config(m0=5, m_max=30, eps1=0.02, eps2=0.5, dynamic_m=True, max_iters=10000, ridge=1e-10,
           assign_path="auto", timing=False, bounded=False, x_refresh=False, comm_always=False,
           fused_comm=False) -> Config:
    """Algorithm 1 settings (m0 = 5 per BASELINE configs, reading R-A18)."""
    c = Config()
    c.m0, c.m_max, c.eps1, c.eps2 = m0, m_max, eps1, eps2
    c.dynamic_m, c.max_iters, c.ridge = int(dynamic_m), max_iters, ridge
    c.assign_path = PATHS[assign_path] if isinstance(assign_path, str) else int(assign_path)
    c.timing = int(timing)
    c.bounded = int(bounded)
    c.x_refresh = int(x_refresh)
    c.comm_always = int(comm_always)
    c.fused_comm = int(fused_comm)
    return c


def broadcast_uid(rank: int, group=None, device=None):
    """Rank 0 draws the 128-byte NCCL unique id (kmeans_nccl_unique_id); every
    rank receives it over the torch process group (gloo: CPU tensor, nccl:
    device tensor).  Returns a ctypes uint8[128]."""
    import torch
    import torch.distributed as dist
    buf = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        raw = (ct.c_uint8 * 128)()
        rc = lib().kmeans_nccl_unique_id(raw)
        if rc != 0:
            raise AAKMError(rc, lib().kmeans_last_error(None).decode())
        buf = torch.tensor(list(raw), dtype=torch.uint8)
    if dist.get_backend(group) == "nccl":
        buf = buf.to(device if device is not None else "cuda")
    dist.broadcast(buf, src=0, group=group)
    return (ct.c_uint8 * 128)(*buf.cpu().tolist())


def _ptr(t):
    return ct.c_void_p(0 if t is None else t.data_ptr())


class KMeans:
    """One rank's handle over its row shard X (torch CUDA float32, n_local x d)."""

    def __init__(self, X, K: int, cfg: Config | None = None, *, n_global: int | None = None,
                 rank: int = 0, nranks: int = 1, group=None, stream=None):
        import torch
        self.torch = torch
        L = lib()
        if X.dtype != torch.float32 or not X.is_cuda or not X.is_contiguous() or X.dim() != 2:
            raise ValueError("X must be a contiguous 2-D float32 CUDA tensor")
        self.X = X
        self.n, self.d = X.shape
        self.K = int(K)
        self.cfg = cfg or config()
        self.device = X.device
        self.stream = stream or torch.cuda.current_stream(self.device)
        self.n_global = int(n_global if n_global is not None else self.n)
        nbytes = ct.c_size_t()
        self._check(L.kmeans_workspace_size(self.n, self.d, self.K, ct.byref(self.cfg), ct.byref(nbytes)), None)
        self.ws = torch.empty(nbytes.value + 256, dtype=torch.uint8, device=self.device)
        base = self.ws.data_ptr()
        self.ws_ptr = (base + 255) & ~255
        uid = None
        if nranks > 1:
            uid = broadcast_uid(rank, group, self.device)
        h = ct.c_void_p()
        with torch.cuda.device(self.device):
            self._check(L.kmeans_create(ct.byref(h), _ptr(X), self.n, self.n_global, self.d, self.K,
                                        ct.byref(self.cfg), ct.c_void_p(self.ws_ptr), nbytes.value, rank, nranks,
                                        uid, ct.c_void_p(self.stream.cuda_stream)), None)
        self.h = h
        self.rank, self.nranks = rank, nranks

    # -- helpers
    def _check(self, rc, h):
        if rc != 0:
            msg = lib().kmeans_last_error(h if h is not None else None)
            raise AAKMError(rc, msg.decode() if msg else "")

    def _c(self, rc):
        self._check(rc, self.h)

    def _f64(self, C):
        """Centroids as a contiguous K x d float64 device tensor (the ABI's fp64 state)."""
        t = self.torch
        C = t.as_tensor(C, dtype=t.float64, device=self.device).reshape(self.K, self.d).contiguous()
        return C

    def _i32(self, L):
        t = self.torch
        return t.as_tensor(L, dtype=t.int32, device=self.device).reshape(self.n).contiguous()

    @property
    def path(self) -> str:
        return lib().kmeans_assign_path_name(self.h).decode()

    def launch_count(self) -> int:
        return lib().kmeans_launch_count(self.h)

    # -- entry points
    def assign(self, C, labels_prev=None):
        """Eq. 3 labels, global E(P, C) and #changed vs labels_prev."""
        t = self.torch
        C = self._f64(C)
        lp = None if labels_prev is None else self._i32(labels_prev)
        out = t.empty(self.n, dtype=t.int32, device=self.device)
        E, ch = ct.c_double(), ct.c_int64()
        self._c(lib().kmeans_assign(self.h, _ptr(C), _ptr(lp), _ptr(out), ct.byref(E), ct.byref(ch)))
        return out, E.value, ch.value

    def update(self, labels, C_prev):
        """Eq. 4 means (global), empty clusters keep C_prev; returns (G, counts)."""
        t = self.torch
        labels = self._i32(labels)
        C_prev = self._f64(C_prev)
        G = t.empty_like(C_prev)
        cnt = t.empty(self.K, dtype=t.int64, device=self.device)
        self._c(lib().kmeans_update(self.h, _ptr(labels), _ptr(C_prev), _ptr(G), _ptr(cnt)))
        return G, cnt

    def update_partials(self, labels, C, labels_prev=None):
        t = self.torch
        labels = self._i32(labels)
        C = self._f64(C)
        lp = None if labels_prev is None else self._i32(labels_prev)
        out = t.empty(self.K * self.d + self.K + 2, dtype=t.float64, device=self.device)
        self._c(lib().kmeans_update_partials(self.h, _ptr(labels), _ptr(lp), _ptr(C), _ptr(out)))
        return out

    def aa_step(self, C0=None, info=True):
        """Algorithm 1 line 1 (C0 given) or one loop pass; returns the pass info dict (or None)."""
        C0 = None if C0 is None else self._f64(C0)
        if not info:
            self._c(lib().kmeans_aa_step(self.h, _ptr(C0), None, None))
            return None
        inf = StepInfo()
        theta = (ct.c_double * KMEANS_M_MAX)()
        self._c(lib().kmeans_aa_step(self.h, _ptr(C0), ct.byref(inf), theta))
        r = _struct(inf)
        r["theta"] = list(theta)[: r["m_t"]]
        return r

    def aa_step_host(self, X_host, chunks=8, info=True):
        """One loop pass with X refreshed from host memory (kmeans_aa_step_host):
        X_host is a CPU float32 tensor of this handle's shape (pin it for overlap);
        the copy streams in `chunks` row blocks under the assignment."""
        t = self.torch
        if not isinstance(X_host, t.Tensor) or X_host.device.type != "cpu":
            raise TypeError("X_host must be a CPU torch tensor")
        if X_host.dtype != t.float32 or not X_host.is_contiguous() or tuple(X_host.shape) != (self.n, self.d):
            raise ValueError("X_host must be a contiguous float32 (n_local, d) tensor")
        self._keep_host = X_host                    # valid until the stream passes this call
        if not info:
            self._c(lib().kmeans_aa_step_host(self.h, ct.c_void_p(X_host.data_ptr()), int(chunks), None, None))
            return None
        inf = StepInfo()
        theta = (ct.c_double * KMEANS_M_MAX)()
        self._c(lib().kmeans_aa_step_host(self.h, ct.c_void_p(X_host.data_ptr()), int(chunks), ct.byref(inf), theta))
        r = _struct(inf)
        r["theta"] = list(theta)[: r["m_t"]]
        return r

    def run(self, C0):
        """Algorithm 1 to convergence (rule R3); returns (C, labels, report dict)."""
        t = self.torch
        C0 = self._f64(C0)
        C = t.empty_like(C0)
        labels = t.empty(self.n, dtype=t.int32, device=self.device)
        rep = Report()
        self._c(lib().kmeans_run(self.h, _ptr(C0), _ptr(C), _ptr(labels), ct.byref(rep)))
        return C, labels, _struct(rep)

    def centroids(self):
        t = self.torch
        C = t.empty(self.K, self.d, dtype=t.float64, device=self.device)
        lab = t.empty(self.n, dtype=t.int32, device=self.device)
        self._c(lib().kmeans_get_centroids(self.h, _ptr(C), _ptr(lab)))
        self.stream.synchronize()
        return C, lab

    def state_export(self):
        H = self.cfg.m_max + 1
        KD = self.K * self.d
        C = np.zeros(KD, np.float64); fb = np.zeros(KD, np.float64)
        Gh = np.zeros(H * KD, np.float64); Fh = np.zeros(H * KD, np.float64)
        lp = np.zeros(max(self.n, 1), np.int32)
        gr = np.zeros(H * H, np.float64)
        s = State()
        s.C, s.fallback, s.Ghist, s.Fhist, s.labels_prev = (C.ctypes.data, fb.ctypes.data, Gh.ctypes.data,
                                                            Fh.ctypes.data, lp.ctypes.data)
        s.gram = gr.ctypes.data
        self._c(lib().kmeans_state_export(self.h, ct.byref(s)))
        r = _struct(s)
        for k in ("C", "fallback", "Ghist", "Fhist", "labels_prev", "gram"):
            r.pop(k)
        hc = r["hist_count"]
        r.update(C=C.reshape(self.K, self.d), fallback=fb.reshape(self.K, self.d),
                 Ghist=Gh.reshape(H, self.K, self.d)[:hc], Fhist=Fh.reshape(H, self.K, self.d)[:hc],
                 labels_prev=lp[: self.n], gram=gr)
        return r

    def state_import(self, st, with_gram=True):
        """Resume Algorithm 1 from a state_export() dict (checkpoint/resume)."""
        KD = self.K * self.d
        hc = int(st["hist_count"])
        H = self.cfg.m_max + 1
        C = np.ascontiguousarray(st["C"], np.float64).reshape(KD)
        fb = np.ascontiguousarray(st["fallback"], np.float64).reshape(KD)
        Gh = np.zeros(H * KD, np.float64); Fh = np.zeros(H * KD, np.float64)
        Gh[: hc * KD] = np.ascontiguousarray(st["Ghist"], np.float64).reshape(-1)[: hc * KD]
        Fh[: hc * KD] = np.ascontiguousarray(st["Fhist"], np.float64).reshape(-1)[: hc * KD]
        lp = np.ascontiguousarray(st["labels_prev"], np.int32).reshape(-1)
        gr = np.ascontiguousarray(st["gram"], np.float64) if with_gram else None
        s = State()
        s.C, s.fallback, s.Ghist, s.Fhist = C.ctypes.data, fb.ctypes.data, Gh.ctypes.data, Fh.ctypes.data
        s.labels_prev = lp.ctypes.data if self.n > 0 else None
        s.gram = gr.ctypes.data if gr is not None else None
        s.hist_count, s.m, s.lloyd, s.done, s.t = hc, int(st["m"]), int(st["lloyd"]), int(st["done"]), int(st["t"])
        s.E1, s.E2 = float(st["E1"]), float(st["E2"])
        s.n_accepted, s.n_rejected, s.n_assign = int(st["n_accepted"]), int(st["n_rejected"]), int(st["n_assign"])
        self._c(lib().kmeans_state_import(self.h, ct.byref(s)))

    def trace(self, cap=8192):
        """The per-pass trace of the current run (kmeans_trace_export): a list of
        step-info dicts, one per loop pass."""
        n = ct.c_int64()
        buf = (StepInfo * max(cap, 1))()
        self._c(lib().kmeans_trace_export(self.h, buf, cap, ct.byref(n)))
        return [_struct(buf[i]) for i in range(min(n.value, cap))]

    def comm_info(self):
        """(mode, lsa_size): -1 no communicator, 0 ncclAllReduce, 1 fused multimem, 2 fused LSA unicast."""
        m, l = ct.c_int32(), ct.c_int32()
        self._c(lib().kmeans_comm_info(self.h, ct.byref(m), ct.byref(l)))
        return m.value, l.value

    def check_canaries(self):
        """(changed canary bytes, canaries) of the checked-workspace mode (AAKM_WS_CANARY=1)."""
        bad, n = ct.c_int64(), ct.c_int64()
        self._c(lib().kmeans_debug_check_canaries(self.h, ct.byref(bad), ct.byref(n)))
        return bad.value, n.value

    def assign_timing(self):
        ms, n = ct.c_double(), ct.c_int64()
        self._c(lib().kmeans_assign_timing(self.h, ct.byref(ms), ct.byref(n)))
        return ms.value, n.value

    def update_timing(self):
        """(ms, launches) of the timed update partials since the last call (cfg.timing)."""
        ms, n = ct.c_double(), ct.c_int64()
        self._c(lib().kmeans_update_timing(self.h, ct.byref(ms), ct.byref(n)))
        return ms.value, n.value

    def bounded_stats(self):
        """(rows run through the assignment engine, rows assigned) since line 1."""
        a, b = ct.c_int64(), ct.c_int64()
        self._c(lib().kmeans_bounded_stats(self.h, ct.byref(a), ct.byref(b)))
        return a.value, b.value

    def update_stats(self):
        """(G-evaluations, of them incremental, their moved rows) since line 1."""
        a, b, c = ct.c_int64(), ct.c_int64(), ct.c_int64()
        self._c(lib().kmeans_update_stats(self.h, ct.byref(a), ct.byref(b), ct.byref(c)))
        return a.value, b.value, c.value

    def seed_pp(self, u):
        """K-Means++ seeding (kmeans_seed_pp) with the caller's K uniforms in [0, 1):
        returns (C0 as a K x d device tensor, the K global sample indices)."""
        import numpy as np
        t = self.torch
        u = np.ascontiguousarray(u, dtype=np.float64)
        if u.shape != (self.K,):
            raise ValueError("u must hold K uniforms")
        C = t.empty((self.K, self.d), dtype=t.float32, device=self.device)
        idx = np.zeros(self.K, dtype=np.int64)
        self._c(lib().kmeans_seed_pp(self.h, u.ctypes.data_as(ct.c_void_p), _ptr(C),
                                     idx.ctypes.data_as(ct.c_void_p)))
        return C, idx

    def debug_scores(self, C):
        """kmeans_debug_scores: per row (b1, b2, tau, i1) of the dense engine on C,
        before the near-tie refine; returns (rows as an n x 4 float32 tensor with the
        index reinterpreted, kind, unit)."""
        t = self.torch
        C = self._f64(C)
        out = t.empty((self.n, 4), dtype=t.float32, device=self.device)
        kind, unit = ct.c_int32(), ct.c_double()
        self._c(lib().kmeans_debug_scores(self.h, _ptr(C), _ptr(out), ct.byref(kind), ct.byref(unit)))
        return out, kind.value, unit.value

    def bounds_export(self):
        """(ub, lb, p2, C_ref) of the bounded engine between passes (kmeans_bounds_export)."""
        t = self.torch
        ub = t.empty(self.n, dtype=t.float32, device=self.device)
        lb = t.empty_like(ub)
        p2 = t.empty(self.n, dtype=t.int32, device=self.device)
        Cr = t.empty((self.K, self.d), dtype=t.float64, device=self.device)
        self._c(lib().kmeans_bounds_export(self.h, _ptr(ub), _ptr(lb), _ptr(p2), _ptr(Cr)))
        return ub, lb, p2, Cr

    def bounds_repeat(self):
        """kmeans_bounds_repeat (destructive): (ub, lb after call 1, rows scored by the two
        calls, labels identical)."""
        t = self.torch
        ub = t.empty(self.n, dtype=t.float32, device=self.device)
        lb = t.empty_like(ub)
        sc = (ct.c_int64 * 2)()
        same = ct.c_int32()
        self._c(lib().kmeans_bounds_repeat(self.h, _ptr(ub), _ptr(lb), sc, ct.byref(same)))
        return ub, lb, (sc[0], sc[1]), bool(same.value)

    def last_flagged(self) -> int:
        v = ct.c_int64()
        self._c(lib().kmeans_last_flagged(self.h, ct.byref(v)))
        return v.value

    def close(self):
        if getattr(self, "h", None):
            lib().kmeans_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
