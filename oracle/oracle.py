"""ctypes wrapper around ``oracle/aakm_oracle.c`` (TEST INFRASTRUCTURE ONLY).

Every function here is argument marshalling; the arithmetic lives in the C
file, which follows PAPER.md step by step (citations there).  The shared
library is built with plain gcc (``-O2 -fopenmp -ffp-contract=off``) into
``oracle/liboracle.so`` by :func:`build` (also called from
``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as ct
import dataclasses
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "aakm_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

M_HIST_MAX = 64  # size of ora_state.theta


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (never nvcc: it shares nothing with the GPU path)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".{os.getpid()}.tmp"
        subprocess.check_call([
            "gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
            "-fPIC", "-shared", "-o", tmp, _SRC, "-lm",
        ])
        os.replace(tmp, _SO)
    return _SO


class _State(ct.Structure):
    _fields_ = [
        ("X", ct.c_void_p), ("N", ct.c_int64), ("d", ct.c_int32), ("K", ct.c_int32),
        ("m_max", ct.c_int32), ("eps1", ct.c_double), ("eps2", ct.c_double),
        ("dynamic_m", ct.c_int32), ("max_iters", ct.c_int64), ("ridge", ct.c_double),
        ("C", ct.c_void_p), ("fallback", ct.c_void_p), ("Ghist", ct.c_void_p),
        ("Fhist", ct.c_void_p), ("hist_count", ct.c_int32),
        ("labels_prev", ct.c_void_p), ("labels", ct.c_void_p),
        ("E1", ct.c_double), ("E2", ct.c_double), ("m", ct.c_int32), ("lloyd", ct.c_int32),
        ("t", ct.c_int64),
        ("n_accepted", ct.c_int64), ("n_rejected", ct.c_int64), ("n_assign", ct.c_int64),
        ("E_cand", ct.c_double), ("E_final", ct.c_double), ("changed", ct.c_int64),
        ("m_t", ct.c_int32), ("rejected_now", ct.c_int32), ("accepted_now", ct.c_int32),
        ("theta", ct.c_double * M_HIST_MAX),
    ]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = ct.CDLL(build())
            P, I64, I32, D = ct.c_void_p, ct.c_int64, ct.c_int32, ct.c_double
            L.ora_sqdist.argtypes = [P, P, I32]; L.ora_sqdist.restype = D
            L.ora_assign.argtypes = [P, I64, I32, P, I32, P]; L.ora_assign.restype = None
            L.ora_best2.argtypes = [P, I64, I32, P, I32, P, P]; L.ora_best2.restype = None
            L.ora_energy.argtypes = [P, I64, I32, P, P]; L.ora_energy.restype = D
            L.ora_update.argtypes = [P, I64, I32, P, I32, P, P, P]; L.ora_update.restype = None
            L.ora_ls_solve.argtypes = [P, P, I64, I32, D, P]; L.ora_ls_solve.restype = I32
            L.ora_adjust_m.argtypes = [I32, I32, D, D, D, D, D]; L.ora_adjust_m.restype = I32
            L.ora_init.argtypes = [ct.POINTER(_State), P, I32]; L.ora_init.restype = None
            L.ora_pass.argtypes = [ct.POINTER(_State)]; L.ora_pass.restype = I32
            L.ora_state_size.restype = I32
            L.ora_seed_pp.argtypes = [P, I64, I32, I32, P, P, P]; L.ora_seed_pp.restype = I32
            assert L.ora_state_size() == ct.sizeof(_State), "ora_state layout mismatch"
            _lib = L
    return _lib


def _f32(X):
    X = np.ascontiguousarray(X, dtype=np.float32)
    if X.ndim == 1:
        X = X[:, None]
    return X


def _f64(C, d=None):
    C = np.ascontiguousarray(C, dtype=np.float64)
    if C.ndim == 1:
        C = C[:, None] if d in (None, 1) else C.reshape(-1, d)
    return C


def _p(a):
    return a.ctypes.data_as(ct.c_void_p)


def sqdist(x, c):
    x = np.ascontiguousarray(x, dtype=np.float32).ravel()
    c = np.ascontiguousarray(c, dtype=np.float64).ravel()
    return lib().ora_sqdist(_p(x), _p(c), x.size)


def assign(X, C):
    """Eq. (3): nearest centroid, lowest index on exact fp64 ties."""
    X = _f32(X); C = _f64(C, X.shape[1])
    out = np.empty(X.shape[0], dtype=np.int32)
    lib().ora_assign(_p(X), X.shape[0], X.shape[1], _p(C), C.shape[0], _p(out))
    return out


def best2(X, C):
    X = _f32(X); C = _f64(C, X.shape[1])
    b1 = np.empty(X.shape[0]); b2 = np.empty(X.shape[0])
    lib().ora_best2(_p(X), X.shape[0], X.shape[1], _p(C), C.shape[0], _p(b1), _p(b2))
    return b1, b2


def energy(X, C, labels):
    """Eq. (1) with a given assignment P (Algorithm 1's E(P, .))."""
    X = _f32(X); C = _f64(C, X.shape[1])
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    return lib().ora_energy(_p(X), X.shape[0], X.shape[1], _p(C), _p(labels))


def update(X, labels, C_prev):
    """Eq. (4): cluster means; empty clusters keep C_prev's row.  Returns (G, counts)."""
    X = _f32(X); C_prev = _f64(C_prev, X.shape[1])
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    K, d = C_prev.shape
    G = np.empty((K, d)); counts = np.empty(K, dtype=np.int64)
    lib().ora_update(_p(X), X.shape[0], d, _p(labels), K, _p(C_prev), _p(G), _p(counts))
    return G, counts


def ls_solve(dF, F, ridge=1e-10):
    """Eq. (7) under reading R-A14.  dF: (m_t, n), row j-1 = dF_j (newest first)."""
    dF = np.ascontiguousarray(dF, dtype=np.float64)
    if dF.ndim == 1:
        dF = dF[None, :]
    F = np.ascontiguousarray(F, dtype=np.float64).ravel()
    m_t, n = dF.shape
    theta = np.zeros(max(m_t, 1))
    used = lib().ora_ls_solve(_p(dF), _p(F), n, m_t, ridge, _p(theta))
    return theta[:m_t], used


def adjust_m(m, m_max, E_t, E1, E2, eps1=0.02, eps2=0.5):
    return lib().ora_adjust_m(m, m_max, E_t, E1, E2, eps1, eps2)


@dataclasses.dataclass
class OracleConfig:
    """Algorithm 1 settings.  Defaults: PAPER.md:177 (eps1, eps2, m_max) and
    reading R-A18 (m0 = 5 on the BASELINE configs; the paper's default is 2)."""
    m0: int = 5
    m_max: int = 30
    eps1: float = 0.02
    eps2: float = 0.5
    dynamic_m: bool = True
    max_iters: int = 10000
    ridge: float = 1e-10


class AAState:
    """Algorithm 1 state (C, fallback, G/F history, P^{t-1}, E's, m, t)."""

    def __init__(self, X, cfg: OracleConfig):
        self.X = _f32(X)
        self.cfg = cfg
        self.N, self.d = self.X.shape
        self.K = None

    def _alloc(self, K):
        self.K = K
        KD = K * self.d
        H = self.cfg.m_max + 1
        self.C = np.zeros((K, self.d)); self.fallback = np.zeros((K, self.d))
        self.Ghist = np.zeros((H, K, self.d)); self.Fhist = np.zeros((H, K, self.d))
        self.labels_prev = np.zeros(self.N, dtype=np.int32)
        self.labels = np.zeros(self.N, dtype=np.int32)
        s = _State()
        s.X = self.X.ctypes.data; s.N = self.N; s.d = self.d; s.K = K
        c = self.cfg
        s.m_max = c.m_max; s.eps1 = c.eps1; s.eps2 = c.eps2; s.dynamic_m = int(c.dynamic_m)
        s.max_iters = c.max_iters; s.ridge = c.ridge
        s.C = self.C.ctypes.data; s.fallback = self.fallback.ctypes.data
        s.Ghist = self.Ghist.ctypes.data; s.Fhist = self.Fhist.ctypes.data
        s.labels_prev = self.labels_prev.ctypes.data; s.labels = self.labels.ctypes.data
        self.s = s
        del KD

    def init(self, C0):
        """Algorithm 1 line 1."""
        C0 = _f64(C0, self.d)
        self._alloc(C0.shape[0])
        lib().ora_init(ct.byref(self.s), _p(C0), self.cfg.m0)

    def load(self, *, C, fallback, Ghist, Fhist, labels_prev, E1, E2, m, lloyd, t,
             n_accepted=0, n_rejected=0, n_assign=0):
        """Set the state from an external snapshot (lockstep parity tests).
        Ghist/Fhist: (count, K, d) newest first."""
        C = _f64(C, self.d)
        self._alloc(C.shape[0])
        self.C[...] = C; self.fallback[...] = _f64(fallback, self.d)
        cnt = len(Ghist)
        self.Ghist[:cnt] = Ghist; self.Fhist[:cnt] = Fhist
        self.labels_prev[...] = labels_prev
        s = self.s
        s.hist_count = cnt; s.E1 = E1; s.E2 = E2; s.m = m; s.lloyd = int(lloyd); s.t = t
        s.n_accepted = n_accepted; s.n_rejected = n_rejected; s.n_assign = n_assign

    def step(self):
        """One loop pass of Algorithm 1; 0 continue, 1 converged, 2 max_iters."""
        return lib().ora_pass(ct.byref(self.s))

    def info(self):
        s = self.s
        return dict(t=s.t, m=s.m, m_t=s.m_t, E_cand=s.E_cand, E=s.E_final, changed=s.changed,
                    accepted=s.accepted_now, rejected=s.rejected_now, lloyd=s.lloyd,
                    theta=list(s.theta[: s.m_t]))


def run(X, C0, cfg: OracleConfig | None = None, trace=False):
    """Algorithm 1 to convergence (R3) or max_iters.  Report fields per R-A19."""
    cfg = cfg or OracleConfig()
    st = AAState(X, cfg)
    st.init(C0)
    tr = []
    while True:
        t = st.s.t
        rc = st.step()
        if trace:
            tr.append(dict(st.info(), t=t))
        if rc != 0:
            break
    s = st.s
    converged = rc == 1
    t_final = t if converged else s.t - 1
    iters = t_final + 1
    return dict(C=st.C.copy(), labels=st.labels.copy(), energy=s.E_final,
                mse=s.E_final / st.N, iters=iters, accepted=s.n_accepted,
                rejected=s.n_rejected, n_assign=s.n_assign, m_final=s.m,
                converged=converged, trace=tr)


def lloyd(X, C0, max_iters=10000, trace=False):
    """Plain Lloyd = Algorithm 1 with fixed m = 0 (every iterate is a Lloyd iterate)."""
    return run(X, C0, OracleConfig(m0=0, dynamic_m=False, max_iters=max_iters), trace=trace)


class SeedError(ValueError):
    """ora_seed_pp status 1 (bad u or k) or 2 (fewer than k distinct samples)."""


def seed_pp(X, k, u, return_d2=False):
    """K-Means++ seeding with the caller's uniforms u[0..k-1] (oracle/aakm_oracle.c
    ora_seed_pp: fixed-point D^2 weights, reading R-A27). Returns the k sample
    indices (int64), and the final fixed-point D2 if asked."""
    X = _f32(X)
    N, d = X.shape
    u = np.ascontiguousarray(u, dtype=np.float64)
    if u.shape != (k,):
        raise SeedError("u must hold k uniforms")
    idx = np.zeros(k, dtype=np.int64)
    d2 = np.zeros(N, dtype=np.int64) if return_d2 else None
    st = lib().ora_seed_pp(_p(X), N, d, int(k), _p(u), _p(idx), _p(d2) if d2 is not None else None)
    if st != 0:
        raise SeedError({1: "u outside [0,1) or k outside [1, N]", 2: "fewer than k distinct samples"}[st])
    return (idx, d2) if return_d2 else idx


def seed_scale(X):
    """t of R-A27: 2^t scales every squared coordinate difference below 2^50."""
    a = float(np.abs(np.asarray(X, dtype=np.float64)).max()) if np.size(X) else 0.0
    if a == 0.0:
        return 50
    return 50 - int(np.frexp(4.0 * a * a)[1])

