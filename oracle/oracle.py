"""ctypes binding of the CPU oracle (oracle.c) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this module.  It marshals workloads.* descriptions into the oracle's
own structs (oracle.h); it shares nothing with the product binding.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
CFLAGS = ["-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-pthread"]


def build(force: bool = False) -> str:
    # PARADL_ORACLE_LIB: a prebuilt oracle (e.g. the ASan/UBSan build of tools/oracle_sanitize.sh)
    if os.environ.get("PARADL_ORACLE_LIB"):
        return os.environ["PARADL_ORACLE_LIB"]
    src = os.path.join(HERE, "oracle.c")
    hdr = os.path.join(HERE, "oracle.h")
    if (not force and os.path.exists(LIB_PATH)
            and os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(src), os.path.getmtime(hdr))):
        return LIB_PATH
    tmp = LIB_PATH + ".tmp"
    subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, src, "-lm"])
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


MAX_TIERS = 4
MAX_STAGES = 64


class Layer(C.Structure):
    _fields_ = [("kind", C.c_int32), ("ndim", C.c_int32),
                ("C", C.c_int64), ("F", C.c_int64),
                ("X", C.c_int64 * 3), ("Y", C.c_int64 * 3), ("K", C.c_int64 * 3),
                ("x", C.c_int64), ("y", C.c_int64), ("w", C.c_int64), ("bi", C.c_int64),
                ("fw", C.c_int64), ("bw", C.c_int64), ("wu", C.c_int64),
                ("flags", C.c_uint32), ("pad_", C.c_uint32)]


class Model(C.Structure):
    _fields_ = [("G", C.c_int32), ("pad_", C.c_int32), ("rows", C.POINTER(Layer)), ("D", C.c_int64)]


class Tier(C.Structure):
    _fields_ = [("max_pes", C.c_int64), ("alpha", C.c_double), ("beta", C.c_double)]


class System(C.Structure):
    _fields_ = [("n_tiers", C.c_int32), ("delta", C.c_int32), ("tiers", Tier * MAX_TIERS),
                ("flops_per_s", C.c_double), ("hbm_bytes", C.c_double), ("gamma", C.c_double),
                ("phi_df", C.c_double), ("tree_threshold", C.c_double),
                ("tree_chunks", C.c_int32), ("filter_rs", C.c_int32),
                ("p2p_alpha_scale", C.c_double), ("p2p_beta_scale", C.c_double),
                ("phi_pd", C.c_double), ("phi_ds", C.c_double)]


class Sub(C.Structure):
    _fields_ = [("family", C.c_int32), ("model", C.c_int32),
                ("part_mode", C.c_int32), ("s_min", C.c_int32), ("s_max", C.c_int32),
                ("n_cap", C.c_int32), ("n_flops", C.c_int32), ("n_b", C.c_int32), ("n_S", C.c_int32),
                ("n_dims", C.c_int32), ("n_Ls", C.c_int32), ("n_alpha", C.c_int32), ("n_beta", C.c_int32),
                ("pad_", C.c_int32),
                ("cap", C.POINTER(C.c_double)), ("flops", C.POINTER(C.c_double)),
                ("b", C.POINTER(C.c_int64)),
                ("S", C.POINTER(C.c_int32)), ("dims", C.POINTER(C.c_int32)), ("Ls", C.POINTER(C.c_int32)),
                ("alpha", C.POINTER(C.c_double)), ("beta", C.POINTER(C.c_double))]


class Spec(C.Structure):
    _fields_ = [("n_sub", C.c_int32), ("pad_", C.c_int32), ("subs", C.POINTER(Sub))]


class Config(C.Structure):
    _fields_ = [("sub", C.c_int32), ("family", C.c_int32), ("model", C.c_int32), ("pad_", C.c_int32),
                ("i_cap", C.c_int64), ("i_flops", C.c_int64), ("i_b", C.c_int64), ("i_S", C.c_int64),
                ("i_dims", C.c_int64), ("i_Ls", C.c_int64), ("i_alpha", C.c_int64), ("i_beta", C.c_int64),
                ("i_part", C.c_uint64),
                ("cap", C.c_double), ("flops", C.c_double), ("b", C.c_int64),
                ("S", C.c_int32), ("Ls", C.c_int32), ("dims", C.c_int32 * 4),
                ("alpha", C.c_double * MAX_TIERS), ("beta", C.c_double * MAX_TIERS),
                ("n_stages", C.c_int32), ("pad2_", C.c_int32), ("stage_end", C.c_int32 * MAX_STAGES)]


class Pred(C.Structure):
    _fields_ = [("t_comp", C.c_double), ("t_ge", C.c_double), ("t_fb_ag", C.c_double),
                ("t_fb_ar", C.c_double), ("t_halo", C.c_double), ("t_p2p", C.c_double),
                ("t_iter", C.c_double), ("t_epoch", C.c_double), ("mem", C.c_double), ("I", C.c_double),
                ("B", C.c_int64), ("p", C.c_int64), ("reason", C.c_uint32), ("feasible", C.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class Hit(C.Structure):
    _fields_ = [("idx", C.c_uint64), ("key", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        L.or_last_error.restype = C.c_char_p
        P = C.POINTER
        L.or_sweep_size.argtypes = [P(Model), C.c_int, P(System), P(Spec), P(C.c_uint64)]
        L.or_decode.argtypes = [P(Model), C.c_int, P(System), P(Spec), C.c_uint64, P(Config)]
        L.or_eval.argtypes = [P(Model), P(System), P(Config), P(Pred)]
        L.or_eval_fold.argtypes = [P(Model), P(System), P(Config), P(Pred)]
        L.or_halo_elements.argtypes = [P(Layer), P(C.c_int32), C.c_int]
        L.or_halo_elements.restype = C.c_int64
        L.or_eval_many.argtypes = [P(Model), C.c_int, P(System), P(Spec), P(C.c_uint64), C.c_int64,
                                   P(C.c_double), P(C.c_double), P(C.c_uint32), P(C.c_double), C.c_int]
        L.or_sweep_dense.argtypes = [P(Model), C.c_int, P(System), P(Spec), C.c_uint64, C.c_uint64,
                                     P(C.c_double), P(C.c_double), P(C.c_uint32), P(C.c_uint8), C.c_int]
        L.or_topk.argtypes = [P(Model), C.c_int, P(System), P(Spec), C.c_uint64, C.c_uint64, C.c_int32,
                              P(Hit), P(C.c_uint64), C.c_int]
    return _lib


class OracleError(RuntimeError):
    def __init__(self, rc):
        super().__init__(f"oracle error {rc}: {lib().or_last_error().decode()}")
        self.rc = rc


def _check(rc):
    if rc != 0:
        raise OracleError(rc)


def make_layer(r) -> Layer:
    L = Layer()
    L.kind, L.ndim, L.C, L.F = r.kind, r.ndim, r.C, r.F
    for a in range(3):
        L.X[a], L.Y[a], L.K[a] = r.X[a], r.Y[a], r.K[a]
    L.x, L.y, L.w, L.bi, L.fw, L.bw, L.wu, L.flags = r.x, r.y, r.w, r.bi, r.fw, r.bw, r.wu, r.flags
    return L


def _arr(ctype, vals):
    vals = list(vals)
    a = (ctype * max(1, len(vals)))(*vals)
    return a


class OracleSweep:
    """Holds the C-side image of a workloads.sweeps.Sweep (keeps buffers alive)."""

    def __init__(self, sweep):
        self.sweep = sweep
        self._keep = []
        ms = sweep.models
        self.models = (Model * len(ms))()
        for i, m in enumerate(ms):
            rows = (Layer * m.G)(*[make_layer(r) for r in m.layers])
            self._keep.append(rows)
            self.models[i].G = m.G
            self.models[i].rows = rows
            self.models[i].D = m.D
        s = sweep.system
        self.system = System()
        self.system.n_tiers = len(s.tiers)
        self.system.delta = s.delta
        for t, tr in enumerate(s.tiers):
            self.system.tiers[t] = Tier(tr.max_pes, tr.alpha, tr.beta)
        self.system.flops_per_s = s.flops_per_s
        self.system.hbm_bytes = s.hbm_bytes
        self.system.gamma = s.gamma
        self.system.phi_df = s.phi_df
        self.system.tree_threshold = s.tree_threshold
        self.system.tree_chunks = s.tree_chunks
        self.system.filter_rs = s.filter_rs
        self.system.p2p_alpha_scale = s.p2p_alpha_scale
        self.system.p2p_beta_scale = s.p2p_beta_scale
        self.system.phi_pd = s.phi_pd
        self.system.phi_ds = s.phi_ds
        subs = (Sub * max(1, len(sweep.subs)))()
        for i, sb in enumerate(sweep.subs):
            x = subs[i]
            x.family, x.model = sb.family, sb.model
            x.part_mode, x.s_min, x.s_max = sb.part_mode, sb.s_min, sb.s_max
            cap = _arr(C.c_double, sb.cap)
            flops = _arr(C.c_double, sb.flops)
            b = _arr(C.c_int64, sb.b)
            S = _arr(C.c_int32, sb.S)
            dims = _arr(C.c_int32, [v for d in sb.dims for v in d])
            Ls = _arr(C.c_int32, sb.Ls)
            alpha = _arr(C.c_double, [v for row in sb.alpha for v in row])
            beta = _arr(C.c_double, [v for row in sb.beta for v in row])
            self._keep += [cap, flops, b, S, dims, Ls, alpha, beta]
            x.n_cap, x.cap = len(sb.cap), cap
            x.n_flops, x.flops = len(sb.flops), flops
            x.n_b, x.b = len(sb.b), b
            x.n_S, x.S = len(sb.S), S
            x.n_dims, x.dims = len(sb.dims), dims
            x.n_Ls, x.Ls = len(sb.Ls), Ls
            x.n_alpha, x.alpha = len(sb.alpha), alpha
            x.n_beta, x.beta = len(sb.beta), beta
        self._keep.append(subs)
        self.spec = Spec()
        self.spec.n_sub = len(sweep.subs)
        self.spec.subs = subs

    # -- thin wrappers ----------------------------------------------------------------
    def size(self) -> int:
        n = C.c_uint64()
        _check(lib().or_sweep_size(self.models, len(self.sweep.models), C.byref(self.system),
                                   C.byref(self.spec), C.byref(n)))
        return n.value

    def decode(self, idx: int) -> Config:
        c = Config()
        _check(lib().or_decode(self.models, len(self.sweep.models), C.byref(self.system),
                               C.byref(self.spec), idx, C.byref(c)))
        return c

    def eval_config(self, cfg: Config, fold: bool = False) -> Pred:
        p = Pred()
        fn = lib().or_eval_fold if fold else lib().or_eval
        _check(fn(self.models, C.byref(self.system), C.byref(cfg), C.byref(p)))
        return p

    def explain(self, idx: int, fold: bool = False) -> Pred:
        return self.eval_config(self.decode(idx), fold)

    def eval_many(self, idx, nthreads: int = 0):
        idx = np.ascontiguousarray(np.asarray(idx, dtype=np.uint64))
        n = len(idx)
        t = np.empty(n, np.float64)
        m = np.empty(n, np.float64)
        r = np.empty(n, np.uint32)
        k = np.empty(n, np.float64)
        P = C.POINTER
        _check(lib().or_eval_many(self.models, len(self.sweep.models), C.byref(self.system),
                                  C.byref(self.spec), idx.ctypes.data_as(P(C.c_uint64)), n,
                                  t.ctypes.data_as(P(C.c_double)), m.ctypes.data_as(P(C.c_double)),
                                  r.ctypes.data_as(P(C.c_uint32)), k.ctypes.data_as(P(C.c_double)),
                                  nthreads))
        return t, m, r, k

    def dense(self, first: int, count: int, nthreads: int = 0):
        t = np.empty(count, np.float64)
        m = np.empty(count, np.float64)
        bits = np.zeros((count + 31) // 32, np.uint32)
        reason = np.empty(count, np.uint8)
        P = C.POINTER
        _check(lib().or_sweep_dense(self.models, len(self.sweep.models), C.byref(self.system),
                                    C.byref(self.spec), first, count,
                                    t.ctypes.data_as(P(C.c_double)), m.ctypes.data_as(P(C.c_double)),
                                    bits.ctypes.data_as(P(C.c_uint32)), reason.ctypes.data_as(P(C.c_uint8)),
                                    nthreads))
        return t, m, bits, reason

    def topk(self, first: int, count: int, k: int, nthreads: int = 0):
        hits = (Hit * k)()
        nf = C.c_uint64()
        _check(lib().or_topk(self.models, len(self.sweep.models), C.byref(self.system),
                             C.byref(self.spec), first, count, k, hits, C.byref(nf), nthreads))
        return [(h.idx, h.key) for h in hits], nf.value

    def halo_elements(self, model: int, row: int, split, which: int) -> int:
        r = make_layer(self.sweep.models[model].layers[row])
        sp = (C.c_int32 * 3)(*split)
        return lib().or_halo_elements(C.byref(r), sp, which)


def halo_elements(layer, split, which) -> int:
    r = make_layer(layer)
    sp = (C.c_int32 * 3)(*split)
    return lib().or_halo_elements(C.byref(r), sp, which)
