"""paper_2104_09075_b200 -- Python binding of libparadl (include/paradl.h).

Argument marshalling only: every step of the ParaDL sweep (decode, Table 2 cost
evaluation, feasibility, selection, dense writes) runs in the CUDA kernels of
csrc/kernels.cu.  There is no CPU fallback: importing works without a GPU (so the
C-ABI can be checked), but every evaluating call needs a CUDA device and raises
ParadlError otherwise.  If libparadl.so is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

from . import _abi as A

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PARADL_LIB") or os.path.join(HERE, "libparadl.so")   # override: experiments only

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                      "or `python paper_2104_09075_b200/build.py` (nvcc, sm_100a). There is no CPU fallback.")

_lib = C.CDLL(LIB_PATH)
A.declare(_lib)

# family / partition constants (same values as include/paradl.h)
SERIAL, DATA, SPATIAL, FILTER, CHANNEL, DF, DS, PIPELINE, LAYERPURE, PD, SPATIAL_AG, GPIPE, DATA_LW, LAYERWISE = range(14)
PART_NONE, PART_COMB, PART_MASK = 0, 1, 2


def lib():
    return _lib


def version() -> str:
    return _lib.paradl_version().decode()


class ParadlError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"paradl {A.STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _arr(ct, vals):
    vals = list(vals)
    return (ct * max(1, len(vals)))(*vals)


def make_layers(layers):
    rows = (A.Layer * len(layers))()
    for i, r in enumerate(layers):
        L = rows[i]
        L.kind, L.ndim, L.C, L.F = r.kind, r.ndim, r.C, r.F
        for a in range(3):
            L.X[a], L.Y[a], L.K[a] = r.X[a], r.Y[a], r.K[a]
        L.x, L.y, L.w, L.bi, L.fw, L.bw, L.wu, L.flags = r.x, r.y, r.w, r.bi, r.fw, r.bw, r.wu, r.flags
    return rows


def make_system(s) -> A.System:
    S = A.System()
    S.n_tiers = len(s.tiers)
    S.delta = s.delta
    for t, tr in enumerate(s.tiers):
        S.tiers[t] = A.Tier(tr.max_pes, tr.alpha, tr.beta)
    S.flops_per_s = s.flops_per_s
    S.hbm_bytes = s.hbm_bytes
    S.gamma = s.gamma
    S.phi_df = s.phi_df
    S.tree_threshold_B = s.tree_threshold
    S.tree_chunks = s.tree_chunks
    S.filter_rs = s.filter_rs
    S.p2p_alpha_scale = getattr(s, "p2p_alpha_scale", 1.0)
    S.p2p_beta_scale = getattr(s, "p2p_beta_scale", 1.0)
    S.phi_pd = getattr(s, "phi_pd", 1.0)
    S.phi_ds = getattr(s, "phi_ds", 1.0)
    return S


class Spec:
    """C image of a list of workloads.sweeps.SubSweep (keeps the arrays alive)."""

    def __init__(self, subs, model_ids):
        self._keep = []
        arr = (A.SubSweep * max(1, len(subs)))()
        for i, sb in enumerate(subs):
            x = arr[i]
            x.family, x.model_id = sb.family, model_ids[sb.model]
            x.part_mode, x.s_min, x.s_max = sb.part_mode, sb.s_min, sb.s_max
            lists = dict(cap=_arr(C.c_double, sb.cap), flops=_arr(C.c_double, sb.flops), b=_arr(C.c_int64, sb.b),
                         S=_arr(C.c_int32, sb.S), dims=_arr(C.c_int32, [v for d in sb.dims for v in d]),
                         Ls=_arr(C.c_int32, sb.Ls), alpha=_arr(C.c_double, [v for r in sb.alpha for v in r]),
                         beta=_arr(C.c_double, [v for r in sb.beta for v in r]))
            self._keep += list(lists.values())
            x.n_cap, x.cap = len(sb.cap), lists["cap"]
            x.n_flops, x.flops = len(sb.flops), lists["flops"]
            x.n_b, x.b = len(sb.b), lists["b"]
            x.n_S, x.S = len(sb.S), lists["S"]
            x.n_dims, x.dims = len(sb.dims), lists["dims"]
            x.n_Ls, x.Ls = len(sb.Ls), lists["Ls"]
            x.n_alpha, x.alpha = len(sb.alpha), lists["alpha"]
            x.n_beta, x.beta = len(sb.beta), lists["beta"]
        self._keep.append(arr)
        self.c = A.SweepSpec()
        self.c.n_sub = len(subs)
        self.c.sub = arr
        self.ref = C.byref(self.c)


class Context:
    """One libparadl context on one CUDA device (device=-1: host-only validation)."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        st = _lib.paradl_create(device, C.byref(self._h))
        if st != 0:
            raise ParadlError(st, f"paradl_create({device}) failed")
        self.device = device

    def close(self):
        if self._h:
            _lib.paradl_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st != 0:
            raise ParadlError(st, _lib.paradl_last_error(self._h).decode())

    # -- inputs ---------------------------------------------------------------
    def load_model(self, model) -> int:
        rows = make_layers(model.layers)
        mid = C.c_int32()
        self._check(_lib.paradl_load_model(self._h, rows, len(model.layers), model.D, C.byref(mid)))
        return mid.value

    def set_system(self, system):
        S = make_system(system)
        self._check(_lib.paradl_set_system(self._h, C.byref(S)))

    def prepare(self, sweep) -> Spec:
        """Loads the sweep's models + system and returns its C spec."""
        ids = [self.load_model(m) for m in sweep.models]
        self.set_system(sweep.system)
        return Spec(sweep.subs, ids)

    # -- calls ----------------------------------------------------------------
    def sweep_size(self, spec: Spec) -> int:
        n = C.c_uint64()
        self._check(_lib.paradl_sweep_size(self._h, spec.ref, C.byref(n)))
        return n.value

    def topk(self, spec: Spec, k: int, first: int = 0, count: int | None = None, stream=None):
        if count is None:
            count = self.sweep_size(spec) - first
        hits = (A.Hit * k)()
        nf = C.c_uint64()
        self._check(_lib.paradl_topk(self._h, spec.ref, first, count, k, hits, C.byref(nf), _stream(stream)))
        return [(h.idx, h.key_epoch_s) for h in hits], nf.value

    def argmin(self, spec: Spec, first: int = 0, count: int | None = None, stream=None):
        if count is None:
            count = self.sweep_size(spec) - first
        h = A.Hit()
        nf = C.c_uint64()
        self._check(_lib.paradl_argmin(self._h, spec.ref, first, count, C.byref(h), C.byref(nf), _stream(stream)))
        return (h.idx, h.key_epoch_s), nf.value

    def topk_async(self, spec: Spec, first: int, count: int, shard: int, n_shards: int, k: int,
                   d_hits_ptr: int, d_count_ptr: int, stream=None):
        self._check(_lib.paradl_topk_async(self._h, spec.ref, first, count, shard, n_shards, k,
                                           C.c_void_p(d_hits_ptr), C.c_void_p(d_count_ptr), _stream(stream)))

    def merge_topk(self, d_lists_ptr: int, n_lists: int, k: int, d_counts_ptr: int, d_out_ptr: int,
                   d_count_out_ptr: int, stream=None):
        self._check(_lib.paradl_merge_topk(self._h, C.c_void_p(d_lists_ptr), n_lists, k, C.c_void_p(d_counts_ptr),
                                           C.c_void_p(d_out_ptr), C.c_void_p(d_count_out_ptr), _stream(stream)))

    def merge_records(self, d_records_ptr: int, n_records: int, k: int, d_out_ptr: int, d_count_out_ptr: int,
                      stream=None):
        self._check(_lib.paradl_merge_records(self._h, C.c_void_p(d_records_ptr), n_records, k,
                                              C.c_void_p(d_out_ptr), C.c_void_p(d_count_out_ptr), _stream(stream)))

    def sweep_dense(self, spec: Spec, first: int, count: int, t_iter_ptr=0, mem_ptr=0, bits_ptr=0, reason_ptr=0,
                    stream=None):
        out = A.DenseOut(t_iter_ptr or None, mem_ptr or None, bits_ptr or None, reason_ptr or None)
        self._check(_lib.paradl_sweep(self._h, spec.ref, first, count, C.byref(out), _stream(stream)))

    def sweep_compact(self, spec: Spec, first: int, count: int, idx_ptr: int, capacity: int, n_ptr: int,
                      t_iter_ptr=0, mem_ptr=0, stream=None):
        """Feasible configurations of [first, first+count) in index order (device outputs)."""
        out = A.CompactOut(idx_ptr, t_iter_ptr or None, mem_ptr or None, capacity, n_ptr)
        self._check(_lib.paradl_sweep_compact(self._h, spec.ref, first, count, C.byref(out), _stream(stream)))

    def stat(self, which: int) -> int:
        """0: H2D bytes, 1: D2H bytes, 2: kernel launches of the last call."""
        return int(_lib.paradl_stat(self._h, which))

    def fp64_peak(self, ms: float = 50.0) -> float:
        """Measured FP64 pipe rate (DFMA instructions / s) on this device."""
        v = C.c_double()
        self._check(_lib.paradl_fp64_peak(self._h, ms, C.byref(v)))
        return v.value

    def decode(self, spec: Spec, idx: int) -> A.Config:
        c = A.Config()
        self._check(_lib.paradl_decode(self._h, spec.ref, idx, C.byref(c)))
        return c

    def explain(self, spec: Spec, idx: int) -> A.Prediction:
        p = A.Prediction()
        self._check(_lib.paradl_explain(self._h, spec.ref, idx, C.byref(p)))
        return p


def _stream(s):
    if s is None:
        return None
    if isinstance(s, int):
        return C.c_void_p(s)
    return C.c_void_p(s.cuda_stream)   # torch.cuda.Stream
