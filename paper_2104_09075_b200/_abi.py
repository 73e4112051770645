"""ctypes mirror of include/paradl.h (layout checked against paradl_struct_size at load)."""
from __future__ import annotations

import ctypes as C

MAX_TIERS = 4
MAX_STAGES = 64
MAX_TOPK = 64

OK, EINVAL, ENOMEM, ECUDA, EOVERFLOW, ERANGE, ESTATE = 0, -1, -2, -3, -4, -5, -6
STATUS_NAMES = {0: "OK", -1: "EINVAL", -2: "ENOMEM", -3: "ECUDA", -4: "EOVERFLOW", -5: "ERANGE", -6: "ESTATE"}

R_SCALING, R_MEMORY, R_SPLIT, R_TIER, R_SEGMENTS = 1, 2, 4, 8, 16


class Layer(C.Structure):
    _fields_ = [("kind", C.c_int32), ("ndim", C.c_int32),
                ("C", C.c_int64), ("F", C.c_int64),
                ("X", C.c_int64 * 3), ("Y", C.c_int64 * 3), ("K", C.c_int64 * 3),
                ("x", C.c_int64), ("y", C.c_int64), ("w", C.c_int64), ("bi", C.c_int64),
                ("fw", C.c_int64), ("bw", C.c_int64), ("wu", C.c_int64),
                ("flags", C.c_uint32), ("reserved", C.c_uint32)]


class Tier(C.Structure):
    _fields_ = [("max_pes", C.c_int64), ("alpha_s", C.c_double), ("beta_s_per_B", C.c_double)]


class System(C.Structure):
    _fields_ = [("n_tiers", C.c_int32), ("delta", C.c_int32), ("tiers", Tier * MAX_TIERS),
                ("flops_per_s", C.c_double), ("hbm_bytes", C.c_double), ("gamma", C.c_double),
                ("phi_df", C.c_double), ("tree_threshold_B", C.c_double),
                ("tree_chunks", C.c_int32), ("filter_rs", C.c_int32),
                ("p2p_alpha_scale", C.c_double), ("p2p_beta_scale", C.c_double),
                ("phi_pd", C.c_double), ("phi_ds", C.c_double)]


class SubSweep(C.Structure):
    _fields_ = [("family", C.c_int32), ("model_id", C.c_int32),
                ("part_mode", C.c_int32), ("s_min", C.c_int32), ("s_max", C.c_int32),
                ("n_cap", C.c_int32), ("n_flops", C.c_int32), ("n_b", C.c_int32), ("n_S", C.c_int32),
                ("n_dims", C.c_int32), ("n_Ls", C.c_int32), ("n_alpha", C.c_int32), ("n_beta", C.c_int32),
                ("reserved", C.c_int32),
                ("cap", C.POINTER(C.c_double)), ("flops", C.POINTER(C.c_double)),
                ("b", C.POINTER(C.c_int64)), ("S", C.POINTER(C.c_int32)),
                ("dims", C.POINTER(C.c_int32)), ("Ls", C.POINTER(C.c_int32)),
                ("alpha", C.POINTER(C.c_double)), ("beta", C.POINTER(C.c_double))]


class SweepSpec(C.Structure):
    _fields_ = [("n_sub", C.c_int32), ("reserved", C.c_int32), ("sub", C.POINTER(SubSweep))]


class DenseOut(C.Structure):
    _fields_ = [("t_iter", C.c_void_p), ("mem", C.c_void_p), ("feasible_bits", C.c_void_p),
                ("reason", C.c_void_p)]


class CompactOut(C.Structure):
    _fields_ = [("idx", C.c_void_p), ("t_iter", C.c_void_p), ("mem", C.c_void_p), ("capacity", C.c_uint64),
                ("n_feasible", C.c_void_p)]


class Hit(C.Structure):
    _fields_ = [("idx", C.c_uint64), ("key_epoch_s", C.c_double)]


class Config(C.Structure):
    _fields_ = [("sub", C.c_int32), ("family", C.c_int32), ("model_id", C.c_int32), ("n_stages", C.c_int32),
                ("i_cap", C.c_int64), ("i_flops", C.c_int64), ("i_b", C.c_int64), ("i_S", C.c_int64),
                ("i_dims", C.c_int64), ("i_Ls", C.c_int64), ("i_alpha", C.c_int64), ("i_beta", C.c_int64),
                ("i_part", C.c_uint64),
                ("cap", C.c_double), ("flops", C.c_double),
                ("b", C.c_int64), ("B", C.c_int64), ("p", C.c_int64),
                ("S", C.c_int32), ("Ls", C.c_int32), ("dims", C.c_int32 * 4),
                ("alpha", C.c_double * MAX_TIERS), ("beta", C.c_double * MAX_TIERS),
                ("stage_end", C.c_int32 * MAX_STAGES)]


class Prediction(C.Structure):
    _fields_ = [("t_comp", C.c_double), ("t_ge", C.c_double), ("t_fb_ag", C.c_double),
                ("t_fb_ar", C.c_double), ("t_halo", C.c_double), ("t_p2p", C.c_double),
                ("t_iter", C.c_double), ("t_epoch", C.c_double), ("mem", C.c_double), ("I", C.c_double),
                ("reason", C.c_uint32), ("feasible", C.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


STRUCTS = [Layer, System, SubSweep, Config, Prediction, Hit]

# every exported symbol of include/paradl.h
EXPORTS = ["paradl_create", "paradl_destroy", "paradl_last_error", "paradl_version", "paradl_load_model",
           "paradl_set_system", "paradl_sweep_size", "paradl_sweep", "paradl_topk", "paradl_argmin",
           "paradl_topk_async", "paradl_merge_topk", "paradl_decode", "paradl_explain", "paradl_struct_size",
           "paradl_stat", "paradl_fp64_peak", "paradl_merge_records", "paradl_sweep_compact"]


def declare(lib):
    P = C.POINTER
    vp = C.c_void_p
    lib.paradl_create.argtypes = [C.c_int32, P(vp)]
    lib.paradl_destroy.argtypes = [vp]
    lib.paradl_destroy.restype = None
    lib.paradl_last_error.argtypes = [vp]
    lib.paradl_last_error.restype = C.c_char_p
    lib.paradl_version.restype = C.c_char_p
    lib.paradl_load_model.argtypes = [vp, P(Layer), C.c_int32, C.c_int64, P(C.c_int32)]
    lib.paradl_set_system.argtypes = [vp, P(System)]
    lib.paradl_sweep_size.argtypes = [vp, P(SweepSpec), P(C.c_uint64)]
    lib.paradl_sweep.argtypes = [vp, P(SweepSpec), C.c_uint64, C.c_uint64, P(DenseOut), vp]
    lib.paradl_sweep_compact.argtypes = [vp, P(SweepSpec), C.c_uint64, C.c_uint64, P(CompactOut), vp]
    lib.paradl_topk.argtypes = [vp, P(SweepSpec), C.c_uint64, C.c_uint64, C.c_int32, P(Hit), P(C.c_uint64), vp]
    lib.paradl_argmin.argtypes = [vp, P(SweepSpec), C.c_uint64, C.c_uint64, P(Hit), P(C.c_uint64), vp]
    lib.paradl_topk_async.argtypes = [vp, P(SweepSpec), C.c_uint64, C.c_uint64, C.c_int32, C.c_int32, C.c_int32,
                                      vp, vp, vp]
    lib.paradl_merge_topk.argtypes = [vp, vp, C.c_int32, C.c_int32, vp, vp, vp, vp]
    lib.paradl_merge_records.argtypes = [vp, vp, C.c_int32, C.c_int32, vp, vp, vp]
    lib.paradl_decode.argtypes = [vp, P(SweepSpec), C.c_uint64, P(Config)]
    lib.paradl_explain.argtypes = [vp, P(SweepSpec), C.c_uint64, P(Prediction)]
    lib.paradl_stat.argtypes = [vp, C.c_int32]
    lib.paradl_stat.restype = C.c_uint64
    lib.paradl_fp64_peak.argtypes = [vp, C.c_double, P(C.c_double)]
    lib.paradl_struct_size.argtypes = [C.c_int32]
    lib.paradl_struct_size.restype = C.c_int32
    for name in EXPORTS:
        f = getattr(lib, name)
        if f.restype is C.c_int and name != "paradl_stat":   # default
            f.restype = C.c_int32
    for i, st in enumerate(STRUCTS):
        n = lib.paradl_struct_size(i)
        if n != C.sizeof(st):
            raise RuntimeError(f"ABI mismatch: {st.__name__} is {C.sizeof(st)} bytes in Python, {n} in C")
