"""ctypes mirror of include/hygro_b200.h (struct layouts and prototypes).

Shared by the product binding (paper_1703_10119_b200.api) and the test-only
oracle bindings (oracle/), so one description of a model drives the CUDA
library, the C restatement and the unmodified reference.
"""
from __future__ import annotations

import ctypes as C

HYG_OK, HYG_EINVAL, HYG_ESCHEMA, HYG_EDIVERGED, HYG_EDOMAIN, HYG_ECONVERGE, HYG_ESCALING, HYG_ECUDA, HYG_ENOTSUP = range(9)
HYG_SIG_CONSTANT, HYG_SIG_SIN, HYG_SIG_SIN2 = 0, 1, 2
HYG_FACE_EXTERIOR, HYG_FACE_ZONE = 0, 1
HYG_MOISTURE_AS_PRINTED, HYG_MOISTURE_FLUX_CONSISTENT = 0, 1
HYG_COEFF_CONSTANT, HYG_COEFF_ANALYTIC_D, HYG_COEFF_MATERIAL = 0, 1, 2
HYG_F64, HYG_F32 = 0, 1
HYG_BOOT_IMPLICIT, HYG_BOOT_EXPLICIT = 0, 1
HYG_SCHEME_DF, HYG_SCHEME_EULER_IMPLICIT, HYG_SCHEME_EULER_EXPLICIT = 0, 1, 2
HYG_TUNE_RING_GRID, HYG_TUNE_RING_KERNEL, HYG_TUNE_MATERIAL_EXACT, HYG_TUNE_TILED_LOAD, HYG_TUNE_RING_DEPTH = 1, 2, 3, 4, 5

dp = C.POINTER(C.c_double)


class WallGroups(C.Structure):
    _fields_ = [("Fo_M", C.c_double), ("Fo_TT", C.c_double), ("Fo_TM", C.c_double), ("gamma", C.c_double)]


class FaceBiot(C.Structure):
    _fields_ = [("Bi_M", C.c_double), ("Bi_TT", C.c_double), ("Bi_TM", C.c_double)]


class Ambient(C.Structure):
    _fields_ = [("u_inf", C.c_double), ("v_inf", C.c_double), ("g_inf", C.c_double), ("q_inf", C.c_double)]


class Window(C.Structure):
    _fields_ = [("from_", C.c_double), ("to", C.c_double), ("value", C.c_double)]


class Signal(C.Structure):
    _fields_ = [("form", C.c_int32), ("n_windows", C.c_int32), ("base", C.c_double),
                ("amplitude", C.c_double), ("period", C.c_double), ("phase", C.c_double),
                ("windows", C.POINTER(Window))]


class Channel(C.Structure):
    _fields_ = [("u_inf", Signal), ("v_inf", Signal), ("g_inf", Signal), ("q_inf", Signal)]


class ZoneSources(C.Structure):
    _fields_ = [("g_o", Signal), ("q_o", Signal), ("q_h", Signal)]


class FaceAttach(C.Structure):
    _fields_ = [("kind", C.c_int32), ("index", C.c_int32)]


class ZoneWallLink(C.Structure):
    _fields_ = [("wall", C.c_int32), ("face", C.c_int32), ("Bi_M", C.c_double), ("Bi_TT", C.c_double),
                ("Bi_TM", C.c_double), ("theta_T", C.c_double), ("theta_M", C.c_double)]


class InterzoneLink(C.Structure):
    _fields_ = [("peer", C.c_int32), ("g_inz", C.c_double), ("q_inz1", C.c_double), ("q_inz2", C.c_double)]


class RadiationLink(C.Structure):
    _fields_ = [("emitter_wall", C.c_int32), ("receiver_wall", C.c_int32), ("view_factor", C.c_double),
                ("emissivity", C.c_double)]


class CoeffSet(C.Structure):
    _fields_ = [("c_M", C.c_double), ("k_M", C.c_double), ("c_TT", C.c_double), ("k_TT", C.c_double),
                ("c_TM", C.c_double), ("k_TM", C.c_double)]


class ZoneDesc(C.Structure):
    _fields_ = [("kappa_a_tt1", C.c_double), ("g_v", C.c_double), ("q_v1", C.c_double), ("q_v2", C.c_double),
                ("sources", C.c_int32), ("moisture_sign", C.c_int32), ("n_walls", C.c_int32),
                ("walls", C.POINTER(ZoneWallLink)), ("n_interzone", C.c_int32),
                ("interzone", C.POINTER(InterzoneLink)), ("n_radiation", C.c_int32),
                ("radiation", C.POINTER(RadiationLink))]


class ModelDesc(C.Structure):
    _fields_ = [("n_walls", C.c_int32), ("n_nodes", C.c_int32), ("dx", C.c_double),
                ("precision", C.c_int32), ("coeff_kind", C.c_int32), ("coeff_params", C.c_double * 4),
                ("groups", C.POINTER(WallGroups)), ("biot", C.POINTER(FaceBiot)),
                ("attach", C.POINTER(FaceAttach)), ("n_channels", C.c_int32),
                ("channels", C.POINTER(Channel)), ("n_zones", C.c_int32), ("zones", C.POINTER(ZoneDesc)),
                ("n_zone_sources", C.c_int32), ("zone_sources", C.POINTER(ZoneSources)),
                ("outdoor_u", Signal), ("outdoor_v", Signal), ("dt", C.c_double),
                ("divergence_norm", C.c_double), ("eta_factor", C.c_double), ("max_subiters", C.c_int32),
                ("device", C.c_int32), ("T_i", C.c_double), ("P_vi", C.c_double),
                ("wall_coeff", C.POINTER(C.c_int32)), ("wall_reference", C.POINTER(CoeffSet)),
                ("wall_thickness", dp), ("wall_k_TT0", dp)]


class Status(C.Structure):
    _fields_ = [("code", C.c_int32), ("wall", C.c_int32), ("zone", C.c_int32), ("subiterations", C.c_int32),
                ("layer", C.c_int64), ("t_star", C.c_double), ("residual", C.c_double),
                ("node", C.c_int32), ("half", C.c_int32), ("message", C.c_char * 256)]


class RunReport(C.Structure):
    _fields_ = [("steps", C.c_int64), ("bootstrap_subiters", C.c_int32), ("max_subiters_seen", C.c_int32),
                ("mean_subiters", C.c_double)]


FRAME_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int64, C.c_double, C.c_void_p)
REDUCE_FN = C.CFUNCTYPE(C.c_double, C.c_void_p, C.c_double)

# name -> (restype, argtypes); every symbol the header declares
PROTOTYPES = {
    "hyg_abi_version": (C.c_int, []),
    "hyg_strerror": (C.c_char_p, [C.c_int]),
    "hyg_create": (C.c_int, [C.POINTER(ModelDesc), C.POINTER(C.c_void_p), C.POINTER(Status)]),
    "hyg_destroy": (None, [C.c_void_p]),
    "hyg_set_state": (C.c_int, [C.c_void_p, dp, dp, dp, dp, dp, dp, C.c_double, C.c_int64]),
    "hyg_get_state": (C.c_int, [C.c_void_p, dp, dp, dp, dp, dp, dp, dp, C.POINTER(C.c_int64)]),
    "hyg_get_cells": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, dp, dp, dp, dp]),
    "hyg_set_cells": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, dp, dp, dp, dp]),
    "hyg_get_zones": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, dp, dp]),
    "hyg_set_zones": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, dp, dp]),
    "hyg_pack_cells": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p]),
    "hyg_unpack_cells": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p]),
    "hyg_pack_zones": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    "hyg_unpack_zones": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    "hyg_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "hyg_set_owned": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "hyg_snapshot": (C.c_int, [C.c_void_p]),
    "hyg_restore": (C.c_int, [C.c_void_p]),
    "hyg_set_channel_table": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_int64, C.POINTER(Ambient)]),
    "hyg_set_source_table": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_int64, dp]),
    "hyg_set_outdoor_table": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, dp]),
    "hyg_bootstrap": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(Status)]),
    "hyg_advance": (C.c_int, [C.c_void_p, C.c_int64, C.c_double, C.POINTER(Status)]),
    "hyg_advance_overlapped": (C.c_int, [C.c_void_p, C.c_int64, C.c_double, C.c_int64, C.c_int64, C.c_void_p,
                                         C.POINTER(Status)]),
    "hyg_set_exchange_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "hyg_run": (C.c_int, [C.c_void_p, C.c_double, C.c_double, C.c_int32, FRAME_FN, C.c_void_p, C.POINTER(Status)]),
    "hyg_run_scheme": (C.c_int, [C.c_void_p, C.c_int32, C.c_double, C.c_double, FRAME_FN, C.c_void_p,
                                 C.POINTER(RunReport), C.POINTER(Status)]),
    "hyg_synchronize": (C.c_int, [C.c_void_p]),
    "hyg_host_register": (C.c_int, [C.c_void_p, C.c_size_t]),
    "hyg_host_unregister": (C.c_int, [C.c_void_p]),
    "hyg_event_record": (C.c_int, [C.c_void_p, C.c_int32]),
    "hyg_event_elapsed_ms": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, dp]),
    "hyg_set_profiling": (C.c_int, [C.c_void_p, C.c_int32]),
    "hyg_kernel_stats_count": (C.c_int, [C.c_void_p]),
    "hyg_kernel_stats": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_char_p), C.POINTER(C.c_int64), dp, dp]),
    "hyg_reset_kernel_stats": (C.c_int, [C.c_void_p]),
    "hyg_launch_count": (C.c_int64, [C.c_void_p]),
    "hyg_set_tuning": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64]),
    "hyg_probe_fp64_peak": (C.c_int, [C.c_int32, dp, dp]),
    "hyg_probe_fp32_peak": (C.c_int, [C.c_int32, dp]),
    "hyg_selftest_fastmath": (C.c_int, [C.c_int32, C.c_int32, dp, dp, dp]),
    "hyg_selftest_dvmath": (C.c_int, [C.c_int32, C.c_int32, dp, dp, dp]),
    "hyg_selftest_fastlog": (C.c_int, [C.c_int32, C.c_int32, dp, dp]),
    "hyg_df_march_linear": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_int64, dp, dp]),
    "hyg_selftest_crmath": (C.c_int, [C.c_int32, C.c_int32, dp, dp, dp]),
    "hyg_saturation_pressure": (C.c_int, [C.c_double, dp]),
    "hyg_material_evaluate": (C.c_int, [C.c_double, C.c_double, C.c_int32, C.POINTER(CoeffSet)]),
    "hyg_scale_wall": (C.c_int, [dp, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                 C.c_double, C.c_double, C.c_double, C.POINTER(WallGroups), C.POINTER(FaceBiot)]),
    "hyg_scale_zone": (C.c_int, [C.c_double] * 8 + [dp]),
    "hyg_attach_wall_to_zone": (C.c_int, [dp] + [C.c_double] * 8 + [dp]),
    "hyg_scale_interzone": (C.c_int, [C.c_double] * 8 + [dp]),
}


def bind(lib: C.CDLL) -> C.CDLL:
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def header_symbols(path) -> list[str]:
    """Function names declared in include/hygro_b200.h."""
    import re
    text = open(path).read()
    return sorted(set(re.findall(r"\b(hyg_[a-z0-9_]+)\s*\(", text)) - {"hyg_frame_fn", "hyg_signal"})
