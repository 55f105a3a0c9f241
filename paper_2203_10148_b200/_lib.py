"""ctypes binding of libpit_b200.so (include/pit_b200.h).

The shared library is built in-tree by __graft_entry__.build() (or
`make -C paper_2203_10148_b200/csrc`).  There is no fallback: if the library
is missing, loading raises ImportError; without a CUDA device every compute
entry point returns PIT_ERR_CUDA, which the API layer raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PIT_LIB") or os.path.join(HERE, "libpit_b200.so")

PIT_OK = 0
PIT_ERR_INVALID_ARGUMENT = 1
PIT_ERR_INNER_SOLVE = 2
PIT_ERR_SLAB = 3
PIT_ERR_CONFIG = 4
PIT_ERR_CUDA = 5

PIT_FINE = 0
PIT_COARSE = 1
PIT_SOURCE_NONE = 0
PIT_SOURCE_SEPARABLE = 1
PIT_SOURCE_TABLE = 2
PIT_GUESS_COARSE_SWEEP = 0
PIT_GUESS_ZERO = 1
PIT_CONVERGED = 0
PIT_MAX_ITERATIONS = 1
PIT_SCHEME_BACKWARD_EULER = 0
PIT_SCHEME_EXPLICIT_EULER = 1

_dp = C.POINTER(C.c_double)


class ProblemDesc(C.Structure):
    _fields_ = [("dimension", C.c_int32), ("interior", C.c_int32), ("grid_lo", C.c_double),
                ("grid_hi", C.c_double), ("band_lo", C.c_double), ("band_diag", C.c_double),
                ("band_up", C.c_double), ("slab_count", C.c_int32), ("total_time", C.c_double),
                ("fine_steps", C.c_int32), ("coarse_steps", C.c_int32),
                ("source_kind", C.c_int32), ("source_amp", C.c_double),
                ("source_omega", C.c_double), ("source_phase", C.c_double),
                ("source_shape", _dp), ("initial_value", _dp), ("device", C.c_int32),
                ("fine_mpt", C.c_int32), ("fine_nsub", C.c_int32), ("fine_nseg", C.c_int32),
                ("fine_warps", C.c_int32), ("coarse_mpt", C.c_int32), ("coarse_nsub", C.c_int32),
                ("coarse_nseg", C.c_int32), ("coarse_warps", C.c_int32),
                ("fine_scheme", C.c_int32), ("coarse_tolerance", C.c_double),
                ("coarse_max_iterations", C.c_int64), ("tile_rows", C.c_int32),
                ("tile_cols", C.c_int32), ("tile_cluster", C.c_int32), ("tile_warps", C.c_int32),
                ("stencil", _dp), ("nonsymmetric", C.c_int32), ("fine_tolerance", C.c_double),
                ("fine_max_iterations", C.c_int64), ("source_table_fine", _dp),
                ("source_table_coarse", _dp)]


class StepCoeffs2DC(C.Structure):
    _fields_ = [("m", C.c_int32), ("fine_steps", C.c_int32), ("coarse_steps", C.c_int32),
                ("ac", C.c_double), ("an", C.c_double), ("scaled", C.c_int32), ("R", C.c_int32),
                ("kappa", C.c_double), ("anR", C.c_double), ("anLast", C.c_double),
                ("D", C.c_double), ("O", C.c_double),
                ("minv", C.c_double), ("rel_tol", C.c_double), ("cap", C.c_int64),
                ("rows", C.c_int32), ("cluster", C.c_int32), ("threads", C.c_int32),
                ("tile_rows", C.c_int32), ("tile_cols", C.c_int32), ("tile_cluster", C.c_int32),
                ("tile_warps", C.c_int32)]


class RunStatsC(C.Structure):
    _fields_ = [("fine_applications", C.c_int64), ("coarse_applications", C.c_int64),
                ("fine_parallel_ms", C.c_double), ("fine_busy_ms", C.c_double),
                ("coarse_sequential_ms", C.c_double)]


class RecordC(C.Structure):
    _fields_ = [("k", C.c_int32), ("residual_norm", C.c_double),
                ("fine_applications", C.c_int64), ("coarse_applications", C.c_int64),
                ("wall_ms", C.c_double), ("error_vs_reference", C.c_double),
                ("has_error", C.c_int32)]


class SolverConfigC(C.Structure):
    _fields_ = [("tolerance", C.c_double), ("restart_tolerance", C.c_double),
                ("max_iterations", C.c_int32), ("initial_guess", C.c_int32)]


class SolveInfoC(C.Structure):
    _fields_ = [("status", C.c_int32), ("restarts", C.c_int32), ("record_count", C.c_int32),
                ("total_records", C.c_int32), ("min_restart_margin", C.c_double),
                ("stats", RunStatsC)]


class StepCoeffsC(C.Structure):
    _fields_ = [("M", C.c_int32), ("mpt", C.c_int32), ("nsub", C.c_int32), ("nseg", C.c_int32),
                ("warps", C.c_int32),
                ("steps", C.c_int32),
                ("delta", C.c_double), ("lam", C.c_double), ("mu", C.c_double),
                ("dstar", C.c_double), ("nl", C.c_double), ("nu", C.c_double),
                ("inv", C.c_double), ("gneg", C.c_double), ("K0", C.c_int32), ("R", C.c_int32),
                ("invR", C.c_double), ("invLast", C.c_double), ("pS", C.c_double),
                ("qS", C.c_double), ("Pseg", C.c_double), ("Qseg", C.c_double),
                ("nlpow", C.c_double * 32), ("pw", C.c_double * 8), ("narrow", C.c_int32),
                ("pp", C.c_double * 5), ("qq", C.c_double * 5),
                ("p32", C.c_double), ("q32", C.c_double), ("plane", C.c_double * 32),
                ("qlane", C.c_double * 32), ("scan_f", C.c_int32), ("scan_b", C.c_int32)]


EXPORTS = [
    "pit_last_error", "pit_last_error_slab", "pit_version", "pit_device_count",
    "pit_context_create", "pit_context_destroy", "pit_context_shape", "pit_step_coefficients",
    "pit_step_correction", "pit_step_positions", "pit_apply_F", "pit_assemble_rhs", "pit_apply_G_inverse",
    "pit_initial_guess", "pit_preconditioned_residual", "pit_sequential_fine_solve",
    "pit_propagate", "pit_block_inner_product", "pit_block_norm_n_inf", "pit_pitsbicg_solve",
    "pit_parareal_solve", "pit_apply_F_device", "pit_residual_device", "pit_coarse_sweep_device",
    "pit_block_partials_device", "pit_block_partials2_device", "pit_update_s_device",
    "pit_update_lr_device", "pit_update_p_device", "pit_axpy_device", "pit_add_device",
    "pit_fine_source_device",
    "pit_sync_status", "pit_pitsbicg_solve_device",
    "pit_seeded_uniform", "pit_seeded_normal", "pit_measure_fp64_peak",
    "pit_step_coefficients_2d", "pit_coarse_iterations", "pit_set_reference",
    "pit_last_error_detail", "pit_set_iterate_observer", "pit_context_slots", "pit_host_alloc",
    "pit_host_free", "pit_comm_nccl_unique_id", "pit_comm_create_nccl", "pit_comm_create_host",
    "pit_comm_destroy", "pit_context_attach_comm", "pit_context_shard",
    "pit_sharded_apply_F_device", "pit_sharded_pitsbicg_solve_device",
    "pit_sharded_parareal_solve_device", "pit_sharded_sync_status",
]

# pit_comm_ops callbacks (host transport)
COMM_SEND = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.c_size_t, C.c_int, C.c_void_p)
COMM_RECV = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.c_size_t, C.c_int, C.c_void_p)
COMM_ALLGATHER = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.c_size_t, C.POINTER(C.c_double),
                             C.c_void_p)


class CommOpsC(C.Structure):
    _fields_ = [("send", COMM_SEND), ("recv", COMM_RECV), ("allgather", COMM_ALLGATHER),
                ("user", C.c_void_p)]

# void (*)(const pit_record*, const double* lambda, int N, int M, void* user)
ITERATE_OBSERVER = C.CFUNCTYPE(None, C.POINTER(RecordC), C.POINTER(C.c_double), C.c_int, C.c_int,
                               C.c_void_p)

_lib = None


def lib():
    """Load libpit_b200.so (raises ImportError when it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(make -C paper_2203_10148_b200/csrc)")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    L.pit_last_error.restype = C.c_char_p
    L.pit_version.restype = C.c_char_p
    L.pit_context_create.argtypes = [C.POINTER(ProblemDesc), C.POINTER(vp)]
    L.pit_context_destroy.argtypes = [vp]
    L.pit_set_reference.argtypes = [vp, _dp]
    L.pit_context_shape.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), _dp]
    L.pit_step_coefficients.argtypes = [C.POINTER(ProblemDesc), C.c_int, C.POINTER(StepCoeffsC)]
    L.pit_step_correction.argtypes = [C.POINTER(ProblemDesc), C.c_int, _dp]
    L.pit_step_positions.argtypes = [C.POINTER(ProblemDesc), C.c_int, _dp, _dp, _dp]
    st = C.POINTER(RunStatsC)
    L.pit_apply_F.argtypes = [vp, _dp, _dp, st]
    L.pit_assemble_rhs.argtypes = [vp, _dp, st]
    L.pit_apply_G_inverse.argtypes = [vp, _dp, _dp, st]
    L.pit_initial_guess.argtypes = [vp, C.c_int, _dp, st]
    L.pit_preconditioned_residual.argtypes = [vp, _dp, _dp, _dp, st]
    L.pit_sequential_fine_solve.argtypes = [vp, _dp]
    L.pit_propagate.argtypes = [vp, C.c_int, C.c_int, _dp, C.c_int, _dp]
    L.pit_block_inner_product.argtypes = [vp, _dp, _dp, _dp]
    L.pit_block_norm_n_inf.argtypes = [vp, _dp, _dp]
    for name in ("pit_pitsbicg_solve", "pit_parareal_solve"):
        getattr(L, name).argtypes = [vp, C.POINTER(SolverConfigC), _dp, _dp, _dp,
                                     C.POINTER(RecordC), C.c_int, C.POINTER(SolveInfoC)]
    L.pit_apply_F_device.argtypes = [vp, vp, vp, vp, C.c_int, C.c_int, vp]
    L.pit_residual_device.argtypes = [vp, vp, vp, vp, vp, C.c_int, C.c_int, vp]
    L.pit_coarse_sweep_device.argtypes = [vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, vp]
    L.pit_block_partials_device.argtypes = [vp, vp, vp, vp, C.c_int, vp]
    L.pit_block_partials2_device.argtypes = [vp, vp, vp, vp, vp, vp, C.c_int, vp]
    L.pit_update_s_device.argtypes = [vp, C.c_double, vp, vp, vp, vp, C.c_int, vp]
    L.pit_update_lr_device.argtypes = [vp, C.c_double, C.c_double, vp, vp, vp, vp, vp, vp, vp,
                                       C.c_int, vp]
    L.pit_update_p_device.argtypes = [vp, C.c_double, C.c_double, vp, vp, vp, C.c_int, vp]
    L.pit_axpy_device.argtypes = [vp, C.c_double, vp, vp, C.c_int, vp]
    L.pit_add_device.argtypes = [vp, vp, vp, C.c_int, vp]
    L.pit_fine_source_device.argtypes = [vp, vp, C.c_int, C.c_int, vp]
    L.pit_sync_status.argtypes = [vp, vp]
    L.pit_pitsbicg_solve_device.argtypes = [vp, C.POINTER(SolverConfigC), vp, vp,
                                            C.POINTER(RecordC), C.c_int, C.POINTER(SolveInfoC), vp]
    L.pit_measure_fp64_peak.argtypes = [C.c_int, _dp]
    L.pit_last_error_detail.argtypes = [_dp, C.POINTER(C.c_int64)]
    L.pit_set_iterate_observer.argtypes = [vp, ITERATE_OBSERVER, vp]
    L.pit_context_slots.argtypes = [vp, C.POINTER(C.c_int)]
    L.pit_host_alloc.argtypes = [C.c_size_t, C.POINTER(vp)]
    L.pit_host_free.argtypes = [vp]
    L.pit_comm_nccl_unique_id.argtypes = [C.c_char_p]
    L.pit_comm_create_nccl.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]
    L.pit_comm_create_host.argtypes = [C.POINTER(CommOpsC), C.c_int, C.c_int, C.POINTER(vp)]
    L.pit_comm_destroy.argtypes = [vp]
    L.pit_context_attach_comm.argtypes = [vp, vp]
    L.pit_context_shard.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.pit_sharded_apply_F_device.argtypes = [vp, vp, vp, vp]
    L.pit_sharded_sync_status.argtypes = [vp, vp]
    for name in ("pit_sharded_pitsbicg_solve_device", "pit_sharded_parareal_solve_device"):
        getattr(L, name).argtypes = [vp, C.POINTER(SolverConfigC), vp, vp, C.POINTER(RecordC),
                                     C.c_int, C.POINTER(SolveInfoC), vp]
    L.pit_step_coefficients_2d.argtypes = [C.POINTER(ProblemDesc), C.POINTER(StepCoeffs2DC)]
    L.pit_coarse_iterations.argtypes = [vp, C.POINTER(C.c_int64)]
    L.pit_seeded_uniform.argtypes = [C.c_uint64, C.c_int64, C.c_double, C.c_double, _dp]
    L.pit_seeded_uniform.restype = None
    L.pit_seeded_normal.argtypes = [C.c_uint64, C.c_int64, C.c_double, C.c_double, _dp]
    L.pit_seeded_normal.restype = None
    _lib = L
    return L


def dptr(a):
    return None if a is None else a.ctypes.data_as(_dp)
