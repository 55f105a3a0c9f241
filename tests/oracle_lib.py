"""ctypes bindings for oracle/libpit_oracle.so and oracle/_ref/libpitref.so.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline leg of bench.py — never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "libpit_oracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libpitref.so")

_dp = C.POINTER(C.c_double)
PROP_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_int, _dp, C.c_int, _dp)

MODE_REFERENCE = 0
MODE_DEVICE = 1


class OrcRecord(C.Structure):
    _fields_ = [("k", C.c_int), ("residual", C.c_double), ("fine_applications", C.c_long),
                ("coarse_applications", C.c_long)]


class OrcHistory(C.Structure):
    _fields_ = [("records", C.POINTER(OrcRecord)), ("max_records", C.c_int), ("count", C.c_int),
                ("converged", C.c_int), ("restarts", C.c_int), ("fine_applications", C.c_long),
                ("coarse_applications", C.c_long), ("min_restart_margin", C.c_double)]


class OrcStepper(C.Structure):
    _fields_ = [("M", C.c_int), ("m", C.c_int), ("nsub", C.c_int), ("nseg", C.c_int), ("warps", C.c_int),
                ("Mp", C.c_int),
                ("steps", C.c_int), ("delta", C.c_double), ("lam", C.c_double), ("mu", C.c_double),
                ("dstar", C.c_double), ("nl", C.c_double), ("nu", C.c_double), ("inv", C.c_double),
                ("gneg", C.c_double), ("K0", C.c_int), ("pS", C.c_double), ("qS", C.c_double),
                ("Pseg", C.c_double), ("Qseg", C.c_double), ("nlpow", C.c_double * 32),
                ("pw", C.c_double * 8), ("narrow", C.c_int), ("pp", C.c_double * 5), ("qq", C.c_double * 5),
                ("p32", C.c_double), ("q32", C.c_double), ("plane", C.c_double * 32),
                ("qlane", C.c_double * 32), ("R", C.c_int), ("invR", C.c_double),
                ("invLast", C.c_double), ("zc", _dp), ("ppos", _dp), ("qpos", _dp),
                ("zt", _dp), ("scan_f", C.c_int), ("scan_b", C.c_int)]


class Orc2Coeffs(C.Structure):
    _fields_ = [("m", C.c_int), ("fine_steps", C.c_int), ("coarse_steps", C.c_int),
                ("ac", C.c_double), ("an", C.c_double), ("scaled", C.c_int), ("R", C.c_int),
                ("kappa", C.c_double), ("anR", C.c_double), ("anLast", C.c_double),
                ("D", C.c_double), ("O", C.c_double),
                ("minv", C.c_double), ("rel_tol", C.c_double), ("cap", C.c_longlong),
                ("rows", C.c_int), ("cluster", C.c_int), ("threads", C.c_int)]


def ensure_built() -> None:
    if not os.path.exists(ORACLE_SO) or (os.path.isdir("/root/reference/proj") and not os.path.exists(REF_SO)):
        subprocess.run(["make", "-s", "-C", ORACLE_DIR, "-j8"], check=True)


_orc = None
_ref = None


def ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def orc():
    global _orc
    if _orc is None:
        ensure_built()
        lib = C.CDLL(ORACLE_SO)
        lib.orc_stepper_init.argtypes = [C.POINTER(OrcStepper), C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                         C.c_double]
        lib.orc_stepper_free.argtypes = [C.POINTER(OrcStepper)]
        lib.orc_stepper_propagate.argtypes = [C.POINTER(OrcStepper), _dp, _dp, _dp, _dp]
        lib.orc_thomas_propagate.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                             C.c_double, _dp, _dp, _dp, _dp]
        lib.orc_1d_create.restype = C.c_void_p
        lib.orc_1d_create.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                      C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                      C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp,
                                      C.c_int, _dp, C.c_double, C.c_double, C.c_double, C.c_int,
                                      C.c_int]
        lib.orc_1d_destroy.argtypes = [C.c_void_p]
        lib.orc_1d_set_source_tables.argtypes = [C.c_void_p, _dp, _dp]
        lib.orc_1d_problem.restype = C.c_void_p
        lib.orc_1d_problem.argtypes = [C.c_void_p]
        lib.orc_1d_stepper.restype = C.POINTER(OrcStepper)
        lib.orc_1d_stepper.argtypes = [C.c_void_p, C.c_int]
        lib.orc_1d_ds.restype = _dp
        lib.orc_1d_ds.argtypes = [C.c_void_p, C.c_int, C.c_int]
        lib.orc_problem_new.restype = C.c_void_p
        lib.orc_problem_new.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, _dp,
                                        C.c_void_p, C.c_void_p]
        lib.orc_problem_delete.argtypes = [C.c_void_p]
        for name in ("orc_apply_F", "orc_apply_G_inverse"):
            getattr(lib, name).argtypes = [C.c_void_p, _dp, _dp, C.POINTER(OrcHistory)]
        lib.orc_assemble_rhs.argtypes = [C.c_void_p, _dp, C.POINTER(OrcHistory)]
        lib.orc_initial_guess.argtypes = [C.c_void_p, C.c_int, _dp, C.POINTER(OrcHistory)]
        lib.orc_sequential_fine.argtypes = [C.c_void_p, _dp]
        lib.orc_preconditioned_residual.argtypes = [C.c_void_p, _dp, _dp, _dp, C.POINTER(OrcHistory)]
        for name in ("orc_pitsbicg", "orc_parareal"):
            getattr(lib, name).argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_int, C.c_int,
                                           _dp, _dp, _dp, C.POINTER(OrcHistory)]
        lib.orc_block_dot.restype = C.c_double
        lib.orc_block_dot.argtypes = [C.c_void_p, _dp, _dp]
        lib.orc_block_norm.restype = C.c_double
        lib.orc_block_norm.argtypes = [C.c_void_p, _dp]
        lib.orc_vec_update_s.argtypes = [C.c_long, C.c_double, _dp, _dp, _dp]
        lib.orc_vec_update_lr.argtypes = [C.c_long, C.c_double, C.c_double, _dp, _dp, _dp, _dp, _dp]
        lib.orc_vec_update_p.argtypes = [C.c_long, C.c_double, C.c_double, _dp, _dp, _dp]
        lib.orc_vec_axpy.argtypes = [C.c_long, C.c_double, _dp, _dp]
        lib.orc_block_partial.restype = C.c_double
        lib.orc_block_partial.argtypes = [C.c_void_p, _dp, _dp]
        lib.orc2_coefficients.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_int,
                                          C.c_int, C.c_int, C.c_double, C.c_longlong,
                                          C.POINTER(Orc2Coeffs)]
        lib.orc2_explicit_propagate.argtypes = [C.POINTER(Orc2Coeffs), _dp, _dp]
        lib.orc2_cg_solve.argtypes = [C.POINTER(Orc2Coeffs), _dp, _dp, C.POINTER(C.c_longlong)]
        lib.orc2_coarse_propagate.argtypes = [C.POINTER(Orc2Coeffs), _dp, _dp,
                                              C.POINTER(C.c_longlong)]
        lib.orc_2d_create.restype = C.c_void_p
        lib.orc_2d_create.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int, C.c_double,
                                      C.c_int, C.c_int, C.c_double, C.c_longlong, _dp, C.c_int]
        lib.orc_2d_destroy.argtypes = [C.c_void_p]
        lib.orc_2d_problem.restype = C.c_void_p
        lib.orc_2d_problem.argtypes = [C.c_void_p]
        lib.orc_2d_coeffs.restype = C.POINTER(Orc2Coeffs)
        lib.orc_2d_coeffs.argtypes = [C.c_void_p]
        lib.orc_2d_coarse_iterations.restype = C.c_longlong
        lib.orc_2d_coarse_iterations.argtypes = [C.c_void_p]
        lib.orc_problem_propagate.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, C.c_int, _dp]
        lib.orc_be2_stencil.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                        C.c_int, _dp]
        lib.orc_be2d_create.restype = C.c_void_p
        lib.orc_be2d_create.argtypes = [C.c_int, C.c_double, C.c_double, _dp, C.c_int, C.c_int,
                                        C.c_double, C.c_int, C.c_int, C.c_double, C.c_longlong,
                                        C.c_double, C.c_longlong, _dp, C.c_int]
        lib.orc_be2d_create_1d.restype = C.c_void_p
        lib.orc_be2d_create_1d.argtypes = [C.c_int, C.c_double, C.c_double, _dp, C.c_int, C.c_int,
                                        C.c_double, C.c_int, C.c_int, C.c_double, C.c_longlong,
                                        C.c_double, C.c_longlong, _dp, C.c_int]
        lib.orc_be2d_destroy.argtypes = [C.c_void_p]
        lib.orc_be2d_set_source_tables.argtypes = [C.c_void_p, _dp, _dp]
        lib.orc_be2d_problem.restype = C.c_void_p
        lib.orc_be2d_problem.argtypes = [C.c_void_p]
        lib.orc_be2d_coarse_iterations.restype = C.c_longlong
        lib.orc_be2d_coarse_iterations.argtypes = [C.c_void_p]
        _orc = lib
    return _orc


def ref_available() -> bool:
    ensure_built()
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        ensure_built()
        lib = C.CDLL(REF_SO)
        lib.pitref_last_error.restype = C.c_char_p
        lib.pitref_create_1d.restype = C.c_void_p
        lib.pitref_create_1d.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                         C.c_int, C.c_double, C.c_double, C.c_double, C.c_int,
                                         C.c_int, C.c_double, C.c_int, C.c_int, _dp, C.c_int, _dp,
                                         C.c_double, C.c_double, C.c_double]
        lib.pitref_create_2d.restype = C.c_void_p
        lib.pitref_create_2d.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                         C.c_int, C.c_double, C.c_int, C.c_int, _dp]
        lib.pitref_create_preset.restype = C.c_void_p
        lib.pitref_create_preset.argtypes = [C.c_int, C.c_int, C.c_int]
        lib.pitref_initial_value.argtypes = [C.c_void_p, _dp]
        lib.pitref_run_experiment.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int), C.c_int,
                                              C.c_int, C.c_double, C.c_char_p]
        lib.pitref_destroy.argtypes = [C.c_void_p]
        lib.pitref_spacing.restype = C.c_double
        lib.pitref_spacing.argtypes = [C.c_void_p]
        lib.pitref_apply_F.argtypes = [C.c_void_p, _dp, _dp, C.c_int]
        lib.pitref_apply_G_inverse.argtypes = [C.c_void_p, _dp, _dp]
        lib.pitref_assemble_rhs.argtypes = [C.c_void_p, _dp, C.c_int]
        lib.pitref_initial_guess.argtypes = [C.c_void_p, _dp]
        lib.pitref_sequential_fine.argtypes = [C.c_void_p, _dp]
        lib.pitref_create_1d_csr.restype = C.c_void_p
        lib.pitref_create_1d_csr.argtypes = [C.c_int, C.c_double, C.c_double, _dp, _dp, _dp, C.c_int,
                                             C.c_int, C.c_double, C.c_int, C.c_int, _dp, C.c_int]
        lib.pitref_propagate.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, C.c_int, _dp]
        lib.pitref_sample_source.argtypes = [C.c_void_p, C.c_double, _dp]
        for name in ("pitref_pitsbicg", "pitref_parareal"):
            getattr(lib, name).argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_int, C.c_int,
                                           C.c_int, _dp, _dp, _dp, C.POINTER(C.c_int), _dp,
                                           C.POINTER(C.c_long), C.POINTER(C.c_long), C.c_int,
                                           C.POINTER(C.c_int), C.POINTER(C.c_int),
                                           C.POINTER(C.c_int)]
        lib.pitref_seeded_normal.argtypes = [C.c_ulonglong, C.c_long, C.c_double, C.c_double, _dp]
        lib.pitref_seeded_uniform.argtypes = [C.c_ulonglong, C.c_long, C.c_double, C.c_double, _dp]
        _ref = lib
    return _ref
