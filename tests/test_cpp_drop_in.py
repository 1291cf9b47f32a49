"""The C++ mirror of the reference API (include/nls2d) compiles and, on the GPU,
reproduces the reference golden state through StepDriver::advance."""
import os
import subprocess

import numpy as np
import pytest

from paper_2003_04345_b200 import configs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_drop_in.cpp")
SRC_HARNESS = os.path.join(ROOT, "tests", "cpp", "test_harness.cpp")
LIBDIR = os.path.join(ROOT, "paper_2003_04345_b200")


def build(out, src=SRC):
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), src, "-o", out,
           "-L", LIBDIR, "-lmb4cu", f"-Wl,-rpath,{LIBDIR}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_cpp_mirror_compiles(tmp_path):
    exe = str(tmp_path / "test_drop_in")
    build(exe)
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_cpp_drop_in_matches_reference_golden(tmp_path):
    exe = str(tmp_path / "test_drop_in")
    build(exe)
    cfg = configs.CONFIGS["cfg1"]
    V, psi = configs.make_inputs(cfg)
    V.tofile(tmp_path / "V.bin")
    psi.tofile(tmp_path / "psi.bin")
    out = tmp_path / "u10.bin"
    r = subprocess.run([exe, str(tmp_path / "V.bin"), str(tmp_path / "psi.bin"), str(cfg.nx), str(cfg.ny),
                        repr(cfg.gamma), repr(cfg.dt), str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    u = np.fromfile(out, dtype=np.complex128)
    g = np.load(os.path.join(ROOT, "tests", "golden", "ref_cfg1_10.npz"))
    ref = g["state_10"]
    assert np.linalg.norm(u - ref) / np.linalg.norm(ref) <= 1e-10


def test_cpp_harness_mirror_compiles(tmp_path):
    exe = str(tmp_path / "test_harness")
    build(exe, SRC_HARNESS)
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_cpp_harness_drop_in_runs(tmp_path):
    # reference-style harness code (RunConfig, parse_config_file, run, compare_methods,
    # convergence_study, parallel_bench) compiled against include/nls2d
    exe = str(tmp_path / "test_harness")
    build(exe, SRC_HARNESS)
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


SRC_SCHEME = os.path.join(ROOT, "tests", "cpp", "test_scheme_api.cpp")


def _exact_table(path):
    import json

    d = json.load(open(os.path.join(ROOT, "tests", "golden", "scheme_exact.json")))
    lines = [f"alpha1 {d['alpha1']!r}", f"A_half_half {d['A_half_half']!r}", f"l3_half {d['l3_half']!r}"]
    for i in range(3):
        for j in range(4):
            lines.append(f"E_{i + 1}_{j} {d['E'][i * 4 + j]!r}")
        lines.append(f"lambda{i + 1} {d['eigenvalues'][i]!r}")
    lines.append(f"W_3_3_3_3 {d['W'][191]!r}")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")


def test_cpp_scheme_surface_matches_reference_cases(tmp_path):
    """eval_A / lagrange_basis / a_coeff / t() / t_inv() / dump / integrate_e and
    split_state / join_state of include/nls2d, checked with the cases of the
    reference's test_mb4_scheme.cpp against its exact-rational tables (host only)."""
    exe = str(tmp_path / "test_scheme_api")
    build(exe, SRC_SCHEME)
    _exact_table(tmp_path / "exact.txt")
    r = subprocess.run([exe, "scheme", str(tmp_path / "exact.txt")], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_newton_solve_matches_oracle(tmp_path):
    """newton_solve (mb4_integrator.hpp:85-95) through include/nls2d on the paper's
    70x70 lx = 2 pi baseline: the three stages against the C oracle's newton_solve,
    U3 against the reference library's step, and the reference's iteration count."""
    from oracle import oracle as O
    from paper_2003_04345_b200 import nls2d

    exe = str(tmp_path / "test_scheme_api")
    build(exe, SRC_SCHEME)
    n, gamma, h = 70, -0.1, 0.01
    g = nls2d.GridSpec(n, n, 2 * np.pi, 2 * np.pi)
    u0 = nls2d.initial_condition(g)
    u0.tofile(tmp_path / "u0.bin")
    r = subprocess.run([exe, "newton", str(tmp_path / "u0.bin"), str(n), repr(gamma), repr(h),
                        str(tmp_path / "stage")], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    iters = int(r.stdout.split()[1])
    stages = [np.fromfile(tmp_path / f"stage{i}.bin", dtype=np.complex128) for i in (1, 2, 3)]
    cx = 1.0 / g.hx() ** 2
    orc = O.Oracle(n, n, gamma, np.zeros(n * n), cx=cx, cy=cx)
    rc, ost, oit, _ = orc.newton_solve(u0, h, eps=1e-13)
    assert rc == 0
    for a, b in zip(stages, ost):
        assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-10
    ref, _, riters, _ = O.ref_run(n, n, 2 * np.pi, 2 * np.pi, gamma, np.zeros(n * n), u0, h, 1, eps=1e-13,
                                  solver="direct", record=False)
    assert np.linalg.norm(stages[2] - ref) / np.linalg.norm(ref) <= 1e-10
    assert iters == int(riters[0])
