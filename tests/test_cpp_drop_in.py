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
