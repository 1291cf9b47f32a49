"""BASELINE.json workload configs and their seeded inputs.

Mapping to the reference model:
  hopping t = 1       -> GridSpec(nx, ny, lx=nx, ly=ny): hx = hy = 1, K diag 4, off-diag -1
  (g/2) sum |psi|^4   -> reference gamma = -g  (H has -(gamma/2) sum |u|^4, lattice.hpp:80)
  defects             -> V = V_d on Bernoulli(frac) sites (counter-based hash of the site index)
  packets             -> normalised (sum |psi|^2 = 1) Gaussian packets, periodic minimum image
  stage tolerance     -> epsilon = 1e-14 for every config (configs 3-5 do not state one)
Unstated choices, fixed here: cfg2 centre (64,128); cfg3 centre (256,512);
cfg4 packet centres uniform on the lattice, momenta uniform in [-pi/2, pi/2]^2;
cfg5 packet centres uniform, momenta uniform in [-pi/4, pi/4]^2, phases uniform.
The inputs are synthetic, seeded; both the oracle and the GPU consume the same arrays.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, replace
from typing import Optional, Tuple

import numpy as np

from . import _lib
from ._lib import dptr


@dataclass(frozen=True)
class LatticeConfig:
    name: str
    nx: int
    ny: int
    dt: float
    steps: int
    g: float                    # BASELINE nonlinearity g; reference gamma = -g
    defect_frac: float
    defect_seed: int
    vd_min: float
    vd_max: float               # > vd_min: uniform V_d in [vd_min, vd_max)
    npackets: int
    sigma: float
    x0: float = 0.0
    y0: float = 0.0
    kx: float = 0.0
    ky: float = 0.0
    random_packets: bool = False
    packet_seed: int = 0
    k_max: float = 0.0
    epsilon: float = 1e-14
    max_iters: int = 50
    max_step_halvings: int = 4

    @property
    def gamma(self) -> float:
        return -self.g

    @property
    def sites(self) -> int:
        return self.nx * self.ny

    def with_lattice(self, nx: int, ny: int) -> "LatticeConfig":
        """Same physics on another lattice (multi-GPU tiling / reduced samples)."""
        return replace(self, nx=nx, ny=ny)


PI = math.pi

CONFIGS = {
    "cfg1": LatticeConfig("cfg1", 64, 64, 0.01, 1000, 1.0, 0.01, 42, 10.0, 10.0, 1, 4.0,
                          x0=16, y0=32, kx=PI / 4, ky=0.0),
    "cfg2": LatticeConfig("cfg2", 256, 256, 0.005, 2000, 2.0, 0.05, 7, 20.0, 20.0, 1, 8.0,
                          x0=64, y0=128, kx=PI / 2, ky=PI / 4),
    "cfg3": LatticeConfig("cfg3", 1024, 1024, 0.005, 500, 1.0, 0.02, 11, 10.0, 10.0, 1, 32.0,
                          x0=256, y0=512, kx=PI / 4, ky=PI / 4),
    "cfg4": LatticeConfig("cfg4", 4096, 4096, 0.002, 200, 1.0, 0.01, 13, 5.0, 50.0, 4, 64.0,
                          random_packets=True, packet_seed=13, k_max=PI / 2),
    "cfg5": LatticeConfig("cfg5", 8192, 8192, 0.002, 100, 1.5, 0.01, 17, 10.0, 10.0, 16, 128.0,
                          random_packets=True, packet_seed=17, k_max=PI / 4),
}


def cfg5_lattice(n_gpus: int) -> Tuple[int, int]:
    """Weak-scaling tiling of cfg5: 8192^2 per GPU (BASELINE configs[4])."""
    return {1: (8192, 8192), 2: (16384, 8192), 4: (16384, 16384), 8: (16384, 32768)}[n_gpus]


def input_spec(cfg: LatticeConfig, threads: int = 0) -> _lib.Inputs:
    s = _lib.Inputs()
    s.gnx, s.gny = cfg.nx, cfg.ny
    s.defect_frac = cfg.defect_frac
    s.defect_seed = cfg.defect_seed
    s.vd_min, s.vd_max = cfg.vd_min, cfg.vd_max
    s.npackets = cfg.npackets
    s.sigma = cfg.sigma
    s.x0, s.y0, s.kx, s.ky = cfg.x0, cfg.y0, cfg.kx, cfg.ky
    s.random_packets = int(cfg.random_packets)
    s.packet_seed = cfg.packet_seed
    s.k_max = cfg.k_max
    s.threads = threads
    return s


def _generator(gen):
    """(make_inputs, scale_state) C entry points: the product library's by default;
    `gen` injects the same generator from another library (bench.py's reference arm
    uses oracle/libinputs.so so that it never maps libmb4cu.so)."""
    if gen is not None:
        return gen
    L = _lib.lib()
    return L.mb4cu_make_inputs, L.mb4cu_scale_state


def make_block(cfg: LatticeConfig, x0: int = 0, y0: int = 0, lnx: Optional[int] = None,
               lny: Optional[int] = None, threads: int = 0, gen=None):
    """(V, psi_unnormalised, sum|psi|^2) of a sub-block of the global lattice."""
    lnx = cfg.nx if lnx is None else lnx
    lny = cfg.ny if lny is None else lny
    V = np.empty(lnx * lny)
    psi = np.empty(lnx * lny, dtype=np.complex128)
    psum = C.c_double(0.0)
    make, _ = _generator(gen)
    spec = input_spec(cfg, threads)
    rc = make(C.byref(spec), x0, y0, lnx, lny, dptr(V), dptr(psi), C.byref(psum))
    if rc != 0:
        raise ValueError(f"make_inputs: invalid lattice / block / packet spec ({rc})")
    return V, psi, psum.value


def make_inputs(cfg: LatticeConfig, threads: int = 0, gen=None):
    """(V, psi) of the whole lattice, psi normalised to sum |psi|^2 = 1."""
    V, psi, psum = make_block(cfg, threads=threads, gen=gen)
    _, scale = _generator(gen)
    scale(dptr(psi), psi.size, 1.0 / math.sqrt(psum), threads)
    return V, psi


def model_for(cfg: LatticeConfig, V: np.ndarray):
    from .nls2d import GridModel, GridSpec

    return GridModel(GridSpec(cfg.nx, cfg.ny, float(cfg.nx), float(cfg.ny)), cfg.gamma, V)


def newton_for(cfg: LatticeConfig):
    from .nls2d import NewtonConfig

    return NewtonConfig(cfg.epsilon, cfg.max_iters, cfg.max_step_halvings)
