"""Multi-GPU MB4 stepping: 2-D block decomposition of the periodic lattice.

One process per GPU (torchrun); torch.distributed is the plumbing (NCCL on the
GPU, gloo for the CPU tests).  Each rank owns a block of the global lattice in
a ghost-padded libmb4cu sub-domain context (mb4cu_problem.ghost = max(mf, m) + 1;
u0 / V halos are mf + 1 wide for the depth-mf first sweep, the stage-set halos
m + 1).  One MB4 step:

    exchange u0 halos (x phase, then y phase: corners propagate)
    for s = 0, 1, ...:
        s > 0: exchange halos of the stage set written by sweep s-1
        local sweep s  (one launch of the production kernel in sub-domain mode)
        r = allreduce_max(local ||r||_inf);  s == 0: allreduce_sum(energy sums of u0)
        r <= eps -> commit (u0 <- U3); non-finite / max_iters -> halve (reference policy)

The convergence test, the halving policy (mb4_integrator.cpp:287-315) and the
energy monitor (lattice.cpp:106-137) are the single-domain ones; only the
reductions become collectives.  The exchange and reduction logic is covered on
the CPU by tests/test_dist_gloo.py (world sizes 2 and 4) with a numpy backend.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np

from . import _lib

WEST, EAST, SOUTH, NORTH = 0, 1, 2, 3
F_U0, F_V, F_SET0, F_SET1 = 0, 1, 2, 3
F_SETFULL0 = 4  # stage set 0 / 1 at the full ghost width (halo-overlap mode)

# Stopping rule, identical to the device kernels (mb4cu_internal.hpp: stage_converged):
# the reference test r <= eps plus a margin on the predicted next update.
STOP_MARGIN = 0.01
STAGNATION = 0.8


def widen_residual(r: float) -> float:
    """The kernels track ||r||_inf on the high 32 bits of |r| and report the largest
    double with that high word (an upper bound within 1 + 2^-20)."""
    import struct

    b = struct.unpack("<Q", struct.pack("<d", abs(r)))[0]
    if b >> 32:
        b = (b & 0xFFFFFFFF00000000) | 0xFFFFFFFF
    return struct.unpack("<d", struct.pack("<Q", b))[0]


def stage_converged(r: float, r_prev: float, s: int, eps: float) -> bool:
    if not r <= eps:
        return False
    if s == 0:
        return r <= STOP_MARGIN * eps
    return r * r <= STOP_MARGIN * eps * r_prev or r >= STAGNATION * r_prev


def choose_grid(n: int, gnx: int, gny: int) -> Tuple[int, int]:
    """px * py = n minimising the halo perimeter per rank (ties: squarest blocks, then
    even splits).  Uneven splits are allowed (blocks differ by at most one column / row)."""
    best = None
    for px in range(1, n + 1):
        if n % px:
            continue
        py = n // px
        if px > gnx or py > gny:
            continue
        lnx, lny = -(-gnx // px), -(-gny // py)  # the largest block
        cost = (lny if px > 1 else 0) + (lnx if py > 1 else 0)
        key = (cost, abs(lnx - lny), int(gnx % px != 0) + int(gny % py != 0), px)
        if best is None or key < best[0]:
            best = (key, (px, py))
    if best is None:
        raise ValueError(f"cannot split {gnx}x{gny} over {n} ranks")
    return best[1]


@dataclass
class Decomposition:
    """Tensor-product block split of the periodic gnx x gny lattice over a px x py torus:
    process column rx owns columns [rx gnx / px, (rx + 1) gnx / px), process row ry the
    rows [ry gny / py, (ry + 1) gny / py) -- so ranks in one process row share the block
    height and ranks in one process column the block width (what the halo strips need)."""
    gnx: int
    gny: int
    px: int
    py: int
    rank: int

    def __post_init__(self):
        if not (1 <= self.px <= self.gnx and 1 <= self.py <= self.gny):
            raise ValueError("process grid larger than the lattice")
        if not 0 <= self.rank < self.px * self.py:
            raise ValueError("rank out of range")

    @property
    def rx(self) -> int:
        return self.rank % self.px

    @property
    def ry(self) -> int:
        return self.rank // self.px

    @property
    def x0(self) -> int:
        return self.rx * self.gnx // self.px

    @property
    def y0(self) -> int:
        return self.ry * self.gny // self.py

    @property
    def lnx(self) -> int:
        return (self.rx + 1) * self.gnx // self.px - self.x0

    @property
    def lny(self) -> int:
        return (self.ry + 1) * self.gny // self.py - self.y0

    def rank_of(self, rx: int, ry: int) -> int:
        return (ry % self.py) * self.px + (rx % self.px)

    def neighbor(self, side: int) -> int:
        dx, dy = {WEST: (-1, 0), EAST: (1, 0), SOUTH: (0, -1), NORTH: (0, 1)}[side]
        return self.rank_of(self.rx + dx, self.ry + dy)

    def block(self, global_array: np.ndarray) -> np.ndarray:
        a = global_array.reshape(self.gny, self.gnx)
        return np.ascontiguousarray(a[self.y0:self.y0 + self.lny, self.x0:self.x0 + self.lnx]).reshape(-1)


class Comm:
    """torch.distributed transport for halos and scalar reductions."""

    def __init__(self, device: str):
        import torch
        import torch.distributed as dist

        self.torch = torch
        self.dist = dist
        self.device = device

    def allreduce_max(self, x: float) -> float:
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def allreduce_max_(self, t) -> None:
        """In-place MAX all-reduce of a device tensor (no host synchronisation)."""
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)

    def allreduce_sum_(self, t) -> None:
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)

    def allreduce_sum(self, xs) -> np.ndarray:
        t = self.torch.tensor(np.asarray(xs, dtype=np.float64), device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return t.cpu().numpy()

    def broadcast_(self, t, src: int) -> None:
        """In-place broadcast of a device tensor from rank src."""
        self.dist.broadcast(t, src=src)

    def exchange(self, pairs):
        """pairs: list of (send_tensor, dst, recv_tensor, src); all posted at once."""
        ops = []
        for send, dst, _, _ in pairs:
            ops.append(self.dist.P2POp(self.dist.isend, send, dst))
        for _, _, recv, src in pairs:
            ops.append(self.dist.P2POp(self.dist.irecv, recv, src))
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()


class HaloExchange:
    """Two-phase (x then y) halo exchange of one field on the process torus."""

    def __init__(self, dec: Decomposition, backend, comm: Comm):
        self.dec, self.b, self.comm = dec, backend, comm
        self.bufs = {}

    def _buf(self, key, n):
        t = self.bufs.get(key)
        if t is None or t.numel() != n:
            t = self.b.new_buffer(n)
            self.bufs[key] = t
        return t

    def exchange(self, field: int):
        d = self.dec
        for lo, hi, extent in ((WEST, EAST, d.px), (SOUTH, NORTH, d.py)):
            n = self.b.halo_count(field, lo)
            s_lo, s_hi = self._buf((field, lo, "s"), n), self._buf((field, hi, "s"), n)
            self.b.pack(field, lo, s_lo)
            self.b.pack(field, hi, s_hi)
            if extent == 1:
                # periodic wrap onto this rank: my low strip is my high ghost and vice versa
                self.b.unpack(field, hi, s_lo)
                self.b.unpack(field, lo, s_hi)
                continue
            r_hi, r_lo = self._buf((field, hi, "r"), n), self._buf((field, lo, "r"), n)
            # order matters for extent == 2 (both neighbours are the same rank):
            # sends [low strip -> low neighbour, high strip -> high neighbour],
            # recvs [high ghost <- high neighbour's low strip, low ghost <- low neighbour's high strip]
            self.b.sync()
            self.comm.exchange([(s_lo, d.neighbor(lo), r_hi, d.neighbor(hi)),
                                (s_hi, d.neighbor(hi), r_lo, d.neighbor(lo))])
            self.b.unpack(field, hi, r_hi)
            self.b.unpack(field, lo, r_lo)


class NonConvergence(RuntimeError):
    def __init__(self, what: str, residual: float):
        super().__init__(what)
        self.last_residual = residual


class DistributedSession:
    """MB4 stepping on one rank's block, collectives over torch.distributed."""

    def __init__(self, dec: Decomposition, backend, comm: Comm, gamma: float, cx: float, cy: float,
                 epsilon: float, max_iters: int = 50, max_step_halvings: int = 4, adaptive_m: bool = False):
        """adaptive_m: the later-sweep depth follows the single-domain policy (the library's
        adapt_neumann): m = 2 once a sub-step needs >= 4 sweeps at m = 1, back to m = 1
        after 64 sub-steps -- decided from sweep counts only, so every rank agrees."""
        self.dec, self.b, self.comm = dec, backend, comm
        self.adaptive_m = adaptive_m
        self._m_steps = 0
        self.gamma, self.cx, self.cy = gamma, cx, cy
        self.eps, self.max_iters, self.max_halvings = epsilon, max_iters, max_step_halvings
        self.halo = HaloExchange(dec, backend, comm)
        self.halo.exchange(F_V)
        self.last_sweeps = 0
        self.entry_sums: Optional[np.ndarray] = None
        # max|u0|^2 of the current sub-step's entry state (all-reduced), measured by its
        # first sweep; the next sub-step's spectral bound uses it, as on one GPU
        self._sub_amax2: Optional[float] = None

    # -- energy monitor: global sums -> Observables (lattice.cpp:113-137)
    def finish(self, sums) -> np.ndarray:
        qr, qi, prob, quart, ext = sums[:5]
        imag_scale = max(abs(qr), (4 * self.cx + 4 * self.cy) * prob)
        if abs(qi) > 1e-12 * imag_scale and imag_scale > 0.0:
            raise RuntimeError("observables: non-real kinetic quadratic form")
        uk, ui = qr, -0.5 * self.gamma * quart
        return np.array([uk, ui, ext, uk + ui + ext, prob, quart / (prob * prob) if prob > 0 else 0.0, quart])

    def observables(self) -> np.ndarray:
        if getattr(self.b, "overlap", False):
            self.b.wait_exchange()
        self.halo.exchange(F_U0)
        return self.finish(self.comm.allreduce_sum(self.b.obs_sums()))

    def _take_entry(self, sums) -> None:
        """Reduced sums of a sub-step's first sweep: the step's energy record (first
        sub-step) and, when the backend reports it, max|u0|^2 of the entry state."""
        if self.entry_sums is None:
            self.entry_sums = np.asarray(sums[:5])
        self._sub_amax2 = float(sums[5]) if len(sums) > 5 else None

    def _commit(self, sweeps: int) -> None:
        """Accept the sub-step; the next one's spectral bound follows the measured
        amplitude (the single-domain rule: mb4cu's per-step max|u0|^2 tracking)."""
        self.b.commit(sweeps)
        if self._sub_amax2 is not None and hasattr(self.b, "set_amax2"):
            self.b.set_amax2(self._sub_amax2)
            self.b.bound_dirty = True

    def _substep(self, h: float) -> Tuple[int, float]:
        self.sync_spectral_bound()
        if getattr(self.b, "overlap", False):
            return self._substep_overlap(h)
        if hasattr(self.b, "sweep_launch"):
            return self._substep_device(h)
        self.halo.exchange(F_U0)
        r = r_prev = float("nan")
        for s in range(self.max_iters):
            if s > 0:
                self.halo.exchange(F_SET0 + ((s - 1) & 1))
            r_loc, sums = self.b.sweep(h, s)
            # NaN -> +inf before the MAX all-reduce (fmax would drop a NaN rank)
            r = self.comm.allreduce_max(r_loc if math.isfinite(r_loc) else math.inf)
            if s == 0:
                red = list(self.comm.allreduce_sum(sums[:5]))
                if len(sums) > 5:
                    red.append(self.comm.allreduce_max(float(sums[5])))
                self._take_entry(red)
            if not math.isfinite(r):
                raise NonConvergence("stage iteration diverged (non-finite update)", math.inf)
            if stage_converged(r, r_prev, s, self.eps):
                self._commit(s + 1)
                return s + 1, r
            r_prev = r
        raise NonConvergence(f"stage iteration: no convergence after {self.max_iters} sweeps", r)

    def _substep_device(self, h: float) -> Tuple[int, float]:
        """Device-side reductions (one host read per sweep) and the speculative final
        sweep: the sweep predicted by the previous sub-step's count stores U3 only and
        is repeated with all stages if the reduced residual does not converge."""
        self.halo.exchange(F_U0)
        guess = getattr(self, "_guess", 0)
        want0 = True  # every sub-step's first sweep: energy sums + max|u0|^2
        finals = {}

        def launch(s):
            # sweep s with its halo exchange and device-side reductions, no host wait
            if s > 0:
                self.halo.exchange(F_SET0 + ((s - 1) & 1))
            finals[s] = s > 0 and s == guess - 1
            self.b.sweep_launch(h, s, finals[s], self.comm, slot=s & 1, want_sums=(s == 0 and want0))

        launch(0)
        launched = 0
        r = r_prev = float("nan")
        for s in range(self.max_iters):
            # look-ahead: a sweep the previous sub-step says will be needed is enqueued
            # before this one's residual is read, so the host round trip overlaps the
            # GPU work (every rank takes the same decision: the guess is global)
            if launched == s and s + 1 < self.max_iters and s + 1 <= guess - 1:
                launch(s + 1)
                launched = s + 1
            r, sums = self.b.sweep_read(slot=s & 1, want_sums=(s == 0 and want0))
            if sums is not None:
                self._take_entry(sums)
            if not math.isfinite(r):
                raise NonConvergence("stage iteration diverged (non-finite update)", math.inf)
            if stage_converged(r, r_prev, s, self.eps):
                self._commit(s + 1)
                self._guess = s + 1
                return s + 1, r
            if finals[s]:
                self.b.sweep_repeat(h, s)
            r_prev = r
            if launched == s and s + 1 < self.max_iters:
                launch(s + 1)
                launched = s + 1
        raise NonConvergence(f"stage iteration: no convergence after {self.max_iters} sweeps", r)

    def _substep_overlap(self, h: float) -> Tuple[int, float]:
        """Halo-exchange overlap: each sweep runs its boundary frame
        first, the frame's halo exchange then proceeds on a side stream while the
        interior is swept, and the next sweep waits for both.  The exchange after the
        last sweep carries U3 at the full ghost width, so the next step's u0 halos
        are already in place.  Device-side reductions, look-ahead and the speculative
        final sweep as in _substep_device."""
        if not self.b.u0_halo_ok:
            self.b.wait_exchange()
            self.halo.exchange(F_U0)
        self.b.u0_halo_ok = False
        guess = getattr(self, "_guess", 0)
        want0 = True  # every sub-step's first sweep: energy sums + max|u0|^2
        finals = {}

        def launch(s, final=None):
            finals[s] = (s > 0 and s == guess - 1) if final is None else final
            self.b.wait_exchange()  # halos of the input (u0 or the previous stage set)
            self.b.sweep_frame(h, s, finals[s])
            self.b.exchange_async(self.halo, F_SETFULL0 + (s & 1))
            self.b.sweep_interior(h, s, finals[s], self.comm, slot=s & 1, want_sums=(s == 0 and want0))

        launch(0)
        launched = 0
        r = r_prev = float("nan")
        for s in range(self.max_iters):
            if launched == s and s + 1 < self.max_iters and s + 1 <= guess - 1:
                launch(s + 1)
                launched = s + 1
            r, sums = self.b.sweep_read(slot=s & 1, want_sums=(s == 0 and want0))
            if sums is not None:
                self._take_entry(sums)
            if not math.isfinite(r):
                raise NonConvergence("stage iteration diverged (non-finite update)", math.inf)
            if stage_converged(r, r_prev, s, self.eps):
                self._commit(s + 1)
                self._guess = s + 1
                # the exchange after sweep s moved U3 ghost-wide: the new u0's halos
                # (a look-ahead sweep s + 1 writes the other stage set; wait_exchange
                # orders every later use after the pending exchanges)
                self.b.u0_halo_ok = True
                return s + 1, r
            if finals[s]:
                launch(s, final=False)  # repeat the missed final sweep with every stage
                self.b.sweep_read(slot=s & 1, want_sums=False)
            r_prev = r
            if launched == s and s + 1 < self.max_iters:
                launch(s + 1)
                launched = s + 1
        raise NonConvergence(f"stage iteration: no convergence after {self.max_iters} sweeps", r)

    def _adapt_m(self, sweeps: int) -> None:
        if not self.adaptive_m:
            return
        m = self.b.neumann_terms()
        if m == 1 and sweeps >= 4:
            self.b.set_neumann_terms(2)
        elif m == 2:
            self._m_steps += 1
            if self._m_steps < 64:
                return
            self.b.set_neumann_terms(1)
        else:
            return
        self._m_steps = 0
        self._guess = 0  # as the library: no speculative final sweep right after a switch

    def sync_spectral_bound(self) -> None:
        """After a state was set: all ranks place the first sweep's Chebyshev polynomial
        on one interval, the max of the ranks' bounds (mb4cu_spectral_bound), which
        equals the bound of the whole lattice (the bounds are rounded up to powers of
        2^(1/16)), so a decomposed run matches the single-domain one."""
        if getattr(self.b, "bound_dirty", False):
            self.b.set_spectral_bound(self.comm.allreduce_max(self.b.spectral_bound()))
            self.b.bound_dirty = False

    def step(self, h: float) -> Tuple[int, int]:
        """One MB4 step with the reference halving policy; returns (sweeps, halvings)."""
        self.sync_spectral_bound()
        self.entry_sums = None
        if getattr(self.b, "overlap", False):
            self.b.wait_exchange()
        last = 0.0
        for hv in range(self.max_halvings + 1):
            sub = 1 << hv
            if hv == 1:
                self.b.save()
            elif hv > 1:
                self.b.restore()
            try:
                total = 0
                for _ in range(sub):
                    n, _ = self._substep(h / sub)
                    total += n
                    self._adapt_m(n)
                self.last_sweeps = total
                return total, hv
            except NonConvergence as e:
                last = e.last_residual
        if self.max_halvings >= 1:
            self.b.restore()
        raise NonConvergence(f"mb4_step: no convergence after {self.max_halvings} step halvings", last)

    def run(self, h: float, nsteps: int):
        """nsteps steps; returns (obs[(nsteps+1),7], sweeps[nsteps]) with the fused energy record."""
        rows, sweeps = [], []
        for _ in range(nsteps):
            n, _ = self.step(h)
            sweeps.append(n)
            rows.append(self.finish(self.entry_sums))
        rows.append(self.observables())
        return np.array(rows), np.array(sweeps)


def nccl_library() -> Optional[str]:
    """Path of the libnccl.so.2 torch loads (its nvidia-nccl wheel); None: the loader's."""
    import os

    try:
        import nvidia.nccl  # noqa: F401

        path = os.path.join(os.path.dirname(nvidia.nccl.__file__), "lib", "libnccl.so.2")
        return path if os.path.exists(path) else None
    except Exception:
        return None


def nccl_unique_id(lib=None) -> bytes:
    """A new NCCL communicator id (rank 0), for NativeSession's broadcast."""
    L = lib or _lib.lib()
    buf = C.create_string_buffer(128)
    path = nccl_library()
    rc = L.mb4cu_nccl_unique_id(path.encode() if path else None, buf)
    if rc:
        raise RuntimeError(L.mb4cu_create_error().decode())
    return buf.raw


class NativeSession:
    """The decomposed MB4 step inside the library (mb4cu_dist_*): NCCL transport opened from
    torch's libnccl, the halo exchange of each sweep's boundary frame concurrent with the
    interior, the residual / energy all-reduces and the stopping test on the device, and one
    host read per step when the previous step's sweep count holds (DistributedSession reads
    once per sweep).  Same step / run / observables interface as DistributedSession, and the
    same trajectory as the single-domain kernel, bit for bit.

    nccl_id: the same 128 bytes on every rank (rank 0's nccl_unique_id(), broadcast by the
    caller, e.g. torch.distributed.broadcast_object_list)."""

    def __init__(self, dec: Decomposition, backend: "CudaBackend", nccl_id: bytes, gamma: float, cx: float,
                 cy: float, adaptive_m: bool = False, force_p2p: bool = False, grid_cap: int = 0):
        self.dec, self.b = dec, backend
        self.L = backend.L
        self.gamma, self.cx, self.cy = gamma, cx, cy
        nb = (C.c_int * 4)(*[dec.neighbor(k) for k in (WEST, EAST, SOUTH, NORTH)])
        path = nccl_library()
        rc = self.L.mb4cu_dist_attach(backend.ctx, path.encode() if path else None, nccl_id, dec.px * dec.py,
                                      dec.rank, nb, dec.px, dec.py, grid_cap, int(force_p2p), int(adaptive_m))
        if rc:
            raise RuntimeError(f"mb4cu_dist_attach: {self.L.mb4cu_last_error(backend.ctx).decode()}")
        self.entry_sums: Optional[np.ndarray] = None

    finish = DistributedSession.finish

    def observables(self) -> np.ndarray:
        sums = np.zeros(5)
        self.b._chk(self.L.mb4cu_dist_observables(self.b.ctx, _lib.dptr(sums)))
        return self.finish(sums)

    def step(self, h: float) -> Tuple[int, int]:
        """One MB4 step with the reference halving policy; returns (sweeps, halvings)."""
        st = _lib.Stats()
        sums = np.zeros(5)
        rc = self.L.mb4cu_dist_step(self.b.ctx, h, C.byref(st), _lib.dptr(sums))
        if rc == _lib.MB4CU_NONCONVERGED:
            raise NonConvergence(self.L.mb4cu_last_error(self.b.ctx).decode(), st.last_residual)
        self.b._chk(rc)
        self.entry_sums = sums
        return st.newton_iters, st.halvings

    def run(self, h: float, nsteps: int):
        """nsteps steps; returns (obs[(nsteps+1),7], sweeps[nsteps]) with the fused energy record."""
        rows, sweeps = [], []
        for _ in range(nsteps):
            n, _ = self.step(h)
            sweeps.append(n)
            rows.append(self.finish(self.entry_sums))
        rows.append(self.observables())
        return np.array(rows), np.array(sweeps)

    def close(self) -> None:
        if self.b.ctx:
            self.L.mb4cu_dist_detach(self.b.ctx)


class CudaBackend:
    """libmb4cu sub-domain context on this rank's GPU (ghost mode)."""

    def __init__(self, dec: Decomposition, V_block: np.ndarray, scheme, gamma: float, cx: float, cy: float,
                 epsilon: float, max_iters: int, neumann_terms: int, device: int,
                 neumann_first: int = 6, overlap: bool = False, reserve_sms: int = 0, max_step_halvings: int = 0):
        """overlap: sweep the boundary frame first and exchange its halos on a side
        stream while the interior is swept (the interior launch leaves reserve_sms
        SMs to the concurrent NCCL kernels)."""
        import torch

        self.torch = torch
        self.L = _lib.lib()
        self.dev = torch.device("cuda", device)
        p = _lib.Problem()
        p.nx, p.ny = dec.lnx, dec.lny
        p.cx, p.cy, p.gamma = cx, cy, gamma
        self._v = np.ascontiguousarray(V_block, dtype=np.float64)
        p.V = _lib.dptr(self._v)
        # (halving: DistributedSession drives it; the native stepper in the library uses this)
        p.epsilon, p.max_iters, p.max_step_halvings = epsilon, max_iters, max_step_halvings
        p.neumann_terms = neumann_terms
        self.m = neumann_terms
        p.neumann_first = neumann_first
        p.first_poly = 0
        p.device = device
        p.kernel = 0
        p.ghost = max(neumann_terms, neumann_first) + 1
        self.ctx = C.c_void_p()
        rc = self.L.mb4cu_create(C.byref(p), C.byref(scheme.raw), C.byref(self.ctx))
        if rc:
            raise RuntimeError(self.L.mb4cu_create_error().decode())
        # run on torch's stream so NCCL and our kernels are ordered
        # torch's default stream reports handle 0, which the C ABI reads as "own
        # stream"; pass cudaStreamLegacy (0x1) for it so that the sweeps, the halo
        # pack/unpack kernels and NCCL are ordered on one stream
        self.L.mb4cu_set_stream(self.ctx, C.c_void_p(torch.cuda.current_stream(self.dev).cuda_stream or 1))
        self.n = dec.lnx * dec.lny
        self._saved = None
        self.bound_dirty = False
        self._red = None
        self._scratch = None
        self.u0_halo_ok = False
        self.overlap = overlap
        self._pending = False
        if overlap:
            # the context runs on `compute` (made torch's current stream, so NCCL
            # collectives order after the sweeps); halo exchanges run on `comms`
            self.compute = torch.cuda.Stream(self.dev)
            self.comms = torch.cuda.Stream(self.dev)
            torch.cuda.set_stream(self.compute)
            self.L.mb4cu_set_stream(self.ctx, C.c_void_p(self.compute.cuda_stream))
            self._ev_frame = torch.cuda.Event()
            self._ev_x = torch.cuda.Event()
            # negative: the library keeps the kernel's own CTAs-per-SM on all but reserve_sms SMs
            self.grid_cap = -reserve_sms if reserve_sms > 0 else 0

    def _chk(self, rc):
        if rc:
            raise RuntimeError(f"mb4cu status {rc}: {self.L.mb4cu_last_error(self.ctx).decode()}")

    def new_buffer(self, n):
        return self.torch.empty(n, dtype=self.torch.float64, device=self.dev)

    def sync(self):
        pass  # same stream as torch.distributed

    def halo_count(self, field, side):
        return int(self.L.mb4cu_halo_count(self.ctx, field, side))

    def pack(self, field, side, buf):
        self._chk(self.L.mb4cu_halo_pack(self.ctx, field, side, C.c_void_p(buf.data_ptr())))

    def unpack(self, field, side, buf):
        self._chk(self.L.mb4cu_halo_unpack(self.ctx, field, side, C.c_void_p(buf.data_ptr())))

    def sweep(self, h, s):
        """Sweep s, waiting for it: (local ||r||_inf, [5 local energy sums, local max|u0|^2])."""
        out = self._red_buf(0)
        self._chk(self.L.mb4cu_sweep_async(self.ctx, h, s, 0, C.c_void_p(out.data_ptr())))
        host = out.cpu().numpy()
        return float(host[0]), host[1:7].copy()

    def set_amax2(self, amax2: float) -> None:
        self._chk(self.L.mb4cu_set_amax2(self.ctx, amax2))
        self._amax2 = amax2

    def sweep_launch(self, h, s, final, comm, slot=0, want_sums=False):
        """Enqueue sweep s and the all-reduce of [residual max, energy sums] into the
        device buffer `slot`, on the stream shared with NCCL (no host wait)."""
        if self._red is None:
            self._red = [self.torch.zeros(7, dtype=self.torch.float64, device=self.dev) for _ in range(2)]
        red = self._red[slot]
        self._chk(self.L.mb4cu_sweep_async(self.ctx, h, s, int(final), C.c_void_p(red.data_ptr())))
        comm.allreduce_max_(red[0:1])
        if want_sums:
            comm.allreduce_sum_(red[1:6])
            comm.allreduce_max_(red[6:7])

    def sweep_read(self, slot=0, want_sums=False):
        """Host read of a launched sweep's reduced [r, 5 sums, max|u0|^2] (waits for it)."""
        host = self._red_buf(slot).cpu().numpy()
        return float(host[0]), (host[1:7].copy() if want_sums else None)

    def sweep_reduce(self, h, s, final, comm, want_sums=False):
        self.sweep_launch(h, s, final, comm, 0, want_sums)
        return self.sweep_read(0, want_sums)

    # ---- halo-exchange overlap (DistributedSession._substep_overlap) -------------
    def _red_buf(self, slot):
        if self._red is None:
            self._red = [self.torch.zeros(7, dtype=self.torch.float64, device=self.dev) for _ in range(2)]
        return self._red[slot]

    def sweep_frame(self, h, s, final):
        """Sweep s on the boundary frame (compute stream); marks it for the exchange."""
        self._chk(self.L.mb4cu_sweep_region(self.ctx, h, s, int(final), 1, 0, None))
        self._ev_frame.record(self.compute)

    def exchange_async(self, halo, field):
        """Exchange the frame just swept on the side stream (pack, NCCL, unpack)."""
        self.comms.wait_event(self._ev_frame)
        self.L.mb4cu_set_stream(self.ctx, C.c_void_p(self.comms.cuda_stream))
        try:
            with self.torch.cuda.stream(self.comms):
                halo.exchange(field)
        finally:
            self.L.mb4cu_set_stream(self.ctx, C.c_void_p(self.compute.cuda_stream))
        self._ev_x.record(self.comms)
        self._pending = True

    def wait_exchange(self):
        if self._pending:
            self.compute.wait_event(self._ev_x)
            self._pending = False

    def sweep_interior(self, h, s, final, comm, slot=0, want_sums=False):
        """Sweep s on the interior (concurrently with the exchange), then the
        device-side reduction of [r, sums] into slot (compute stream)."""
        red = self._red_buf(slot)
        self._chk(self.L.mb4cu_sweep_region(self.ctx, h, s, int(final), 2, self.grid_cap,
                                            C.c_void_p(red.data_ptr())))
        comm.allreduce_max_(red[0:1])
        if want_sums:
            comm.allreduce_sum_(red[1:6])
            comm.allreduce_max_(red[6:7])

    def sweep_repeat(self, h, s):
        """Repeat sweep s storing every stage (after a missed final guess)."""
        if self._scratch is None:
            self._scratch = self.torch.zeros(7, dtype=self.torch.float64, device=self.dev)
        self._chk(self.L.mb4cu_sweep_async(self.ctx, h, s, 0, C.c_void_p(self._scratch.data_ptr())))

    def commit(self, sweeps):
        self._chk(self.L.mb4cu_commit_step(self.ctx, sweeps))

    def obs_sums(self):
        sums = np.zeros(5)
        self._chk(self.L.mb4cu_observables_sums(self.ctx, _lib.dptr(sums)))
        return sums

    def set_state(self, u_block):
        self.u0_halo_ok = False
        if self.overlap:
            self.wait_exchange()
        u = np.ascontiguousarray(u_block, dtype=np.complex128)
        self._chk(self.L.mb4cu_set_state(self.ctx, _lib.dptr(u)))
        self.bound_dirty = True
        self._amax2 = None  # the library measures a newly set state itself

    def neumann_terms(self) -> int:
        return self.m

    def set_neumann_terms(self, m: int) -> None:
        self._chk(self.L.mb4cu_set_neumann_terms(self.ctx, m))
        self.m = m

    def spectral_bound(self) -> float:
        rho = C.c_double(0.0)
        self._chk(self.L.mb4cu_spectral_bound(self.ctx, C.byref(rho)))
        return rho.value

    def set_spectral_bound(self, rho: float) -> None:
        self._chk(self.L.mb4cu_set_spectral_bound(self.ctx, rho))

    def get_state(self):
        out = np.empty(self.n, dtype=np.complex128)
        self._chk(self.L.mb4cu_get_state(self.ctx, _lib.dptr(out)))
        return out

    def save(self):
        self._saved = self.get_state()

    def restore(self):
        dirty = getattr(self, "bound_dirty", False)  # an internal restore keeps the step's bound
        amax2 = getattr(self, "_amax2", None)
        self.set_state(self._saved)
        if amax2 is not None:  # as on one GPU: a restore keeps the tracked amplitude
            self.set_amax2(amax2)
        self.bound_dirty = dirty

    def profile(self, on=True):
        self.L.mb4cu_profile_enable(self.ctx, int(on))

    def close(self):
        if self.ctx:
            self.L.mb4cu_destroy(self.ctx)
            self.ctx = None


class StageSplitSession:
    """The paper's stage partition on GPUs: every rank holds the
    whole lattice in its own context, and the three decoupled stage systems
    (I - h lam_k J) x_k = b_k of each simplified-Newton iteration (the reference's
    WorkerPool tasks, mb4_integrator.cpp:221-229; the paper's per-node solves) are solved
    on different ranks: rank r owns the systems k with k % world == r.  The corrections
    are broadcast from their owners and every rank applies the same update, so all ranks
    hold the same iterate -- bit-identical to the single-context Newton-Krylov step
    (kernel 3).  This is the stiff-regime (paper-scale) partition; the matrix-free sweep
    path shards the lattice instead (DistributedSession).  No step halving: a step that
    does not converge raises NonConvergence with the state unchanged."""

    def __init__(self, session, comm, rank: int, world: int, epsilon: float, max_iters: int = 50,
                 lib=None, device=None):
        """lib / device: injection points for the CPU tests (a numpy stand-in of the
        mb4cu_ns_* entry points and host buffers)."""
        import torch

        self.s, self.comm, self.rank, self.world = session, comm, rank, world
        self.eps, self.max_iters = epsilon, max_iters
        self.L = lib if lib is not None else _lib.lib()
        self.torch = torch
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        if dev.type == "cuda":
            # the context runs on torch's stream so the collectives order after its kernels
            self.L.mb4cu_set_stream(session._ctx, C.c_void_p(torch.cuda.current_stream(dev).cuda_stream or 1))
        self.buf = [torch.empty(2 * session.n, dtype=torch.float64, device=dev) for _ in range(3)]

    def _chk(self, rc):
        if rc:
            raise RuntimeError(f"mb4cu status {rc}: {self.L.mb4cu_last_error(self.s._ctx).decode()}")

    def owner(self, k: int) -> int:
        return k % self.world

    def step(self, h: float) -> int:
        """One MB4 step; returns the Newton iterations."""
        ctx = self.s._ctx
        self._chk(self.L.mb4cu_ns_begin(ctx, h))
        r = math.inf
        for it in range(1, self.max_iters + 1):
            self._chk(self.L.mb4cu_ns_phibar(ctx))
            for k in range(3):
                if self.owner(k) == self.rank:
                    self._chk(self.L.mb4cu_ns_solve(ctx, k))
                    self._chk(self.L.mb4cu_ns_get_correction(ctx, k, C.c_void_p(self.buf[k].data_ptr())))
            for k in range(3):
                self.comm.broadcast_(self.buf[k], self.owner(k))
                if self.owner(k) != self.rank:
                    self._chk(self.L.mb4cu_ns_set_correction(ctx, k, C.c_void_p(self.buf[k].data_ptr())))
            rv = C.c_double(0.0)
            self._chk(self.L.mb4cu_ns_update(ctx, C.byref(rv)))
            r = rv.value
            if not math.isfinite(r):
                raise NonConvergence("newton_solve: iteration diverged (non-finite update)", math.inf)
            if r <= self.eps:  # the reference test (mb4_integrator.cpp:250)
                self._chk(self.L.mb4cu_ns_commit(ctx))
                return it
        raise NonConvergence(f"newton_solve: no convergence after {self.max_iters} iterations", r)
