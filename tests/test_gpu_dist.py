"""GPU tests of the sub-domain (multi-GPU) path on ONE GPU.

Ranks are emulated by threads in one process, each owning a libmb4cu sub-domain
context (ghost mode) on cuda:0; a host-side loopback transport stands in for
NCCL.  Kernels never wait on each other (the exchange is host-mediated between
launches), so this is safe on a single GPU.  The decomposed run must reproduce
the single-domain production kernel bit for bit.
"""
import threading

import numpy as np
import pytest
import torch

from paper_2003_04345_b200 import configs, dist as D, nls2d

pytestmark = pytest.mark.gpu


class Hub:
    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world)
        self.vals = [None] * world
        self.mail = {}
        self.lock = threading.Lock()


class LoopbackComm:
    def __init__(self, hub, rank):
        self.h, self.rank = hub, rank

    def _gather(self, x):
        self.h.vals[self.rank] = x
        self.h.bar.wait()
        v = list(self.h.vals)
        self.h.bar.wait()
        return v

    def allreduce_max(self, x):
        return float(max(self._gather(x)))

    def allreduce_sum(self, xs):
        vals = self._gather(np.asarray(xs, dtype=np.float64))
        acc = np.zeros_like(vals[0])
        for v in vals:  # fixed rank order
            acc = acc + v
        return acc

    # device-tensor variants used by the production path (dist.CudaBackend.sweep_reduce)
    def allreduce_max_(self, t):
        t.copy_(torch.from_numpy(np.max(np.stack(self._gather(t.cpu().numpy().copy())), axis=0)))

    def allreduce_sum_(self, t):
        t.copy_(torch.from_numpy(self.allreduce_sum(t.cpu().numpy().copy())))

    def exchange(self, pairs):
        torch.cuda.synchronize()
        counts = {}
        with self.h.lock:
            for send, dst, _, _ in pairs:
                k = counts.get(dst, 0)
                counts[dst] = k + 1
                self.h.mail[(self.rank, dst, k)] = send.clone()
        torch.cuda.synchronize()
        self.h.bar.wait()
        counts = {}
        for _, _, recv, src in pairs:
            k = counts.get(src, 0)
            counts[src] = k + 1
            recv.copy_(self.h.mail[(src, self.rank, k)])
        torch.cuda.synchronize()
        self.h.bar.wait()
        with self.h.lock:
            self.h.mail.clear()
        self.h.bar.wait()


def _run_decomposed(name, px, py, m, nsteps, overlap=False, hs=None, reserve_sms=0, adaptive_m=False):
    cfg = configs.CONFIGS[name]
    V, psi = configs.make_inputs(cfg)
    world = px * py
    hub = Hub(world)
    out = [None] * world
    errs = []

    def work(rank):
        try:
            torch.cuda.set_device(0)
            dec = D.Decomposition(cfg.nx, cfg.ny, px, py, rank)
            be = D.CudaBackend(dec, dec.block(V), nls2d.Mb4Scheme(), cfg.gamma, 1.0, 1.0, cfg.epsilon,
                               cfg.max_iters, m, 0, overlap=overlap, reserve_sms=reserve_sms)
            be.set_state(dec.block(psi))
            sess = D.DistributedSession(dec, be, LoopbackComm(hub, rank), cfg.gamma, 1.0, 1.0, cfg.epsilon,
                                        adaptive_m=adaptive_m)
            if hs is None:
                obs, sweeps = sess.run(cfg.dt, nsteps)
            else:
                sweeps = [sess.step(h)[0] for h in hs]
                obs = None
            out[rank] = (dec, be.get_state(), obs, sweeps)
            be.close()
        except Exception as exc:  # surface thread failures
            errs.append(exc)
            hub.bar.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    glob = np.zeros((cfg.ny, cfg.nx), dtype=np.complex128)
    for dec, u, _, _ in out:
        glob[dec.y0:dec.y0 + dec.lny, dec.x0:dec.x0 + dec.lnx] = u.reshape(dec.lny, dec.lnx)
    return glob.reshape(-1), out[0][2], out[0][3]


@pytest.mark.parametrize("px,py,m", [(1, 1, 1), (2, 1, 1), (1, 2, 2), (2, 2, 1), (2, 2, 2), (3, 1, 1), (1, 3, 2)])
def test_subdomain_path_matches_single_domain(px, py, m):
    name, nsteps = "cfg2", 4
    cfg = configs.CONFIGS[name]
    u_dec, obs_dec, sweeps_dec = _run_decomposed(name, px, py, m, nsteps)
    V, psi = configs.make_inputs(cfg)
    with nls2d.Session(configs.model_for(cfg, V), nls2d.Mb4Scheme(), configs.newton_for(cfg),
                       neumann_terms=m) as s:
        s.set_state(psi)
        obs, sweeps = s.run(cfg.dt, nsteps)
        u = s.get_state()
    assert list(sweeps_dec) == list(sweeps)
    assert np.array_equal(u_dec, u), np.abs(u_dec - u).max()
    H = obs_dec[:, 3]
    assert np.abs(H - obs[:, 3]).max() <= 1e-14 * abs(H[0])
    assert np.abs(H - H[0]).max() / abs(H[0]) <= 1e-13


@pytest.mark.parametrize("px,py,reserve", [(1, 1, 0), (2, 1, 0), (2, 2, 0), (2, 1, 8)])
def test_halo_overlap_path_matches_single_domain(px, py, reserve):
    """Boundary frame first, its halo exchange on a side stream while the interior
    is swept (mb4cu_sweep_region), U3 halos carried into the next step: the same
    trajectory bit for bit as the single-domain kernel, including a step that misses
    its predicted final sweep (the longer third step)."""
    name = "cfg2"
    cfg = configs.CONFIGS[name]
    hs = [cfg.dt, cfg.dt, 2 * cfg.dt, cfg.dt]
    # reserve > 0: the interior launches leave that many SMs free (the NCCL overlap setting)
    u_dec, _, sweeps_dec = _run_decomposed(name, px, py, 1, len(hs), overlap=True, hs=hs, reserve_sms=reserve)
    V, psi = configs.make_inputs(cfg)
    with nls2d.Session(configs.model_for(cfg, V), nls2d.Mb4Scheme(), configs.newton_for(cfg),
                       neumann_terms=1) as s:
        s.set_state(psi)
        sweeps = []
        for h in hs:
            st = nls2d.StepStats()
            s.step(h, st)
            sweeps.append(st.newton_iters)
        u = s.get_state()
    assert list(sweeps_dec) == sweeps
    assert np.array_equal(u_dec, u), np.abs(u_dec - u).max()


class LoopbackBroadcast(LoopbackComm):
    def broadcast_(self, t, src):
        torch.cuda.synchronize()
        vals = self._gather(t.cpu().clone() if self.rank == src else None)
        t.copy_(vals[src].to(t.device))
        torch.cuda.synchronize()


@pytest.mark.parametrize("world", [1, 2, 3])
def test_stage_split_matches_single_context_newton_krylov(world):
    """The paper's stage partition (dist.StageSplitSession): each rank solves the stage
    systems it owns and the corrections are broadcast -- here `world` thread-loopback ranks,
    each with its own context on one GPU -- reproduces the single-context Newton-Krylov step
    (kernel 3) bit for bit, with the same Newton iteration counts."""
    n, gamma = 70, 0.1
    g = nls2d.GridSpec(n, n, 2 * np.pi, 2 * np.pi)
    model = nls2d.GridModel(g, gamma)
    u0 = nls2d.initial_condition(g)
    cfg = nls2d.NewtonConfig()
    hs = [0.01, 0.01]
    with nls2d.Session(model, nls2d.Mb4Scheme(), cfg, kernel=3) as s:
        s.set_state(u0)
        its = []
        for h in hs:
            st = nls2d.StepStats()
            s.step(h, st)
            its.append(st.newton_iters)
        ref = s.get_state()
    hub = Hub(world)
    out = [None] * world
    errs = []

    def work(rank):
        try:
            torch.cuda.set_device(0)
            with nls2d.Session(model, nls2d.Mb4Scheme(), cfg, kernel=3) as s:
                s.set_state(u0)
                sess = D.StageSplitSession(s, LoopbackBroadcast(hub, rank), rank, world, cfg.epsilon, cfg.max_iters)
                got_its = [sess.step(h) for h in hs]
                out[rank] = (s.get_state(), got_its)
        except Exception as exc:
            errs.append(exc)
            hub.bar.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    for u, got_its in out:
        assert got_its == its
        assert np.array_equal(u, ref)
    # anchor to the reference itself (not only to the single-context GPU path): the
    # reference's stage solves (mb4_integrator.cpp:221-229, direct LU), same inputs
    from oracle import oracle as O

    oref, _, oits, _ = O.ref_run(n, n, 2 * np.pi, 2 * np.pi, gamma, np.zeros(n * n), u0, hs[0], len(hs),
                                 eps=cfg.epsilon, max_iters=cfg.max_iters, solver="direct")
    for u, got_its in out:
        assert np.linalg.norm(u - oref) / np.linalg.norm(oref) <= 1e-10
        assert got_its == list(oits)  # the reference's simplified-Newton iteration counts


@pytest.mark.parametrize("overlap", [False, True])
def test_adaptive_depth_matches_single_domain(overlap):
    """DistributedSession(adaptive_m=True) applies the library's adaptive later-sweep depth
    (m = 2 once a step needs >= 4 sweeps at m = 1): the decomposed cfg1 run switches where the
    single-domain default does and reproduces it bit for bit."""
    name, nsteps = "cfg1", 4
    cfg = configs.CONFIGS[name]
    u_dec, _, sweeps_dec = _run_decomposed(name, 2, 2, 1, nsteps, overlap=overlap, adaptive_m=True)
    V, psi = configs.make_inputs(cfg)
    with nls2d.Session(configs.model_for(cfg, V), nls2d.Mb4Scheme(), configs.newton_for(cfg)) as s:
        s.set_state(psi)
        _, sweeps = s.run(cfg.dt, nsteps)
        u = s.get_state()
    assert sweeps[0] >= 4  # the switch happens
    assert list(sweeps_dec) == list(sweeps)
    assert np.array_equal(u_dec, u), np.abs(u_dec - u).max()


def test_set_neumann_terms_validation():
    """mb4cu_set_neumann_terms accepts the compiled (neumann_first, m) pairs within the ghost
    width and rejects the rest; the stage-split entry points refuse to run without ns_begin."""
    import ctypes as C

    from paper_2003_04345_b200 import _lib

    cfg = configs.CONFIGS["cfg1"]
    V, psi = configs.make_inputs(cfg)
    L = _lib.lib()
    with nls2d.Session(configs.model_for(cfg, V), nls2d.Mb4Scheme(), configs.newton_for(cfg)) as s:
        assert L.mb4cu_set_neumann_terms(s._ctx, 2) == 0
        assert L.mb4cu_set_neumann_terms(s._ctx, 3) == _lib.MB4CU_INVALID
        assert L.mb4cu_set_neumann_terms(s._ctx, -1) == _lib.MB4CU_INVALID
        r = C.c_double(0.0)
        assert L.mb4cu_ns_update(s._ctx, C.byref(r)) == _lib.MB4CU_INVALID
        assert L.mb4cu_ns_solve(s._ctx, 0) == _lib.MB4CU_INVALID
        s.set_state(psi)
        s.step(cfg.dt)  # still steps normally at the fixed depth


class FmaxLoopbackComm(LoopbackComm):
    """MAX all-reduce with NCCL / gloo semantics (fmax: a NaN operand is dropped)."""

    def allreduce_max(self, x):
        return float(np.fmax.reduce(np.asarray(self._gather(x), dtype=np.float64)))

    def allreduce_max_(self, t):
        t.copy_(torch.from_numpy(np.fmax.reduce(np.stack(self._gather(t.cpu().numpy().copy())), axis=0)))


@pytest.mark.parametrize("overlap", [False, True])
def test_nan_block_on_one_rank_is_reported_by_every_rank(overlap):
    """A NaN in one rank's sub-domain must not be lost in the MAX all-reduce (fmax drops
    NaN operands): the library reports a non-finite local residual as +inf, so every
    rank sees the divergence and no rank commits a step (dist.py)."""
    cfg = configs.CONFIGS["cfg2"]
    V, psi = configs.make_inputs(cfg)
    px, py, world = 2, 1, 2
    hub = Hub(world)
    res = [None] * world
    errs = []

    def work(rank):
        try:
            torch.cuda.set_device(0)
            dec = D.Decomposition(cfg.nx, cfg.ny, px, py, rank)
            be = D.CudaBackend(dec, dec.block(V), nls2d.Mb4Scheme(), cfg.gamma, 1.0, 1.0, cfg.epsilon,
                               cfg.max_iters, 1, 0, overlap=overlap)
            blk = dec.block(psi).copy()
            if rank == 1:
                blk[blk.size // 2] = np.nan
            be.set_state(blk)
            sess = D.DistributedSession(dec, be, FmaxLoopbackComm(hub, rank), cfg.gamma, 1.0, 1.0, cfg.epsilon,
                                        max_step_halvings=0)
            try:
                sess.step(cfg.dt)
                res[rank] = "committed"
            except D.NonConvergence:
                res[rank] = "diverged"
            be.close()
        except Exception as exc:
            errs.append(exc)
            hub.bar.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    assert res == ["diverged", "diverged"]


@pytest.mark.parametrize("name,force_p2p,adaptive", [("cfg2", False, False), ("cfg2", True, False),
                                                     ("cfg1", True, True)])
def test_native_nccl_stepper_matches_single_domain(name, force_p2p, adaptive):
    """The decomposed step inside the library (dist.NativeSession / mb4cu_dist_*: NCCL
    transport, device-side stopping test, one host read per step) on a 1-rank NCCL
    communicator -- with force_p2p the periodic halos go through NCCL send / recv to
    oneself -- reproduces the single-domain production kernel bit for bit (cfg2 changes its
    sweep count from step to step: predicted-sweep misses and repeated final sweeps; cfg1
    with the adaptive depth crosses the m switch)."""
    cfg = configs.CONFIGS[name]
    nsteps = 6
    V, psi = configs.make_inputs(cfg)
    dec = D.Decomposition(cfg.nx, cfg.ny, 1, 1, 0)
    be = D.CudaBackend(dec, V, nls2d.Mb4Scheme(), cfg.gamma, 1.0, 1.0, cfg.epsilon, cfg.max_iters, 1, 0,
                       max_step_halvings=cfg.max_step_halvings)
    be.set_state(psi)
    ns = D.NativeSession(dec, be, D.nccl_unique_id(), cfg.gamma, 1.0, 1.0, adaptive_m=adaptive,
                         force_p2p=force_p2p)
    obs_d, sweeps_d = ns.run(cfg.dt, nsteps)
    u_d = be.get_state()
    ns.close()
    be.close()
    with nls2d.Session(configs.model_for(cfg, V), nls2d.Mb4Scheme(), configs.newton_for(cfg),
                       neumann_terms=None if adaptive else 1) as s:
        s.set_state(psi)
        obs, sweeps = s.run(cfg.dt, nsteps)
        u = s.get_state()
    assert list(sweeps_d) == list(sweeps)
    assert np.array_equal(u_d, u), np.abs(u_d - u).max()
    H = obs[:, 3]
    assert np.abs(obs_d[:, 3] - H).max() <= 1e-14 * abs(H[0])


def test_native_nccl_stepper_halving_and_divergence():
    """The native stepper's failure paths: with max_iters = 3 some cfg2 steps need more
    sweeps, fail on the device (one host read) and are halved -- the same trajectory, sweep
    and halving counts as the Python-driven decomposed loop (DistributedSession, which halves
    the same way; the single-domain library would first try Newton-Krylov); a NaN in the state
    is reported as non-convergence."""
    cfg = configs.CONFIGS["cfg2"]
    V, psi = configs.make_inputs(cfg)
    dec = D.Decomposition(cfg.nx, cfg.ny, 1, 1, 0)

    def backend():
        be = D.CudaBackend(dec, V, nls2d.Mb4Scheme(), cfg.gamma, 1.0, 1.0, cfg.epsilon, 3, 1, 0,
                           max_step_halvings=4)
        be.set_state(psi)
        return be

    be = backend()
    ns = D.NativeSession(dec, be, D.nccl_unique_id(), cfg.gamma, 1.0, 1.0, force_p2p=True)
    got = [ns.step(cfg.dt) for _ in range(3)]
    u_d = be.get_state()
    bad = psi.copy()
    bad[5] = np.nan
    be.set_state(bad)
    with pytest.raises(D.NonConvergence):
        ns.step(cfg.dt)
    ns.close()
    be.close()
    be = backend()
    ps = D.DistributedSession(dec, be, LoopbackComm(Hub(1), 0), cfg.gamma, 1.0, 1.0, cfg.epsilon, max_iters=3,
                              max_step_halvings=4)
    ref = [ps.step(cfg.dt) for _ in range(3)]
    u = be.get_state()
    be.close()
    assert got == ref and max(hv for _, hv in got) >= 1
    assert np.array_equal(u_d, u)
