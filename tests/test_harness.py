"""Harness drop-in: RunConfig parsing/validation on the CPU,
run() + trajectory CSV + snapshots on the GPU (compared with the reference)."""
import os

import numpy as np
import pytest

from paper_2003_04345_b200 import harness as Hn

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_parse_config_file_and_overrides(tmp_path):
    p = tmp_path / "run.cfg"
    p.write_text("# comment\nnx = 32\nny = 16  # trailing\nlx = 6.5\nmethod = mb4\n"
                 "snapshot_times = 0.1, 0.2\nsolver = gmres\nworkers = 3\n")
    cfg = Hn.parse_config_file(str(p))
    assert (cfg.nx, cfg.ny, cfg.lx, cfg.solver, cfg.workers) == (32, 16, 6.5, "gmres", 3)
    assert cfg.snapshot_times == [0.1, 0.2]
    Hn.apply_key_value(cfg, "dt", "0.005")
    assert cfg.dt == 0.005
    with pytest.raises(Hn.ConfigError):
        Hn.apply_key_value(cfg, "no_such_key", "1")
    with pytest.raises(Hn.ConfigError):
        Hn.apply_key_value(cfg, "nx", "abc")
    bad = tmp_path / "bad.cfg"
    bad.write_text("nx 32\n")
    with pytest.raises(Hn.ConfigError):
        Hn.parse_config_file(str(bad))


@pytest.mark.parametrize("field,val", [("nx", 1), ("dt", 0.0), ("t_end", 0.001), ("epsilon", 0.0),
                                       ("max_iters", 0), ("max_halvings", -1), ("workers", 4),
                                       ("method", "leapfrog")])
def test_validate_rejects(field, val):
    cfg = Hn.RunConfig()
    setattr(cfg, field, val)
    with pytest.raises(Hn.ConfigError):
        cfg.validate()


def test_baseline_key_sets_the_lattice():
    cfg = Hn.RunConfig()
    Hn.apply_key_value(cfg, "baseline", "cfg2")
    assert (cfg.nx, cfg.ny, cfg.lx, cfg.dt, cfg.gamma) == (256, 256, 256.0, 0.005, -2.0)
    assert Hn.step_count(cfg.t_end, cfg.dt) == 2000
    assert Hn.step_count(1.0, 0.3) == 4


@pytest.mark.gpu
def test_run_writes_reference_compatible_csv(tmp_path):
    cfg = Hn.RunConfig()
    Hn.apply_key_value(cfg, "baseline", "cfg1")
    cfg.t_end = 0.1  # 10 steps
    cfg.snapshot_times = [0.0, 0.05]
    cfg.out_dir = str(tmp_path)
    rec = Hn.run(cfg)
    g = np.load(os.path.join(GOLD, "ref_cfg1_10.npz"))
    H = np.array([r.total_energy for r in rec.rows])
    assert len(rec.rows) == 11
    assert np.abs(H - g["obs"][:, 3]).max() <= 1e-13 * abs(H[0])
    assert np.linalg.norm(rec.final_state - g["state_10"]) / np.linalg.norm(g["state_10"]) <= 1e-10
    assert rec.max_energy_drift() <= 1e-13
    lines = (tmp_path / "trajectory.csv").read_text().splitlines()
    assert lines[0] == "t,UK,UI,UE,H,prob,participation,newton_iters,wall_s"
    assert len(lines) == 12
    t, uk, ui, ue, h = (float(x) for x in lines[1].split(",")[:5])
    assert t == 0.0 and abs(h - (uk + ui + ue)) <= 1e-15 * abs(h)
    assert os.path.exists(tmp_path / "snapshot_0.txt") and os.path.exists(tmp_path / "snapshot_0.05.txt")
    snap = (tmp_path / "snapshot_0.05.txt").read_text().splitlines()
    assert snap[0].startswith("# 0.05") and len(snap) == 1 + 64


@pytest.mark.gpu
def test_run_last_short_step_and_paper_style_config(tmp_path):
    # t_end not a multiple of dt: the last step is shorter (harness.cpp:107-110)
    cfg = Hn.RunConfig(nx=16, ny=16, lx=16.0, ly=16.0, t_end=0.025, dt=0.01, gamma=-0.5, v0=2.0,
                       epsilon=1e-14)
    rec = Hn.run(cfg)
    ts = [r.t for r in rec.rows]
    assert len(ts) == 4 and abs(ts[-1] - 0.025) < 1e-15
    from oracle import oracle as O

    model = cfg.make_model()
    u0 = cfg.make_initial(model)
    o = O.Oracle(16, 16, -0.5, model.potential())
    u, _, _ = o.run(u0, 0.01, 2, eps=1e-14)
    u, _, _ = o.run(u, 0.005, 1, eps=1e-14)
    assert np.linalg.norm(rec.final_state - u) / np.linalg.norm(u) <= 1e-10


@pytest.mark.gpu
def test_compare_methods_and_convergence_study():
    # harness.cpp:147-196 / 272-316 on the GPU: every method, the reference's
    # conservation classes and orders on a short paper-scale run
    cfg = Hn.RunConfig(nx=16, ny=16, t_end=0.1, dt=0.01, gamma=0.1)
    rep = Hn.compare_methods(cfg, ["gauss2", "gauss4", "avf2", "avf4", "mb4", "rk4"])
    d = {m.method: m for m in rep.methods}
    for m in ("mb4", "avf2", "avf4"):
        assert d[m].energy_drift <= 1e-11
    for m in ("gauss2", "gauss4"):
        assert d[m].probability_drift <= 1e-12
    assert d["rk4"].total_newton_iters == 0 and d["mb4"].total_newton_iters > 0
    assert rep.mb4_over_gauss2 > 0.0
    import io
    buf = io.StringIO()
    rep.write(buf)
    assert buf.getvalue().startswith("method  energy_drift")
    conv = Hn.convergence_study(Hn.RunConfig(nx=16, ny=16, t_end=0.2, gamma=0.1), ["avf2", "gauss4"],
                                [0.02, 0.01, 0.005])
    slopes = {e.method: e.slope for e in conv.entries}
    assert 1.8 <= slopes["avf2"] <= 2.2
    assert 3.6 <= slopes["gauss4"] <= 4.4
    bench = Hn.parallel_bench(Hn.RunConfig(nx=16, ny=16, t_end=0.05, dt=0.01))
    assert bench.trajectories_identical
