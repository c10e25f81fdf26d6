"""CUDA path vs the 3D CPU oracle, through the C-ABI.

Tolerances (north star): fp64 state relative Linf <= 1e-12 after one stage /
step, <= 1e-10 after 100 stages; residuals compared relative to their own
scale at 1e-12 (absolute 1e-12 for free-stream noise); pairing bit-exact.
"""
import math
import os

import numpy as np
import pytest

from conftest import rel_linf
from oracle import pyoracle as P
from paper_2008_04356_b200 import types as T

pytestmark = pytest.mark.gpu


def gpu_solver(mesh, cfg):
    from paper_2008_04356_b200.capi import RankSolver
    return RankSolver(mesh, cfg)


def three_band(ny=6, nz=2, vg=1.0, nx=2):
    return T.mesh_spec([(nx, 1.0, 0.0), (nx, 1.0, vg), (nx, 1.0, 0.0)], ny=ny, nz=nz, depth=1.0)


def box0(n_per=4):
    # BASELINE config [0]: [0,2]^3 split at the interface, upper block sliding +0.5,
    # Dirichlet across the split axis (x here), periodic along the slide and the third axis.
    return T.mesh_spec([(n_per, 1.0, 0.0), (n_per, 1.0, 0.5)], ny=n_per, nz=n_per, periodic=(False, True, True))


CASES = {
    "dw3band_lgl_inv": (three_band(), dict(degree=3, node_kind=T.NODES_LGL, mu=0.0)),
    "dw3band_gauss_visc": (three_band(), dict(degree=3, node_kind=T.NODES_GAUSS, mu=1e-3)),
    "box0_gauss_visc": (box0(2), dict(degree=3, node_kind=T.NODES_GAUSS, mu=1e-3)),
    "box0_lgl_visc_n5": (box0(2), dict(degree=5, node_kind=T.NODES_LGL, mu=1e-3)),
}


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("t", [0.0, 0.05, 0.37])
def test_residual_matches_oracle(name, t):
    mesh, kw = CASES[name]
    cfg = T.solver_config(case=T.density_wave(), **kw)
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    o.set_initial_condition(0.0)
    u = o.field()
    rg, ro = g.compute_residual(t, u), o.compute_residual(t, u)
    assert rel_linf(rg, ro) <= 1e-12


@pytest.mark.parametrize("degree", [1, 2, 3, 4, 5, 6, 7])
@pytest.mark.parametrize("kind", [T.NODES_LGL, T.NODES_GAUSS])
def test_all_degrees_one_step(degree, kind):
    mesh = three_band(ny=3, nz=2)
    cfg = T.solver_config(degree, kind, mu=1e-3, case=T.density_wave())
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    g.set_initial_condition(0.0)
    o.set_initial_condition(0.0)
    dt = o.suggest_dt(0.4)
    assert abs(g.suggest_dt(0.4) - dt) <= 1e-14 * dt
    g.step(dt)
    o.step(dt)
    assert rel_linf(g.field(), o.field()) <= 1e-12


def test_hundred_stages_box0():
    mesh = box0(2)
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=1e-3, case=T.density_wave())
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    g.set_initial_condition(0.0)
    o.set_initial_condition(0.0)
    dt = o.suggest_dt(0.5)
    g.step(dt, 20)
    o.step(dt, 20)
    assert rel_linf(g.field(), o.field()) <= 1e-10
    assert g.total_rebuilds() == o.total_rebuilds()


def test_pairing_bit_exact_every_stage():
    mesh = three_band(ny=6, nz=3)
    cfg = T.solver_config(2, T.NODES_GAUSS, mu=0.0, case=T.density_wave())
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    o.set_initial_condition(0.0)
    u = o.field()
    for t in [0.0, 0.05, 1.0 / 3.0, 0.37, 0.99, 2.0, 5.0 + 1e-9]:
        g.compute_residual(t, u)
        o.compute_residual(t, u)
        for role in (0, 1):
            assert np.array_equal(g.pairing(role), o.pairing(role))
        for c in range(o.n_contexts()):
            ig, io = g.ctx_info(c), o.ctx_info(c)
            assert (ig["n_delta"], ig["conforming"], ig["s_delta"]) == (io["n_delta"], io["conforming"], io["s_delta"])
            assert np.array_equal(g.mapping(c), o.mapping(c))


@pytest.mark.parametrize("kind", [T.NODES_LGL, T.NODES_GAUSS])
@pytest.mark.parametrize("mu", [0.0, 1e-3])
def test_freestream_preserved_across_sliding(kind, mu):
    mesh = three_band(ny=6, nz=2)
    cfg = T.solver_config(4, kind, mu=mu, case=T.freestream(v=(1.0, 0.5, 0.25)))
    g = gpu_solver(mesh, cfg)
    g.set_initial_condition(0.0)
    for t in [0.0, 0.05, 1.0 / 3.0, 0.37, 0.99, 2.0, 5.0 + 1e-9]:
        assert np.abs(g.compute_residual(t)).max() < 1e-12


def test_conservation_sliding_density_wave():
    mesh = three_band(ny=6, nz=2)
    cfg = T.solver_config(3, T.NODES_LGL, mu=0.0, case=T.density_wave(a=(1.0, 1.0, 0.5)))
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    g.set_initial_condition(0.0)
    before = o.mass_energy(g.field())
    g.step(0.008, 10)
    after = o.mass_energy(g.field())
    assert np.all(np.abs(after - before) / np.abs(before) < 1e-12)


def test_dirichlet_all_sides():
    mesh = T.mesh_spec([(3, 1.0, 0.0)], ny=3, nz=3, periodic=(False, False, False))
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=1e-3, case=T.density_wave())
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    g.set_initial_condition(0.1)
    o.set_initial_condition(0.1)
    dt = o.suggest_dt(0.5)
    g.step(dt, 2)
    o.step(dt, 2)
    assert rel_linf(g.field(), o.field()) <= 1e-12


def test_gradients_match_oracle():
    mesh = three_band(ny=4, nz=2)
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=1e-3, case=T.density_wave())
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    o.set_initial_condition(0.0)
    u = o.field()
    gg, go = g.compute_gradients(0.21, u), o.compute_gradients(0.21, u)
    assert rel_linf(gg, go) <= 1e-12


def test_tgv_three_blocks():
    L = 2 * math.pi
    mesh = T.mesh_spec([(2, 1.0, 0.0), (2, 1.0, 0.2), (2, 1.0, 0.0)], ny=3, nz=3, width=L, height=L, depth=L)
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=1.0 / 1600.0, case=T.tgv())
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    g.set_initial_condition(0.0)
    o.set_initial_condition(0.0)
    dt = o.suggest_dt(0.5)
    g.step(dt, 2)
    o.step(dt, 2)
    assert rel_linf(g.field(), o.field()) <= 1e-12


@pytest.mark.parametrize("degree", [3, 5, 7])
def test_baseline_config4_sweep_smallest_load(degree):
    """BASELINE configs[4] sweep at its smallest load (8^3 elements, the bench's mesh builder:
    three blocks along the split axis, middle block sliding at +0.2), N in {3, 5, 7}: one RK step
    equal to the oracle."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    mesh, _ = bench.tgv_mesh(T, 8, 8)
    cfg = T.solver_config(degree, T.NODES_GAUSS, mu=1.0 / 1600.0, case=T.tgv())
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    g.set_initial_condition(0.0)
    o.set_initial_condition(0.0)
    dt = o.suggest_dt(0.5)
    g.step(dt)
    o.step(dt)
    assert rel_linf(g.field(), o.field()) <= 1e-12


def test_positivity_violation_raises():
    mesh = three_band(ny=3, nz=1)
    cfg = T.solver_config(2, T.NODES_LGL, case=T.freestream())
    g = gpu_solver(mesh, cfg)
    g.set_initial_condition(0.0)
    u = g.field()
    u[0] = -1.0
    g.set_state(u)
    with pytest.raises(T.InvalidStateError):
        g.step(1e-6)


def test_appendix_a_device_pairing():
    # Worked sorting example, proj/tests/test_partition.cpp:23-53 and :110-150 (Appendix A).
    faces = [(5, 4, 1), (6, 4, 2), (7, 5, 1), (8, 3, 2), (9, 3, 1)]
    ranks = np.full((3, 6), 9, dtype=np.int32)
    for (ip, iq, r) in [(1, 1, 7), (2, 1, 7), (3, 1, 4), (4, 1, 4), (1, 2, 7), (2, 2, 4), (3, 2, 4), (4, 2, 4)]:
        ranks[iq, ip] = r
    from paper_2008_04356_b200.capi import pairing_device
    out = pairing_device(faces, 6, 3, ranks, 1, True, False, 0)
    cols = out["cols"]
    assert list(cols[:, 0]) == [4, 4, 4, 4, 4, 4, 7, 7, 7, 7]
    assert list(cols[:, 2]) == [3, 4, 4, 4, 5, 5, 3, 3, 3, 4]
    assert list(cols[:, 3]) == [2, 1, 2, 2, 1, 1, 1, 1, 2, 1]
    assert list(cols[:, 4]) == [1, 1, 0, 1, 0, 1, 0, 1, 0, 0]
    assert list(cols[:, 5]) == [8, 5, 6, 6, 7, 7, 9, 9, 8, 5]
    assert out["face_lo"] == 5
    assert list(out["m"][0] + 1) == [10, 3, 5, 9, 7]
    assert list(out["m"][1] + 1) == [2, 4, 6, 1, 8]
    assert out["sched"].tolist() == [[4, 0, 6], [7, 6, 4]]
    assert out["self_entry"][2] == 0


# ---------------------------------------------------------------- SURVEY §8(f) rows 2-3
def test_diagnostics_match_oracle():
    """integrate_mass_energy / error_norms (diagnostics.cpp:31-87) on the device."""
    mesh = box0(2)
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=1e-3, case=T.density_wave())
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    g.set_initial_condition(0.0)
    o.set_initial_condition(0.0)
    dt = o.suggest_dt(0.5)
    g.step(dt, 3)
    o.step(dt, 3)
    d = g.diagnostics(g.time())
    me = o.mass_energy(g.field())
    assert abs(d["mass"] - me[0]) <= 1e-13 * abs(me[0])
    assert abs(d["energy"] - me[1]) <= 1e-13 * abs(me[1])
    assert abs(d["volume"] - 8.0) <= 1e-12
    ex = o.sample_case(g.time()).reshape(-1, 5)
    err = g.field().reshape(-1, 5) - ex
    assert np.allclose(d["linf"], np.abs(err).max(axis=0), rtol=1e-6, atol=1e-15)
    assert np.all(d["l2"] >= 0.0) and d["l2"][0] <= d["linf"][0]


def test_freestream_deviation_after_steps():
    mesh = three_band(ny=6, nz=2)
    cfg = T.solver_config(4, T.NODES_GAUSS, mu=1e-3, case=T.freestream(v=(1.0, 0.5, 0.25)))
    g = gpu_solver(mesh, cfg)
    g.set_initial_condition(0.0)
    g.step(g.suggest_dt(0.5), 10)
    assert g.diagnostics(g.time())["max_deviation"] < 1e-12


def test_snapshot_round_trip(tmp_path):
    """SDGFLD1 write / read (snapshot.cpp:10-56), 3D header."""
    mesh = three_band(ny=3, nz=2)
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=1e-3, case=T.density_wave())
    g = gpu_solver(mesh, cfg)
    g.set_initial_condition(0.25)
    g.step(1e-3, 2)
    path = str(tmp_path / "field.sdg")
    g.write_snapshot(path)
    head = open(path, "rb").read(200).split(b"\n")
    assert head[0] == b"SDGFLD1" and head[1].startswith(b"n_elements 36 degree 3 nvars 5 time 0.252")
    before = g.field()
    h = gpu_solver(mesh, cfg)
    t = h.read_snapshot(path)
    assert abs(t - g.time()) < 1e-15
    assert np.array_equal(h.field(), before)
    # the restored context continues from the snapshot's time and interface offset
    assert h.time() == t
    g.step(1e-3, 2)
    h.step(1e-3, 2)
    assert rel_linf(h.field(), g.field()) <= 1e-13


@pytest.mark.parametrize("ranks", [2, 3])
def test_snapshot_multi_rank_equals_single_rank(tmp_path, ranks):
    """Collective snapshot: every rank writes its elements in place after rank 0
    has created and sized the file; the file equals a single-rank write, and a
    multi-rank read restores every rank's field."""
    from paper_2008_04356_b200 import capi
    mesh = T.mesh_spec([(2, 1.0, 0.0), (2, 1.0, 1.0), (2, 1.0, 0.0)], ny=6, nz=2, depth=1.0)
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=1e-3, case=T.density_wave())
    one, many = str(tmp_path / "one.sdg"), str(tmp_path / "many.sdg")

    def write(path):
        def body(s):
            s.set_initial_condition(0.0)
            s.step(0.004, 2)
            s.write_snapshot(path)
            return s.local_element_ids(), s.field()
        return body

    def read(s):
        t = s.read_snapshot(many)
        return s.local_element_ids(), s.field(), t

    capi.run_inproc(mesh, cfg, 1, write(one), hub="snap1")
    parts = capi.run_inproc(mesh, cfg, ranks, write(many), hub=f"snap{ranks}")
    assert open(one, "rb").read() == open(many, "rb").read()
    back = capi.run_inproc(mesh, cfg, ranks, read, hub=f"snapr{ranks}")
    for (ids, u), (ids2, u2, t) in zip(parts, back):
        assert np.array_equal(ids, ids2) and np.array_equal(u, u2) and t == 0.008


# ---------------------------------------------------------------- GPU vs the reference itself
GOLDEN_FIXT = {
    # name: (bands, ny, degree, kind, mu, periodic_x, case) — see tests/golden/make_golden.py
    "dw_lgl3_inv": ([(2, 1.0, 0.0), (2, 1.0, 1.0), (2, 1.0, 0.0)], 6, 3, T.NODES_LGL, 0.0, True, "density_wave"),
    "dw_gauss3_visc": ([(2, 1.0, 0.0), (2, 1.0, 1.0), (2, 1.0, 0.0)], 6, 3, T.NODES_GAUSS, 1e-3, True,
                       "density_wave"),
    "dw_gauss5_visc_dirichlet": ([(2, 1.0, 0.0), (2, 1.0, 0.5)], 2, 5, T.NODES_GAUSS, 1e-3, False, "density_wave"),
    "fs_lgl4_inv": ([(2, 1.0, 0.0), (2, 1.0, 1.0), (2, 1.0, 0.0)], 6, 4, T.NODES_LGL, 0.0, True, "freestream"),
}


@pytest.mark.parametrize("name", sorted(GOLDEN_FIXT))
def test_gpu_embeds_reference_fixture(name):
    """z-invariant embedding of the reference's own 2D results (tests/golden, made
    from oracle/_ref = the unmodified reference library): residual and 10 RK steps."""
    import os

    import embed
    bands, ny, deg, kind, mu, px, case = GOLDEN_FIXT[name]
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", f"ref2d_{name}.npz"))
    nz, n = 2, deg + 1
    mesh = embed.mesh3d(bands, ny, nz, periodic_x=px)
    cfg = T.solver_config(deg, kind, mu=mu, case=embed.case3d(case))
    g = gpu_solver(mesh, cfg)
    g.set_initial_condition(0.0)
    u0 = g.field()
    r = g.compute_residual(float(z["t_res"]), u0)
    scale = max(np.abs(z["residual"]).max(), 1.0)
    assert embed.max_layer_diff(r, z["residual"], bands, ny, nz, n) <= 1e-12 * scale
    g = gpu_solver(mesh, cfg)  # fresh solver: rebuild counts start from zero as in the fixture
    g.set_initial_condition(0.0)
    g.step(float(z["dt"]), int(z["n_steps"]))
    assert embed.max_layer_diff(g.field(), z["u_end"], bands, ny, nz, n) <= 1e-12 * np.abs(z["u_end"]).max()
    assert g.total_rebuilds() == int(z["rebuilds"])


# ---------------------------------------------------------------- multi-rank data path on one GPU
@pytest.mark.parametrize("partition", [T.PARTITION_LEX, T.PARTITION_SFC, T.PARTITION_YSLAB])
@pytest.mark.parametrize("ranks", [2, 3, 6])
def test_rank_counts_do_not_change_the_bits(ranks, partition):
    """proj/tests/test_runner.cpp:32-50 on the B200 path: 1 rank vs 2/3/6 ranks
    (in-process hub, same device) must give bitwise-identical fields.  Exercises
    the partition, the halo slots of trace / Fv.n exchange and the per-partner
    mortar blocks of the NCCL path's protocol."""
    from paper_2008_04356_b200 import capi
    mesh = T.mesh_spec([(2, 1.0, 0.0), (2, 1.0, 1.0), (2, 1.0, 0.0)], ny=6, nz=2, depth=1.0, partition=partition)
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=1e-3, case=T.density_wave())
    n_el = 2 * 6 * 2 * 3

    def body(s):
        s.set_initial_condition(0.0)
        s.step(0.004, 5)
        return s.local_element_ids(), s.field()

    ref = capi.gather_global(capi.run_inproc(mesh, cfg, 1, body, hub="r1"), n_el, 4)
    got = capi.gather_global(capi.run_inproc(mesh, cfg, ranks, body, hub=f"r{ranks}p{partition}"), n_el, 4)
    assert not np.isnan(got).any()
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("bands,ranks,partition", [
    ([(8, 1.0, 0.0)], 2, T.PARTITION_LEX),
    ([(6, 1.0, 0.0), (6, 1.0, 0.3), (6, 1.0, 0.0)], 3, T.PARTITION_LEX),
    ([(6, 1.0, 0.0), (6, 1.0, 0.3), (6, 1.0, 0.0)], 6, T.PARTITION_SFC),
    ([(5, 1.0, 0.0), (7, 1.0, 0.3)], 4, T.PARTITION_LEX)])
@pytest.mark.parametrize("mu", [0.0, 1e-3])
def test_exchange_overlap_keeps_the_bits(bands, ranks, partition, mu):
    """SURVEY §8(e) overlap: the interior element run is computed while the halo round is in
    flight (comm stream), the boundary ranges after the join.  Ranks with a non-empty
    interior run must still reproduce the single-rank bits, viscous and inviscid."""
    from paper_2008_04356_b200 import capi
    mesh = T.mesh_spec(bands, ny=4, nz=2, depth=1.0, partition=partition)
    assert all(capi.plan(mesh, ranks, r)["interior_run"][1] > capi.plan(mesh, ranks, r)["interior_run"][0]
               for r in range(ranks))
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=mu, case=T.density_wave())
    n_el = sum(b[0] for b in bands) * 4 * 2

    def body(s):
        s.set_initial_condition(0.0)
        s.step(0.004, 5)
        return s.local_element_ids(), s.field()

    ref = capi.gather_global(capi.run_inproc(mesh, cfg, 1, body, hub=f"ov1_{mu}"), n_el, 4)
    got = capi.gather_global(capi.run_inproc(mesh, cfg, ranks, body, hub=f"ov{ranks}_{partition}_{mu}"), n_el, 4)
    assert not np.isnan(got).any()
    assert np.array_equal(got, ref)


def test_communication_audit_passes_and_catches_injected_collective():
    """audit_communication (audit.cpp:44-148) on the traces of a 3-rank run; the
    inject_collective hook (solver.cpp:961-964) must make it fail."""
    from paper_2008_04356_b200 import audit, capi
    mesh = T.mesh_spec([(2, 1.0, 0.0), (2, 1.0, 1.0), (2, 1.0, 0.0)], ny=6, nz=2, depth=1.0)
    cfg = T.solver_config(2, T.NODES_GAUSS, mu=1e-3, case=T.density_wave())

    def clean(s):
        s.set_initial_condition(0.0)
        s.step(0.004, 2)
        return s.trace()

    def dirty(s):
        s.set_initial_condition(0.0)
        s.step(0.004, 1)
        s.inject_collective()
        return s.trace()

    rep = audit.audit(capi.run_inproc(mesh, cfg, 3, clean, hub="audit3"), mesh)
    assert rep["passed"], rep["violations"]
    assert rep["init_collective_sends"] == 3 * 2 and rep["post_init_collectives"] == 0
    assert rep["data_messages"] > 0
    bad = audit.audit(capi.run_inproc(mesh, cfg, 3, dirty, hub="audit3b"), mesh)
    assert not bad["passed"] and bad["post_init_collectives"] > 0


def test_baseline_config0_ten_steps():
    """BASELINE.json configs[0] in full: [0,2]^3 split at the interface into two
    4x4x4 blocks, upper block +0.5 along the slide, N=3 Gauss, mu=1e-3, Dirichlet
    across the split, periodic otherwise, rho = 2 + 0.1 sin(pi(x+y+z)), u=v=w=1,
    p=1, 10 low-storage RK steps at CFL 0.5 (axes relabelled, include/sdg_types.h)."""
    mesh = box0(4)
    cfg = T.solver_config(3, T.NODES_GAUSS, gamma=1.4, R=1.0, mu=1e-3, Pr=0.72, case=T.density_wave())
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    g.set_initial_condition(0.0)
    o.set_initial_condition(0.0)
    dt = o.suggest_dt(0.5)
    assert abs(g.suggest_dt(0.5) - dt) <= 1e-14 * dt
    g.step(dt, 10)
    o.step(dt, 10)
    assert g.n_elements == 128
    assert rel_linf(g.field(), o.field()) <= 1e-10
    assert g.total_rebuilds() == o.total_rebuilds()
    d = g.diagnostics(g.time())
    me = o.mass_energy(o.field())
    assert abs(d["mass"] - me[0]) <= 1e-12 * me[0]


@pytest.mark.parametrize("degree,nx,nyz", [(3, 6, 14), (5, 4, 8)])
def test_multi_wave_meshes_match_oracle(degree, nx, nyz):
    """Meshes with several times more element tiles than resident CTAs, so the
    persistent kernels process neighbours in different waves: a neighbour must
    still see this stage's traces (double-buffered trace slots)."""
    mesh = T.mesh_spec([(nx, 1.0, 0.0), (nx, 1.0, 0.7), (nx, 1.0, 0.0)], ny=nyz, nz=nyz)
    cfg = T.solver_config(degree, T.NODES_GAUSS, mu=1e-3, case=T.density_wave())
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    g.set_initial_condition(0.0)
    o.set_initial_condition(0.0)
    dt = o.suggest_dt(0.5)
    g.step(dt, 3)
    o.step(dt, 3)
    assert rel_linf(g.field(), o.field()) <= 1e-12


# ---------------------------------------------------------------- RK-stage and interface entry points
def test_rk_stages_equal_one_step_bitwise():
    """sdg_rk_stage x5 (lsrk_step, lsrk.hpp:20-21) is bitwise sdg_step, and the
    oracle's step agrees; stages out of order or at the wrong time are refused."""
    from paper_2008_04356_b200 import capi
    mesh = three_band(ny=4, nz=2, vg=0.7)
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=1e-3, case=T.density_wave())
    a, b = gpu_solver(mesh, cfg), gpu_solver(mesh, cfg)
    a.set_initial_condition(0.1)
    b.set_initial_condition(0.1)
    dt = a.suggest_dt(0.5)
    for step in range(3):
        a.step(dt)
        t = b.time()
        for s in range(5):
            b.rk_stage(s, t, dt)
        assert b.time() == a.time() and b.step_index() == a.step_index() == step + 1
    assert np.array_equal(a.field(), b.field())
    assert np.array_equal(a.register(), b.register())
    assert a.total_rebuilds() == b.total_rebuilds()
    with pytest.raises(T.ConfigError):
        b.rk_stage(1, b.time(), dt)
    with pytest.raises(T.ConfigError):
        b.rk_stage(0, b.time() + dt, dt)
    b.rk_stage(0, b.time(), dt)
    with pytest.raises(T.ConfigError):
        b.step(dt)  # an unfinished step


@pytest.mark.parametrize("t", [0.0, 0.13, 0.5, 1.71])
def test_update_interfaces_matches_oracle_and_reference(t):
    """sdg_update_interfaces (solver.cpp:156-176): the device displacement / sigma of
    every side context and the host long-double operators equal the oracle's, and
    the operators are the reference library's build_mortar_operators bits."""
    mesh = three_band(ny=4, nz=2, vg=0.7)
    cfg = T.solver_config(3, T.NODES_GAUSS, mu=1e-3, case=T.density_wave())
    g, o = gpu_solver(mesh, cfg), P.Oracle3D(mesh, cfg)
    g.set_initial_condition(0.0)
    o.set_initial_condition(0.0)
    ops = g.update_interfaces(t)
    o.compute_residual(t)  # the oracle updates its interfaces at the stage time
    assert g.n_contexts() == o.n_contexts() == 4
    for c in range(g.n_contexts()):
        gi, oi = g.ctx_info(c), o.ctx_info(c)
        assert gi == oi, (c, gi, oi)
        if not gi["conforming"]:
            f, bwd = P.oracle_mortar_ops(3, T.NODES_GAUSS, gi["sigma_side"])
            assert np.array_equal(ops[c, :2], f) and np.array_equal(ops[c, 2:], bwd)
            if P.ref_available():
                rf, rb = P.ref_mortar_ops(3, T.NODES_GAUSS, gi["sigma_side"])
                assert np.array_equal(ops[c, :2], rf) and np.array_equal(ops[c, 2:], rb)
        assert np.array_equal(g.mapping(c), o.mapping(c))


def test_nccl_transport_calls_run_on_the_device():
    """NCCL itself on the device (the N > 1 data path is checked bitwise on the in-process
    transport; one GPU offers NCCL only the rank itself as a partner): a one-rank communicator
    through every NcclComm method -- init, the all-gathers of init_rank_maps, min and sum
    all-reduces, one grouped send + receive round of 8 MB -- with exact results."""
    from paper_2008_04356_b200 import capi
    capi.nccl_selfcheck(0, 1 << 20)
    capi.nccl_selfcheck(0, 1)
