"""GPU parity of the synchronous path (K1) against the oracle -- bit-exact.

Mirrors proj/tests/test_sync.cpp and acceptance.cpp criteria 4-6, called
through the C-ABI (paper_1510_08982_b200.heat -> libheat_b200.so)."""
import numpy as np
import pytest

from helpers import SplitMix64, bits_equal, fnv1a64, random_field, sine_field

pytestmark = pytest.mark.gpu

DIR, PER = 0, 1


@pytest.fixture(scope="module")
def H(gpu):
    from paper_1510_08982_b200 import heat
    return heat


def test_sync_step_dirichlet_kat(H):
    # test_sync.cpp:31-36
    out = H.sync_step(H.TemperatureField([1.0, 0.0, 0.0]), H.SolverParams.from_r(0.5),
                      H.BoundaryCondition.dirichlet(1.0, 0.0))
    assert list(out.values()) == [1.0, 0.5, 0.0]


def test_sync_step_rejects_mismatched_ends(H):
    # test_sync.cpp:38-43
    with pytest.raises(H.InvalidArgument):
        H.sync_step(H.TemperatureField([0.5, 0.0, 0.0]), H.SolverParams.from_r(0.5),
                    H.BoundaryCondition.dirichlet(1.0, 0.0))


def test_sync_step_periodic_kat(H):
    # test_sync.cpp:45-52
    out = H.sync_step(H.TemperatureField([2.0, 0.0, 1.0]), H.SolverParams.from_r(0.25),
                      H.BoundaryCondition.periodic())
    assert out.values() == pytest.approx([1.25, 0.75, 1.0], rel=1e-15)


def test_recording_stride_and_k0(H):
    # test_sync.cpp:54-70
    u0 = H.cosine_init(10)
    t0 = H.sync_run(u0, H.SolverParams.from_r(0.5), H.BoundaryCondition.dirichlet(1.0, 0.0), 0)
    assert t0.steps == [0] and len(t0.snapshots) == 1
    assert t0.initial()[0] == 1.0 and t0.initial()[9] == 0.0
    t = H.sync_run(u0, H.SolverParams.from_r(0.5), H.BoundaryCondition.dirichlet(1.0, 0.0), 10, 3)
    assert t.steps == [0, 3, 6, 9, 10]


def test_cfg1_golden_hash(H, port):
    # BASELINE configs[0]: N=1024, r=0.25, Dirichlet(0,0), sine IC, 1000 steps.
    u0 = port.prepare_initial(port.sine_init(1024), DIR, 0.0, 0.0)
    fin = H.sync_final(u0, H.SolverParams.from_r(0.25), H.BoundaryCondition.dirichlet(0, 0), 1000)
    assert fnv1a64(fin) == 0xC2C466B7716F830A
    assert fin[512] == 0.99764390050177021


@pytest.mark.parametrize("seed", [20260824, 555, 77])
def test_random_small_trajectories_bit_exact(H, port, seed):
    # acceptance.cpp:67-99 style: N in [3, 63], r in (0, 0.5], both BCs, stride 1.
    gen = SplitMix64(seed)
    for _ in range(25):
        n = 3 + gen.next_bounded(60)
        r = 0.5 * (gen.next_double() * 0.999 + 0.001)
        periodic = gen.next() & 1
        u0 = random_field(gen, n)
        k_end = 1 + gen.next_bounded(120)
        if periodic:
            bc = H.BoundaryCondition.periodic()
        else:
            bc = H.BoundaryCondition.dirichlet(u0[0], u0[-1])
        p = H.SolverParams.from_r(r)
        t = H.sync_run(H.TemperatureField(u0), p, bc, k_end, 1)
        steps, snaps = port.sync_run(u0, p.r(), bc.kind, bc.c1, bc.c2, k_end, 1, record=True)
        assert t.steps == steps
        for j, s in enumerate(t.snapshots):
            assert bits_equal(s.values(), snaps[j]), (n, r, periodic, k_end, j)


@pytest.mark.parametrize("n", [959, 960, 961, 1024, 1921, 4097, 30000, 65536 + 7, 1 << 20])
@pytest.mark.parametrize("bc", [DIR, PER])
def test_tile_boundaries_bit_exact(H, port, n, bc):
    # N straddling warp-tile sizes (30*32 = 960 points per tile), odd sizes,
    # and a 2^20 field; K crosses several 32-step passes plus a remainder.
    gen = SplitMix64(n * 31 + bc)
    u0 = random_field(gen, n)
    b = H.BoundaryCondition.periodic() if bc else H.BoundaryCondition.dirichlet(u0[0], u0[-1])
    k = 100 if n <= 65543 else 70
    p = H.SolverParams.from_r(0.4)
    fin = H.sync_final(u0, p, b, k)
    exp = port.sync_run(u0, p.r(), b.kind, b.c1, b.c2, k)
    assert bits_equal(fin, exp)


def test_f32_bit_exact_vs_port(H, port):
    # sync_run_f32 (sync_solver.cpp:87-91) and test_sync.cpp:164-171.
    u0 = H.cosine_init(100)
    p = H.SolverParams.from_r(0.5)
    bc = H.BoundaryCondition.dirichlet(1.0, 0.0)
    f32 = H.sync_run_f32(u0, p, bc, 2000, 2000)
    exp = port.sync_run_f32(u0.values(), p.r(), 0, 1.0, 0.0, 2000)
    assert bits_equal(f32.final().values(), exp)
    f64 = H.sync_run(u0, p, bc, 2000, 2000)
    assert np.max(np.abs(f64.final().values() - f32.final().values())) <= 1e-3
    gen = SplitMix64(9)
    u = random_field(gen, 5000)
    pb = H.BoundaryCondition.periodic()
    got = H.sync_run_f32(H.TemperatureField(u), H.SolverParams.from_r(0.3), pb, 77, 77)
    assert bits_equal(got.final().values(), port.sync_run_f32(u, 0.3, 1, 0, 0, 77))


@pytest.mark.parametrize("periodic", [False, True])
def test_f32_large_bit_exact_vs_port(H, port, periodic):
    # many K1 f32 tiles (64-point lanes), two full passes and a partial one
    n = (1 << 20) + 777
    gen = SplitMix64(31 + periodic)
    u = random_field(gen, n)
    c1, c2 = (0.0, 0.0) if periodic else (float(u[0]), float(u[-1]))
    bc = H.BoundaryCondition.periodic() if periodic else H.BoundaryCondition.dirichlet(c1, c2)
    got = H.sync_run_f32(H.TemperatureField(u), H.SolverParams.from_r(0.45), bc, 150, 150)
    exp = port.sync_run_f32(u, 0.45, 1 if periodic else 0, c1, c2, 150)
    assert bits_equal(got.final().values(), exp)


def test_divergence_errors(H):
    # test_sync.cpp:151-162 (strict) and the TemperatureField ctor (non-strict).
    v = np.zeros(8)
    v[3], v[4] = 1e308, -1e308
    p = H.SolverParams.from_r(100.0, True)
    bc = H.BoundaryCondition.dirichlet(0.0, 0.0)
    H.set_strict_finite_checks(True)
    try:
        with pytest.raises(H.DivergenceError):
            H.sync_run(H.TemperatureField(v), p, bc, 50, 1)
    finally:
        H.set_strict_finite_checks(False)
    with pytest.raises(H.DomainError):
        H.sync_run(H.TemperatureField(v), p, bc, 50, 50)


def test_unstable_r_diverges(H):
    # test_sync.cpp:128-138
    v = np.zeros(32)
    v[1:-1] = [(-1.0 if i % 2 == 0 else 1.0) for i in range(1, 31)]
    t = H.sync_run(H.TemperatureField(v), H.SolverParams.from_r(0.6, True),
                   H.BoundaryCondition.dirichlet(0, 0), 100, 1)
    assert max(np.max(np.abs(s.values())) for s in t.snapshots) > 10.0


def test_periodic_conservation_and_steady_state(H):
    # test_sync.cpp:72-106 (long runs reach steady state / conserve heat)
    u0 = H.cosine_init(100)
    t = H.sync_run(u0, H.SolverParams.from_r(0.5), H.BoundaryCondition.dirichlet(1.0, 0.0),
                   100000, 100000)
    steady = H.linear_steady_state(100, 1.0, 0.0)
    assert np.max(np.abs(t.final().values() - steady.values())) <= 1e-6
    mean = H.total_heat(u0) / 100.0
    t = H.sync_run(u0, H.SolverParams.from_r(0.45), H.BoundaryCondition.periodic(), 100000,
                   100000)
    assert np.max(np.abs(t.final().values() - mean)) <= 1e-6


def test_sine_1k_matches_helper(port):
    # the sine IC helper agrees bit-for-bit with the oracle's libm sin
    assert bits_equal(sine_field(1024), port.prepare_initial(port.sine_init(1024), 0, 0.0, 0.0))


@pytest.mark.parametrize("periodic", [False, True])
def test_large_trajectory_overlapped_snapshots(H, periodic):
    # N >= 2^20 with a trajectory: snapshots staged device-to-device and
    # downloaded on the copy stream while the next segment computes
    # (sync_run_overlapped); every row must equal an independent run to its step
    n = (1 << 20) + 333
    gen = SplitMix64(77 + periodic)
    u = random_field(gen, n)
    c1, c2 = (0.0, 0.0) if periodic else (float(u[0]), float(u[-1]))
    bc = H.BoundaryCondition.periodic() if periodic else H.BoundaryCondition.dirichlet(c1, c2)
    p = H.SolverParams.from_r(0.41)
    t = H.sync_run(H.TemperatureField(u), p, bc, 250, 64)
    assert t.steps == [0, 64, 128, 192, 250]
    assert bits_equal(t.snapshots[0].values(), u)  # the prepared field (ends already exact)
    for k, snap in zip(t.steps[1:], t.snapshots[1:]):
        assert bits_equal(snap.values(), H.sync_final(u, p, bc, k)), k
