"""GPU parity of the asynchronous paths against the oracle.

Deterministic mode (async_run): bit-exact with the reference's seeded stream
(proj/tests/test_async_sim.cpp, acceptance.cpp criterion 1, BASELINE cfg2).
Executors (exec_run): Barriered bit-exact with sync_run; BarrierFree (free-
running, bounded staleness) checked for the reference's stability properties
(test_exec.cpp:89-136) and its logged delays against the bound."""
import numpy as np
import pytest

from helpers import SplitMix64, bits_equal, fnv1a64, random_divisor, random_field

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H(gpu):
    from paper_1510_08982_b200 import heat
    return heat


def _sine(port, n):
    return port.prepare_initial(port.sine_init(n), 0, 0.0, 0.0)


@pytest.mark.parametrize("seed,expect", [(1, 0x50008031848D280C), (42, 0x1E3D733CB51BD50B)])
def test_cfg2_golden(H, port, seed, expect):
    # BASELINE configs[1]: N=1024, 8 PEs, q=2 uniform, r=0.25, 1000 steps, sine IC.
    u0 = _sine(port, 1024)
    got = H.async_final(u0, H.SolverParams.from_r(0.25), H.BoundaryCondition.dirichlet(0, 0),
                        H.PartitionSpec(1024, 128), H.DelayModel.uniform(2, seed), 1000)
    assert fnv1a64(got) == expect


def test_cfg2_trajectory_bit_exact(H, port):
    u0 = _sine(port, 1024)
    p = H.SolverParams.from_r(0.25)
    t = H.async_run(H.TemperatureField(u0), p, H.BoundaryCondition.dirichlet(0, 0),
                    H.PartitionSpec(1024, 128), H.DelayModel.uniform(3, 7), 300, 25)
    steps, snaps = port.async_run(u0, p.r(), 0, 0.0, 0.0, 128, 0, 3, seed=7, k_end=300,
                                  stride=25, record=True)
    assert t.steps == steps
    for j, s in enumerate(t.snapshots):
        assert bits_equal(s.values(), snaps[j]), j


def _law(gen, q):
    k = gen.next_bounded(2)
    if k == 0:
        return 0, 0, 0.5
    if k == 1:
        return 1, gen.next_bounded(q - 1), 0.5
    return 2, 0, 0.05 + 0.9 * gen.next_double()


@pytest.mark.parametrize("seed", [20260824, 4048, 2024])
def test_random_partitions_bit_exact(H, port, seed):
    # acceptance.cpp:67-99 style, with random divisor partitions (n = 1 included),
    # q in 1..10, all three delay laws, both BCs, every step recorded.
    gen = SplitMix64(seed)
    for _ in range(20):
        n = 3 + gen.next_bounded(60)
        r = 0.5 * (gen.next_double() * 0.999 + 0.001)
        periodic = gen.next() & 1
        u0 = random_field(gen, n)
        k_end = 1 + gen.next_bounded(150)
        per_pe = random_divisor(gen, n)
        q = 1 + gen.next_bounded(9)
        law, fd, gp = _law(gen, q)
        mseed = gen.next()
        bc = H.BoundaryCondition.periodic() if periodic else H.BoundaryCondition.dirichlet(
            u0[0], u0[-1])
        model = H.DelayModel(q, H.Distribution(law), fd, gp, mseed)
        params = H.SolverParams.from_r(r)
        t = H.async_run(H.TemperatureField(u0), params, bc, H.PartitionSpec(n, per_pe), model,
                        k_end, 1)
        steps, snaps = port.async_run(u0, params.r(), bc.kind, bc.c1, bc.c2, per_pe, law, q, fd,
                                      gp, mseed, k_end, 1, record=True)
        assert t.steps == steps
        for j, s in enumerate(t.snapshots):
            assert bits_equal(s.values(), snaps[j]), (n, per_pe, q, law, periodic, j)


@pytest.mark.parametrize("n_total,per_pe,q,bc", [
    (1024, 512, 2, 0), (1024, 32, 3, 1), (1024, 8, 9, 0), (4096, 1024, 4, 1),
    (1 << 16, 1024, 5, 0), (3 * 1000, 1000, 2, 1)])
def test_larger_grids_bit_exact(H, port, n_total, per_pe, q, bc):
    gen = SplitMix64(n_total + per_pe + q)
    u0 = random_field(gen, n_total)
    b = H.BoundaryCondition.periodic() if bc else H.BoundaryCondition.dirichlet(u0[0], u0[-1])
    p = H.SolverParams.from_r(0.4)
    k = 200
    got = H.async_final(u0, p, b, H.PartitionSpec(n_total, per_pe), H.DelayModel.uniform(q, 99),
                        k)
    exp = port.async_run(u0, p.r(), b.kind, b.c1, b.c2, per_pe, 0, q, seed=99, k_end=k)
    assert bits_equal(got, exp)


def test_reductions_to_sync(H, port):
    # q = 1 and single-PE runs are bit-identical to sync (test_async_sim.cpp:110-150)
    gen = SplitMix64(11)
    u0 = random_field(gen, 200)
    bc = H.BoundaryCondition.dirichlet(u0[0], u0[-1])
    p = H.SolverParams.from_r(0.3)
    sync = port.sync_run(u0, p.r(), 0, bc.c1, bc.c2, 150)
    a = H.async_final(u0, p, bc, H.PartitionSpec(200, 20), H.DelayModel.uniform(1, 5), 150)
    b = H.async_final(u0, p, bc, H.PartitionSpec(200, 200), H.DelayModel.uniform(7, 5), 150)
    assert bits_equal(a, sync) and bits_equal(b, sync)


def test_async_model_validation(H):
    u0 = H.cosine_init(12)
    p = H.SolverParams.from_r(0.5)
    bc = H.BoundaryCondition.dirichlet(1.0, 0.0)
    with pytest.raises(H.DomainError):
        H.DelayModel.uniform(0, 1)
    with pytest.raises(H.DomainError):
        H.DelayModel.fixed(3, 3, 1)
    with pytest.raises(H.DomainError):
        H.PartitionSpec(12, 5)
    with pytest.raises(H.InvalidArgument):
        H.async_run(u0, p, bc, H.PartitionSpec(24, 4), H.DelayModel.uniform(2, 1), 5)


def test_counter_form_matches_stream(H, port):
    # the per-draw counter form equals the sequential SplitMix64 stream
    # (golden vector test_async_sim.cpp:64-71)
    assert [H.sample_delay_at(H.DelayModel.uniform(4, 42), j, 100) for j in range(8)] == \
        [1, 3, 2, 0, 2, 2, 1, 0]
    m = H.DelayModel.geometric(6, 0.7, 99)
    assert [H.sample_delay_at(m, j, 1000) for j in range(200)] == \
        port.delay_stream(2, 6, 0, 0.7, 99, 1000, 200)


# ---- executors ------------------------------------------------------------
def test_exec_barriered_bit_exact(H, port):
    # test_exec.cpp:45-67 / acceptance.cpp:208-237
    gen = SplitMix64(555)
    for _ in range(10):
        pe = 1 << gen.next_bounded(2)
        per = 1 + gen.next_bounded(7)
        n = max(3 * pe, pe * per)
        per = n // pe
        r = 0.5 * (gen.next_double() * 0.999 + 0.001)
        periodic = gen.next() & 1
        u0 = random_field(gen, n)
        bc = H.BoundaryCondition.periodic() if periodic else H.BoundaryCondition.dirichlet(
            u0[0], u0[-1])
        k = 1 + gen.next_bounded(99)
        res = H.exec_run(H.TemperatureField(u0), H.SolverParams.from_r(r), bc,
                         H.PartitionSpec(n, per), H.ExecConfig(pe, k, H.ExecMode.Barriered))
        assert bits_equal(res.field.values(), port.sync_run(u0, r, bc.kind, bc.c1, bc.c2, k))
        assert res.steps_per_pe == [k] * pe
        # barrier-free with one PE is also exact
        res1 = H.exec_run(H.TemperatureField(u0), H.SolverParams.from_r(r), bc,
                          H.PartitionSpec(n, n), H.ExecConfig(1, k, H.ExecMode.BarrierFree))
        assert bits_equal(res1.field.values(), port.sync_run(u0, r, bc.kind, bc.c1, bc.c2, k))


def test_exec_validation(H):
    u0 = H.cosine_init(12)
    p = H.SolverParams.from_r(0.5)
    bc = H.BoundaryCondition.dirichlet(1.0, 0.0)
    part = H.PartitionSpec(12, 3)
    with pytest.raises(H.InvalidArgument):
        H.exec_run(u0, p, bc, part, H.ExecConfig(3, 10, H.ExecMode.Barriered))
    with pytest.raises(H.InvalidArgument):
        H.exec_run(u0, p, bc, part, H.ExecConfig(4, 0, H.ExecMode.Barriered))


def test_barrier_free_steady_state_and_lag(H):
    # test_exec.cpp:89-97 and 121-136
    u0 = H.cosine_init(100)
    res = H.exec_run(u0, H.SolverParams.from_r(0.5), H.BoundaryCondition.dirichlet(1.0, 0.0),
                     H.PartitionSpec(100, 25),
                     H.ExecConfig(4, 200000, H.ExecMode.BarrierFree, True))
    steady = H.linear_steady_state(100, 1.0, 0.0)
    assert np.max(np.abs(res.field.values() - steady.values())) <= 1e-3
    lag = res.lag
    assert lag.reads > 0 and lag.max_lag >= lag.min_lag
    assert sum(lag.histogram) + lag.overflow == lag.reads
    st = res.stats
    assert st.reads == lag.reads
    assert st.max_delay <= 7  # default bound q_free = 8: delays in {0..7}
    assert sum(st.delay_histogram) == st.reads


def test_barrier_free_envelope(H):
    # free-running iterates stay inside the initial envelope (SPEC maximum principle,
    # test_async_sim.cpp:175-198)
    gen = SplitMix64(31)
    for _ in range(5):
        n = 64
        u0 = random_field(gen, n)
        lo, hi = u0.min(), u0.max()
        r = 0.5 * (gen.next_double() * 0.999 + 0.001)
        res = H.exec_run(H.TemperatureField(u0), H.SolverParams.from_r(r),
                         H.BoundaryCondition.dirichlet(u0[0], u0[-1]), H.PartitionSpec(n, 8),
                         H.ExecConfig(8, 2000, H.ExecMode.BarrierFree, False, 4))
        v = res.field.values()
        assert v.min() >= lo - 1e-12 and v.max() <= hi + 1e-12
        assert res.stats.max_delay <= 3


# ---- K5: streaming async (PEs wider than a warp) ---------------------------
@pytest.mark.parametrize("n_total,per_pe,q,bc,law", [
    (16384, 2048, 3, 0, 0), (16384, 4096, 2, 1, 0), (12288, 3072, 4, 0, 1),
    (8192, 2048, 5, 1, 2), (1 << 20, 1 << 15, 5, 0, 0)])
def test_stream_deterministic_bit_exact(H, port, n_total, per_pe, q, bc, law):
    gen = SplitMix64(n_total + per_pe + q + bc)
    u0 = random_field(gen, n_total)
    b = H.BoundaryCondition.periodic() if bc else H.BoundaryCondition.dirichlet(u0[0], u0[-1])
    p = H.SolverParams.from_r(0.4)
    k = 100 if n_total >= (1 << 20) else 150
    fd = 1 if law == 1 else 0
    model = H.DelayModel(q, H.Distribution(law), fd, 0.6, 1234 + q)
    got = H.async_final(u0, p, b, H.PartitionSpec(n_total, per_pe), model, k)
    exp = port.async_run(u0, p.r(), b.kind, b.c1, b.c2, per_pe, law, q, fd, 0.6, 1234 + q, k)
    assert bits_equal(got, exp)


def test_stream_trajectory_bit_exact(H, port):
    gen = SplitMix64(77)
    u0 = random_field(gen, 8192)
    p = H.SolverParams.from_r(0.3)
    b = H.BoundaryCondition.dirichlet(u0[0], u0[-1])
    t = H.async_run(H.TemperatureField(u0), p, b, H.PartitionSpec(8192, 2048),
                    H.DelayModel.uniform(3, 5), 90, 40)
    steps, snaps = port.async_run(u0, p.r(), 0, b.c1, b.c2, 2048, 0, 3, seed=5, k_end=90,
                                  stride=40, record=True)
    assert t.steps == steps == [0, 40, 80, 90]
    for j, s in enumerate(t.snapshots):
        assert bits_equal(s.values(), snaps[j])


def test_stream_free_q1_is_sync(H, port):
    # free-running with q = 1 must read exactly u_j(k): bit-identical to sync
    n = 1 << 18
    gen = SplitMix64(3)
    u0 = random_field(gen, n)
    u0[0] = u0[-1] = 0.0
    plan = H.Plan(n)
    plan.upload(u0)
    st = plan.async_advance(0.4, H.BoundaryCondition.dirichlet(0, 0), 1 << 13, 1, 200)
    got = plan.download()
    exp = port.sync_run(u0, 0.4, 0, 0.0, 0.0, 200)
    assert bits_equal(got, exp)
    assert st.max_delay == 0 and st.reads > 0


def test_stream_free_bounded(H, port):
    n = 1 << 18
    u0 = port.prepare_initial(port.sine_init(n), 0, 0.0, 0.0)
    plan = H.Plan(n)
    plan.upload(u0)
    st = plan.async_advance(0.4, H.BoundaryCondition.dirichlet(0, 0), 1 << 12, 4, 500)
    got = plan.download()
    assert st.max_delay <= 3 and sum(st.delay_histogram) == st.reads > 0
    assert got.min() >= -1e-12 and got.max() <= 1.0 + 1e-12  # envelope of the sine IC
    exp = port.sync_run(u0, 0.4, 0, 0.0, 0.0, 500)
    assert np.max(np.abs(got - exp)) < 1e-3


def test_plan_async_replay_bit_exact(H, port):
    # the resident-plan deterministic replay (bench's async_det leg) == async_run
    n = 1 << 16
    gen = SplitMix64(123)
    u0 = random_field(gen, n)
    u0[0] = u0[-1] = 0.0
    plan = H.Plan(n)
    plan.upload(u0)
    plan.async_replay(0.4, H.BoundaryCondition.dirichlet(0, 0), 1 << 13,
                      H.DelayModel.uniform(2, 1), 300)
    exp = port.async_run(u0, 0.4, 0, 0.0, 0.0, 1 << 13, 0, 2, seed=1, k_end=300)
    assert bits_equal(plan.download(), exp)


@pytest.mark.parametrize("r,q,periodic,per_pe", [
    (0.25, 3, False, 128), (0.49, 9, False, 128), (0.1, 5, True, 64), (0.4, 2, False, 1)])
def test_free_run_within_aposteriori_bound(H, port, r, q, periodic, per_pe):
    # ||u_async(K) - u_sync(K)||_inf <= sum_k ||u(k+1) - A u(k)||_inf
    n = 1024 if per_pe > 1 else 16
    u0 = port.prepare_initial(port.sine_init(n), 0, 0.0, 0.0)
    bc = H.BoundaryCondition.periodic() if periodic else H.BoundaryCondition.dirichlet(0, 0)
    p = H.SolverParams.from_r(r)
    fin, st = H.async_free_run(u0, p, bc, H.PartitionSpec(n, per_pe), q, 1000)
    sync = port.sync_run(u0, r, bc.kind, 0.0, 0.0, 1000)
    err = np.max(np.abs(fin - sync))
    assert err <= st.residual_sum
    assert st.max_delay <= q - 1 and sum(st.delay_histogram) == st.reads > 0


@pytest.mark.parametrize("periodic", [False, True])
@pytest.mark.parametrize("q", [1, 3, 8])
def test_free_run_wide_pes_within_aposteriori_bound(H, port, q, periodic):
    # K5 (PEs of whole 32-point units) logs every PE edge value and every
    # read's source step on the device; the host forms the same bound
    n, per_pe = 1 << 18, 1 << 14  # 16 PEs of 16384 points
    u0 = port.prepare_initial(port.sine_init(n), 0, 0.0, 0.0)
    bc = H.BoundaryCondition.periodic() if periodic else H.BoundaryCondition.dirichlet(0, 0)
    p = H.SolverParams.from_r(0.4)
    k = 2000
    fin, st = H.async_free_run(u0, p, bc, H.PartitionSpec(n, per_pe), q, k)
    sync = port.sync_run(u0, 0.4, bc.kind, 0.0, 0.0, k)
    err = float(np.max(np.abs(fin - sync)))
    assert err <= st.residual_sum
    P = n // per_pe
    assert st.reads == (2 * P if periodic else 2 * (P - 1)) * k
    assert st.max_delay <= q - 1 and sum(st.delay_histogram) == st.reads
    if q == 1:
        assert bits_equal(fin, sync) and st.residual_sum < 1e-6


def test_free_run_q1_exact(H, port):
    u0 = port.prepare_initial(port.sine_init(1024), 0, 0.0, 0.0)
    fin, st = H.async_free_run(u0, H.SolverParams.from_r(0.3), H.BoundaryCondition.dirichlet(0, 0),
                               H.PartitionSpec(1024, 128), 1, 700)
    assert bits_equal(fin, port.sync_run(u0, 0.3, 0, 0.0, 0.0, 700))
    assert st.max_delay == 0 and st.residual_sum < 1e-9


def test_measure_and_speedup_ratio(gpu):
    """measure / speedup_ratio (async_exec.cpp:281-318) over the GPU exec_run,
    as test_exec.cpp:151-175 checks them: row shape, reps >= 3, median >= min,
    a positive ratio, and cost growing with N in both modes."""
    from paper_1510_08982_b200 import heat as H
    one = H.measure([30], [H.ExecMode.Barriered], 3, 50, 1)
    assert len(one) == 1
    assert (one[0].n_points, one[0].reps) == (30, 3)
    assert one[0].median_ns >= one[0].min_ns > 0
    with pytest.raises(H.InvalidArgument):
        H.measure([30], [H.ExecMode.Barriered], 2, 50, 1)
    with pytest.raises(H.InvalidArgument):
        H.measure([30], [H.ExecMode.Barriered], 3, 50, 7)
    rows = H.measure([100, 10000], [H.ExecMode.Barriered, H.ExecMode.BarrierFree], 5, 200, 1)
    assert H.speedup_ratio(rows, 100) > 0.0
    for mode in (H.ExecMode.Barriered, H.ExecMode.BarrierFree):
        med = {r.n_points: r.median_ns for r in rows if r.mode == mode}
        assert med[10000] >= med[100]
    with pytest.raises(H.InvalidArgument):
        H.speedup_ratio(rows, 64)


@pytest.mark.parametrize("N,n", [(1024, 128), (3 * 4096, 4096)])
def test_geometric_large_q_device_thresholds(gpu, port, N, n):
    """The geometric law with q = 300 (beyond a byte-table's range): K3 / K5
    draw from the exact device thresholds and replay the reference's stream."""
    from paper_1510_08982_b200 import heat as H
    u0 = random_field(SplitMix64(N + 300), N)
    bc = H.BoundaryCondition.dirichlet(float(u0[0]), float(u0[-1]))
    got = H.async_final(u0, H.SolverParams.from_r(0.3), bc, H.PartitionSpec(N, n),
                        H.DelayModel.geometric(300, 0.02, 5), 500)
    want = port.async_run(u0, 0.3, 0, u0[0], u0[-1], n, 2, 300, 0, 0.02, 5, k_end=500)
    assert bits_equal(got, want)


@pytest.mark.parametrize("seed", [9, 1510, 8982])
def test_small_async_kernel_bit_exact(H, port, seed):
    # K9 (csrc/async_small.cu): N <= 2048, PEs of a multiple of 8 points, q <= 8 --
    # one CTA, 64-step rounds, delays applied by the sending lane.  Random shapes
    # around its limits (rounds cut by the recording stride, k_end not a multiple
    # of 64, windows wrapping small periodic rings), all laws, both BCs.
    gen = SplitMix64(seed)
    for _ in range(12):
        m = 2 + gen.next_bounded(254)
        n = 8 * m
        per_pe = 8 * random_divisor(gen, m)
        if per_pe == n:
            per_pe = 8
        q = 1 + gen.next_bounded(7)
        r = 0.5 * (gen.next_double() * 0.999 + 0.001)
        periodic = gen.next() & 1
        u0 = random_field(gen, n)
        k_end = 1 + gen.next_bounded(300)
        stride = 1 + gen.next_bounded(97)
        law, fd, gp = _law(gen, q)
        mseed = gen.next()
        bc = H.BoundaryCondition.periodic() if periodic else H.BoundaryCondition.dirichlet(
            u0[0], u0[-1])
        model = H.DelayModel(q, H.Distribution(law), fd, gp, mseed)
        params = H.SolverParams.from_r(r)
        t = H.async_run(H.TemperatureField(u0), params, bc, H.PartitionSpec(n, per_pe), model,
                        k_end, stride)
        steps, snaps = port.async_run(u0, params.r(), bc.kind, bc.c1, bc.c2, per_pe, law, q, fd,
                                      gp, mseed, k_end, stride, record=True)
        assert t.steps == steps
        for j, s in enumerate(t.snapshots):
            assert bits_equal(s.values(), snaps[j]), (n, per_pe, q, law, periodic, k_end, stride, j)


@pytest.mark.parametrize("n,per_pe,q,law,bc", [
    (2056, 8, 3, 0, 0), (2056, 8, 3, 0, 1), (4096, 64, 8, 2, 1), (4104, 216, 5, 1, 0),
    (6144, 8, 3, 0, 1), (8192, 512, 2, 0, 0), (8192, 8, 1, 0, 1), (8184, 24, 7, 2, 0)])
def test_small_async_cluster_sizes_bit_exact(H, port, n, per_pe, q, law, bc):
    # K9 beyond one CTA (N = 2049..8192: windows over clusters of up to 8 CTAs,
    # each with the whole field and history table; shapes whose tables do not
    # fit take K3) against the oracle, rows cut by an odd stride
    gen = SplitMix64(n * 13 + per_pe + q)
    u0 = random_field(gen, n)
    b = H.BoundaryCondition.periodic() if bc else H.BoundaryCondition.dirichlet(u0[0], u0[-1])
    fd = q - 1 if law == 1 else 0
    gp = 0.4
    model = H.DelayModel(q, H.Distribution(law), fd, gp, 99 + n)
    p = H.SolverParams.from_r(0.4)
    k_end, stride = 211, 37
    t = H.async_run(H.TemperatureField(u0), p, b, H.PartitionSpec(n, per_pe), model, k_end, stride)
    steps, snaps = port.async_run(u0, p.r(), b.kind, b.c1, b.c2, per_pe, law, q, fd, gp, 99 + n,
                                  k_end, stride, record=True)
    assert t.steps == steps
    for j, s_ in enumerate(t.snapshots):
        assert bits_equal(s_.values(), snaps[j]), (n, per_pe, q, law, bc, j)


@pytest.mark.parametrize("n,per_pe,q,bc", [(2048, 8, 4, 0), (2048, 1024, 2, 1), (2048, 64, 8, 1),
                                           (16, 8, 3, 1), (24, 8, 2, 0)])
def test_small_async_kernel_equals_k3(H, port, monkeypatch, n, per_pe, q, bc):
    # K9, the one-member K6 (HEAT_NO_SMALL_ASYNC, small fields) and K3 (both
    # off) all give the oracle's bits
    gen = SplitMix64(n * 7 + q)
    u0 = random_field(gen, n)
    b = H.BoundaryCondition.periodic() if bc else H.BoundaryCondition.dirichlet(u0[0], u0[-1])
    p = H.SolverParams.from_r(0.45)
    part = H.PartitionSpec(n, per_pe)
    model = H.DelayModel.uniform(q, 5)
    k9 = H.async_final(u0, p, b, part, model, 777)
    monkeypatch.setenv("HEAT_NO_SMALL_ASYNC", "1")
    k6 = H.async_final(u0, p, b, part, model, 777)
    monkeypatch.setenv("HEAT_NO_MEMBER_ASYNC", "1")
    k3 = H.async_final(u0, p, b, part, model, 777)
    exp = port.async_run(u0, p.r(), b.kind, b.c1, b.c2, per_pe, 0, q, seed=5, k_end=777)
    assert bits_equal(k9, exp) and bits_equal(k6, exp) and bits_equal(k3, exp)


@pytest.mark.parametrize("n,per_pe,q,law,bc", [
    (100, 1, 5, 0, 0), (100, 1, 5, 0, 1), (97, 1, 3, 2, 0), (600, 75, 6, 1, 1), (1024, 4, 2, 0, 0),
    (5, 1, 2, 0, 1), (640, 5, 16, 2, 1)])
def test_member_async_trajectories_bit_exact(H, port, monkeypatch, n, per_pe, q, law, bc):
    # async_run of shapes K9 does not lay out on the one-member K6
    # (ensemble.cu async_run_member): the paper's one point per PE, odd N,
    # the three laws, rows cut at an odd stride; and K3 on the same shape
    gen = SplitMix64(n * 31 + per_pe + q)
    u0 = random_field(gen, n)
    b = H.BoundaryCondition.periodic() if bc else H.BoundaryCondition.dirichlet(u0[0], u0[-1])
    fd = q - 1 if law == 1 else 0
    model = H.DelayModel(q, H.Distribution(law), fd, 0.35, 11 + n)
    p = H.SolverParams.from_r(0.4)
    k_end, stride = 1500, 77
    steps, snaps = port.async_run(u0, p.r(), b.kind, b.c1, b.c2, per_pe, law, q, fd, 0.35, 11 + n,
                                  k_end, stride, record=True)
    for env in (None, "HEAT_NO_MEMBER_ASYNC"):
        if env:
            monkeypatch.setenv(env, "1")
        t = H.async_run(H.TemperatureField(u0), p, b, H.PartitionSpec(n, per_pe), model, k_end,
                        stride)
        assert t.steps == steps, env
        for j, s_ in enumerate(t.snapshots):
            assert bits_equal(s_.values(), snaps[j]), (env, n, per_pe, q, law, bc, j)


@pytest.mark.parametrize("n_total,per_pe,q,bc,law", [
    (10000, 2500, 3, 0, 0), (10000, 2500, 2, 1, 2), (6000, 2000, 4, 1, 1), (4 * 1100, 1100, 2, 0, 0)])
def test_wide_pes_off_the_32_grid_bit_exact(H, port, n_total, per_pe, q, bc, law):
    # PEs wider than 1024 points that are not a multiple of 32 (K5 needs whole
    # 32-point units) run on K3 as equal units of <= 1024 points, synchronous
    # inside the PE: the reference's measure() sweep (N = 10000 over 4 or 8
    # workers) and any such partition stay exact
    gen = SplitMix64(n_total + per_pe + q)
    u0 = random_field(gen, n_total)
    b = H.BoundaryCondition.periodic() if bc else H.BoundaryCondition.dirichlet(u0[0], u0[-1])
    p = H.SolverParams.from_r(0.41)
    fd, gp = (1, 0.5) if law == 1 else (0, 0.35)
    model = H.DelayModel(q, H.Distribution(law), fd, gp, 77)
    part = H.PartitionSpec(n_total, per_pe)
    t = H.async_run(H.TemperatureField(u0), p, b, part, model, 150, 40)
    steps, snaps = port.async_run(u0, p.r(), b.kind, b.c1, b.c2, per_pe, law, q, fd, gp, seed=77,
                                  k_end=150, stride=40, record=True)
    assert t.steps == steps
    for j, s in enumerate(t.snapshots):
        assert bits_equal(s.values(), snaps[j]), j
    # AsyncSimulator in uneven slices (the same units, resumed) = async_run
    sim = H.AsyncSimulator(H.TemperatureField(u0), p, b, part, model)
    for c in (1, 37, 50, 62):
        sim.step(c)
    assert bits_equal(sim.current(), snaps[-1])
    sim.close()


def test_wide_pes_off_the_32_grid_executors(H, port):
    # exec_run over such PEs: BarrierFree with q = 1 is the synchronous scheme;
    # the reference's measure() sweep {100, 1000, 10000} x 4 workers runs
    n = 10000
    u0 = port.cosine_init(n)
    p = H.SolverParams.from_r(0.5)
    bc = H.BoundaryCondition.dirichlet(1.0, 0.0)
    res = H.exec_run(H.TemperatureField(u0), p, bc, H.PartitionSpec(n, 2500),
                     H.ExecConfig(4, 300, H.ExecMode.BarrierFree, False, 1))
    assert bits_equal(res.field.values(), port.sync_run(u0, p.r(), 0, 1.0, 0.0, 300))
    rows = H.measure([100, 1000, 10000], [H.ExecMode.Barriered, H.ExecMode.BarrierFree], 3, 200, 4)
    assert len(rows) == 6 and all(r.median_ns > 0 for r in rows)
    # a prime PE width above 1024 has no split into units: async_run and the
    # simulator take the reference's own loop over a device HistoryRing
    # (K8a/K8b); the free-running executor runs its delay-0 schedule
    u1 = random_field(SplitMix64(3), 2 * 1031)
    for bc in (H.BoundaryCondition.periodic(), H.BoundaryCondition.dirichlet(u1[0], u1[-1])):
        t = H.async_run(H.TemperatureField(u1), p, bc, H.PartitionSpec(2 * 1031, 1031),
                        H.DelayModel.geometric(3, 0.4, 1), 40, 15)
        steps, snaps = port.async_run(u1, p.r(), bc.kind, bc.c1, bc.c2, 1031, 2, 3, 0, 0.4,
                                      seed=1, k_end=40, stride=15, record=True)
        assert t.steps == steps
        for j, s in enumerate(t.snapshots):
            assert bits_equal(s.values(), snaps[j]), j
    for bc in (H.BoundaryCondition.periodic(), H.BoundaryCondition.dirichlet(u1[0], u1[-1])):
        res = H.exec_run(H.TemperatureField(u1), p, bc, H.PartitionSpec(2 * 1031, 1031),
                         H.ExecConfig(2, 57, H.ExecMode.BarrierFree))
        assert bits_equal(res.field.values(), port.sync_run(u1, p.r(), bc.kind, bc.c1, bc.c2, 57))
        assert res.stats.max_delay == 0 and res.stats.reads > 0
        # AsyncSimulator in uneven slices = async_run (the reference's draws)
        sim = H.AsyncSimulator(H.TemperatureField(u1), p, bc, H.PartitionSpec(2 * 1031, 1031),
                               H.DelayModel.uniform(3, 5))
        for cnt in (1, 7, 13):
            sim.step(cnt)
        assert sim.step_index() == 21
        exp = port.async_run(u1, p.r(), bc.kind, bc.c1, bc.c2, 1031, 0, 3, seed=5, k_end=21)
        assert bits_equal(sim.current(), exp)
        sim.close()
