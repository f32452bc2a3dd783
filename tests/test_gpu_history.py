"""HistoryRing in HBM and async_step on the GPU (csrc/history.cu, kernels
K8a/K8b) against the oracle:

* the ring's read contract (test_async_sim.cpp:95-108);
* async_step over arbitrary rings (random step, depth, partition, BC, law and
  stream position): the field bit-exact, the status, and the SplitMix64
  state after the call -- D draws for a completed step, only through the
  failing draw when a delay reaches past the ring (logic_error);
* HistoryRing(q, prepare_initial(u0)) + K x push_async_step is async_run(K)
  (AsyncSimulator::step, async_sim.cpp:136-140), up to a 2^20-point field;
* the reference's errors: partition mismatch, DelayModel / PartitionSpec
  domain errors, strict finite checks (DivergenceError, ring unchanged)."""
import numpy as np
import pytest

from helpers import SplitMix64, async_step_cases, bits_equal, random_field

pytestmark = pytest.mark.gpu

GAMMA = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


@pytest.fixture(scope="module")
def H(gpu):
    from paper_1510_08982_b200 import heat
    return heat


def test_history_ring_read_contract(H):
    ring = H.HistoryRing(3, [1.0, 2.0, 3.0])
    assert ring.read(1, 0) == 2.0
    with pytest.raises(H.LogicError):
        ring.read(1, 1)  # d > k
    ring.push([4.0, 5.0, 6.0])
    assert ring.current_step() == 1
    assert ring.read(0, 0) == 4.0
    assert ring.read(0, 1) == 1.0
    ring.push([7.0, 8.0, 9.0])
    ring.push([10.0, 11.0, 12.0])
    assert ring.read(2, 0) == 12.0
    assert ring.read(2, 2) == 6.0
    with pytest.raises(H.LogicError):
        ring.read(0, 3)  # d >= q
    with pytest.raises(H.LogicError):
        ring.push([1.0, 2.0])  # size mismatch
    assert list(ring.snapshot(1)) == [7.0, 8.0, 9.0]
    assert (ring.depth(), ring.grid_size()) == (3, 3)
    with pytest.raises(H.DomainError):
        H.HistoryRing(0, [1.0, 2.0, 3.0])
    with pytest.raises(H.DomainError):
        H.HistoryRing(2, [1.0, 2.0])
    ring.close()


def _ring_at(H, c):
    return H.HistoryRing.at_step(c["depth"], c["step"], c["snaps"])


def _model(H, c):
    return H.DelayModel(c["q"], H.Distribution(c["law"]), c["fixed_d"], c["p"], 0)


def _bc(H, c):
    return H.BoundaryCondition.periodic() if c["bc"] else H.BoundaryCondition.dirichlet(c["c1"], c["c2"])


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_async_step_matches_oracle(H, port, seed):
    errors = 0
    for c in async_step_cases(seed, 60):
        sp, fp, rp = port.async_step(**c)
        ring = _ring_at(H, c)
        rng = H.SplitMix64(c["rng_state"])
        params = H.SolverParams.from_r(c["r"])
        part = H.PartitionSpec(c["part_total"], c["per_pe"])
        if sp == 3:
            with pytest.raises(H.LogicError):
                H.async_step(ring, params, _bc(H, c), part, _model(H, c), rng)
            errors += 1
        else:
            assert sp == 0
            got = H.async_step(ring, params, _bc(H, c), part, _model(H, c), rng)
            assert bits_equal(got.values(), fp)
        assert rng.state == rp
        assert ring.current_step() == c["step"]  # async_step leaves the ring alone
        ring.close()
    assert errors > 0


@pytest.mark.parametrize("N,n,law,q", [(1024, 128, 0, 2), (1024, 128, 2, 4), (300, 1, 0, 3),
                                       (4096, 4096, 0, 3), (3 * 4096, 4096, 1, 4),
                                       (1 << 20, 1 << 14, 0, 3)])
@pytest.mark.parametrize("periodic", [False, True])
def test_push_async_step_is_async_run(H, port, N, n, law, q, periodic):
    gen = SplitMix64(N + n + law + periodic)
    u0 = random_field(gen, N)
    c1, c2 = (0.0, 0.0) if periodic else (float(u0[0]), float(u0[-1]))
    bc = H.BoundaryCondition.periodic() if periodic else H.BoundaryCondition.dirichlet(c1, c2)
    seed = 777 + N
    model = H.DelayModel(q, H.Distribution(law), 1 if law == 1 else 0, 0.6, seed)
    params = H.SolverParams.from_r(0.4)
    part = H.PartitionSpec(N, n)
    ring = H.HistoryRing(q, H.prepare_initial(H.TemperatureField(u0), bc))
    rng = H.SplitMix64(seed)
    K = 12 if N >= 1 << 20 else 40
    for _ in range(K):
        ring.push_async_step(params, bc, part, model, rng)
    assert ring.current_step() == K
    want = port.async_run(u0, 0.4, int(periodic), c1, c2, n, law, q, model.fixed_delay, 0.6, seed,
                          k_end=K)
    assert bits_equal(ring.snapshot(0), want)
    P = N // n
    D = 0 if P == 1 else (2 * P if periodic else (2 * (N - 2) if n == 1 else 2 * (P - 1)))
    assert rng.state == (seed + K * D * GAMMA) & M64
    ring.close()


def test_async_step_errors(H):
    u = np.linspace(0.0, 1.0, 64)
    ring = H.HistoryRing(2, u)
    params = H.SolverParams.from_r(0.4)
    bc = H.BoundaryCondition.dirichlet(0.0, 1.0)
    rng = H.SplitMix64(5)
    with pytest.raises(H.InvalidArgument):  # async_sim.cpp:113-114
        H.async_step(ring, params, bc, H.PartitionSpec(32, 8), H.DelayModel.uniform(2, 0), rng)
    assert rng.state == 5
    with pytest.raises(H.DomainError):
        H.PartitionSpec(64, 7)
    # strict finite checks: an unstable r on an alternating field overflows
    big = np.array([1.7e308 * (-1.0) ** i for i in range(64)])
    ring2 = H.HistoryRing(1, big)
    H.set_strict_finite_checks(True)
    try:
        with pytest.raises(H.DivergenceError):
            ring2.push_async_step(H.SolverParams.from_r(0.6, True), H.BoundaryCondition.periodic(),
                                  H.PartitionSpec(64, 16), H.DelayModel.uniform(1, 0), rng)
        assert ring2.current_step() == 0
    finally:
        H.set_strict_finite_checks(False)
    # without strict checks the non-finite result still cannot form a TemperatureField
    with pytest.raises(H.DomainError):
        H.async_step(ring2, H.SolverParams.from_r(0.6, True), H.BoundaryCondition.periodic(),
                     H.PartitionSpec(64, 16), H.DelayModel.uniform(1, 0), rng)
    ring.close()
    ring2.close()


def test_sample_delay_stream(H):
    """sample_delay(rng, model, k) consumes one draw (async_sim.cpp:57-73):
    test_async_sim.cpp:64-71's golden vector, and the fixed law's clamp."""
    model = H.DelayModel.uniform(4, 42)
    rng = H.SplitMix64(model.seed)
    assert [H.sample_delay(rng, model, 100) for _ in range(8)] == [1, 3, 2, 0, 2, 2, 1, 0]
    model = H.DelayModel.fixed(4, 2, 77)
    rng = H.SplitMix64(model.seed)
    assert [H.sample_delay(rng, model, k) for k in (0, 1, 2, 100)] == [0, 1, 2, 2]
    assert rng.state == (77 + 4 * GAMMA) & M64


def test_reference_binding_async_step(gpu):
    """heat::async_step and heat::AsyncSimulator::step through
    integration/heat_core_b200.cpp (the reference's own types, GPU ring +
    K8a/K8b) print exactly what the reference prints: exception class, result
    hash, and the caller's stream position after the call for 200 seeded rings;
    field hashes and the step index of 60 seeded simulators stepped 1-40 times
    (oracle/binding_check.cpp)."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    bins = [os.path.join(root, "oracle", "_ref", f"binding_check_{w}") for w in ("ref", "b200")]
    if not all(os.path.exists(b) for b in bins):
        pytest.skip("oracle/_ref/binding_check_* not built (needs /root/reference at build time)")
    ref, b200 = (subprocess.run([b], capture_output=True, text=True, timeout=300, check=True).stdout
                 for b in bins)
    assert len(ref.splitlines()) == 260
    assert "logic_error" in ref and sum(l.startswith("sim ") for l in ref.splitlines()) == 60
    assert b200 == ref
