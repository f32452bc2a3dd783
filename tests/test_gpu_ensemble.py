"""GPU ensembles (K6, csrc/ensemble.cu) against the reference's ensemble_run
(analysis.cpp:51-104): fixtures produced by the reference itself
(tests/golden/golden.json) -- bit-exact norms, terminal fields, mean and std
series -- plus the paper's experiment as acceptance.cpp criteria 2-3 run it
(50 members, N = 100, one point per PE, q = 5, 2e5 steps)."""
import json
import os

import numpy as np
import pytest

from helpers import bits_equal, fnv1a64

pytestmark = pytest.mark.gpu

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def unhex(v):
    return np.array([float.fromhex(x) for x in v], np.float64)


@pytest.fixture(scope="module")
def H(gpu):
    from paper_1510_08982_b200 import heat
    return heat


def _cfg(H, port, e):
    u0 = port.cosine_init(100)
    p = H.SolverParams.checked(0.5, 0.01, 0.1)
    bc = H.BoundaryCondition.periodic() if e["bc"] else H.BoundaryCondition.dirichlet(e["c1"],
                                                                                       e["c2"])
    model = H.DelayModel(e["q"], H.Distribution(e["law"]), e["d"], 0.5, 0)
    return H.EnsembleConfig(H.TemperatureField(u0), p, bc, H.PartitionSpec(100, e["per_pe"]),
                            model, e["k"], e["stride"])


@pytest.mark.parametrize("idx", [0, 1, 2])
def test_ensemble_matches_reference_fixture(H, port, idx):
    e = G["ensembles"][idx]
    res = H.ensemble_run(_cfg(H, port, e), e["runs"], e["base"])
    assert res.steps == e["steps"]
    for j in range(e["runs"]):
        assert bits_equal(np.array(res.norm_series[j]), unhex(e["norms"][j])), j
        assert fnv1a64(res.terminal_fields[j].values()) == e["terminal_fnv"][j]
    assert bits_equal(np.array(res.mean_series), unhex(e["mean"]))
    assert bits_equal(np.array(res.std_series), unhex(e["std"]))


def test_ensemble_member_is_async_run(H, port):
    # member j is async_run with seed base + j (analysis.cpp:16-38)
    e = G["ensembles"][0]
    res = H.ensemble_run(_cfg(H, port, e), 2, 555)
    u0 = port.cosine_init(100)
    r = H.SolverParams.checked(0.5, 0.01, 0.1).r()
    for j in range(2):
        fin = port.async_run(u0, r, 0, 1.0, 0.0, 1, 0, 5, seed=555 + j, k_end=e["k"])
        assert bits_equal(res.terminal_fields[j].values(), fin)


def test_paper_ensembles_acceptance_criteria_2_3(H, port):
    # acceptance.cpp:103-137: Dirichlet members all reach the linear steady
    # state (<= 1e-4); the periodic terminal mean temperature spreads (> 10x)
    crit = G["acceptance_ensembles"]
    out = {}
    for name, bc in (("dirichlet", H.BoundaryCondition.dirichlet(1.0, 0.0)),
                     ("periodic", H.BoundaryCondition.periodic())):
        cfg = H.EnsembleConfig(H.cosine_init(100), H.SolverParams.checked(0.5, 0.01, 0.1), bc,
                               H.PartitionSpec(100, 1), H.DelayModel.uniform(5, 0), 200000,
                               200000)
        res = H.ensemble_run(cfg, 50, 1000)
        assert [fnv1a64(t.values()) for t in res.terminal_fields] == crit[name]["terminal_fnv"]
        sm, sn = H.terminal_spread(res)
        assert sm == float.fromhex(crit[name]["spread_mean_temp"])
        assert sn == float.fromhex(crit[name]["spread_norm"])
        out[name] = (res, sm)
    steady = H.linear_steady_state(100, 1.0, 0.0).values()
    worst = max(np.max(np.abs(f.values() - steady)) for f in out["dirichlet"][0].terminal_fields)
    assert worst <= 1e-4
    assert out["periodic"][1] > 1e-6 and out["periodic"][1] > 10 * out["dirichlet"][1]


def test_ensemble_validation(H):
    cfg = H.EnsembleConfig(H.cosine_init(100), H.SolverParams.from_r(0.5),
                           H.BoundaryCondition.dirichlet(1, 0), H.PartitionSpec(100, 1),
                           H.DelayModel.uniform(5, 0), 10, 10)
    with pytest.raises(H.DomainError):
        H.ensemble_run(cfg, 0, 1)
    cfg.model = H.DelayModel.geometric(5, 0.5, 0)
    assert len(H.ensemble_run(cfg, 2, 1).terminal_fields) == 2  # every law runs on the GPU


def test_paper_ensemble_speed_vs_reference(H, ref):
    # The paper's Fig. 6 ensemble (M = 50, N = 100, q = 5, 2e5 steps, periodic)
    # through the reference's own ensemble_run on this host and through the
    # GPU; identical terminal means, GPU time printed for profiles/.
    import time
    cos = ref.cosine_init(100)
    r = ref.checked_r(0.5, 0.01, 0.1)
    from oracle import oracle as O
    t0 = time.perf_counter()
    steps, norms, terms, mean, std, spread = ref.ensemble_run(
        cos, r, O.PERIODIC, 0.0, 0.0, 1, O.UNIFORM, 5, 0, 200000, 200000, 50, 1000)
    t_ref = time.perf_counter() - t0
    cfg = H.EnsembleConfig(H.cosine_init(100), H.SolverParams.checked(0.5, 0.01, 0.1),
                           H.BoundaryCondition.periodic(), H.PartitionSpec(100, 1),
                           H.DelayModel.uniform(5, 0), 200000, 200000)
    H.ensemble_run(cfg, 2, 1)  # context + module load
    t0 = time.perf_counter()
    res = H.ensemble_run(cfg, 50, 1000)
    t_gpu = time.perf_counter() - t0
    assert [fnv1a64(t.values()) for t in res.terminal_fields] == [fnv1a64(t) for t in terms]
    print(f"\npaper ensemble (M=50, N=100, q=5, 2e5 steps): reference {t_ref:.3f} s, "
          f"GPU {t_gpu:.4f} s, x{t_ref / t_gpu:.0f}")
    assert t_gpu < t_ref


def _check_against_reference(H, ref, u0, r, bc, per_pe, law, q, d, p, k_end, stride, runs, base):
    from oracle import oracle as O
    bck = O.PERIODIC if not bc.is_dirichlet() else O.DIRICHLET
    steps, norms, terms, mean, std, _ = ref.ensemble_run(u0, r, bck, bc.c1, bc.c2, per_pe, law, q,
                                                         d, k_end, stride, runs, base, p=p)
    cfg = H.EnsembleConfig(H.TemperatureField(u0), H.SolverParams.from_r(r), bc,
                           H.PartitionSpec(u0.size, per_pe),
                           H.DelayModel(q, H.Distribution(law), d, p, 0), k_end, stride)
    res = H.ensemble_run(cfg, runs, base)
    assert res.steps == steps
    assert bits_equal(np.array(res.norm_series), norms)
    for j in range(runs):
        assert bits_equal(res.terminal_fields[j].values(), terms[j]), j
    assert bits_equal(np.array(res.mean_series), mean)
    assert bits_equal(np.array(res.std_series), std)


@pytest.mark.parametrize("periodic", [False, True])
@pytest.mark.parametrize("per_pe,q,p", [(1, 5, 0.6), (10, 3, 0.3), (25, 8, 0.05)])
def test_geometric_ensemble_matches_reference(H, ref, periodic, per_pe, q, p):
    """The geometric law on K6: delays from the device thresholds
    (geometric_thresholds) -- the reference's own ensemble_run, bit for bit."""
    u0 = ref.cosine_init(100)
    bc = H.BoundaryCondition.periodic() if periodic else H.BoundaryCondition.dirichlet(1.0, 0.0)
    _check_against_reference(H, ref, u0, 0.45, bc, per_pe, 2, q, 0, p, 3000, 250, 6, 77)


@pytest.mark.parametrize("N,per_pe,law,q", [(6000, 1000, 0, 3), (6144, 2048, 2, 4),
                                            (4096, 512, 1, 7)])
def test_ensemble_beyond_shared_memory_matches_reference(H, ref, N, per_pe, law, q):
    """Members whose history does not fit one CTA (N > 4096, or (q+1)*N*8 > 200 KB)
    run on AsyncSimulator handles (K3/K5): same results as the reference."""
    from helpers import SplitMix64, random_field
    u0 = random_field(SplitMix64(N + q), N)
    bc = H.BoundaryCondition.dirichlet(float(u0[0]), float(u0[-1]))
    _check_against_reference(H, ref, u0, 0.4, bc, per_pe, law, q, 2 if law == 1 else 0, 0.5, 400,
                             150, 3, 9)


def test_sharded_ensemble_one_rank_equals_ensemble_run(gpu, port):
    # multigpu.ensemble_run_sharded on one process (no process group): the GPU
    # members on the device heat_set_device picked, statistics formed on the
    # host in the reference's order -- identical to heat.ensemble_run
    from paper_1510_08982_b200 import heat as H
    from paper_1510_08982_b200 import multigpu as M
    cfg = H.EnsembleConfig(H.cosine_init(100), H.SolverParams.from_r(0.45),
                           H.BoundaryCondition.periodic(), H.PartitionSpec(100, 1),
                           H.DelayModel.uniform(3, 0), k_end=2000, stride=100)
    a = M.ensemble_run_sharded(cfg, 9, 42, device=0)
    b = H.ensemble_run(cfg, 9, 42)
    assert a.steps == b.steps and a.seeds == b.seeds
    assert np.array_equal(np.array(a.norm_series).view(np.uint64),
                          np.array(b.norm_series).view(np.uint64))
    assert np.array_equal(np.array(a.mean_series).view(np.uint64),
                          np.array(b.mean_series).view(np.uint64))
    assert np.array_equal(np.array(a.std_series).view(np.uint64),
                          np.array(b.std_series).view(np.uint64))
    with pytest.raises(H.InvalidArgument):
        H.set_device(4096)
