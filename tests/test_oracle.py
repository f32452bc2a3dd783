"""CPU: the oracle port (oracle/heat_oracle.c) pinned against the reference.

(a) golden fixtures produced by the reference itself (tests/golden/golden.json,
    made by tests/golden/gen_golden.py through oracle/_ref), and the KATs of
    the reference's unit tests (test_sync.cpp, test_async_sim.cpp, test_core.cpp);
(b) live side-by-side runs against oracle/_ref when it is built here."""
import json
import os

import numpy as np
import pytest

from helpers import SplitMix64, bits_equal, fnv1a64, random_divisor, random_field, sine_field

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def unhex(v):
    return np.array([float.fromhex(x) for x in v], np.float64)


def test_delay_stream_goldens(port):
    for s in G["delay_streams"]:
        assert port.delay_stream(s["law"], s["q"], s["d"], s["p"], s["seed"], s["k"],
                                 s["count"]) == s["values"]
    # test_async_sim.cpp:64-71 literal
    assert port.delay_stream(0, 4, 0, 0.5, 42, 100, 8) == [1, 3, 2, 0, 2, 2, 1, 0]
    # test_async_sim.cpp:55-62: fixed law clamps to k
    st = [port.delay_stream(1, 4, 2, 0.5, 77, k, 1)[0] for k in (0, 1, 2, 100)]
    assert st[:3] == [0, 1, 2]


def test_core_goldens(port):
    assert fnv1a64(port.cosine_init(100)) == G["cosine_init_100_fnv"]
    # test_core.cpp:101
    assert port.l2_norm(port.cosine_init(100)) == pytest.approx(6.1339220731926485, rel=1e-14)
    assert port.total_heat(port.cosine_init(100)) == pytest.approx(50.0, rel=1e-13)
    assert fnv1a64(port.prepare_initial(port.sine_init(1024), 0, 0.0, 0.0)) == G["sine_1024_fnv"]
    assert bits_equal(sine_field(1024), port.prepare_initial(port.sine_init(1024), 0, 0, 0))


def test_cfg1_cfg2_goldens(port):
    u = port.prepare_initial(port.sine_init(1024), 0, 0.0, 0.0)
    fin = port.sync_run(u, 0.25, 0, 0.0, 0.0, 1000)
    assert fnv1a64(fin) == G["cfg1"]["fnv"] == 0xC2C466B7716F830A
    assert fin[512].hex() == G["cfg1"]["u512"]
    for c in G["cfg2"]:
        fin = port.async_run(u, 0.25, 0, 0.0, 0.0, 128, 0, c["q"], seed=c["seed"], k_end=1000)
        assert fnv1a64(fin) == c["fnv"]


def test_small_case_goldens(port):
    for c in G["cases"]:
        u0 = unhex(c["u0"])
        r = float.fromhex(c["r"])
        c1, c2 = float.fromhex(c["c1"]), float.fromhex(c["c2"])
        s = port.sync_run(u0, r, c["bc"], c1, c2, c["k"])
        assert bits_equal(s, unhex(c["sync_final"]))
        a = port.async_run(u0, r, c["bc"], c1, c2, c["per_pe"], c["law"], c["q"], c["d"],
                           float.fromhex(c["p"]), c["seed"], c["k"])
        assert bits_equal(a, unhex(c["async_final"]))


def test_sync_kats(port):
    assert list(port.sync_step([1.0, 0.0, 0.0], 0.5, 0, 1.0, 0.0)) == [1.0, 0.5, 0.0]
    assert bits_equal(port.sync_step([1.0, 0.0, 0.0], 0.5, 0, 1.0, 0.0),
                      unhex(G["kat_sync_step_dirichlet"]))
    assert bits_equal(port.sync_step([2.0, 0.0, 1.0], 0.25, 1), unhex(G["kat_sync_step_periodic"]))
    steps, _ = port.sync_run(port.cosine_init(10), 0.5, 0, 1.0, 0.0, 10, 3, record=True)
    assert steps == [0, 3, 6, 9, 10]  # test_sync.cpp:65-70


def test_errors(port):
    from oracle.oracle import OracleError
    with pytest.raises(OracleError) as e:
        port.sync_run([0.5, 0.0, 0.0], 0.5, 0, 1.0, 0.0, 1)
    assert e.value.code == 2  # std::invalid_argument
    with pytest.raises(OracleError) as e:
        port.async_run(np.zeros(12), 0.5, 0, 0, 0, 5, 0, 2, k_end=1)
    assert e.value.code == 1  # PartitionSpec: domain_error
    v = np.zeros(8)
    v[3], v[4] = 1e308, -1e308
    with pytest.raises(OracleError) as e:
        port.sync_run(v, 100.0, 0, 0, 0, 50, 1, strict=True)
    assert e.value.code == 4  # DivergenceError


def test_lightcone_windows(port):
    # a window of half-width K+1 reproduces the centre bit-exactly
    gen = SplitMix64(5)
    n = 1 << 14
    u = random_field(gen, n)
    u[0], u[-1] = 0.0, 0.0
    k = 300
    full = port.sync_run(u, 0.4, 0, 0.0, 0.0, k)
    for c in (0, 5, 299, 8000, n - 2, n - 1):
        assert port.sync_lightcone(u, 0.4, 0, 0.0, 0.0, k, c) == full[c]


# ---- live against the reference library ------------------------------------
@pytest.mark.parametrize("seed", [2026, 7])
def test_port_vs_reference_random(port, ref, seed):
    gen = SplitMix64(seed)
    for _ in range(30):
        n = 3 + gen.next_bounded(60)
        r = 0.5 * (gen.next_double() * 0.999 + 0.001)
        periodic = int(gen.next() & 1)
        u0 = random_field(gen, n)
        c1, c2 = (0.0, 0.0) if periodic else (u0[0], u0[-1])
        k = 1 + gen.next_bounded(300)
        per = random_divisor(gen, n)
        q = 1 + gen.next_bounded(9)
        law = int(gen.next_bounded(2))
        fd = int(gen.next_bounded(q - 1)) if law == 1 else 0
        gp = 0.05 + 0.9 * gen.next_double()
        sd = gen.next()
        st_p, sn_p = port.sync_run(u0, r, periodic, c1, c2, k, 1, record=True)
        st_r, sn_r = ref.sync_run(u0, r, periodic, c1, c2, k, 1, record=True)
        assert st_p == st_r and bits_equal(sn_p, sn_r)
        a_p = port.async_run(u0, r, periodic, c1, c2, per, law, q, fd, gp, sd, k)
        a_r = ref.async_run(u0, r, periodic, c1, c2, per, law, q, fd, gp, sd, k)
        assert bits_equal(a_p, a_r)
        f_p = port.sync_run_f32(u0, r, periodic, c1, c2, k)
        f_r = ref.sync_run_f32(u0, r, periodic, c1, c2, k)
        assert bits_equal(f_p, f_r)


def test_port_exec_vs_reference(port, ref):
    u = port.cosine_init(96)
    fp, _ = port.exec_run(u, 0.5, 0, 1.0, 0.0, 24, 4, 500)
    fr, _, _ = ref.exec_run(u, 0.5, 0, 1.0, 0.0, 24, 4, 500)
    assert bits_equal(fp, fr)
    # barrier-free with one PE is exact in both
    fp, _ = port.exec_run(u, 0.5, 0, 1.0, 0.0, 96, 1, 500, mode=1)
    fr, _, _ = ref.exec_run(u, 0.5, 0, 1.0, 0.0, 96, 1, 500, mode=1)
    assert bits_equal(fp, fr)


@pytest.mark.parametrize("seed", [11, 12])
def test_port_async_step_vs_reference(port, ref, seed):
    """async_step over arbitrary rings: values, status and the stream position
    after the call (D draws, or through the failing draw on a logic_error)."""
    from helpers import async_step_cases
    errors = 0
    for c in async_step_cases(seed, 60):
        sp, fp, rp = port.async_step(**c)
        sr, fr, rr = ref.async_step(**c)
        assert (sp, rp) == (sr, rr)
        errors += sp == 3
        if sp == 0:
            assert bits_equal(fp, fr)
    assert errors > 0  # the logic_error path was exercised


@pytest.mark.parametrize("law,q,fd,gp", [(0, 2, 0, 0.5), (0, 3, 0, 0.5), (1, 4, 2, 0.5),
                                         (2, 5, 0, 0.3)])
def test_async_lightcone_windows(port, law, q, fd, gp):
    # the deterministic async run's light cone (orc_async_lightcone) equals the
    # full async_run at PE boundaries, interior points and near the true ends
    n, per_pe, k, seed = 4096, 256, 120, 99 + q
    gen = SplitMix64(n + q)
    u0 = random_field(gen, n)
    u0[0], u0[-1] = 0.0, 0.0
    full = port.async_run(u0, 0.4, 0, 0.0, 0.0, per_pe, law, q, fd, gp, seed=seed, k_end=k)
    for c in [0, 1, 5, 255, 256, 257, 1023, 1024, 2000, 3839, 3840, n - 2, n - 1]:
        lo, hi = max(0, c - k - 2), min(n, c + k + 3)
        got = port.async_lightcone(u0[lo:hi], lo, n, 0.4, 0.0, 0.0, per_pe, law, q, fd, gp,
                                   seed, k, c)
        assert got == full[c], (c, got, full[c])


@pytest.mark.parametrize("seed", [3, 11])
def test_window_runs_vs_reference(port, ref, seed):
    """orc_sync_window / orc_async_window (the bench's at-scale checkers):
    every point more than k from a held window end equals the reference's own
    full sync_run / async_run; true domain ends are pinned."""
    rng = np.random.default_rng(seed)
    n, per_pe, k = 2048, 256, 200
    u0 = random_field(SplitMix64(seed), n)
    u0[0], u0[-1] = 0.0, 0.0
    full_s = ref.sync_run(u0, 0.4, 0, 0.0, 0.0, k)
    full_a = ref.async_run(u0, 0.4, 0, 0.0, 0.0, per_pe, 0, 3, seed=seed, k_end=k)
    for lo, w in [(0, 700), (n - 600, 600), (int(rng.integers(1, n - 900)), 900)]:
        a = 0 if lo == 0 else k + 1
        b = w if lo + w == n else w - k - 1
        got = port.sync_window(u0[lo:lo + w], lo, n, 0.4, 0.0, 0.0, k)
        assert bits_equal(got[a:b], np.asarray(full_s)[lo + a:lo + b]), ("sync", lo, w)
        got = port.async_window(u0[lo:lo + w], lo, n, 0.4, 0.0, 0.0, per_pe, 0, 3, seed=seed, k=k)
        assert bits_equal(got[a:b], np.asarray(full_a)[lo + a:lo + b]), ("async", lo, w)
