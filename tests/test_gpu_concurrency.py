"""Thread safety of the C-ABI (include/heat_b200.h: "every entry point may be
called from any host thread"): the reference's ensemble_run runs its members
on many std::threads at once (analysis.cpp:68-85), and a drop-in caller may do
the same with sync_run / async_run / exec_run.  Ten host threads call the
library concurrently (ctypes releases the GIL for the duration of each call)
on different fields, sizes and partitions, repeatedly, and every result must be
bit-identical with the oracle -- no shared scratch, tile counter or flag word
may leak between calls."""
import threading

import numpy as np
import pytest

from helpers import SplitMix64, bits_equal, random_field
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H(gpu):
    from paper_1510_08982_b200 import heat
    return heat


def _case(i):
    gen = SplitMix64(1000 + i)
    kind = i % 5
    N = [1024, 5000, 1 << 17, 3 << 12, 1024][kind]
    u0 = random_field(gen, N)
    r = 0.1 + 0.39 * gen.next_double()
    return kind, N, u0, r


def _work(H, port, i, reps, errors):
    kind, N, u0, r = _case(i)
    c1, c2 = float(u0[0]), float(u0[-1])
    bc = H.BoundaryCondition.dirichlet(c1, c2)
    p = H.SolverParams.from_r(r)
    try:
        for rep in range(reps):
            k = 50 + 37 * rep + i
            if kind in (0, 2):  # sync_run (K7c cluster + zero-copy staging / K1)
                got = H.sync_final(u0, p, bc, k)
                exp = port.sync_run(u0, r, O.DIRICHLET, c1, c2, k)
            elif kind in (1, 4):  # deterministic async_run (K3 / K9 cluster + zero-copy)
                n = N // 8
                got = H.async_final(u0, p, bc, H.PartitionSpec(N, n), H.DelayModel.uniform(3, 7 + i), k)
                exp = port.async_run(u0, r, O.DIRICHLET, c1, c2, n, O.UNIFORM, 3, seed=7 + i, k_end=k)
            else:  # exec_run(Barriered) and BarrierFree with q = 1 (exact)
                n = N // 4
                mode = H.ExecMode.Barriered if rep % 2 == 0 else H.ExecMode.BarrierFree
                res = H.exec_run(H.TemperatureField(u0), p, bc, H.PartitionSpec(N, n),
                                 H.ExecConfig(4, k, mode, False, 1))
                got = res.field.values()
                exp = port.sync_run(u0, r, O.DIRICHLET, c1, c2, k)
            if not bits_equal(got, exp):
                errors.append(f"thread {i} rep {rep} kind {kind}: mismatch")
    except Exception as e:  # noqa: BLE001 - reported below
        errors.append(f"thread {i}: {type(e).__name__}: {e}")


def test_eight_threads_bit_exact(H, port):
    errors = []
    threads = [threading.Thread(target=_work, args=(H, port, i, 4, errors)) for i in range(10)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


def test_threads_match_serial(H, port):
    """The same calls serially and concurrently give the same bits (no hidden
    state carried from one call into another)."""
    serial_err = []
    for i in range(4):
        _work(H, port, i, 2, serial_err)
    assert not serial_err, serial_err
    errors = []
    threads = [threading.Thread(target=_work, args=(H, port, i, 2, errors)) for i in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
