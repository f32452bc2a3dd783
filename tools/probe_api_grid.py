"""Discovery sweep of unusual shapes through the public API against the C
port (bit-exact), reporting every failure instead of stopping at the first."""
import numpy as np

from oracle import oracle as O
from paper_1510_08982_b200 import heat as H

port = O.port()
rng = np.random.default_rng(7)
cases = []
for N, n in [(5000, 1), (3000, 3), (4098, 2049), (40000, 8), (40000, 40000 // 3 * 0 + 5000),
             (65536 * 3, 65536), (100000, 20000), (12345 * 2, 12345), (2 * 1031, 1031),
             (1 << 20, 1 << 10), (1 << 16, 1 << 15), (96, 32), (3, 1), (6, 2)]:
    if N % n:
        continue
    for bc in (0, 1):
        for q, law in ((1, 0), (3, 0), (5, 2), (16, 0), (9, 1)):
            cases.append((N, n, bc, q, law))
bad = 0
for N, n, bc, q, law in cases:
    u0 = rng.uniform(-1, 1, N)
    b = H.BoundaryCondition.periodic() if bc else H.BoundaryCondition.dirichlet(u0[0], u0[-1])
    p = H.SolverParams.from_r(0.37)
    fd, gp = (min(2, q - 1), 0.3)
    k = 70
    try:
        got = H.async_final(u0, p, b, H.PartitionSpec(N, n), H.DelayModel(q, H.Distribution(law), fd, gp, 5), k)
        exp = port.async_run(u0, p.r(), b.kind, b.c1, b.c2, n, law, q, fd, gp, seed=5, k_end=k)
        ok = np.array_equal(got.view(np.uint64), exp.view(np.uint64))
        msg = "ok" if ok else "MISMATCH"
    except Exception as e:  # noqa: BLE001
        ok, msg = False, f"{type(e).__name__}: {e}"
    if not ok:
        bad += 1
        print(f"async N={N} n={n} bc={bc} q={q} law={law}: {msg}")
for N, n, mode in [(5000, 1, 1), (3000, 3, 1), (100000, 20000, 1), (12345 * 2, 12345, 1),
                   (1 << 20, 1 << 10, 1), (5000, 5000, 1)]:
    u0 = rng.uniform(-1, 1, N)
    b = H.BoundaryCondition.dirichlet(u0[0], u0[-1])
    try:
        r = H.exec_run(H.TemperatureField(u0), H.SolverParams.from_r(0.3), b, H.PartitionSpec(N, n),
                       H.ExecConfig(N // n, 50, H.ExecMode(mode), False, 1))
        exp = port.sync_run(u0, 0.3, 0, b.c1, b.c2, 50)
        ok = np.array_equal(r.field.values().view(np.uint64), exp.view(np.uint64))
        msg = "ok" if ok else "MISMATCH (free q=1 should equal sync)"
    except Exception as e:  # noqa: BLE001
        ok, msg = False, f"{type(e).__name__}: {e}"
    if not ok:
        bad += 1
        print(f"exec N={N} n={n}: {msg}")
print("cases", len(cases) + 6, "bad", bad)
