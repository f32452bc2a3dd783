"""Discovery sweep of sync / f32 / ensemble shapes through the public API
against the C port and the reference's algorithm, reporting every failure."""
import numpy as np

from oracle import oracle as O
from paper_1510_08982_b200 import heat as H

port = O.port()
rng = np.random.default_rng(11)
bad = 0
total = 0
for N in (3, 4, 7, 63, 64, 65, 1000, 1023, 1025, 4095, 4097, 16383, 16384, 16385, 100003,
          (1 << 20) + 7, (1 << 24) + 5):
    for bc in (0, 1):
        for k, stride in ((1, 1), (65, 13), (300, 0)):
            total += 1
            u0 = rng.uniform(-1, 1, N)
            b = H.BoundaryCondition.periodic() if bc else H.BoundaryCondition.dirichlet(u0[0], u0[-1])
            p = H.SolverParams.from_r(0.43)
            try:
                t = H.sync_run(H.TemperatureField(u0), p, b, k, stride)
                steps, snaps = port.sync_run(u0, p.r(), b.kind, b.c1, b.c2, k, stride, record=True)
                ok = t.steps == steps and all(
                    np.array_equal(s.values().view(np.uint64), snaps[j].view(np.uint64))
                    for j, s in enumerate(t.snapshots))
                f = H.sync_run_f32(H.TemperatureField(u0), p, b, k, k).final().values()
                ok &= np.array_equal(f.view(np.uint64),
                                     port.sync_run_f32(u0, p.r(), b.kind, b.c1, b.c2, k).view(np.uint64))
                msg = "ok" if ok else "MISMATCH"
            except Exception as e:  # noqa: BLE001
                ok, msg = False, f"{type(e).__name__}: {e}"
            if not ok:
                bad += 1
                print(f"sync N={N} bc={bc} k={k} stride={stride}: {msg}")
# ensembles beyond one CTA's history (simulator path) and odd PE widths
ref = O.ref() if O.Ref.available() else None
for N, n, q in ((5000, 1, 2), (6000, 1500, 3), (2048, 2048 // 8, 9)):
    total += 1
    u0 = port.cosine_init(N)
    cfg = H.EnsembleConfig(H.TemperatureField(u0), H.SolverParams.from_r(0.4),
                           H.BoundaryCondition.dirichlet(1.0, 0.0), H.PartitionSpec(N, n),
                           H.DelayModel.uniform(q, 0), k_end=60, stride=20)
    try:
        res = H.ensemble_run(cfg, 3, 9)
        ok = len(res.norm_series) == 3 and len(res.steps) == 4
        if ref is not None:
            st, nr, _, mean, std, _ = ref.ensemble_run(u0, 0.4, 0, 1.0, 0.0, n, 0, q, 0, 60, 20, 3, 9)
            ok &= np.array_equal(np.array(res.norm_series).view(np.uint64), nr.view(np.uint64))
        msg = "ok" if ok else "MISMATCH"
    except Exception as e:  # noqa: BLE001
        ok, msg = False, f"{type(e).__name__}: {e}"
    if not ok:
        bad += 1
        print(f"ensemble N={N} n={n} q={q}: {msg}")
print("cases", total, "bad", bad)
