"""BASELINE configs[4]: stability/error sweep, r in {0.1,0.25,0.4,0.49} x delay bound
q in {0,1,2,4,8} (reference buffer length q_ref = q+1), N=1024, 8 PEs, sine IC,
Dirichlet(0,0), K steps.  Deterministic async (seeds 1..5) and free-running async,
L-inf distance to the synchronous solution vs the a-posteriori bound."""
import sys
import numpy as np
from paper_1510_08982_b200 import heat as H

K = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
out = sys.argv[2] if len(sys.argv) > 2 else None
n, P = 1024, 8
u0 = np.sin(np.pi * np.arange(n) / (n - 1)); u0[0] = 0.0; u0[-1] = 0.0
bc = H.BoundaryCondition.dirichlet(0, 0)
part = H.PartitionSpec(n, n // P)
rows = ["| r | q (max delay) | q_ref | det: max L∞(async−sync), 5 seeds | free: L∞(async−sync) | free: bound Σ‖u(k+1)−Au(k)‖∞ | bound/L∞ | free: max delay | free: waits/reads |",
        "|---|---|---|---|---|---|---|---|---|"]
ok = True
for r in (0.1, 0.25, 0.4, 0.49):
    p = H.SolverParams.from_r(r)
    sync = H.sync_final(u0, p, bc, K)
    for q in (0, 1, 2, 4, 8):
        qr = q + 1
        det = max(float(np.max(np.abs(H.async_final(u0, p, bc, part, H.DelayModel.uniform(qr, s), K) - sync)))
                  for s in range(1, 6))
        fin, st = H.async_free_run(u0, p, bc, part, qr, K)
        err = float(np.max(np.abs(fin - sync)))
        ok &= err <= st.residual_sum and st.max_delay <= q
        ratio = (st.residual_sum / err) if err > 0 else float("inf")
        rows.append(f"| {r} | {q} | {qr} | {det:.3e} | {err:.3e} | {st.residual_sum:.3e} | {ratio:.1f} | {st.max_delay} | {st.waits}/{st.reads} |")
text = "\n".join(rows) + f"\n\nK={K}, all free-running errors within the bound and delays within q: {ok}\n"
print(text)
if out:
    open(out, "w").write(text)
