"""The reference's own methodology on the GPU path: measure() over N in
{100, 1000, 10000} x {Barriered, BarrierFree}, 5 reps, 2000 steps, 4 PEs
(async_exec.cpp:281-320, device time), and speedup_ratio per N."""
from paper_1510_08982_b200 import heat as H

rows = H.measure([100, 1000, 10000], [H.ExecMode.Barriered, H.ExecMode.BarrierFree], 5, 2000, 4)
for r in rows:
    print(f"N={r.n_points:6d} {H.to_string(r.mode):13s} median {r.median_ns / 2000:8.1f} ns/step")
for n in (100, 1000, 10000):
    print(f"speedup_ratio(N={n}) = {H.speedup_ratio(rows, n):.3f}")
