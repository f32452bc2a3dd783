"""Device-time probe of the streaming async kernel (free-running) at N=2^30."""
import sys
import torch
from paper_1510_08982_b200 import heat as H

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 320
P = int(sys.argv[3]) if len(sys.argv) > 3 else 512
q = int(sys.argv[4]) if len(sys.argv) > 4 else 8
s = torch.cuda.Stream()
p = H.Plan(n, 0)
p.set_stream(s.cuda_stream)
p.fill_sine()
bc = H.BoundaryCondition.dirichlet(0, 0)
r = H.SolverParams.from_r(0.4).r()
p.async_advance(r, bc, n // P, q, 64)
p.sync_advance(r, bc, 128)  # both kernels warmed up (first-launch setup is not timed)
p.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for mode in ("async", "sync", "async"):
    e0.record(s)
    if mode == "async":
        st = p.async_advance(r, bc, n // P, q, steps)
    else:
        p.sync_advance(r, bc, steps)
    e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    extra = f" reads={st.reads} waits={st.waits} maxdelay={st.max_delay}" if mode == "async" else ""
    print(f"{mode:5s} N={n} P={P} q={q} steps={steps} ms={ms:.2f} GLUPS={n*steps/(ms*1e-3)/1e9:.1f}{extra}")
p.synchronize()
