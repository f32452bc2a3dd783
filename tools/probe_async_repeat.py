"""K5 back-to-back on one plan, the bench's call sequence: per-call device time."""
import sys
import torch
from paper_1510_08982_b200 import heat as H

n = 1 << 30
P = 512
s = torch.cuda.Stream()
p = H.Plan(n, 0)
p.set_stream(s.cuda_stream)
bc = H.BoundaryCondition.dirichlet(0, 0)
r = H.SolverParams.from_r(0.4).r()
mode = sys.argv[1] if len(sys.argv) > 1 else "free"
p.fill_sine()
for i in range(8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    if mode == "free":
        st = p.async_advance(r, bc, n // P, 8, 1000)
    else:
        st = p.async_replay(r, bc, n // P, H.DelayModel.uniform(2, 1), 1000)
    e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{mode} call {i}: {ms:.1f} ms  {n * 1000 / (ms * 1e-3) / 1e9:.0f} GLUPS waits={st.waits}")
