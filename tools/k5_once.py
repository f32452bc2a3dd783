"""One K5 free-running launch at N=2^30, 512 PEs, q=8 (profiler capture)."""
import sys
import torch
from paper_1510_08982_b200 import heat as H

n = 1 << 30
s = torch.cuda.Stream()
p = H.Plan(n, 0)
p.set_stream(s.cuda_stream)
p.fill_sine()
st = p.async_advance(H.SolverParams.from_r(0.4).r(), H.BoundaryCondition.dirichlet(0, 0), n // 512, 8, int(sys.argv[1]) if len(sys.argv) > 1 else 320)
p.synchronize()
print("reads", st.reads, "waits", st.waits, "max_delay", st.max_delay)
