"""Quick device-time probe of the sync path at BASELINE cfg3 size (N=2^30)."""
import sys, time
import torch
from paper_1510_08982_b200 import heat as H

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 320
s = torch.cuda.Stream()
p = H.Plan(n, 0)
p.set_stream(s.cuda_stream)
p.fill_sine()
bc = H.BoundaryCondition.dirichlet(0, 0)
r = H.SolverParams.from_r(0.4).r()
p.sync_advance(r, bc, 32)
p.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(3):
    e0.record(s)
    p.sync_advance(r, bc, steps)
    e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    glups = n * steps / (ms * 1e-3) / 1e9
    print(f"N={n} steps={steps} ms={ms:.2f} GLUPS={glups:.1f} frac_of_roofline={glups*16/6541.8:.3f}")
p.synchronize()
print("launches", H.kernel_launches())
