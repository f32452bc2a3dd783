#!/bin/bash
export PYTHONPATH=.
timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python -c "
import numpy as np
from paper_1510_08982_b200 import heat as H
n=1024
u0=np.sin(np.pi*np.arange(n)/(n-1)); u0[-1]=0
print(H.async_run(H.TemperatureField(u0),H.SolverParams.from_r(0.25),H.BoundaryCondition.dirichlet(0,0),H.PartitionSpec(n,n//8),H.DelayModel.uniform(2,1),100,50).final()[:4])
" 2>&1 | head -60
