import os, sys, time
sys.path.insert(0, '/root/repo')
import torch
from paper_1501_03105_b200 import build, irls as I
from synthetic import generators as gen
build.build()
spec = gen.config4()
stream = torch.cuda.current_stream().cuda_stream
for use_torch in (False, True, True, False):
    mem = I.TorchDeviceMemory(0) if use_torch else None
    comm = I.comm_desc(1, 0, 0, None, stream, memory=mem)
    for it in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        m = I.MinCut.from_spec(spec, I.options(T=50), comm)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        m.irls_solve(I.IRLS_FROM_SCRATCH, T=50, reports=False)
        torch.cuda.synchronize(); t2 = time.perf_counter()
        m.irls_sweep_cut(side=False)
        torch.cuda.synchronize(); t3 = time.perf_counter()
        m.close(); torch.cuda.synchronize(); t4 = time.perf_counter()
        print(f"torch={use_torch} it={it}: create {1e3*(t1-t0):.1f} solve {1e3*(t2-t1):.1f} sweep {1e3*(t3-t2):.1f} destroy {1e3*(t4-t3):.1f}  reserved {torch.cuda.memory_reserved()/1e9:.1f} GB", flush=True)
