import sys, os, json
sys.path.insert(0, "/root/repo")
import torch
from paper_1501_03105_b200 import build, irls as I
from synthetic import generators as gen
build.build()
spec = gen.config4()
st = torch.cuda.current_stream()
m = I.MinCut.from_spec(spec, I.options(T=50), I.comm_desc(1, 0, 0, None, st.cuda_stream))
m.irls_solve(I.IRLS_FROM_SCRATCH, T=50, reports=False)
for rep in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(st)
    reps, tot = m.irls_solve(I.IRLS_FROM_SCRATCH, T=50)
    e1.record(st); torch.cuda.synchronize()
    print("total ms", e0.elapsed_time(e1), "sum report ms", sum(r["ms"] for r in reps))
    print([(r["cg_iters"], round(r["ms"], 3), round(r["ms_assemble"], 3)) for r in reps])
