"""Host-timed breakdown of one end-to-end call sequence on config 4."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import torch  # noqa: E402

from paper_1501_03105_b200 import build, irls as I  # noqa: E402
from synthetic import generators as gen  # noqa: E402

build.build()
spec = gen.config4()
pinned = {}
for name in ("cx", "cy", "cz", "cs", "ct"):
    t = torch.empty(spec[name].shape[0], dtype=torch.float64, pin_memory=True)
    t.numpy()[:] = spec[name]
    pinned[name] = t.numpy()
side = torch.empty(spec["cx"].shape[0] + 2, dtype=torch.uint8, pin_memory=True).numpy()
opts = I.options(T=50)
stream = torch.cuda.current_stream().cuda_stream
comm = I.comm_desc(1, 0, 0, None, stream)
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m = I.MinCut.irls_mincut_create_stencil(512, 512, 256, pinned["cx"], pinned["cy"], pinned["cz"], pinned["cs"],
                                            pinned["ct"], opts, comm)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    m.irls_init()
    t2 = time.perf_counter()
    m.irls_step()
    t3 = time.perf_counter()
    _, tot = m.irls_solve(I.IRLS_FROM_SCRATCH, T=50, reports=False)
    t4 = time.perf_counter()
    k, cut = C.c_int64(), C.c_double()
    I.lib().irls_sweep_cut(m.h, side.ctypes.data_as(C.c_void_p), None, C.byref(k), C.byref(cut))
    t5 = time.perf_counter()
    m.close()
    torch.cuda.synchronize()
    t6 = time.perf_counter()
    print(f"iter {it}: create {1e3*(t1-t0):.1f}  init(+graph) {1e3*(t2-t1):.1f}  step(+graph) {1e3*(t3-t2):.1f}  "
          f"solve {1e3*(t4-t3):.1f}  sweep+D2H {1e3*(t5-t4):.1f}  destroy {1e3*(t6-t5):.1f} ms")
