"""Host enqueue rate vs device time of the step chain: wall time of kpm_moments_ex with
KPM_DEVICE_OUT (returns without waiting for the GPU) against the device time the library's events
measure, for L2-resident small-R shapes.  usage: launch_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import kpm_inputs as ki  # noqa: E402
from paper_1105_5481_b200 import kpm  # noqa: E402

for name, R, opts in [("c2", 2, {}), ("c2", 8, {}), ("c2", 8, {"no_pdl": 1}), ("c2", 64, {})]:
    cfg = ki.CONFIGS[name]
    lat = ki.lattice(cfg)
    a, b = kpm.kpm_gershgorin_stencil(lat["ndim"], lat["L"], lat["t"], onsite=lat["onsite"], flux=lat["flux"])
    h = kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b, onsite=lat["onsite"], flux=lat["flux"])
    if opts:
        h.set_plan_opts(**opts)
    N = cfg["N"]
    out = torch.empty(N, dtype=torch.float64, device="cuda")
    h.moments(N, R, 1)
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h.moments_ex(N, R, 1, flags=kpm.KPM_DEVICE_OUT, out=out.data_ptr())
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        ms, sl, tl = h.last_timing()
    print(f"{name} R={R} {opts}: host enqueue {1e3*(t1-t0):.2f} ms for {tl} launches "
          f"({1e6*(t1-t0)/tl:.1f} us each), wall to sync {1e3*(t2-t0):.2f} ms, device steps {ms:.2f} ms", flush=True)
    h.close()
