"""Where the end-to-end time goes: kpm_create_stencil, the first and a second kpm_moments call on
the handle, kpm_destroy (wall clock, host-synchronous), per config.  usage: e2e_probe.py c3 [c4 ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import kpm_inputs as ki  # noqa: E402
from paper_1105_5481_b200 import kpm  # noqa: E402

for name in sys.argv[1:]:
    cfg = ki.CONFIGS[name]
    lat = ki.lattice(cfg)
    a, b = kpm.kpm_gershgorin_stencil(lat["ndim"], lat["L"], lat["t"], onsite=lat["onsite"], flux=lat["flux"])
    on = None if lat["onsite"] is None else torch.from_numpy(lat["onsite"]).pin_memory().numpy()
    for rep in range(3):
        t0 = time.perf_counter()
        h = kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b, onsite=on, flux=lat["flux"])
        t1 = time.perf_counter()
        h.moments(cfg["N"], cfg["R"], cfg["seed"])
        t2 = time.perf_counter()
        ms1, sl, tl = h.last_timing()
        h.moments(cfg["N"], cfg["R"], cfg["seed"])
        t3 = time.perf_counter()
        ms2, _, _ = h.last_timing()
        h.close()
        t4 = time.perf_counter()
        print(f"{name} rep{rep}: create {1e3*(t1-t0):.1f} ms, moments#1 {1e3*(t2-t1):.1f} ms (steps {ms1:.1f}), "
              f"moments#2 {1e3*(t3-t2):.1f} ms (steps {ms2:.1f}), destroy {1e3*(t4-t3):.1f} ms", flush=True)
