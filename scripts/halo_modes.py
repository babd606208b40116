"""Row partition in one process (kpm_moments_group) on the GPUs present: fused halo (kernels store
boundary planes into the neighbours' ghost planes) vs plane copies vs the unpartitioned lattice.
usage: python scripts/halo_modes.py [config] [slabs]   (wall time per call, after one warm-up)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kpm_inputs as ki
from paper_1105_5481_b200 import kpm

cfg = ki.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
G = int(sys.argv[2]) if len(sys.argv) > 2 else 4
lat = ki.lattice(cfg)
import torch
ndev = max(torch.cuda.device_count(), 1)
a, b = kpm.kpm_gershgorin_stencil(lat["ndim"], lat["L"], lat["t"], onsite=lat["onsite"], flux=lat["flux"])
N, R, seed = cfg["N"], cfg["R"], cfg["seed"]


def timed(fn, reps=2):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        mu = fn()
    return (time.perf_counter() - t0) / reps * 1e3, mu


whole = kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b, onsite=lat["onsite"], flux=lat["flux"])
t_whole, mu_whole = timed(lambda: whole.moments(N, R, seed))
whole.close()
hs = [kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b, onsite=lat["onsite"], flux=lat["flux"],
                             device=rk % ndev, dist=(kpm.KPM_PART_ROWS, rk, G, kpm.KPM_COMM_LOCAL)) for rk in range(G)]
res = {}
for mode in ("0", "1"):
    hs[0].set_plan_opts(no_fused_halo=int(mode))
    t, mu = timed(lambda: kpm.kpm_moments_group(hs, N, R, seed))
    res["fused" if mode == "0" else "copies"] = (t, float(abs(mu - mu_whole).max()), hs[0].last_stats())
print({"config": sys.argv[1] if len(sys.argv) > 1 else "c3", "slabs": G, "devices": ndev, "whole_ms": t_whole, **res})
