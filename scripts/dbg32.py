"""Debug driver: one small 3D lattice through the 3D two-step kernel (kpm_tma32.cuh)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kpm_inputs as ki
from paper_1105_5481_b200 import kpm

W = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0
L = (16, 16, 8)
D = L[0] * L[1] * L[2]
on = ki.anderson_onsite(5, D, W) if W else None
a, b = kpm.kpm_gershgorin_stencil(3, L, -1.0, onsite=on)
h = kpm.kpm_create_stencil(3, L, -1.0, a, b, onsite=on)
os.environ["KPM_NO_SMALL"] = "1"
print("plan", h.plan_info(12, 16))
mu = h.moments(12, 16, 3)
os.environ["KPM_NO_TMA32"] = "1"
mu1 = h.moments(12, 16, 3)
print("W", W, "max diff vs single-step", np.abs(mu - mu1).max())
