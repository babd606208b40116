import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# The persistent L2-resident kernel (kpm_persist.cuh) is opt-in (KPM_PERSIST=1); its own tests
# (test_persistent_kernel_matches_oracle) switch it on, everything else runs the per-step kernels.
os.environ.setdefault("KPM_NO_PERSIST", "1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running (full-size sampled parity)")
