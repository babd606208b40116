"""Compile a variant of csrc/ (a copy under scratch/) into a .so for A/B runs (scripts/r02_var.sh).
usage: build_variant.py <csrc dir> <out.so> [-Dmacro ...]"""
import os, subprocess, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "paper_1105_5481_b200"))
import build  # noqa: E402
src, out, extra = sys.argv[1], sys.argv[2], tuple(sys.argv[3:])
cmd = build._cmd(out, extra)
cmd[cmd.index(os.path.join(build.HERE, "csrc", "kpm_capi.cu"))] = os.path.join(src, "kpm_capi.cu")
subprocess.check_call(cmd)
os.replace(out + ".tmp", out)
