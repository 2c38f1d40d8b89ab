"""Build a libosmpm variant with extra -D flags for A/B runs:
  python scripts/build_variant.py <out.so> -DOSMPM_SW_DEFER=0 ..."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2605_09097_b200"))
import build as B  # noqa: E402

out = sys.argv[1]
cmd = [B.NVCC, *B.FLAGS, *sys.argv[2:], *[os.path.join(B.CSRC, s) for s in B.SOURCES], "-o", out]
subprocess.check_call(cmd)
print(out)
