"""Build a tuning variant of libtp.so with extra -D flags (select it with TP_LIB_PATH).

usage: python tools/build_variant.py NAME -DMACRO=VALUE ...   -> paper_2408_05235_b200/libtp_NAME.so
"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as G  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(G.PKG, f"libtp_{name}.so")
srcs = sorted(glob.glob(os.path.join(G.PKG, "csrc", "*.cu")))
subprocess.check_call([G._nvcc()] + G.NVCC_FLAGS + defs + ["-I" + os.path.join(ROOT, "include"), "-o", out] + srcs)
print(out)
