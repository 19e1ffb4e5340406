"""Build a tuning variant of libtp.so with extra -D flags (select it with TP_LIB_PATH).

usage: python tools/build_variant.py NAME [--only file.cu ...] -DMACRO=VALUE ...
       -> paper_2408_05235_b200/libtp_NAME.so
With --only, just those sources are recompiled with the flags; the rest link from the objects of the
regular build (csrc/build, produced by __graft_entry__.build_lib()).
"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as G  # noqa: E402

args = sys.argv[1:]
name = args.pop(0)
only = []
while args and args[0] == "--only":
    args.pop(0)
    only.append(args.pop(0))
defs = args
out = os.path.join(G.PKG, f"libtp_{name}.so")
srcs = sorted(glob.glob(os.path.join(G.PKG, "csrc", "*.cu")))
if not only:
    subprocess.check_call([G._nvcc()] + G.NVCC_FLAGS + defs + ["-I" + os.path.join(ROOT, "include"), "-o", out] + srcs)
else:
    G.build_lib()
    cflags = [f for f in G.NVCC_FLAGS if f != "-shared"]
    objs = []
    for src in srcs:
        base = os.path.basename(src)[:-3]
        if os.path.basename(src) in only:
            obj = os.path.join(G.PKG, "csrc", "build", f"{base}_{name}.o")
            subprocess.check_call([G._nvcc()] + cflags + defs + ["-I" + os.path.join(ROOT, "include"), "-c", src,
                                   "-o", obj])
        else:
            obj = os.path.join(G.PKG, "csrc", "build", f"{base}.o")
        objs.append(obj)
    subprocess.check_call([G._nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out] + objs)
print(out)
