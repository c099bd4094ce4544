"""Build an A/B variant of libhmx.so with extra nvcc flags (e.g. -D...).

python tools/build_variant.py SUFFIX [nvcc flags...]  ->  paper_1911_07531_b200/libhmxSUFFIX.so
Load it with HMX_LIB=$PWD/paper_1911_07531_b200/libhmxSUFFIX.so (tools only).
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_07531_b200 import _build as B  # noqa: E402

suf, extra = sys.argv[1], sys.argv[2:]
objs = []
for s in B.SOURCES:
    o = os.path.join("/tmp", f"{os.path.splitext(s)[0]}{suf}.o")
    subprocess.check_call([B._nvcc(), *B.NVCC_FLAGS, *extra, "-c", "-o", o, os.path.join(B.CSRC, s)],
                          stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    objs.append(o)
out = os.path.join(B.HERE, f"libhmx{suf}.so")
subprocess.check_call([B._nvcc(), *B.ARCH, "-shared", "-o", out, *objs])
print(out)
