"""Build a variant of librsw.so with extra nvcc defines, for A/B measurements on the GPU box
(select it there with RSW_LIB=<path>).  Not part of the product build.

  python tools/build_variant.py OUT.so -DRSW_FINE_TWT=0 [-D...]
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1303_6615_b200 import build as b  # noqa: E402


def main(out, defines):
    objdir = os.path.join(os.path.dirname(os.path.abspath(out)), "build_" + os.path.basename(out).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    jobs, objs = [], []
    for src in b.SOURCES:
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        objs.append(obj)
        cmd = b.compile_cmd(os.path.join(b.CSRC, src), obj)
        cmd[-4:-4] = defines
        jobs.append((subprocess.Popen(cmd), cmd))
    for p, cmd in jobs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, cmd)
    subprocess.check_call(b.link_cmd(objs, out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
