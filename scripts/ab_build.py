"""Experiment builds: libseed variant with extra nvcc defines for one source -> ab/<name>.so
    python scripts/ab_build.py NAME SRC.cu|all -DFOO=1 ...   (then SEED_LIB=ab/NAME.so python ...)"""
import os
import subprocess
import sys

sys.path.insert(0, os.getcwd())
from paper_2406_18200_b200 import build as b

name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
b.build()
os.makedirs("ab", exist_ok=True)
srcs = [s for s in b.SOURCES if s.endswith(".cu")] if src == "all" else [src]
for one in srcs:
    r = subprocess.run([b.NVCC] + b.CU_FLAGS + defs + ["-c", os.path.join(b.CSRC, one), "-o", f"ab/{name}.{one}.o"],
                       capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stderr)
objs = [f"ab/{name}.{s}.o" if s in srcs else os.path.join(b.OBJ, s + ".o") for s in b.SOURCES]
r = subprocess.run([b.NVCC] + b.ARCH + ["-shared", "-cudart", "static", "-o", f"ab/{name}.so"] + objs +
                   ["-ldl", "-lpthread", "-lrt"], capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
print(f"ab/{name}.so")
