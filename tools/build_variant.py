"""Build an A/B variant of libhcg.so with extra nvcc defines for search.cu
(tuning experiments; load it with HCG_LIB_OVERRIDE=<path>).

    python tools/build_variant.py minb3 -DHCG_NU_MINB4=3 -DHCG_NU_MINB8=3
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1209_0410_b200 import _build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
B.build()
out_dir = os.path.join(B.CSRC, "build-" + name)
os.makedirs(out_dir, exist_ok=True)
obj = os.path.join(out_dir, "search.cu.o")
subprocess.run([B._nvcc()] + B.NVCC_FLAGS + defs + ["-c", os.path.join(B.CSRC, "search.cu"), "-o", obj], check=True)
objs = [obj if s == "search.cu" else os.path.join(B.OBJ, s + ".o") for s in B.CU + B.CPP]
lib = os.path.join(out_dir, f"libhcg_{name}.so")
subprocess.run([B._nvcc(), "-shared"] + B.ARCH + ["-cudart", "static", "-o", lib] + objs + ["-ldl"], check=True)
print(lib)
