"""Build an A/B variant of libhcg.so with extra nvcc defines and the tuning
switches (HCG_NO_UNIONLESS, HCG_NO_QSORT, ... read from the environment, which
the release library ignores) compiled in; load it with HCG_LIB_OVERRIDE=<path>.

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
# every .cu with the defines (and the A/B environment switches compiled in)
objs = []
for s in B.CU:
    o = os.path.join(out_dir, s + ".o")
    subprocess.run([B._nvcc()] + B.NVCC_FLAGS + ["-DHCG_TUNING_KNOBS"] + defs + ["-c", os.path.join(B.CSRC, s), "-o", o],
                   check=True)
    objs.append(o)
objs += [os.path.join(B.OBJ, s + ".o") for s in B.CPP]
lib = os.path.join(out_dir, f"libhcg_{name}.so")
subprocess.run([B._nvcc(), "-shared"] + B.ARCH + ["-cudart", "static", "-o", lib] + objs + ["-ldl"], check=True)
print(lib)
