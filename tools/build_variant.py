"""Build a libqgear_b200 variant with extra nvcc defines for fused.cu (dev tool):
    python tools/build_variant.py NAME -DFOO=1 ...   -> gpu_variants/libqgear_b200_NAME.so
Load it with QG_LIB_PATH=gpu_variants/libqgear_b200_NAME.so."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_03967_b200 import build as B

name, defs = sys.argv[1], sys.argv[2:]
B.build()
out_dir = os.path.join(B.ROOT, "gpu_variants")  # not under build/: must travel with gpurun
os.makedirs(out_dir, exist_ok=True)
obj = os.path.join(out_dir, f"fused_{name}.o")
r = subprocess.run([B.NVCC, *B.ARCH, *B.FLAGS, *defs, "-c", os.path.join(B.CSRC, "fused.cu"), "-o", obj],
                   capture_output=True, text=True)
assert r.returncode == 0, r.stderr
objs = [os.path.join(B.BUILD, os.path.splitext(s)[0] + ".o") for s in B.SOURCES if s != "fused.cu"] + [obj]
lib = os.path.join(out_dir, f"libqgear_b200_{name}.so")
r = subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", lib, *objs, "-cudart", "static"], capture_output=True, text=True)
assert r.returncode == 0, r.stderr
print(lib)
