"""Experiments only: build libhcspmm.so with extra -D flags into tools/exp_libs/<name>/ (load it
with HCS_LIB_PATH).  Usage: python tools/build_variant.py NAME -DFLAG ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_08902_b200 import _build as b

name, flags = sys.argv[1], sys.argv[2:]
out = os.path.join(b.ROOT, "tools", "exp_libs", name)
os.makedirs(out, exist_ok=True)
b.BUILD = os.path.join(out, "obj")
b.LIB = os.path.join(out, "libhcspmm.so")
b.NVCC_FLAGS = b.NVCC_FLAGS + flags
print(b.build())
