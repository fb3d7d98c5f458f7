"""Build a variant of libnsg with extra nvcc defines into tools/libnsg_<name>.so (timing experiments).

usage: python tools/build_variant.py NAME [-DMACRO[=V] ...]
Run it with NSG_LIB_PATH_DEV=tools/libnsg_<name>.so to load the variant instead of the product build.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_03653_b200 import _lib  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "tools", f"libnsg_{name}.so")
subprocess.check_call(["nvcc", *_lib.NVCC_FLAGS, *defs, "-I", os.path.join(ROOT, "include"), "-o", out, _lib.SOURCES[0]])
print(out)
