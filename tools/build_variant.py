"""Diagnostic build of libmoa with extra nvcc defines (kernel tuning A/B runs).

    python tools/build_variant.py NAME -DMACRO=VALUE ...   -> tools/bin/libmoa_NAME.so

Load it with MOA_LIB=tools/bin/libmoa_NAME.so (tools only; the product loads the in-tree
paper_2406_14909_b200/libmoa.so).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2406_14909_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
b.NVCC_FLAGS = b.NVCC_FLAGS + defs
b.BUILD = os.path.join(ROOT, "tools", "bin", f"build_{name}")
b.LIB = os.path.join(ROOT, "tools", "bin", f"libmoa_{name}.so")
print(b.build())
