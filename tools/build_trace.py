"""Diagnostic build: libmoa with the decode kernel's %globaltimer trace (-DMOA_DEC_TRACE).

    python tools/build_trace.py      -> tools/bin/libmoa_trace.so

Load it with MOA_LIB=tools/bin/libmoa_trace.so (tools only; the product loads the in-tree
paper_2406_14909_b200/libmoa.so) and read the stamps with moa_debug_decode_trace().
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2406_14909_b200 import build as b  # noqa: E402

b.NVCC_FLAGS = b.NVCC_FLAGS + ["-DMOA_DEC_TRACE"]
b.BUILD = os.path.join(ROOT, "tools", "bin", "trace_build")
b.LIB = os.path.join(ROOT, "tools", "bin", "libmoa_trace.so")
print(b.build())
