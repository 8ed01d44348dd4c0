"""Build an experimental variant of libmlk (extra nvcc defines) as the in-tree
libmlk_<name>.so, loaded with MLK_LIB_VARIANT=<name> (A/B timing on one GPU box).

    python tools/build_variant.py occ5 -DMLK_K5A_OCC5
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1701_00285_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
B.OBJ = os.path.join(B.HERE, "build_" + name)
B.LIB = os.path.join(B.HERE, "libmlk_%s.so" % name)
B.FLAGS = B.FLAGS + defs
print(B.build(verbose=False))
