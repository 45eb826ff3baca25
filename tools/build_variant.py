"""Build an A/B variant of the library with extra nvcc flags:
python tools/build_variant.py TAG -DH2G_X=Y ...  ->  paper_2502_02395_b200/libh2ulv_b200_TAG.so
(select it at run time with H2G_LIB_PATH)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2502_02395_b200 import _build as b  # noqa: E402

tag, extra = sys.argv[1], sys.argv[2:]
b.LIB = os.path.join(b.HERE, f"libh2ulv_b200_{tag}.so")
b.OBJ_DIR = os.path.join(b.HERE, "build", tag)
print(b.build(force=True, extra=extra))
