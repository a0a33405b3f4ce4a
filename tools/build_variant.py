"""Build a tuning variant of libnulpa.so next to the product library, for A/B runs on the
GPU box without rebuilding there:

    python tools/build_variant.py NAME "-DNULPA_X=1 -DNULPA_Y=2"
    NULPA_LIB=paper_2411_11468_b200/var/libnulpa_NAME.so python bench.py ...

Only the sources compiled with nvcc are rebuilt (into build/var_NAME/); the C++ host
objects are shared with the product build.
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_11468_b200 import build as b  # noqa: E402

name, flags = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
b.EXTRA_NVCC = flags.split()
b.OBJ = b.ROOT / "build" / f"var_{name}"
out = b.PKG / "var"
out.mkdir(exist_ok=True)
b.LIB = out / f"libnulpa_{name}.so"
b.build_library()
print(b.LIB, os.path.getsize(b.LIB))
