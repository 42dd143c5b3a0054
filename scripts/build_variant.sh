#!/bin/bash
# build libbfgpu.so with extra nvcc defines into variants/libbfgpu_$1.so
set -e
cd /root/repo
name=$1; shift
python - "$@" <<'PY'
import sys
from paper_2505_07829_b200 import _build
_build.NVCC_FLAGS = _build.NVCC_FLAGS + sys.argv[1:]
_build.OBJDIR = _build.ROOT / "build" / "obj_var"
_build.LIB = _build.LIBDIR / "libbfgpu_var.so"
print(_build.build())
PY
mv paper_2505_07829_b200/lib/libbfgpu_var.so variants/libbfgpu_$name.so
