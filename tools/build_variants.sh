#!/bin/bash
# Dev only: build libib_b200 variants with extra -D flags into build_variants/<name>.so
# usage: tools/build_variants.sh name "-DFOO -DBAR" [name2 "flags2" ...]
set -e
cd "$(dirname "$0")/.."
mkdir -p build_variants
while [ $# -ge 2 ]; do
  python -c "
import sys; sys.path.insert(0, '.')
from paper_math_0301321_b200 import _build
_build.build(force=True, extra='$2'.split(), out='build_variants/$1.so')" 2>&1 | grep -v Remark | grep -E "error" || true
  echo "built build_variants/$1.so"
  shift 2
done
