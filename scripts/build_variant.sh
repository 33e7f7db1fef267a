#!/bin/bash
# Build an experimental variant of liblkv.so (build-time defines only; the
# shipped library has no runtime switches) into build/variants/<name>/.
#   bash scripts/build_variant.sh trace "-DLKV_PREFILL_TRACE=1"   (scripts/prefill_trace.py)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; DEFS=$2
make -s -C "$ROOT/paper_2410_00428_b200" -j8 BUILD="$ROOT/build/variants/$NAME/obj" \
  LIB="$ROOT/build/variants/$NAME/liblkv.so" EXTRA_NVFLAGS="$DEFS"
echo "$ROOT/build/variants/$NAME/liblkv.so"
