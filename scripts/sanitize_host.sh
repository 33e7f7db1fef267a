#!/bin/bash
# Host-side sanitizer runs: the CPU test suite
# against an ASan+UBSan build of liblkv.so, and the host-tier concurrency
# stress (scripts/tier_stress.cpp) under TSan and under ASan+UBSan.
# The product library and package are not modified: the instrumented
# library is linked into a scratch copy of the repo under /tmp.
#   bash scripts/sanitize_host.sh [out_dir]
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=${1:-$ROOT/gpurun_out}
mkdir -p "$OUT"
CUDA=/usr/local/cuda
SAN=/tmp/lkv_san
rm -rf $SAN && mkdir -p $SAN/obj
INC="-I$ROOT/include -I$ROOT/paper_2410_00428_b200/csrc -I$CUDA/include"
FL="-fsanitize=address,undefined -fno-omit-frame-pointer -fno-sanitize-recover=undefined -g -O1"
cd "$ROOT/paper_2410_00428_b200/csrc"
for f in kv_manager cost_model interconnect prefill_span capi serve_trace serve_sched serve_engine; do
  g++ -std=c++20 -fPIC $FL $INC -c $f.cpp -o $SAN/obj/$f.o || exit 1
done
for f in device serve_device; do
  $CUDA/bin/nvcc -std=c++20 -O1 -g -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr \
    -Xcompiler -fPIC,-fsanitize=address,-fsanitize=undefined,-fno-omit-frame-pointer $INC -c $f.cu -o $SAN/obj/$f.o || exit 1
done
# scratch repo copy with the instrumented library in the product's place
tar -C "$ROOT" --exclude=.git --exclude=gpurun_out --exclude=build --exclude='*.so' -cf - . | (mkdir -p $SAN/repo && tar -C $SAN/repo -xf -)
cp -r "$ROOT/oracle/_ref" "$ROOT/oracle/_build" $SAN/repo/oracle/ 2>/dev/null
$CUDA/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $SAN/repo/paper_2410_00428_b200/liblkv.so $SAN/obj/*.o \
  -Xcompiler -fsanitize=address,-fsanitize=undefined -L$CUDA/lib64 -lcublas -lcudart -Xlinker -rpath=$CUDA/lib64 -lpthread -ldl -lrt || exit 1
ASAN_RT=$(g++ -print-file-name=libasan.so)
UBSAN_RT=$(g++ -print-file-name=libubsan.so)
{
  echo "== CPU suite (pytest -m 'not gpu') against liblkv.so built with $FL"
  cd $SAN/repo && LD_PRELOAD="$ASAN_RT $UBSAN_RT" ASAN_OPTIONS=detect_leaks=0:protect_shadow_gap=0:halt_on_error=1 \
    UBSAN_OPTIONS=print_stacktrace=1:halt_on_error=1 timeout 1800 python -m pytest tests -q -m "not gpu" -p no:cacheprovider 2>&1 | tail -15
  echo "rc=${PIPESTATUS[0]}"
} > "$OUT/sanitize_asan_ubsan_cpu_suite.txt" 2>&1
# host-tier stress: real HostTier code, CUDA calls replaced by a host-side stub
for mode in thread address; do
  extra=""; [ $mode = address ] && extra="-fsanitize=undefined"
  g++ -std=c++20 -O1 -g -fsanitize=$mode $extra -fno-omit-frame-pointer -I$ROOT/scripts/cuda_stub \
    -I$ROOT/paper_2410_00428_b200/csrc "$ROOT/scripts/tier_stress.cpp" -o $SAN/tier_stress_$mode -lpthread || exit 1
  {
    echo "== host-tier stress under -fsanitize=$mode $extra (scripts/tier_stress.cpp)"
    TSAN_OPTIONS=halt_on_error=1 ASAN_OPTIONS=halt_on_error=1 UBSAN_OPTIONS=halt_on_error=1:print_stacktrace=1 \
      timeout 900 $SAN/tier_stress_$mode 2>&1 | tail -30
    echo "rc=${PIPESTATUS[0]}"
  } > "$OUT/sanitize_tier_stress_$mode.txt" 2>&1
done
echo "sanitizer logs in $OUT"
