#!/bin/bash
# Mutation check of the decode parity tests (VERDICT r1 "what's weak" 1): each
# mutant breaks one running-max path of the decode kernels; the peaked-softmax
# tests must fail on it, and the uniform-q ragged test shows what the round-1
# suite alone would have missed. Run on a GPU box from the repo root:
#   bash scripts/mutation_check.sh > gpurun_out/mutation.txt 2>&1
set -u
ROOT=$(pwd)
T_TC_RISING='tests/test_device_gpu.py::test_attention_parity_peaked_softmax[4-16-rising]'
T_TC_EXTREME='tests/test_device_gpu.py::test_attention_parity_peaked_softmax[4-16-extreme]'
T_G1_RISING='tests/test_device_gpu.py::test_attention_parity_peaked_softmax[1-16-rising]'
T_UNIFORM='tests/test_device_gpu.py::test_attention_parity_ragged[4-16] tests/test_device_gpu.py::test_attention_parity_ragged[1-16]'
T_LONG_RISING='tests/test_device_gpu.py::test_attention_parity_peaked_long_units[4-rising]'
T_LONG_EXTREME='tests/test_device_gpu.py::test_attention_parity_peaked_long_units[4-extreme]'
T_G1_BENCH='tests/test_device_gpu.py::test_attention_parity_bench_shape_g1[rising]'
mutate() {  # name file sed-expr tests...
  local name=$1 file=$2 expr=$3; shift 3
  local dir=/tmp/mut_$name
  rm -rf $dir; mkdir -p $dir
  tar -C $ROOT --exclude=.git --exclude=gpurun_out --exclude=build -cf - . | tar -C $dir -xf -
  rm -f $dir/paper_2410_00428_b200/liblkv.so
  sed -i "$expr" $dir/$file
  if cmp -s $ROOT/$file $dir/$file; then echo "== $name: sed did not apply"; return; fi
  echo "== mutant $name: $(diff $ROOT/$file $dir/$file | grep '^>' | head -2 | tr -s ' ')"
  (cd $dir && make -s -C paper_2410_00428_b200 -j16 > /dev/null 2>&1) || { echo "build failed"; return; }
  for t in "$@"; do
    (cd $dir && timeout 600 python -m pytest $t -m gpu -q -p no:cacheprovider 2>&1 | tail -1 | sed "s|^|   $t: |")
  done
}
echo "== unmutated"
for t in "$T_TC_RISING" "$T_TC_EXTREME" "$T_G1_RISING" "$T_LONG_RISING" "$T_LONG_EXTREME" "$T_G1_BENCH" "$T_UNIFORM"; do
  timeout 600 python -m pytest $t -m gpu -q -p no:cacheprovider 2>&1 | tail -1 | sed "s|^|   $t: |"
done
# M1: the tcgen05 tile's lazy max never re-bases after the first tile (scores may exceed fp32's range)
mutate lazy_never paper_2410_00428_b200/csrc/decode_gqa_tc.cuh \
  's/raise |= s\[g\] > m_run\[g\] + kLazyMax;/raise |= (m_run[g] == -INFINITY) \&\& (s[g] > -INFINITY);/' \
  "$T_TC_RISING" "$T_TC_EXTREME" "$T_LONG_RISING" "$T_LONG_EXTREME" "$T_UNIFORM"
# M2: the tile's correction factor is dropped when the running max moves
mutate corr_one paper_2410_00428_b200/csrc/decode_gqa_tc.cuh \
  's/corr\[g\] = (m_run\[g\] == -INFINITY) ? 0.f : exp2f(m_run\[g\] - mnew);/corr[g] = (m_run[g] == -INFINITY) ? 0.f : 1.f;/' \
  "$T_TC_RISING" "$T_TC_EXTREME" "$T_LONG_RISING" "$T_LONG_EXTREME" "$T_UNIFORM"
# M3: the split merge stops rescaling its accumulator when a later partial has a larger max
mutate merge_rescale paper_2410_00428_b200/csrc/decode_attn.cuh \
  's/const float cs = (M == -INFINITY) ? 0.f : exp2f(M - mb);/const float cs = (M == -INFINITY) ? 0.f : 1.f;/' \
  "$T_TC_RISING" "$T_G1_RISING" "$T_UNIFORM"
# M4: the CUDA-core G=1 kernel (decode_attn_v2) drops its per-block correction
mutate v2_corr paper_2410_00428_b200/csrc/decode_attn.cuh \
  's/const float corr = (mrun\[g\] == -INFINITY) ? 0.f : exp2f(mrun\[g\] - mnew);/const float corr = (mrun[g] == -INFINITY) ? 0.f : 1.f;/' \
  "$T_G1_RISING" "$T_G1_BENCH" "$T_UNIFORM"
