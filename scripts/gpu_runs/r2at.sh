#!/bin/bash
# round 2: S split (product: lower half of S(j+1) issued once the softmax holds S(j), P in the upper half; MMA warpgroup 80 registers) against the shipped kernel (nossplit)

O=gpurun_out; mkdir -p $O
timeout 300 python -m pytest tests/test_prefill_attention.py -m gpu -q -x > $O/r2at_pytest.txt 2>&1; echo "pytest rc=$?"
for rep in 1 2 3; do
for T in 4096 16384 32768; do
  for v in nossplit product; do
    lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
    timeout 120 python scripts/prefill_micro.py --tokens $T --iters 5 $lib --label $v >> $O/r2at_prefill_micro.jsonl 2>> $O/r2at_prefill_micro.err
  done
done
done
