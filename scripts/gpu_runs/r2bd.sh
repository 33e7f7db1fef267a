#!/bin/bash
# round 2: S loaded in two halves, the first half's max under the second half's load (product) vs one bulk load (sload1)

O=gpurun_out; mkdir -p $O
timeout 300 python -m pytest tests/test_prefill_attention.py -m gpu -q -x > $O/r2bd_pytest.txt 2>&1; echo "pytest rc=$?"
for rep in 1 2 3; do
for T in 4096 16384 32768; do
  for v in sload1 product; do
    lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
    timeout 120 python scripts/prefill_micro.py --tokens $T --iters 5 $lib --label $v >> $O/r2bd_prefill_micro.jsonl 2>> $O/r2bd_prefill_micro.err
  done
done
done
