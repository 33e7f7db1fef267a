#!/bin/bash
# round 2: row max as 16 independent 3-input chains + tree (product) against
# the 4-chain max (nomaxtree); prefill parity on the product
O=gpurun_out; mkdir -p $O
timeout 300 python -m pytest tests/test_prefill_attention.py -m gpu -q -x > $O/r2ar_pytest.txt 2>&1; echo "pytest rc=$?"
for rep in 1 2 3; do
for T in 4096 16384 32768; do
  for v in nomaxtree product; do
    lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
    timeout 120 python scripts/prefill_micro.py --tokens $T --iters 5 $lib --label $v >> $O/r2ar_prefill_micro.jsonl 2>> $O/r2ar_prefill_micro.err
  done
done
done
