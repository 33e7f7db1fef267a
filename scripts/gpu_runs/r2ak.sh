#!/bin/bash
# round 2: P handed to the PV MMAs in 1 / 2 / 4 parts per KV tile (pc1, pc2, product = 4) against the committed kernel (base)
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_prefill_attention.py -m gpu -q -x > $O/r2ak_pytest.txt 2>&1; echo "pytest rc=$?"
for rep in 1 2; do
for T in 4096 16384 32768; do
  for v in base pc1 pc2 product; do
    lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
    timeout 300 python scripts/prefill_micro.py --tokens $T --iters 5 $lib --label $v >> $O/r2ak_prefill_micro.jsonl 2>> $O/r2ak_prefill_micro.err
  done
done
done
