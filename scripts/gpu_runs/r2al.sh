#!/bin/bash
# round 2: softmax ping-pong (product: pp + P in 2 parts; pp1, pp4) against pc2 (no ping-pong) and base (committed)
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_prefill_attention.py -m gpu -q -x > $O/r2al_pytest.txt 2>&1; echo "pytest rc=$?"
for rep in 1 2; do
for T in 4096 16384 32768; do
  for v in base pc2 pp1 pp4 product; do
    lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
    timeout 300 python scripts/prefill_micro.py --tokens $T --iters 5 $lib --label $v >> $O/r2al_prefill_micro.jsonl 2>> $O/r2al_prefill_micro.err
  done
done
done
