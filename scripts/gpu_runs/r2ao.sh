#!/bin/bash
# round 2 (r2an hung: setmaxnreg.inc 112 exceeded what warpgroup 0 released; now 104): two softmax warpgroups per query tile (product: 640 threads, 64
# columns each, P in 2 parts; s2pc4: P in 4 parts) against one per tile (s1 =
# the r2ak pc2 kernel) and the committed kernel (base); prefill parity on the product
O=gpurun_out; mkdir -p $O
timeout 300 python -m pytest tests/test_prefill_attention.py -m gpu -q -x > $O/r2ao_pytest.txt 2>&1; echo "pytest rc=$?"
for rep in 1 2; do
for T in 4096 16384 32768; do
  for v in base s1 s2pc4 product; do
    lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
    timeout 120 python scripts/prefill_micro.py --tokens $T --iters 5 $lib --label $v >> $O/r2ao_prefill_micro.jsonl 2>> $O/r2ao_prefill_micro.err
  done
done
done
