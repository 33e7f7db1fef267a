#!/bin/bash
# round 2: on the WG3 kernel (now the product): packed-poly share 1/4 (p1),
# speculative exps (spec), both (specp1).
O=gpurun_out; mkdir -p $O
for v in p1 spec specp1; do
  rm -rf /tmp/v_$v && mkdir -p /tmp/v_$v && tar --exclude=.git --exclude=gpurun_out -cf - . | tar -C /tmp/v_$v -xf -
  cp build/variants/$v/liblkv.so /tmp/v_$v/paper_2410_00428_b200/liblkv.so
  (cd /tmp/v_$v && timeout 600 python -m pytest tests/test_prefill_attention.py -m gpu -q -p no:cacheprovider 2>&1 | tail -1) > $O/r2p_pytest_prefill_$v.txt
done
for rep in 1 2; do
for T in 4096 16384 32768; do
  for v in product p1 spec specp1; do
    lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
    timeout 300 python scripts/prefill_micro.py --tokens $T --iters 5 $lib --label $v >> $O/r2p_prefill_micro.jsonl 2>> $O/r2p_prefill_micro.err
  done
done
done
