#!/bin/bash
# round 2: prefill kernel on per-CTA item lists — product (one item per CTA)
# and the persistent LPT variant: parity, micro at 4k / 16k / 32k / 16k MHA.
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_prefill_attention.py -m gpu -q -p no:cacheprovider > $O/r2y_pytest_prefill_product.txt 2>&1; echo "product parity rc=$?"
v=persist
rm -rf /tmp/v_$v && mkdir -p /tmp/v_$v && tar --exclude=.git --exclude=gpurun_out -cf - . | tar -C /tmp/v_$v -xf -
cp build/variants/$v/liblkv.so /tmp/v_$v/paper_2410_00428_b200/liblkv.so
(cd /tmp/v_$v && timeout 600 python -m pytest tests/test_prefill_attention.py -m gpu -q -p no:cacheprovider 2>&1 | tail -3) > $O/r2y_pytest_prefill_$v.txt
for rep in 1 2; do
for T in 4096 8192 16384 32768; do
  for v in product persist; do
    lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
    timeout 300 python scripts/prefill_micro.py --tokens $T --iters 5 $lib --label $v >> $O/r2y_prefill_micro.jsonl 2>> $O/r2y_prefill_micro.err
  done
done
done
for v in product persist; do
  lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
  timeout 300 python scripts/prefill_micro.py --tokens 16384 --hkv 32 --iters 5 $lib --label $v >> $O/r2y_prefill_micro.jsonl 2>> $O/r2y_prefill_micro.err
done
