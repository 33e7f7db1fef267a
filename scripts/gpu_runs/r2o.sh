#!/bin/bash
# round 2: prefill with three aligned warpgroups + setmaxnreg (WG3, no spills)
# against the product kernel; tier read-ahead slack 1 (ra1) against 2.
O=gpurun_out; mkdir -p $O
v=wg3
rm -rf /tmp/v_$v && mkdir -p /tmp/v_$v && tar --exclude=.git --exclude=gpurun_out -cf - . | tar -C /tmp/v_$v -xf -
cp build/variants/$v/liblkv.so /tmp/v_$v/paper_2410_00428_b200/liblkv.so
(cd /tmp/v_$v && timeout 600 python -m pytest tests/test_prefill_attention.py -m gpu -q -p no:cacheprovider 2>&1 | tail -3) > $O/r2o_pytest_prefill_$v.txt
for rep in 1 2; do
for T in 4096 16384 32768; do
  for v in product wg3; do
    lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
    timeout 300 python scripts/prefill_micro.py --tokens $T --iters 5 $lib --label $v >> $O/r2o_prefill_micro.jsonl 2>> $O/r2o_prefill_micro.err
  done
done
done
for v in product wg3; do
  lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
  timeout 300 python scripts/prefill_micro.py --tokens 16384 --hkv 32 --iters 5 $lib --label $v >> $O/r2o_prefill_micro.jsonl 2>> $O/r2o_prefill_micro.err
done
v=ra1
rm -rf /tmp/v_$v && mkdir -p /tmp/v_$v && tar --exclude=.git --exclude=gpurun_out -cf - . | tar -C /tmp/v_$v -xf -
cp build/variants/$v/liblkv.so /tmp/v_$v/paper_2410_00428_b200/liblkv.so
for rep in 1 2; do
  timeout 300 python scripts/tier_micro.py >> $O/r2o_tier_micro_product.jsonl 2>> $O/r2o_tier.err
  (cd /tmp/v_$v && timeout 300 python scripts/tier_micro.py) >> $O/r2o_tier_micro_ra1.jsonl 2>> $O/r2o_tier.err
done
