#!/bin/bash
# round 2: prefill dispatch-chunk L2 budget (4 / 48 / 256 MB of K+V per chunk
# vs the shipped 16) on MHA (7B heads, Hq = Hkv = 32) at 4k / 16k / 32k
O=gpurun_out; mkdir -p $O
for rep in 1 2; do
for T in 4096 16384 32768; do
  for v in l2_4 l2_48 l2_256 product; do
    lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
    timeout 120 python scripts/prefill_micro.py --tokens $T --hq 32 --hkv 32 --iters 5 $lib --label $v >> $O/r2bh_prefill_micro.jsonl 2>> $O/r2bh_prefill_micro.err
  done
done
done
