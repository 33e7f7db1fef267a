#!/bin/bash
# round 2: split-merge warps per CTA (w2, w8) against the shipped 4, on the
# headline G=1 shape (7 x 16k, 7B) and the 70B TP8 shard (G=8, 64 x 32k):
# attention + merge as one event interval per layer
O=gpurun_out; mkdir -p $O
for rep in 1 2 3; do
  for v in w2 w8 product; do
    lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
    timeout 300 python scripts/attn_micro.py --group 1 --batch 7 --ctx 16384 --layers 4 $lib --label $v >> $O/r2az_attn_micro.jsonl 2>> $O/r2az_attn_micro.err
    timeout 300 python scripts/attn_micro.py --group 8 --hkv 1 --batch 64 --ctx 32768 --layers 2 $lib --label $v >> $O/r2az_attn_micro.jsonl 2>> $O/r2az_attn_micro.err
  done
done
