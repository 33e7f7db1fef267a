#!/bin/bash
# round 2: where the MMA warp waits (V / K arrival) and whether L2-resident K/V
# (every CTA on KV head 0) changes the period
O=gpurun_out; mkdir -p $O
for v in trace samekv; do
  for T in 16384 32768; do
    timeout 300 python scripts/prefill_trace.py --lib build/variants/$v/liblkv.so --tokens $T | sed "s/^/{\"lib\": \"$v\", \"trace\": /; s/\$/}/" >> $O/r2ad_prefill_trace.jsonl 2>> $O/r2ad.err
    timeout 300 python scripts/prefill_micro.py --lib build/variants/$v/liblkv.so --tokens $T --iters 5 --label $v >> $O/r2ad_prefill_micro.jsonl 2>> $O/r2ad.err
  done
done
