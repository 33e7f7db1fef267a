#!/bin/bash
# round 2: clocks / power during back-to-back prefill attention (product, poly 1/4)
O=gpurun_out; mkdir -p $O
nvidia-smi -q -d POWER > $O/r2w_power_limits.txt 2>&1
for T in 16384 32768; do
  timeout 120 python scripts/prefill_clocks.py --tokens $T >> $O/r2w_prefill_clocks.jsonl 2>> $O/r2w.err
  timeout 120 python scripts/prefill_clocks.py --tokens $T --lib build/variants/p1/liblkv.so --label p1 >> $O/r2w_prefill_clocks.jsonl 2>> $O/r2w.err
done
