#!/bin/bash
# round 2: prefill per-CTA timeline (%globaltimer) at 4k / 16k / 32k
O=gpurun_out; mkdir -p $O
for T in 4096 16384 32768; do
  timeout 300 python scripts/prefill_trace.py --lib build/variants/trace/liblkv.so --tokens $T >> $O/r2x_prefill_trace.jsonl 2>> $O/r2x.err
done
