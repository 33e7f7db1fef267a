#!/bin/bash
# round 2: prefill phase trace (clock64) of CTA 0 at 16k and 32k
O=gpurun_out; mkdir -p $O
for T in 16384 32768; do
  timeout 300 python scripts/prefill_trace.py --lib build/variants/trace/liblkv.so --tokens $T >> $O/r2u_prefill_trace.jsonl 2>> $O/r2u_prefill_trace.err
done
