#!/bin/bash
# round 2: clock64 phase trace of the softmax ping-pong (trace_pp) against the
# same kernel without it (trace_nopp), 16k and 32k
O=gpurun_out; mkdir -p $O
for T in 16384 32768; do
  for v in trace_pp trace_nopp; do
    echo "{\"variant\": \"$v\"}" >> $O/r2am_prefill_trace.jsonl
    timeout 300 python scripts/prefill_trace.py --lib build/variants/$v/liblkv.so --tokens $T >> $O/r2am_prefill_trace.jsonl 2>> $O/r2am_prefill_trace.err
  done
done
