#!/bin/bash
# round 2: prefill phase trace with the poly share 0 / 1/4 / 1/2
O=gpurun_out; mkdir -p $O
for v in trace tracep1 tracep2; do
  timeout 300 python scripts/prefill_trace.py --lib build/variants/$v/liblkv.so --tokens 32768 | sed "s/^/{\"lib\": \"$v\", \"trace\": /; s/\$/}/" >> $O/r2v_prefill_trace.jsonl 2>> $O/r2v_prefill_trace.err
done
