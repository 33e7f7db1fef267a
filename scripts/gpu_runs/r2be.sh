#!/bin/bash
# round 2: sustained (back to back, 4 s, power-capped) prefill attention, ours
# against cuDNN SDPA on the same shape, with clocks and power
O=gpurun_out; mkdir -p $O
for rep in 1 2; do
for T in 16384 32768; do
  timeout 120 python scripts/prefill_clocks.py --tokens $T --seconds 4 >> $O/r2be_prefill_sustained.jsonl 2>> $O/r2be.err
  timeout 120 python scripts/prefill_clocks.py --tokens $T --seconds 4 --cudnn --label cudnn >> $O/r2be_prefill_sustained.jsonl 2>> $O/r2be.err
done
done
