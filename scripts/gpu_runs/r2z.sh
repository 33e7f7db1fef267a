#!/bin/bash
# round 2: same-box A/B of the prefill launch forms: head (grid of pairs,
# in-kernel dispatch order), product (per-CTA item lists, one item each),
# persist (persistent LPT lists)
O=gpurun_out; mkdir -p $O
for rep in 1 2 3; do
for T in 4096 16384 32768; do
  for v in head product persist; do
    lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
    timeout 300 python scripts/prefill_micro.py --tokens $T --iters 5 $lib --label $v >> $O/r2z_prefill_micro.jsonl 2>> $O/r2z_prefill_micro.err
  done
done
done
