#!/bin/bash
# round 2: timing probe — does switching the MMA operand format between the
# bf16 QK^T and the fp16 PV cost tensor throughput? pvbf16: PV issued as bf16,
# sf16: QK^T issued as fp16 (both wrong numerics, same data movement), against
# the shipped kernel (mixed)
O=gpurun_out; mkdir -p $O
for rep in 1 2 3; do
for T in 4096 16384 32768; do
  for v in pvbf16 sf16 product; do
    lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
    timeout 120 python scripts/prefill_micro.py --tokens $T --iters 5 $lib --label $v >> $O/r2ay_prefill_micro.jsonl 2>> $O/r2ay_prefill_micro.err
  done
done
done
