#!/bin/bash
# round 2: speculative exponentials with the bulk S load (spec2) vs product:
# parity, micro (burst), sustained clocks, phase trace
O=gpurun_out; mkdir -p $O
v=spec2
rm -rf /tmp/v_$v && mkdir -p /tmp/v_$v && tar --exclude=.git --exclude=gpurun_out -cf - . | tar -C /tmp/v_$v -xf -
cp build/variants/$v/liblkv.so /tmp/v_$v/paper_2410_00428_b200/liblkv.so
(cd /tmp/v_$v && timeout 600 python -m pytest tests/test_prefill_attention.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2) > $O/r2ag_pytest_$v.txt
for rep in 1 2; do
for T in 4096 16384 32768; do
  for v in product spec2; do
    lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
    timeout 300 python scripts/prefill_micro.py --tokens $T --iters 5 $lib --label $v >> $O/r2ag_prefill_micro.jsonl 2>> $O/r2ag.err
  done
done
done
for v in product spec2; do
  lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
  timeout 120 python scripts/prefill_clocks.py --tokens 16384 $lib --label $v >> $O/r2ag_prefill_clocks.jsonl 2>> $O/r2ag.err
done
for v in trace spec2trace; do
  timeout 300 python scripts/prefill_trace.py --lib build/variants/$v/liblkv.so --tokens 16384 | sed "s/^/{\"lib\": \"$v\", \"trace\": /; s/\$/}/" >> $O/r2ag_prefill_trace.jsonl 2>> $O/r2ag.err
done
