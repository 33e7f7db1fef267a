#!/bin/bash
# round 2: prefill A/B on the restored two-tile kernel — packed-poly share
# (POLY 1/2) and the register budget (maxnreg 200, no spills) — plus an ncu
# source capture of the product kernel; then sanitizers, mutation check and
# the N=2-ranks-on-one-GPU bench path (r2g).
O=gpurun_out; mkdir -p $O
timeout 900 python bench.py > $O/r2i_bench.json 2> $O/r2i_bench.err; echo "bench rc=$?"
for rep in 1 2; do
for T in 4096 16384 32768; do
  for v in product poly1 poly2 r200 r200p1; do
    lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
    timeout 300 python scripts/prefill_micro.py --tokens $T --iters 5 $lib --label $v >> $O/r2i_prefill_micro.jsonl 2>> $O/r2i_prefill_micro.err
  done
done
done
for v in product poly1 r200 r200p1; do
  lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
  timeout 300 python scripts/prefill_micro.py --tokens 16384 --hkv 32 --iters 5 $lib --label $v >> $O/r2i_prefill_micro.jsonl 2>> $O/r2i_prefill_micro.err
done
for v in poly1 r200 r200p1; do  # parity of each variant: a repo copy with its library in the product's place
  rm -rf /tmp/v_$v && mkdir -p /tmp/v_$v && tar --exclude=.git --exclude=gpurun_out -cf - . | tar -C /tmp/v_$v -xf -
  cp build/variants/$v/liblkv.so /tmp/v_$v/paper_2410_00428_b200/liblkv.so
  (cd /tmp/v_$v && timeout 600 python -m pytest tests/test_prefill_attention.py -m gpu -q -p no:cacheprovider 2>&1 | tail -3) > $O/r2i_pytest_prefill_$v.txt
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_attn2 -c 1 \
  -o $O/r2i_prefill_attn2 -f python scripts/prefill_micro.py --tokens 16384 --iters 1 > $O/r2i_ncu_pf.log 2>&1; echo "ncu rc=$?"
bash scripts/gpu_runs/r2g.sh
