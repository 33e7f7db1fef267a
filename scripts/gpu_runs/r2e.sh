#!/bin/bash
# round 2: prefill attention rework — pipe-rate probe, parity of the new kernel
# (product = POLY 0) and its POLY 1/2 variants, A/B micro against the round-1
# kernel (build/variants/attn2_r1), ncu capture of the new kernel.
O=gpurun_out; mkdir -p $O
timeout 300 ./build/pipe_probe > $O/r2e_pipe_probe.jsonl 2>&1; echo "probe rc=$?"
timeout 900 python -m pytest tests/test_prefill_attention.py -m gpu -q > $O/r2e_pytest_prefill.txt 2>&1; echo "pytest prefill rc=$?"
for v in poly1 poly2 gridall; do
  rm -rf /tmp/v_$v && mkdir -p /tmp/v_$v && tar --exclude=.git --exclude=gpurun_out -cf - . | tar -C /tmp/v_$v -xf -
  cp build/variants/$v/liblkv.so /tmp/v_$v/paper_2410_00428_b200/liblkv.so
  (cd /tmp/v_$v && timeout 900 python -m pytest tests/test_prefill_attention.py -m gpu -q -p no:cacheprovider 2>&1 | tail -3) > $O/r2e_pytest_prefill_$v.txt; echo "pytest $v done"
done
for T in 4096 16384 32768; do
  for v in attn2_r1 product poly1 poly2 gridall poly1_gridall; do
    lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
    timeout 300 python scripts/prefill_micro.py --tokens $T --iters 5 $lib --label $v >> $O/r2e_prefill_micro.jsonl 2>> $O/r2e_prefill_micro.err
  done
done
for v in attn2_r1 product poly1 gridall; do
  lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
  timeout 300 python scripts/prefill_micro.py --tokens 16384 --hkv 32 --iters 5 $lib --label $v >> $O/r2e_prefill_micro.jsonl 2>> $O/r2e_prefill_micro.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_attn2 -c 1 \
  -o $O/r2e_prefill_attn2 -f python scripts/prefill_micro.py --tokens 8192 --iters 1 > $O/r2e_ncu_pf.log 2>&1; echo "ncu rc=$?"
