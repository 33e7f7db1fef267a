#!/bin/bash
# round 2 (re-entry): full GPU suite + smoke on HEAD (prefill rework), prefill
# A/B against the pre-rework kernel (build/variants/attn2_r1), bench both arms,
# ncu launch list and one full capture of the new prefill kernel.
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/r2f_gpu.txt 2>&1
timeout 900 python -m pytest tests/test_prefill_attention.py -m gpu -q > $O/r2f_pytest_prefill.txt 2>&1; echo "pytest prefill rc=$?"
for T in 4096 16384 32768; do
  for v in attn2_r1 product poly1 gridall; do
    lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
    timeout 300 python scripts/prefill_micro.py --tokens $T --iters 5 $lib --label $v >> $O/r2f_prefill_micro.jsonl 2>> $O/r2f_prefill_micro.err
  done
done
for v in attn2_r1 product; do
  lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
  timeout 300 python scripts/prefill_micro.py --tokens 16384 --hkv 32 --iters 5 $lib --label $v >> $O/r2f_prefill_micro.jsonl 2>> $O/r2f_prefill_micro.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_attn2 -c 1 \
  -o $O/r2f_prefill_attn2 -f python scripts/prefill_micro.py --tokens 16384 --iters 1 > $O/r2f_ncu_pf.log 2>&1; echo "ncu rc=$?"
timeout 1500 python -m pytest tests -m gpu -q > $O/r2f_pytest.txt 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2f_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/r2f_bench.json 2> $O/r2f_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $O/r2f_bench_ref.json 2> $O/r2f_bench_ref.err; echo "ref rc=$?"
