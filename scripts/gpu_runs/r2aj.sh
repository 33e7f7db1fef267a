#!/bin/bash
# round 2: library prefill attention (cuDNN SDPA, flashinfer backends) on the
# prefill_micro shapes, beside the shipped kernel on the same box; smoke + bench
# on the restored tree
O=gpurun_out; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2aj_smoke.txt 2>&1; echo "smoke rc=$?"
for T in 4096 16384 32768; do
  timeout 300 python scripts/prefill_micro.py --tokens $T --iters 5 >> $O/r2aj_prefill_libs.jsonl 2>> $O/r2aj_prefill_libs.err
  for b in cudnn flashinfer-trtllm-gen flashinfer-cutlass flashinfer-auto flashinfer-cudnn; do
    timeout 400 python scripts/prefill_libs.py --backend $b --tokens $T >> $O/r2aj_prefill_libs.jsonl 2>> $O/r2aj_prefill_libs.err; echo "$b $T rc=$?"
  done
done
timeout 900 python bench.py > $O/r2aj_bench.json 2> $O/r2aj_bench.err; echo "bench rc=$?"
