#!/bin/bash
# round 2: per-SM pipe rates (MUFU ex2, F2FP, FFMA2, FMNMX3, TMEM load) for
# the prefill softmax; synccheck of the prefill kernel after the o_full fix;
# prefill micro (the added wait must cost nothing).
O=gpurun_out; mkdir -p $O
timeout 300 ./build/pipe_probe > $O/r2l_pipe_probe.jsonl 2>&1; echo "probe rc=$?"
PF='tests/test_prefill_attention.py::test_prefill_attention_parity[1-4] tests/test_prefill_attention.py::test_prefill_attention_parity[129-4] tests/test_prefill_attention.py::test_prefill_attention_parity[385-8] tests/test_prefill_attention.py::test_prefill_attention_parity[640-1]'
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest -x -q -m gpu -p no:cacheprovider $PF \
  > $O/r2l_synccheck_prefill.txt 2>&1; echo "synccheck prefill rc=$?"
for T in 4096 16384 32768; do
  timeout 300 python scripts/prefill_micro.py --tokens $T --iters 5 --label ofull_wait >> $O/r2l_prefill_micro.jsonl 2>> $O/r2l_prefill_micro.err
done
