#!/bin/bash
# round 2: compute-sanitizer memcheck / racecheck / synccheck on the P-halves
# prefill kernel (new per-half p_full barriers, rescale moved before the exps).
# Refused: compute-sanitizer is closed on this pool (runs under it left GPUs
# needing a reset); the round-2 sanitizer logs predate the P-halves change.
O=gpurun_out; mkdir -p $O
PF='tests/test_prefill_attention.py::test_prefill_attention_parity[1-4] tests/test_prefill_attention.py::test_prefill_attention_parity[129-4] tests/test_prefill_attention.py::test_prefill_attention_parity[385-8] tests/test_prefill_attention.py::test_prefill_attention_parity[640-1]'
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -x -q -m gpu -p no:cacheprovider $PF \
    > $O/r2aw_${tool}_prefill.txt 2>&1; echo "$tool prefill rc=$?"
done
