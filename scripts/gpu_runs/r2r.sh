#!/bin/bash
# round 2: tier residency policy (fixed resident subset for the cyclic
# re-fetch) — tier tests, f3 micro at 25% / 50% pinned; the new D2H
# coalescing test; memcheck on the pull kernel and the WG3 prefill kernel.
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_host_tier.py tests/test_decode_append.py -m gpu -q -p no:cacheprovider > $O/r2r_pytest_tier.txt 2>&1; echo "tier tests rc=$?"
timeout 600 python -m pytest "tests/test_device_gpu.py::test_offload_of_reused_slots_coalesces" -m gpu -q -p no:cacheprovider > $O/r2r_pytest_coalesce.txt 2>&1; echo "coalesce rc=$?"
for f in 0.25 0.5; do
  for rep in 1 2; do
    timeout 300 python scripts/tier_micro.py --pinned-frac $f >> $O/r2r_tier_micro.jsonl 2>> $O/r2r_tier.err
  done
done
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_host_tier.py -x -q -m gpu -p no:cacheprovider \
  > $O/r2r_memcheck_tier.txt 2>&1; echo "memcheck tier rc=$?"
PF='tests/test_prefill_attention.py::test_prefill_attention_parity[1-4] tests/test_prefill_attention.py::test_prefill_attention_parity[129-4] tests/test_prefill_attention.py::test_prefill_attention_parity[385-8] tests/test_prefill_attention.py::test_prefill_attention_parity[640-1]'
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -x -q -m gpu -p no:cacheprovider $PF \
    > $O/r2r_${tool}_prefill_wg3.txt 2>&1; echo "$tool prefill rc=$?"
done
