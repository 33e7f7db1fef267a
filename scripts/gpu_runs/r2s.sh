#!/bin/bash
# round 2: tier residency policy, rebuilt with the intended budget formula
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_host_tier.py tests/test_decode_append.py -m gpu -q -p no:cacheprovider > $O/r2s_pytest_tier.txt 2>&1; echo "tier tests rc=$?"
for f in 0.25 0.5; do
  for rep in 1 2; do
    timeout 300 python scripts/tier_micro.py --pinned-frac $f >> $O/r2s_tier_micro.jsonl 2>> $O/r2s_tier.err
  done
done
