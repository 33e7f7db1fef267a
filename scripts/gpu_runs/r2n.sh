#!/bin/bash
# round 2: TMEM load probes (4 x ld32 one wait, 2 x ld64), the full GPU suite
# after the reversed-pack / sorted-escalation staging change, the tier micro at
# 25% and 50% pinned with the new read-ahead bound, and the bench.
O=gpurun_out; mkdir -p $O
timeout 300 ./build/pipe_probe > $O/r2n_pipe_probe.jsonl 2>&1; echo "probe rc=$?"
timeout 300 python scripts/tier_micro.py > $O/r2n_tier_micro.json 2> $O/r2n_tier_micro.err; echo "tier micro rc=$?"
timeout 300 python scripts/tier_micro.py --pinned-frac 0.5 >> $O/r2n_tier_micro.json 2>> $O/r2n_tier_micro.err
timeout 1800 python -m pytest tests -m gpu -q -rs --timeout 600 > $O/r2n_pytest.txt 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py > $O/r2n_bench.json 2> $O/r2n_bench.err; echo "bench rc=$?"
