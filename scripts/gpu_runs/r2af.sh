#!/bin/bash
# round 2: bench rows after the sustained-prefill and link-peak changes
O=gpurun_out; mkdir -p $O
timeout 900 python bench.py --no-cpu-baseline --steps 2 --warmup 3 --rows prefill,config3_offload > $O/r2af_bench.json 2> $O/r2af_bench.err; echo "bench rc=$?"
timeout 600 python -m pytest tests/test_bench_contract.py -m gpu -q -p no:cacheprovider > $O/r2af_pytest_contract.txt 2>&1; echo "contract rc=$?"
