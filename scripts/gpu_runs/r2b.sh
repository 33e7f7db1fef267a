#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_device_gpu.py -m gpu -q -k "peaked or bench_shape" > $O/r2b_pytest.txt 2>&1; echo "pytest rc=$?"
timeout 2400 bash scripts/mutation_check.sh > $O/r2b_mutation.txt 2>&1; echo "mutation rc=$?"
