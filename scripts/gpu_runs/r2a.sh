#!/bin/bash
# round 2, first GPU call: new config-coverage device tests + config3_offload row
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_serve_device.py -m gpu -x -q -k "cfg3 or cfg4_b200 or cfg5" > $O/r2a_pytest.txt 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py --rows config3_offload --no-cpu-baseline > $O/r2a_bench.json 2> $O/r2a_bench.err; echo "bench rc=$?"
free -g >> $O/r2a_bench.err
