#!/bin/bash
# round 2: bench with cuDNN beside the 7B MHA a20 row too
O=gpurun_out; mkdir -p $O
timeout 900 python bench.py > $O/r2bg_bench.json 2> $O/r2bg_bench.err; echo "bench rc=$?"
