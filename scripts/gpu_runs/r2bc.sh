#!/bin/bash
# round 2: decode parity at the 70B TP8 shard (G=8 tcgen05 tile, 12 x 32k, rank 7)
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_device_gpu.py -m gpu -q -rs -k "70b_tp8_shard or bench_shape" --timeout 600 > $O/r2bc_pytest.txt 2>&1; echo "pytest rc=$?"
