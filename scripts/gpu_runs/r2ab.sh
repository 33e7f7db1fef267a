#!/bin/bash
# round 2: serving loop over the tiered host memory (f1 x f3), device-virtual parity
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_serve_device.py -m gpu -q -p no:cacheprovider -k tiered -rs > $O/r2ab_pytest_serve_tiered.txt 2>&1; echo "rc=$?"
