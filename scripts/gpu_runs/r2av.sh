#!/bin/bash
# round 2: transfer_log.csv and decision_log.csv from the device-virtual executor (f4) + the serve suite
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_serve_device.py -m gpu -q -rs --timeout 900 > $O/r2av_pytest.txt 2>&1; echo "pytest rc=$?"
