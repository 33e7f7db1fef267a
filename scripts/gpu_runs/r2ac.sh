#!/bin/bash
# round 2: serving-loop fuzz on the GPU against the live compiled reference
# (with and without the tier); tier tests after the writer-waits-for-clean fix
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_serve_fuzz_gpu.py tests/test_serve_device.py tests/test_host_tier.py -m gpu -q -rs --timeout 900 --durations 8 -p no:cacheprovider > $O/r2ac_pytest.txt 2>&1; echo "rc=$?"
timeout 300 python scripts/tier_micro.py > $O/r2ac_tier_micro.json 2>> $O/r2ac.err
