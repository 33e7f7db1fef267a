#!/bin/bash
# round 2: serving soak again after the resident-subset yield fix; tier + serve suites
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_host_tier.py tests/test_serve_fuzz_gpu.py -m gpu -q -p no:cacheprovider -k "tier or fuzz" > $O/r2ai_pytest.txt 2>&1; echo "pytest rc=$?"
timeout 3000 python scripts/serve_soak.py --n 24 > $O/r2ai_serve_soak.jsonl 2> $O/r2ai.err; echo "soak rc=$?"
