#!/bin/bash
# round 2: serving-loop soak against the live reference (24 random traces)
O=gpurun_out; mkdir -p $O
timeout 2400 python scripts/serve_soak.py --n 24 > $O/r2ah_serve_soak.jsonl 2> $O/r2ah.err; echo "soak rc=$?"
