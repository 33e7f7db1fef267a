#!/bin/bash
# round 2: serving soak on the final code with the CLI logs compared too:
# 16 random traces (7B / 8B GQA / 70B TP8 shards, block sizes 16-64, tiers)
O=gpurun_out; mkdir -p $O
timeout 2400 python scripts/serve_soak.py --n 16 --seed0 3000 --models > $O/r2bf_serve_soak.jsonl 2> $O/r2bf_serve_soak.err; echo "soak rc=$?"
