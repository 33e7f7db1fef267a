make -s -C paper_2410_00428_b200 -j8 >/dev/null
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_host_tier.py -x -q > gpurun_out/pytest_g8.txt 2>&1; echo "pytest rc=$?"
for NT in 1 0 1 0; do LKV_TIER_NT=$NT timeout 300 python scripts/tier_micro.py >> gpurun_out/tier_g8.jsonl; done
lscpu | grep -iE "model name|flags" | cut -c1-300 > gpurun_out/lscpu_g8.txt
