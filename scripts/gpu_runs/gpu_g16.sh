make -s -C paper_2410_00428_b200 -j8 >/dev/null
mkdir -p gpurun_out
cat /sys/kernel/mm/transparent_hugepage/enabled > gpurun_out/thp_g16.txt 2>&1
timeout 300 python -m pytest tests/test_host_tier.py tests/test_prefill_attention.py -x -q > gpurun_out/pytest_g16.txt 2>&1; echo "pytest rc=$?"
for T in 1 0 1 0; do LKV_TIER_THP=$T timeout 300 python scripts/tier_micro.py | sed "s/^{/{\"thp\": $T, /" >> gpurun_out/tier_g16.jsonl; done
