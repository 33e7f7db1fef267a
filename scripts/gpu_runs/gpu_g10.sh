make -s -C paper_2410_00428_b200 -j8 >/dev/null
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_prefill_attention.py -x -q > gpurun_out/pytest_g10.txt 2>&1; echo "pytest rc=$?"
run() { env LKV_PREFILL_L2_MB=$M timeout 200 python scripts/prefill_micro.py "$@" | sed "s/^{/{\"l2_mb\": $M, /" >> gpurun_out/prefill_g10.jsonl; }
for M in 16 48 96 100000; do
  run --tokens 32768
  run --tokens 16384 --hq 32 --hkv 32
  run --tokens 16384
  run --tokens 4096
done
