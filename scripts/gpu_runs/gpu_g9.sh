make -s -C paper_2410_00428_b200 -j8 >/dev/null
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_prefill_attention.py -x -q > gpurun_out/pytest_g9.txt 2>&1; echo "pytest rc=$?"
for T in 1024 4096 8192 16384 32768; do timeout 200 python scripts/prefill_micro.py --tokens $T >> gpurun_out/prefill_g9.jsonl; done
timeout 200 python scripts/prefill_micro.py --tokens 16384 --hq 32 --hkv 32 >> gpurun_out/prefill_g9.jsonl
