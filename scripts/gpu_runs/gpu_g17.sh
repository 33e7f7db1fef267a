make -s -C paper_2410_00428_b200 -j8 >/dev/null
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_device_gpu.py tests/test_fused_gather.py -x -q > gpurun_out/pytest_g17.txt 2>&1; echo "pytest rc=$?"
run() { timeout 200 python scripts/attn_micro.py "$@" | sed "s/^{/{\"args\": \"$*\", /" >> gpurun_out/span_g17.jsonl; }
run --group 1 --ctx 16384 --batch 7 --layers 4
run --group 1 --ctx 16384 --batch 7 --layers 4 --offloaded
run --group 8 --hkv 1 --ctx 32768 --batch 64 --layers 2
timeout 600 python bench.py --no-rows --no-cpu-baseline > gpurun_out/bench_g17.json 2> gpurun_out/bench_g17.err; echo "bench rc=$?"
