make -s -C paper_2410_00428_b200 -j8 >/dev/null
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_device_gpu.py tests/test_decode_append.py -x -q > gpurun_out/pytest_g12.txt 2>&1; echo "pytest rc=$?"
run() { timeout 200 python scripts/attn_micro.py "$@" | sed "s/^{/{\"args\": \"$*\", /" >> gpurun_out/split_g12.jsonl; }
for rep in 1 2; do
run --group 8 --hkv 1 --ctx 32768 --batch 64 --layers 2
run --group 4 --hkv 8 --ctx 32768 --batch 16 --layers 2
run --group 2 --hkv 8 --ctx 32768 --batch 16 --layers 2
run --group 8 --hkv 8 --ctx 16384 --batch 8 --layers 2
run --group 4 --hkv 8 --ctx 32768 --batch 64 --layers 2
done
