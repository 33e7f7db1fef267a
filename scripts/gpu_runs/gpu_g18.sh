make -s -C paper_2410_00428_b200 -j8 >/dev/null
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_gpu.py tests/test_decode_append.py tests/test_serve_device.py tests/test_fused_gather.py -x -q > gpurun_out/pytest_g18.txt 2>&1; echo "pytest rc=$?"
run() { env $E timeout 200 python scripts/attn_micro.py "$@" | sed "s/^{/{\"env\": \"$E\", \"args\": \"$*\", /" >> gpurun_out/fuse_g18.jsonl; }
for E in LKV_TC_FUSED_MERGE=1 LKV_TC_FUSED_MERGE=0 LKV_TC_FUSED_MERGE=1 LKV_TC_FUSED_MERGE=0; do
run --group 8 --hkv 1 --ctx 32768 --batch 64 --layers 2
run --group 4 --hkv 8 --ctx 32768 --batch 16 --layers 2
run --group 4 --hkv 8 --ctx 32768 --batch 64 --layers 2
done
