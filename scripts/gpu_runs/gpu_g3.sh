make -s -C paper_2410_00428_b200 -j8 >/dev/null
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_device_gpu.py tests/test_decode_append.py tests/test_serve_device.py tests/test_full_size.py -x -q > gpurun_out/pytest_g3.txt 2>&1; echo "pytest rc=$?"
for i in 1 2; do
timeout 120 python scripts/attn_micro.py --group 8 --hkv 1 --ctx 32768 --batch 64 --layers 2 >> gpurun_out/gqa_g3.jsonl
timeout 120 python scripts/attn_micro.py --group 4 --hkv 8 --ctx 32768 --batch 16 --layers 2 >> gpurun_out/gqa_g3.jsonl
timeout 120 python scripts/attn_micro.py --group 8 --hkv 8 --ctx 16384 --batch 8 --layers 2 >> gpurun_out/gqa_g3.jsonl
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_gqa_tc -s 2 -c 1 -o gpurun_out/gqa_tp8_g3 -f python scripts/attn_micro.py --group 8 --hkv 1 --ctx 32768 --batch 64 --layers 2 --iters 1 > gpurun_out/ncu_gqa_g3.log 2>&1; echo "ncu rc=$?"
