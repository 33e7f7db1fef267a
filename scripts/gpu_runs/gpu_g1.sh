make -s -C paper_2410_00428_b200 -j8 >/dev/null
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_device_gpu.py -x -q > gpurun_out/pytest_g1.txt 2>&1; echo "pytest rc=$?"
for M in 4 5; do
  LKV_MERGE=$M timeout 120 python scripts/attn_micro.py --group 1 --ctx 16384 --batch 7 --layers 4 >> gpurun_out/merge_g1.jsonl
  LKV_MERGE=$M timeout 120 python scripts/attn_micro.py --group 1 --ctx 16384 --batch 2 --layers 4 >> gpurun_out/merge_g1.jsonl
  LKV_MERGE=$M timeout 120 python scripts/attn_micro.py --group 8 --hkv 1 --ctx 32768 --batch 64 --layers 2 >> gpurun_out/merge_g1.jsonl
  LKV_MERGE=$M timeout 120 python scripts/attn_micro.py --group 4 --hkv 8 --ctx 32768 --batch 16 --layers 2 >> gpurun_out/merge_g1.jsonl
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_gqa_tc -s 2 -c 1 -o gpurun_out/gqa_tp8_g1 -f python scripts/attn_micro.py --group 8 --hkv 1 --ctx 32768 --batch 64 --layers 2 --iters 1 > gpurun_out/ncu_gqa_g1.log 2>&1; echo "ncu rc=$?"
