make -s -C paper_2410_00428_b200 -j8 >/dev/null
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_device_gpu.py tests/test_decode_append.py tests/test_fused_gather.py -x -q > gpurun_out/pytest_g2.txt 2>&1; echo "pytest rc=$?"
for G in 8 4 2; do
  H=$((8 / (G == 8 ? 8 : 1))); [ $G = 8 ] && H=1 || H=8
  B=$([ $G = 8 ] && echo 64 || echo 16)
  timeout 120 python scripts/attn_micro.py --group $G --hkv $H --ctx 32768 --batch $B --layers 2 >> gpurun_out/gqa_g2.jsonl
done
timeout 120 python scripts/attn_micro.py --group 8 --hkv 8 --ctx 16384 --batch 8 --layers 2 >> gpurun_out/gqa_g2.jsonl
for M in 4 5; do
  LKV_MERGE=$M timeout 600 python bench.py --no-rows --no-cpu-baseline > gpurun_out/bench_m${M}_g2.json 2>gpurun_out/bench_m${M}_g2.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_gqa_tc -s 2 -c 1 -o gpurun_out/gqa_tp8_g2 -f python scripts/attn_micro.py --group 8 --hkv 1 --ctx 32768 --batch 64 --layers 2 --iters 1 > gpurun_out/ncu_gqa_g2.log 2>&1; echo "ncu rc=$?"
