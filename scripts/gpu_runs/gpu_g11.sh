make -s -C paper_2410_00428_b200 -j8 >/dev/null
mkdir -p gpurun_out
run() { env LKV_PREFILL_L2_MB=$M timeout 200 python scripts/prefill_micro.py "$@" | sed "s/^{/{\"l2_mb\": $M, /" >> gpurun_out/prefill_g11.jsonl; }
for rep in 1 2 3; do
for M in 0 16 100000; do
  run --tokens 32768 --iters 10
  run --tokens 16384 --hq 32 --hkv 32 --iters 10
  run --tokens 4096 --iters 20
done
done
