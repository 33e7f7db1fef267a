make -s -C paper_2410_00428_b200 -j8 >/dev/null
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_prefill_attention.py -x -q -k "64-key or rescales" > gpurun_out/pytest_g15.txt 2>&1; echo "pytest rc=$?"
if grep -q passed gpurun_out/pytest_g15.txt && ! grep -q failed gpurun_out/pytest_g15.txt; then
for rep in 1 2; do
for K in 2 3; do
for T in 4096 16384 32768; do
  LKV_PREFILL_KERNEL=$K timeout 120 python scripts/prefill_micro.py --tokens $T --iters 10 | sed "s/^{/{\"kernel\": $K, /" >> gpurun_out/pf3_g15.jsonl
done
LKV_PREFILL_KERNEL=$K timeout 120 python scripts/prefill_micro.py --tokens 16384 --hkv 32 --iters 10 | sed "s/^{/{\"kernel\": $K, /" >> gpurun_out/pf3_g15.jsonl
done
done
fi
