make -s -C paper_2410_00428_b200 -j8 >/dev/null
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_prefill_attention.py -x -q > gpurun_out/pytest_g21.txt 2>&1; echo "pytest rc=$?"
for rep in 1 2; do
for P in 1 0; do
for T in 4096 16384 32768; do LKV_PDL=$P timeout 120 python scripts/prefill_micro.py --tokens $T --iters 10 | sed "s/^{/{\"pdl\": $P, /" >> gpurun_out/pf_g21.jsonl; done
LKV_PDL=$P timeout 120 python scripts/prefill_micro.py --tokens 16384 --hkv 32 --iters 10 | sed "s/^{/{\"pdl\": $P, /" >> gpurun_out/pf_g21.jsonl
done
done
