make -s -C paper_2410_00428_b200 -j8 >/dev/null
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_device_gpu.py -x -q -k "parity" > gpurun_out/pytest_g7.txt 2>&1; echo "pytest rc=$?"
run() { env $E timeout 200 python scripts/attn_micro.py "$@" | sed "s/^{/{\"env\": \"$E\", \"args\": \"$*\", /" >> gpurun_out/pf_g7.jsonl; }
for P in 0 2 4 8 12; do
E="LKV_TC_PREFETCH=$P"
run --group 8 --hkv 1 --ctx 32768 --batch 64 --layers 2
run --group 4 --hkv 8 --ctx 32768 --batch 16 --layers 2
run --group 8 --hkv 8 --ctx 16384 --batch 8 --layers 2
done
E="LKV_TC_PREFETCH=4"
run --group 4 --hkv 8 --ctx 32768 --batch 16 --layers 2 --offloaded
E="LKV_TC_PREFETCH=0"
run --group 4 --hkv 8 --ctx 32768 --batch 16 --layers 2 --offloaded
