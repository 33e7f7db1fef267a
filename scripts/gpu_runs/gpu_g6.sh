mkdir -p gpurun_out
run() { timeout 200 python scripts/attn_micro.py "$@" | sed "s/^{/{\"args\": \"$*\", /" >> gpurun_out/tp8_g6.jsonl; }
run --group 8 --hkv 1 --ctx 32768 --batch 64 --layers 2
run --group 8 --hkv 1 --ctx 32768 --batch 64 --layers 1
run --group 8 --hkv 1 --ctx 32768 --batch 64 --layers 4
run --group 8 --hkv 8 --ctx 32768 --batch 8 --layers 2
run --group 4 --hkv 1 --ctx 32768 --batch 64 --layers 2
run --group 4 --hkv 2 --ctx 32768 --batch 32 --layers 2
LKV_UNITS_PER_WORKER=8 run --group 8 --hkv 1 --ctx 32768 --batch 64 --layers 2
LKV_UNITS_PER_WORKER=2 run --group 8 --hkv 1 --ctx 32768 --batch 64 --layers 2
cat /proc/meminfo | head -3 > gpurun_out/meminfo_g6.txt; nproc >> gpurun_out/meminfo_g6.txt; numactl -H >> gpurun_out/meminfo_g6.txt 2>&1
