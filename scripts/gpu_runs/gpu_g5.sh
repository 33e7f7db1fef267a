make -s -C paper_2410_00428_b200 -j8 >/dev/null
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_device_gpu.py tests/test_fused_gather.py -x -q > gpurun_out/pytest_g5.txt 2>&1; echo "pytest rc=$?"
A="--group 1 --ctx 16384 --batch 7 --layers 4"
run() { env "$@" timeout 200 python scripts/attn_micro.py $A $X | sed "s/^{/{\"env\": \"$*\", /" >> gpurun_out/pdl_g5.jsonl; }
X=--offloaded
run LKV_PDL=0 LKV_SPLIT_TIMING=1 LKV_MERGE_WARPS=8
run LKV_PDL=1 LKV_SPLIT_TIMING=1 LKV_MERGE_WARPS=4
run LKV_PDL=1 LKV_SPLIT_TIMING=0 LKV_MERGE_WARPS=4
run LKV_PDL=0 LKV_SPLIT_TIMING=0 LKV_MERGE_WARPS=4
run LKV_PDL=1 LKV_SPLIT_TIMING=0 LKV_MERGE_WARPS=8
run LKV_PDL=0 LKV_SPLIT_TIMING=0 LKV_MERGE_WARPS=8
X=
run LKV_PDL=1 LKV_SPLIT_TIMING=0 LKV_MERGE_WARPS=4
run LKV_PDL=0 LKV_SPLIT_TIMING=0 LKV_MERGE_WARPS=4
run LKV_PDL=0 LKV_SPLIT_TIMING=0 LKV_MERGE_WARPS=8
A="--group 8 --hkv 1 --ctx 32768 --batch 64 --layers 2"
run LKV_PDL=1 LKV_SPLIT_TIMING=0 LKV_MERGE_WARPS=4
run LKV_PDL=0 LKV_SPLIT_TIMING=0 LKV_MERGE_WARPS=8
run LKV_PDL=1 LKV_SPLIT_TIMING=1 LKV_MERGE_WARPS=4
