make -s -C paper_2410_00428_b200 -j8 >/dev/null
mkdir -p gpurun_out
run() { env $E timeout 200 python scripts/attn_micro.py "$@" | sed "s/^{/{\"env\": \"$E\", \"args\": \"$*\", /" >> gpurun_out/upw_g20.jsonl; }
for rep in 1 2; do
for E in LKV_UNITS_PER_WORKER=8 LKV_UNITS_PER_WORKER=4 LKV_UNITS_PER_WORKER=2; do
run --group 1 --ctx 16384 --batch 7 --layers 4 --offloaded
run --group 1 --ctx 16384 --batch 2 --layers 4
done
done
