make -s -C paper_2410_00428_b200 -j8 >/dev/null
mkdir -p gpurun_out
run() { timeout 200 python scripts/attn_micro.py "$@" | sed "s/^{/{\"args\": \"$*\", /" >> gpurun_out/bs_g14.jsonl; }
for BS in 16 32 64; do
run --group 1 --ctx 16384 --batch 7 --layers 4 --bs $BS
run --group 4 --hkv 8 --ctx 32768 --batch 16 --layers 2 --bs $BS
run --group 8 --hkv 1 --ctx 32768 --batch 64 --layers 2 --bs $BS
done
