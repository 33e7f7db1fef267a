#!/bin/bash
# One GPU session: bench (both arms), ncu launch list, full captures of the decode kernel and the tcgen05 kernels.
# Usage: scripts/gpu_round.sh <tag>
TAG=${1:-r1}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi_$TAG.txt 2>&1
timeout 900 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $O/bench_ref_$TAG.json 2> $O/bench_ref_$TAG.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_list_$TAG.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 33 -c 2 \
  -o $O/decode_attn_$TAG -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-rows > $O/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_attn2 -c 1 \
  -o $O/prefill_attn2_$TAG -f python scripts/prefill_micro.py --tokens 8192 --iters 1 > $O/ncu_pf_$TAG.log 2>&1; echo "ncu prefill rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_gqa_tc -c 1 \
  -o $O/decode_gqa_tc_$TAG -f python scripts/attn_micro.py --group 8 --hkv 1 --ctx 32768 --batch 64 --layers 1 --iters 1 > $O/ncu_gqa_$TAG.log 2>&1; echo "ncu gqa rc=$?"
ls -la $O
