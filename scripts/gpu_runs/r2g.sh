#!/bin/bash
# round 2: compute-sanitizer racecheck / synccheck on the tcgen05 / TMA kernels
# (decode tile, G=1 kernel, merge, reworked prefill), the decode mutation check,
# and the N=2 bench path with both ranks on one GPU (gather_verified).
O=gpurun_out; mkdir -p $O
PF='tests/test_prefill_attention.py::test_prefill_attention_parity[1-4] tests/test_prefill_attention.py::test_prefill_attention_parity[129-4] tests/test_prefill_attention.py::test_prefill_attention_parity[385-8] tests/test_prefill_attention.py::test_prefill_attention_parity[640-1]'
LKV_BENCH_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --no-rows --no-cpu-baseline > $O/r2g_bench_2r1g.json 2> $O/r2g_bench_2r1g.err; echo "2r1g rc=$?"
for tool in racecheck synccheck; do
  extra=""; [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1200 compute-sanitizer --tool $tool $extra --print-limit 20 python -m pytest tests/test_device_gpu.py -x -q -m gpu \
    -k "each_kernel or merge_many" -p no:cacheprovider > $O/r2g_${tool}_decode.txt 2>&1; echo "$tool decode rc=$?"
  timeout 900 compute-sanitizer --tool $tool $extra --print-limit 20 python -m pytest -x -q -m gpu -p no:cacheprovider $PF \
    > $O/r2g_${tool}_prefill.txt 2>&1; echo "$tool prefill rc=$?"
done
timeout 2400 bash scripts/mutation_check.sh > $O/r2g_mutation.txt 2>&1; echo "mutation rc=$?"
