#!/bin/bash
# round 2, last GPU check on the final code: full GPU suite, smoke, both bench arms
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -rs --timeout 900 > $O/r2last_pytest.txt 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2last_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/r2last_bench.json 2> $O/r2last_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/r2last_bench_ref.json 2> $O/r2last_bench_ref.err; echo "ref rc=$?"
LKV_BENCH_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29537 bench.py --gpus 2 --steps 2 --warmup 3 --no-rows --no-cpu-baseline > $O/r2last_bench_2r1g.json 2> $O/r2last_bench_2r1g.err; echo "2r1g rc=$?"
