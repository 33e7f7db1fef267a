#!/bin/bash
# round 2: verify hygiene + a4 fix + tier read-ahead + N>1 checks; bench both arms;
# sanitizer racecheck / synccheck on the tcgen05 / TMA kernels.
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/r2d_pytest.txt 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2d_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/r2d_bench.json 2> $O/r2d_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $O/r2d_bench_ref.json 2> $O/r2d_bench_ref.err; echo "ref rc=$?"
LKV_BENCH_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --no-rows --no-cpu-baseline > $O/r2d_bench_2r1g.json 2> $O/r2d_bench_2r1g.err; echo "2r1g rc=$?"
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 python -m pytest tests/test_device_gpu.py -x -q -m gpu \
  -k "each_kernel or merge_many" > $O/r2d_racecheck_decode.txt 2>&1; echo "racecheck decode rc=$?"
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 python -m pytest -x -q -m gpu \
  'tests/test_prefill_attention.py::test_prefill_attention_parity[1-4]' 'tests/test_prefill_attention.py::test_prefill_attention_parity[129-4]' 'tests/test_prefill_attention.py::test_prefill_attention_parity[385-8]' 'tests/test_prefill_attention.py::test_prefill_attention_parity[640-1]' > $O/r2d_racecheck_prefill.txt 2>&1; echo "racecheck prefill rc=$?"
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_device_gpu.py -x -q -m gpu \
  -k "each_kernel or merge_many" > $O/r2d_synccheck_decode.txt 2>&1; echo "synccheck decode rc=$?"
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest -x -q -m gpu \
  'tests/test_prefill_attention.py::test_prefill_attention_parity[1-4]' 'tests/test_prefill_attention.py::test_prefill_attention_parity[129-4]' 'tests/test_prefill_attention.py::test_prefill_attention_parity[385-8]' 'tests/test_prefill_attention.py::test_prefill_attention_parity[640-1]' > $O/r2d_synccheck_prefill.txt 2>&1; echo "synccheck prefill rc=$?"
timeout 2400 bash scripts/mutation_check.sh > $O/r2d_mutation.txt 2>&1; echo "mutation rc=$?"
