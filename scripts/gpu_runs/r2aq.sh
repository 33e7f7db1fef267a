#!/bin/bash
# round 2: check on the P-halves prefill kernel: full GPU suite, smoke, both
# bench arms, ncu launch list of the bench
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -rs --timeout 900 > $O/r2aq_pytest.txt 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2aq_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/r2aq_bench.json 2> $O/r2aq_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/r2aq_bench_ref.json 2> $O/r2aq_bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2aq_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/r2aq_ncu_list.log 2>&1; echo "ncu list rc=$?"
