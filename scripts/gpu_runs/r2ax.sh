#!/bin/bash
# round 2: last check on the final code (serve logs, tests): full GPU suite,
# smoke, both bench arms
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -rs --timeout 900 > $O/r2ax_pytest.txt 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2ax_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/r2ax_bench.json 2> $O/r2ax_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/r2ax_bench_ref.json 2> $O/r2ax_bench_ref.err; echo "ref rc=$?"
