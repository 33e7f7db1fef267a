#!/bin/bash
# round 2: after reverting the prefill rework (slower: profiles/r2f_prefill_micro.jsonl)
# and fixing the host-tier deadlock: full GPU suite (per-test timeout), smoke,
# prefill micro of the restored kernel, bench both arms.
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -rs --timeout 600 --durations 15 > $O/r2h_pytest.txt 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2h_smoke.txt 2>&1; echo "smoke rc=$?"
for T in 4096 16384 32768; do
  timeout 300 python scripts/prefill_micro.py --tokens $T --iters 5 --label restored >> $O/r2h_prefill_micro.jsonl 2>> $O/r2h_prefill_micro.err
done
timeout 1200 python bench.py > $O/r2h_bench.json 2> $O/r2h_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $O/r2h_bench_ref.json 2> $O/r2h_bench_ref.err; echo "ref rc=$?"
