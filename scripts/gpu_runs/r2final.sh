#!/bin/bash
# round 2 final checkpoint on the committed code: GPU suite, smoke, bench both
# arms, ncu launch list + captures (scripts/gpu_round.sh), prefill sanitizers
# after the hygiene pass, and the config-5 sweep.
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -rs --timeout 600 > $O/r2final_pytest.txt 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2final_smoke.txt 2>&1; echo "smoke rc=$?"
bash scripts/gpu_round.sh r2final
PF='tests/test_prefill_attention.py::test_prefill_attention_parity[1-4] tests/test_prefill_attention.py::test_prefill_attention_parity[129-4] tests/test_prefill_attention.py::test_prefill_attention_parity[385-8] tests/test_prefill_attention.py::test_prefill_attention_parity[640-1]'
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -x -q -m gpu -p no:cacheprovider $PF \
    > $O/r2final_${tool}_prefill.txt 2>&1; echo "$tool prefill rc=$?"
done
timeout 1500 python scripts/sweep_offload.py > $O/r2final_sweep_offload.jsonl 2> $O/r2final_sweep.err; echo "sweep rc=$?"
