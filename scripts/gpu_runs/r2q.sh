#!/bin/bash
# round 2 checkpoint: GPU suite, smoke, both bench arms, ncu launch list and
# full captures (decode attention, WG3 prefill, GQA decode tile, pull kernel).
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -rs --timeout 600 > $O/r2q_pytest.txt 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2q_smoke.txt 2>&1; echo "smoke rc=$?"
bash scripts/gpu_round.sh r2q
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pull_frames -c 2 \
  -o $O/pull_frames_r2q -f python scripts/tier_micro.py > $O/ncu_pull_r2q.log 2>&1; echo "ncu pull rc=$?"
