#!/bin/bash
# round 2 (re-entry): verify the a4 device free-list mirror + peaked-softmax tests on the GPU,
# full -m gpu suite, smoke, and the decode mutation check.
O=gpurun_out; mkdir -p $O
nproc > $O/r2c_host.txt; lscpu | head -20 >> $O/r2c_host.txt; nvidia-smi topo -m >> $O/r2c_host.txt 2>&1; numactl -H >> $O/r2c_host.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/r2c_pytest.txt 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2c_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 2400 bash scripts/mutation_check.sh > $O/r2c_mutation.txt 2>&1; echo "mutation rc=$?"
