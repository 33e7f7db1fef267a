#!/bin/bash
# round 2: ncu --set full of cuDNN's SDPA kernel and of ours at 16k GQA
# (launch shape, pipe utilisation, MUFU vs FMA instruction mix)
O=gpurun_out; mkdir -p $O
timeout 600 ncu --set full --clock-control none -k regex:'cudnn|sm100|fmha|flash|attn|sdpa' -c 1 -s 2 \
  -o $O/r2ap_cudnn_16k -f python scripts/prefill_libs.py --backend cudnn --tokens 16384 --iters 1 > $O/r2ap_ncu_cudnn.log 2>&1; echo "cudnn rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_attn2 -c 1 -s 1 \
  -o $O/r2ap_ours_16k -f python scripts/prefill_micro.py --tokens 16384 --iters 1 > $O/r2ap_ncu_ours.log 2>&1; echo "ours rc=$?"
