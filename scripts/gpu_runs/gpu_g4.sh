mkdir -p gpurun_out
A="--group 1 --ctx 16384 --batch 7 --layers 4"
timeout 200 python scripts/attn_micro.py $A >> gpurun_out/idle_g4.jsonl
timeout 200 python scripts/attn_micro.py $A --idle-ms 30 >> gpurun_out/idle_g4.jsonl
timeout 200 python scripts/attn_micro.py $A --offloaded >> gpurun_out/idle_g4.jsonl
timeout 200 python scripts/attn_micro.py $A --idle-ms 2 >> gpurun_out/idle_g4.jsonl
nvidia-smi -q -d PERFORMANCE,CLOCK > gpurun_out/smi_g4.txt
