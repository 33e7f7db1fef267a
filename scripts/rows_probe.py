import json, sys, os
sys.path.insert(0, os.getcwd())
import torch, bench
dev = torch.device("cuda:0")
print(json.dumps({"a6_a8": bench.scatter_gather_row(torch, dev, 6543.4)}))
print(json.dumps({"a20_c3": bench.gqa_prefill_row(torch, dev, 1641.4)}))
