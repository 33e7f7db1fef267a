"""f3 row alone (development aid): tiered host memory decode step.

  python scripts/tier_micro.py [--pinned-frac 0.25]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--pinned-frac", type=float, default=0.25)
    a = p.parse_args()
    dev = torch.device("cuda:0")
    link = bench.host_link_peak(torch, dev)
    row = bench.tiered_host_row(torch, dev, link, pinned_frac=a.pinned_frac)
    print(json.dumps(row))


if __name__ == "__main__":
    main()
