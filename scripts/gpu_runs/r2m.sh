#!/bin/bash
# round 2: (1) prefill speculative-exps variant A/B (parity + micro);
# (2) tiered prefetch through pull_frames_kernel: host-tier GPU tests + f3 row.
O=gpurun_out; mkdir -p $O
for v in spec specp1; do
  rm -rf /tmp/v_$v && mkdir -p /tmp/v_$v && tar --exclude=.git --exclude=gpurun_out -cf - . | tar -C /tmp/v_$v -xf -
  cp build/variants/$v/liblkv.so /tmp/v_$v/paper_2410_00428_b200/liblkv.so
  (cd /tmp/v_$v && timeout 600 python -m pytest tests/test_prefill_attention.py -m gpu -q -p no:cacheprovider 2>&1 | tail -3) > $O/r2m_pytest_prefill_$v.txt
done
for rep in 1 2; do
for T in 4096 16384 32768; do
  for v in product spec specp1; do
    lib=""; [ $v != product ] && lib="--lib build/variants/$v/liblkv.so"
    timeout 300 python scripts/prefill_micro.py --tokens $T --iters 5 $lib --label $v >> $O/r2m_prefill_micro.jsonl 2>> $O/r2m_prefill_micro.err
  done
done
done
timeout 900 python -m pytest tests/test_host_tier.py tests/test_decode_append.py -m gpu -q -p no:cacheprovider > $O/r2m_pytest_tier.txt 2>&1; echo "tier tests rc=$?"
timeout 300 python scripts/tier_micro.py > $O/r2m_tier_micro.json 2> $O/r2m_tier_micro.err; echo "tier micro rc=$?"
timeout 300 python scripts/tier_micro.py --pinned-frac 0.5 >> $O/r2m_tier_micro.json 2>> $O/r2m_tier_micro.err
