#!/bin/bash
# round 2: tier read-ahead cap (6 = product, 4, 2) at 25% and 50% pinned
O=gpurun_out; mkdir -p $O
for v in ramax2 ramax4; do
  rm -rf /tmp/v_$v && mkdir -p /tmp/v_$v && tar --exclude=.git --exclude=gpurun_out -cf - . | tar -C /tmp/v_$v -xf -
  cp build/variants/$v/liblkv.so /tmp/v_$v/paper_2410_00428_b200/liblkv.so
done
for f in 0.25 0.5; do
  for rep in 1 2; do
    timeout 300 python scripts/tier_micro.py --pinned-frac $f | sed 's/^/{"lib": "product", "row": /; s/$/}/' >> $O/r2t_tier_micro.jsonl 2>> $O/r2t_tier.err
    for v in ramax2 ramax4; do
      (cd /tmp/v_$v && timeout 300 python scripts/tier_micro.py --pinned-frac $f) | sed "s/^/{\"lib\": \"$v\", \"row\": /; s/\$/}/" >> $O/r2t_tier_micro.jsonl 2>> $O/r2t_tier.err
    done
  done
done
