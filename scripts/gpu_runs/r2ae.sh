#!/bin/bash
# round 2: units per CTA of the tcgen05 decode tile (4 = product, 2, 1) on
# the a18 rows (config 3 batch 64, 70B TP8 shard)
O=gpurun_out; mkdir -p $O
for v in u2 u1; do
  rm -rf /tmp/v_$v && mkdir -p /tmp/v_$v && tar --exclude=.git --exclude=gpurun_out -cf - . | tar -C /tmp/v_$v -xf -
  cp build/variants/$v/liblkv.so /tmp/v_$v/paper_2410_00428_b200/liblkv.so
done
for rep in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline --steps 2 --warmup 3 --rows a18_gqa_decode,a18_gqa_decode_70b_tp8_shard | sed 's/^/{"lib": "product", "line": /; s/$/}/' >> $O/r2ae.jsonl 2>> $O/r2ae.err
  for v in u2 u1; do
    (cd /tmp/v_$v && timeout 300 python bench.py --no-cpu-baseline --steps 2 --warmup 3 --rows a18_gqa_decode,a18_gqa_decode_70b_tp8_shard) | sed "s/^/{\"lib\": \"$v\", \"line\": /; s/\$/}/" >> $O/r2ae.jsonl 2>> $O/r2ae.err
  done
done
v=u2
(cd /tmp/v_$v && timeout 900 python -m pytest tests/test_device_gpu.py -m gpu -q -p no:cacheprovider -k "each_kernel or peaked or ragged" 2>&1 | tail -2) > $O/r2ae_pytest_$v.txt
