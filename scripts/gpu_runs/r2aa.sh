#!/bin/bash
# round 2: split merge inside the G=1 attention kernel (last arriver per row)
# vs the PDL merge kernel: decode parity with the variant, headline bench A/B
O=gpurun_out; mkdir -p $O
v=mik
rm -rf /tmp/v_$v && mkdir -p /tmp/v_$v && tar --exclude=.git --exclude=gpurun_out -cf - . | tar -C /tmp/v_$v -xf -
cp build/variants/$v/liblkv.so /tmp/v_$v/paper_2410_00428_b200/liblkv.so
(cd /tmp/v_$v && timeout 1200 python -m pytest tests/test_device_gpu.py tests/test_decode_append.py tests/test_full_size.py tests/test_host_tier.py -m gpu -q -p no:cacheprovider 2>&1 | tail -3) > $O/r2aa_pytest_$v.txt
for rep in 1 2 3; do
  timeout 300 python bench.py --no-rows --no-cpu-baseline --steps 5 --warmup 3 > $O/r2aa_bench_product_$rep.json 2>/dev/null
  (cd /tmp/v_$v && timeout 300 python bench.py --no-rows --no-cpu-baseline --steps 5 --warmup 3) > $O/r2aa_bench_${v}_$rep.json 2>/dev/null
done
