make -s -C paper_2410_00428_b200 -j8 >/dev/null
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r1aa.txt 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r1aa.txt 2>&1; echo "smoke rc=$?"
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_device_gpu.py -x -q -k "each_merge or each_kernel" > gpurun_out/sanitizer_r1aa.txt 2>&1; echo "memcheck rc=$?"
timeout 900 python bench.py > gpurun_out/bench_r1aa.json 2> gpurun_out/bench_r1aa.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_r1aa.json 2> gpurun_out/bench_ref_r1aa.err; echo "ref rc=$?"
