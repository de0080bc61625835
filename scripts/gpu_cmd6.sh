python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r6_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_tc.py tests/test_gpu_stress.py tests/test_gpu_dist.py tests/test_gpu_fast.py -q -x > gpurun_out/r6_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r6_tests.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r6_bench.json 2>/dev/null
PE_TC_UPC=0 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r6_bench_upc0.json 2>/dev/null
timeout 900 python scripts/partition_probe.py --reps 5 > gpurun_out/r6_partition.jsonl 2> gpurun_out/r6_partition.err
for u in 0 4 16; do PE_TC_UPC=$u timeout 600 python scripts/fast_sweep.py --reps 3 --cfg 3 > gpurun_out/r6_sweep3_upc$u.jsonl 2>/dev/null; done
timeout 600 python scripts/fast_sweep.py --reps 3 --cfg 5 > gpurun_out/r6_sweep5.jsonl 2>/dev/null
echo done
