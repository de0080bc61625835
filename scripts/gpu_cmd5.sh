python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r5_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_tc.py tests/test_gpu_stress.py tests/test_gpu_dist.py -q -x > gpurun_out/r5_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r5_tests.log
timeout 900 python scripts/partition_probe.py --reps 5 > gpurun_out/r5_partition.jsonl 2> gpurun_out/r5_partition.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/tc_prof.py --cfg 5 --fast > gpurun_out/r5_fast_launches.csv 2> gpurun_out/r5_fast_launches.err
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r5_bench.json 2>/dev/null
echo done
