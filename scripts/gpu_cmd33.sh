python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1800 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x > gpurun_out/r33_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r33_tests.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/shard_prof.py > gpurun_out/r33_shard.csv 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:fixup python scripts/tc_prof.py --cfg 5 > gpurun_out/r33_fix5.csv 2>&1
timeout 900 python scripts/partition_probe.py --reps 5 > gpurun_out/r33_partition.jsonl 2> gpurun_out/r33_partition.err
echo done
