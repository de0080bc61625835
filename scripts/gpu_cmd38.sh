python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/r38_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r38_tests.log
timeout 1200 python scripts/partition_probe.py --reps 5 > gpurun_out/r38_partition.jsonl 2> gpurun_out/r38_partition.err
echo done
