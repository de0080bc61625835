python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4_build.log 2>&1
timeout 900 python scripts/fast_sweep.py --reps 3 > gpurun_out/r4_fast_sweep.jsonl 2> gpurun_out/r4_fast_sweep.err
timeout 900 python scripts/partition_probe.py --reps 5 > gpurun_out/r4_partition.jsonl 2> gpurun_out/r4_partition.err
echo done
