python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r7_build.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r7_bench.json 2>/dev/null
timeout 900 python scripts/partition_probe.py --reps 5 > gpurun_out/r7_partition.jsonl 2> gpurun_out/r7_partition.err
for u in 4 6 8; do PE_TC_UPC=$u timeout 600 python scripts/fast_sweep.py --reps 5 --cfg 3 --only-tc --T 1024,4096,8192 > gpurun_out/r7_tc3_upc$u.jsonl 2>/dev/null; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/tc_prof.py --cfg 5 --fast > gpurun_out/r7_fast_launches.csv 2> gpurun_out/r7_fast_launches.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/tc_prof.py --cfg 3 --fast --T 65536 > gpurun_out/r7_fast3_launches.csv 2> gpurun_out/r7_fast3_launches.err
echo done
