python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r16_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_fast.py -q -x > gpurun_out/r16_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r16_tests.log
timeout 1200 python scripts/fast_sweep.py --reps 3 --cfg 3,5 > gpurun_out/r16_sweep.jsonl 2> gpurun_out/r16_sweep.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/tc_prof.py --cfg 5 --fast > gpurun_out/r16_fast_launches.csv 2> gpurun_out/r16_fast_launches.err
echo done
