python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r10_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fast.py -q -x > gpurun_out/r10_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r10_tests.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/tc_prof.py --cfg 5 --fast > gpurun_out/r10_fast_launches.csv 2> gpurun_out/r10_fast_launches.err
timeout 600 ncu --set full --clock-control none --import-source on -k k_fast_merge_fused -s 0 -c 1 -o gpurun_out/r10_fused -f python scripts/tc_prof.py --cfg 5 --fast > gpurun_out/r10_ncu_fused.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k k_fast_fwd -s 40 -c 1 -o gpurun_out/r10_fwd -f python scripts/tc_prof.py --cfg 5 --fast > gpurun_out/r10_ncu_fwd.log 2>&1
echo done
