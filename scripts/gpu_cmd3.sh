python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fast.py -q -x > gpurun_out/r3_fast_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r3_fast_tests.log
timeout 600 ncu --set full --clock-control none --import-source on -k k_tc -s 1 -c 1 -o gpurun_out/r3_ktc_disc1 -f python scripts/tc_prof.py --cfg 5 > gpurun_out/r3_ncu_disc1.log 2>&1
PE_TC_DISCARD=0 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k k_tc -s 1 -c 1 --csv python scripts/tc_prof.py --cfg 5 > gpurun_out/r3_ncu_disc0.csv 2>&1
echo done
