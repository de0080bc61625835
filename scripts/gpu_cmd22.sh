python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r22_build.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_fast.py -q > gpurun_out/r22_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r22_tests.log
echo done
