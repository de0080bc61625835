python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r15_smoke.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_fast.py tests/test_gpu_stress.py -q > gpurun_out/r15_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r15_tests.log
echo done
