python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r23_smoke.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py -q -x > gpurun_out/r23_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r23_tests.log
timeout 600 python bench.py --no-cpu > gpurun_out/r23_bench.json 2> gpurun_out/r23_bench.err
echo done
