python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r26_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r26_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r26_tests.log
PE_CREATE_PROF=1 timeout 300 python scripts/e2e_breakdown.py > gpurun_out/r26_e2e.txt 2>&1
timeout 600 python bench.py > gpurun_out/r26_bench.json 2> gpurun_out/r26_bench.err
echo done
