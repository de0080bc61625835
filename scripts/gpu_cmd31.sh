python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r31_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r31_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r31_tests.log
PE_CREATE_PROF=1 timeout 300 python scripts/e2e_breakdown.py > gpurun_out/r31_e2e.txt 2>&1
timeout 300 python scripts/eval_host_probe.py > gpurun_out/r31_probe.txt 2>&1
timeout 600 python bench.py --no-cpu > gpurun_out/r31_bench.json 2> gpurun_out/r31_bench.err
echo done
