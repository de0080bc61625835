python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r20_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/r20_gputests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r20_gputests.log
timeout 600 python bench.py --no-cpu > gpurun_out/r20_bench.json 2> gpurun_out/r20_bench.err
timeout 300 python scripts/e2e_breakdown.py > gpurun_out/r20_e2e.txt 2>&1
echo done
