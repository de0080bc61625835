python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r19_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r19_gputests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r19_gputests.log
timeout 600 python bench.py > gpurun_out/r19_bench.json 2> gpurun_out/r19_bench.err
timeout 300 python bench.py --no-e2e --no-cpu --sustain-s 4 > gpurun_out/r19_bench_sustained.json 2>/dev/null
echo done
