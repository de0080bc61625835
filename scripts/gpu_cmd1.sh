nproc > gpurun_out/r2_nproc.txt; lscpu | grep "Model name" >> gpurun_out/r2_nproc.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/r2_gputests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2_gputests.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err
echo "bench rc=$?"
