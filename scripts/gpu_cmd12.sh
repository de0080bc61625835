python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r12_build.log 2>&1
timeout 1200 python scripts/fast_sweep.py --reps 3 --with-step --cfg 3 > gpurun_out/r12_sweep3.jsonl 2> gpurun_out/r12_sweep3.err
timeout 1200 python scripts/fast_sweep.py --reps 3 --with-step --step-max 16384 --cfg 5 > gpurun_out/r12_sweep5.jsonl 2> gpurun_out/r12_sweep5.err
echo done
