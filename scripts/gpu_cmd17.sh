timeout 1200 python scripts/fast_sweep.py --reps 3 --with-step --cfg 3 > gpurun_out/r17_sweep3.jsonl 2> gpurun_out/r17_sweep3.err
timeout 1200 python scripts/fast_sweep.py --reps 3 --with-step --step-max 16384 --cfg 5 > gpurun_out/r17_sweep5.jsonl 2> gpurun_out/r17_sweep5.err
echo done
