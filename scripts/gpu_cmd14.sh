python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r14_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r14_bench.json 2> gpurun_out/r14_bench.err
timeout 300 python bench.py --no-e2e --no-cpu --sustain-s 3 > gpurun_out/r14_bench_sustained.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r14_launches.csv 2> gpurun_out/r14_launches.err
timeout 600 ncu --set full --clock-control none --import-source on -k k_tc -s 1 -c 1 -o gpurun_out/r14_ktc -f python scripts/tc_prof.py --cfg 5 > gpurun_out/r14_ncu_ktc.log 2>&1
echo done
