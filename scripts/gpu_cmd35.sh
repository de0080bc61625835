python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r35_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r35_gputests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r35_gputests.log
timeout 900 python bench.py > gpurun_out/r35_bench.json 2> gpurun_out/r35_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k k_tc -s 1 -c 1 -o gpurun_out/r35_ktc -f python scripts/tc_prof.py --cfg 5 > gpurun_out/r35_ncu_ktc.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r35_launches.csv 2> gpurun_out/r35_launches.err
echo done
