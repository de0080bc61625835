# round-2 GPU pass: tests, discard A/B, ncu capture of k_tc, launch list
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=30 > gpurun_out/r2_gputests2.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2_gputests2.log
for i in 1 2; do
  PE_TC_DISCARD=0 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2_ab_disc0_$i.json 2>/dev/null
  PE_TC_DISCARD=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2_ab_disc1_$i.json 2>/dev/null
done
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --sustain-s 4 > gpurun_out/r2_sustain.json 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc -s 1 -c 1 -o gpurun_out/r2_ktc_disc1 -f python scripts/tc_prof.py --cfg 5 > gpurun_out/r2_ncu_disc1.log 2>&1
PE_TC_DISCARD=0 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_tc -s 1 -c 1 --csv python scripts/tc_prof.py --cfg 5 > gpurun_out/r2_ncu_disc0.csv 2>&1
echo done
