python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r13_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r13_gputests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r13_gputests.log
timeout 900 python scripts/ktc_ab.py --rounds 6 --n 10 "PE_TC_SLEEP=32,64,64" "PE_TC_SLEEP=0,64,64" "PE_TC_SLEEP=0,0,0" "PE_TC_SLEEP=16,32,32" "PE_TC_SLEEP=64,128,128" "PE_TC_DISCARD=0" > gpurun_out/r13_ab.jsonl 2> gpurun_out/r13_ab.err
echo done
