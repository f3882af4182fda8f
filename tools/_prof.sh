python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -1 gpurun_out/bench_c5.json
ncu --set full --clock-control none -k regex:resid_ent --launch-skip 100 --launch-count 1 -o gpurun_out/resid_ent -f python tools/profile_round.py --config c5 --mode order --reps 1 > gpurun_out/ncu_resid.log 2>&1
tail -1 gpurun_out/ncu_resid.log
