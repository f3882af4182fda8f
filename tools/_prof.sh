python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -1 gpurun_out/bench_c5.json | cut -c1-300
ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 2600 --launch-count 1300 --csv --log-file gpurun_out/win_early.csv python tools/profile_round.py --config c5 --mode order --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:prune_pairs --launch-skip 602 --launch-count 1 -o gpurun_out/prune_pairs_full -f python tools/profile_round.py --config c5 --mode order --reps 1 > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
