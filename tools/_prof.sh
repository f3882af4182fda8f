set -x
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
tail -2 gpurun_out/bench_c5.json
ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 40 --launch-count 1000 --csv --log-file gpurun_out/launches_prune.csv python tools/profile_round.py --config c5 --mode order --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:prune_pairs --launch-skip 12 --launch-count 1 -o gpurun_out/prune_pairs -f python tools/profile_round.py --config c5 --mode order --reps 1 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
