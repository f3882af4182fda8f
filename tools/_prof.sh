python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python tools/prune_sweep.py --config c5 --specs "4:2:0.02,0.05,0.12,0.25" 0
ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 2600 --launch-count 1300 --csv --log-file gpurun_out/win_early.csv python tools/profile_round.py --config c5 --mode order --reps 1 > /dev/null 2>&1
