python -m pytest tests/test_gpu_prune.py tests/test_gpu_parity.py tests/test_gpu_kernels_var.py -q -x 2>&1 | tail -1
python tools/prune_sweep.py --config c5 --specs "3:1:0.05,0.25" "3:1:0.03,0.1,0.3"
ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 2200 --launch-count 1000 --csv --log-file gpurun_out/win_early.csv python tools/profile_round.py --config c5 --mode order --reps 1 > /dev/null 2>&1
