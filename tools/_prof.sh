python -m pytest tests/test_gpu_prune.py -q 2>&1 | tail -2
python tools/prune_sweep.py --config c5 --specs "4:2:0.02,0.05,0.12,0.25"
