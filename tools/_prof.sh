for v in 0 1 2; do PLG_LIST_VAR=$v python tools/prune_sweep.py --config c5 --specs "3:1:0.05,0.25"; done
