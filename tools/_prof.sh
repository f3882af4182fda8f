for sm in 0 1; do PLG_SEG_MAJOR=$sm python tools/prune_sweep.py --config c5 --specs "3:1:0.03,0.1,0.3"; done
PLG_SEG_MAJOR=1 PLG_PRUNE_SEGLEN=256 python tools/prune_sweep.py --config c5 --specs "3:1:0.03,0.1,0.3"
