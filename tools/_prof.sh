export PLG_PRUNE_SEGLEN=128
for b in 0.8 0.9 1.0 1.05; do PLG_PRUNE_BETA=$b python tools/prune_sweep.py --config c5 --specs "4:2:0.02,0.05,0.12,0.25"; done
PLG_PRUNE_BETA=1.0 python tools/prune_sweep.py --config c5 --specs "4:2:0.01,0.03,0.08,0.2" "4:2:0.02,0.05,0.1,0.2,0.35" "4:2:0.04,0.12,0.3" "4:3:0.02,0.05,0.12,0.25" "2:2:0.02,0.05,0.12,0.25"
