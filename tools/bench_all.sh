# Round bench lines for profiles/: every BASELINE config, the exhaustive rounds, the Gaussian
# worst case and the reference arm where a whole CPU fit is short. Run on the GPU box:
#   bash tools/bench_all.sh <round tag>   -> gpurun_out/bench_<tag>/*.json
set -u
tag="${1:-r2}"
out="gpurun_out/bench_$tag"
mkdir -p "$out"
run() {  # name, args...
  local name="$1"; shift
  timeout 1800 python bench.py "$@" > "$out/$name.log" 2>&1
  echo "$name rc=$?"
  tail -1 "$out/$name.log" > "$out/$name.json"
}
run c5 --config c5 --steps 5 --warmup 3
run c5_noprune --config c5 --steps 2 --warmup 3 --no-prune --no-cpu --no-ncu
run c5g --config c5g --steps 2 --warmup 3 --no-cpu
run c3 --config c3 --steps 5 --warmup 3 --no-cpu
run c4 --config c4 --steps 5 --warmup 3 --no-cpu --no-ncu
run c2 --config c2 --steps 100 --warmup 5 --no-cpu --no-ncu
run c1 --config c1 --steps 2000 --warmup 20 --no-cpu --no-ncu
run ref_c5 --impl reference --config c5 --steps 1 --warmup 1
run ref_c2 --impl reference --config c2 --steps 1 --warmup 1
run ref_c1 --impl reference --config c1 --steps 3 --warmup 1
lscpu > "$out/lscpu.txt" 2>&1
nproc > "$out/nproc.txt"
