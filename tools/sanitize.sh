# compute-sanitizer over every hot-path kernel family (tools/sanitize_run.py), one tool at a
# time, each bounded by a timeout. Logs under gpurun_out/san/ (summaries go to profiles/).
set -x
mkdir -p gpurun_out/san
: "${SAN_D:=160}" "${SAN_N:=1024}" "${SAN_TIMEOUT:=1500}"
export SAN_D SAN_N
# small pair-list batches: the grid-barrier (multi-batch) path of prune_pairs_kernel runs too
export PLG_PRUNE_BATCH="${PLG_PRUNE_BATCH:-2048}"
nvidia-smi --query-gpu=name,clocks.sm --format=csv
python tools/sanitize_run.py > gpurun_out/san/plain.log 2>&1; echo plain rc=$?
for tool in memcheck synccheck initcheck racecheck; do
  timeout "$SAN_TIMEOUT" compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
    python tools/sanitize_run.py > gpurun_out/san/$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/san/summary.txt
  tail -3 gpurun_out/san/$tool.log
done
