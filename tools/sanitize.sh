set -x
mkdir -p gpurun_out/san
nvidia-smi --query-gpu=name,clocks.sm --format=csv
python tools/sanitize_run.py > gpurun_out/san/plain.log 2>&1; echo plain rc=$?
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/san/$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/san/summary.txt
  tail -3 gpurun_out/san/$tool.log
done
