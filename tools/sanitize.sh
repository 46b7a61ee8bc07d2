# compute-sanitizer over tools/sanitize_run.py (one GPU call); summaries in gpurun_out/san_*.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/san_$tool.txt 2>&1
  echo "$tool exit=$?" >> gpurun_out/san_summary.txt
  tail -3 gpurun_out/san_$tool.txt >> gpurun_out/san_summary.txt
done
