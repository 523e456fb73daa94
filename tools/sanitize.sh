# compute-sanitizer over tools/sanitize_step.py (tiny + small MNIST-shaped step); logs in gpurun_out/san
mkdir -p gpurun_out/san
for tool in memcheck synccheck initcheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --kernel-name-exclude kns=k_fill --print-limit 20 \
    python tools/sanitize_step.py > gpurun_out/san/$tool.txt 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/$tool.txt | tail -1)"
done
