# compute-sanitizer over tools/sanitize_cases.py: memcheck, racecheck, synccheck, initcheck
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck initcheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize cases done|Error" gpurun_out/sanitize_$tool.log | head -8
done
