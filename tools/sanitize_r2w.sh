# Sanitizer pass over the round-2 additions (run under gpurun): the four tools over
# tools/sanitize_cases.py (now with the split backward in the P-worker executor), then
# memcheck / racecheck / synccheck with every forward on the CTA-pair kernel
# (DA_FWD_KERNEL=pair), then the 32K runtime parity cases with the split backward.
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck initcheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python tools/sanitize_cases.py > gpurun_out/sanitize_r2w_$tool.log 2>&1
  echo "rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize cases done" gpurun_out/sanitize_r2w_$tool.log | head -4
done
for tool in memcheck synccheck racecheck; do
  echo "== $tool (pair forward)"
  DA_FWD_KERNEL=pair timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python tools/sanitize_cases.py > gpurun_out/sanitize_r2w_pairfwd_$tool.log 2>&1
  echo "rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize cases done" gpurun_out/sanitize_r2w_pairfwd_$tool.log | head -4
done
timeout 1200 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_runtime_scale.py 2>&1 | tail -2
