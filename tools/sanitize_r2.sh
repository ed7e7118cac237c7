# Round-2 sanitizer pass (run under gpurun): the four compute-sanitizer tools over
# tools/sanitize_cases.py with the product library, then racecheck again with the
# evidence build lib_vecsglobal.so (DA_BWD_VECS_FROM_GLOBAL: the backward's P / dS
# warps read -lse / -D from global memory instead of the loader's mbarrier-ordered
# shared-memory ring) and the backward parity tests on that build.
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck initcheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python tools/sanitize_cases.py > gpurun_out/sanitize_r2_$tool.log 2>&1
  echo "rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize cases done|Error" gpurun_out/sanitize_r2_$tool.log | head -8
done
echo "== racecheck, vecs-from-global evidence build"
DISTATTN_B200_LIB=paper_2310_03294_b200/variants/lib_vecsglobal.so timeout 900 \
  compute-sanitizer --tool racecheck --target-processes all --print-limit 20 \
  python tools/sanitize_cases.py > gpurun_out/sanitize_r2_racecheck_vecsglobal.log 2>&1
echo "rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize cases done|Error" gpurun_out/sanitize_r2_racecheck_vecsglobal.log | head -8
DISTATTN_B200_LIB=paper_2310_03294_b200/variants/lib_vecsglobal.so timeout 600 \
  python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "bwd" > gpurun_out/sanitize_r2_vecsglobal_parity.log 2>&1
echo "vecsglobal parity rc=$?"; tail -2 gpurun_out/sanitize_r2_vecsglobal_parity.log
