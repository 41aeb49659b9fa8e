# compute-sanitizer over the GPU path: memcheck on the smoke and the DAS /
# envelope / pipeline parity tests, racecheck and synccheck on the smoke
# (one small invocation of every hot kernel).  Run under gpurun; logs land in
# gpurun_out/sanitize_*.log and are summarised into profiles/.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SMOKE='import __graft_entry__ as g; g.smoke(); print("SMOKE OK")'
timeout 300 $CS --tool memcheck --error-exitcode 9 python -c "$SMOKE" \
    > gpurun_out/sanitize_memcheck_smoke.log 2>&1; echo "memcheck smoke rc=$?"
timeout 300 $CS --tool racecheck --racecheck-report all --error-exitcode 9 python -c "$SMOKE" \
    > gpurun_out/sanitize_racecheck_smoke.log 2>&1; echo "racecheck smoke rc=$?"
timeout 300 $CS --tool synccheck --error-exitcode 9 python -c "$SMOKE" \
    > gpurun_out/sanitize_synccheck_smoke.log 2>&1; echo "synccheck smoke rc=$?"
timeout 600 $CS --tool memcheck --error-exitcode 9 python -m pytest -q -x -m gpu \
    tests/test_gpu_das.py tests/test_gpu_sigproc.py tests/test_gpu_pipeline.py \
    -k "not fuzz and not full_size" \
    > gpurun_out/sanitize_memcheck_tests.log 2>&1; echo "memcheck tests rc=$?"
for tool in memcheck racecheck synccheck; do
  timeout 300 $CS --tool $tool --error-exitcode 9 python tools/sanitize_batch.py \
      > gpurun_out/sanitize_${tool}_batch.log 2>&1; echo "$tool batch rc=$?"
done
