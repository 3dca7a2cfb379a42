# GPU box: the three compute-sanitizer tools over tools/sanitize_kernels.py with the default
# (tcgen05 whole-row) attention backend only.
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all python tools/sanitize_kernels.py > gpurun_out/sanitize_${tool}_tc.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|all launches done' gpurun_out/sanitize_${tool}_tc.log | tr '\n' ' ')"
done
# synccheck stops the application at its report in the no-size tcgen05 attention instance (profiles/r02c_sanitizer.md),
# so the kernels launched after it get a second synccheck pass with the mma.sync attention backend
TA_ATTENTION_BACKEND=mma timeout 1500 compute-sanitizer --tool synccheck --target-processes all python tools/sanitize_kernels.py > gpurun_out/sanitize_synccheck_mma.log 2>&1
echo "synccheck (attention mma) rc=$? $(grep -E 'ERROR SUMMARY|all launches done' gpurun_out/sanitize_synccheck_mma.log | tr '\n' ' ')"
