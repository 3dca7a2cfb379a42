# GPU box: the three compute-sanitizer tools over tools/sanitize_kernels.py with the default
# (tcgen05 whole-row) attention backend only.
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all python tools/sanitize_kernels.py > gpurun_out/sanitize_${tool}_tc.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|all launches done' gpurun_out/sanitize_${tool}_tc.log | tr '\n' ' ')"
done
