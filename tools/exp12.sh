timeout 1500 compute-sanitizer --tool racecheck --print-limit 2000 --target-processes all python tools/sanitize_kernels.py > gpurun_out/sanitize_racecheck_tc_full.log 2>&1
grep -E "RACECHECK SUMMARY" gpurun_out/sanitize_racecheck_tc_full.log
grep -E "access at" gpurun_out/sanitize_racecheck_tc_full.log | sed 's/+0x[0-9a-f]*//g; s/\[[0-9]* hazards\]//' | sort | uniq -c | sort -rn | head -20
bash tools/exp11.sh
