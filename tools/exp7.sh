NCU="ncu --clock-control none --profile-from-start off --kernel-name-base demangled"
cap() { timeout 300 $NCU --set full --import-source on -k "regex:$3" -s $4 -c 1 -o gpurun_out/x_$1 -f python tools/launch_list.py $2 > /dev/null 2>&1; }
cap projmerge -8 'pair_kernel<\(int\)8' 2
cap fixup -8 'merge_fixup' 2
for r in projmerge fixup; do
  python tools/ncu_stalls.py gpurun_out/x_$r.ncu-rep 25 > gpurun_out/x_stalls_$r.txt 2>&1
  ncu -i gpurun_out/x_$r.ncu-rep --page raw --csv > gpurun_out/x_raw_$r.csv 2>&1
done
rm -f gpurun_out/x_*.ncu-rep
