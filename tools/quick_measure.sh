# GPU box: two default bench lines (no CPU / fp32 legs) and launch lists at the given gammas.
for i in 1 2; do
python bench.py --no-cpu --no-fp32 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('bench', d['value'], d['clocks']['sm_mhz'], ' '.join('%s:%.0f/%.3f'%(g,v['images_per_s'],v['roofline_frac']) for g,v in d['per_gamma'].items()), 'dom', d['roofline']['achieved'], d['roofline']['frac'])"
done
for G in ${GAMMAS:--16 0 16}; do
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qm_$G.csv python tools/launch_list.py $G > /dev/null 2>&1
  python tools/launch_table.py gpurun_out/qm_$G.csv -v > gpurun_out/qm_$G.txt; echo "g=$G"; head -8 gpurun_out/qm_$G.txt
done
